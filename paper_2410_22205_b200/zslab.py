"""z-slab decomposition of the SL step across GPUs.

Rank r owns the z-planes [cuts[r], cuts[r+1]) — z is the slowest axis of the
x-fastest layout (grid.hpp:19-21), so a slab and its halo planes are
contiguous — and keeps planes [cuts[r] - H, cuts[r+1] + H) resident. Cuts are
placed on the cumulative per-plane ACTIVE count so every rank gets the same
share of node-updates (equal z-slabs leave most ranks idle on a sphere band).

One step on rank r: update the owned ACTIVE ids (the unchanged SL kernel in
slab mode, `lsr_cuda_sl_step_device`; stencils leaving the resident planes are
counted, never read), then exchange H planes of phi^{n+1} with each neighbour
(point-to-point send/recv; NCCL on GPUs, gloo on CPU for the tests), then
swap buffers. The update of a node depends only on phi^n, d and E_p, so the
decomposition changes no arithmetic: results are bit-identical to one GPU.

The exchange is written against torch.distributed so the same code drives
NCCL over NVLink and the CPU (gloo) tests; the compute is a callable.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def plan_cuts(active: np.ndarray, nxy: int, nz: int, world: int, min_planes: int = 1) -> np.ndarray:
    """Band-balanced cuts (world + 1 plane indices, cuts[0] = 0, cuts[-1] = nz):
    cut r sits where the cumulative per-plane ACTIVE count reaches r/world of
    the total; every slab is at least `min_planes` thick (the halo exchange
    sends owned planes only)."""
    k = np.asarray(active, dtype=np.int64) // nxy
    per_plane = np.bincount(k, minlength=nz)
    cum = np.cumsum(per_plane)
    total = int(cum[-1]) if cum.size else 0
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, total * r / world, side="left")) + 1
        cuts.append(c)
    cuts.append(nz)
    cuts = np.array(cuts, dtype=np.int64)
    # enforce monotone, min thickness, inside [0, nz]
    for r in range(1, world + 1):
        cuts[r] = max(cuts[r], cuts[r - 1] + min_planes)
    if cuts[-1] != nz:
        cuts[-1] = nz
        for r in range(world - 1, 0, -1):
            cuts[r] = min(cuts[r], cuts[r + 1] - min_planes)
    if np.any(np.diff(cuts) < min_planes) or cuts[0] != 0:
        raise ValueError(f"grid of {nz} planes cannot hold {world} slabs of >= {min_planes} planes")
    return cuts


@dataclass
class Slab:
    rank: int
    world: int
    lo: int          # first owned plane
    hi: int          # one past the last owned plane
    z_base: int      # first resident plane
    z_planes: int    # resident planes
    nxy: int

    @property
    def n_resident(self) -> int:
        return self.z_planes * self.nxy

    def local(self, plane: int) -> int:
        """Offset of a global plane in the resident buffer."""
        return (plane - self.z_base) * self.nxy


def make_slab(cuts: np.ndarray, rank: int, halo: int, nxy: int, nz: int) -> Slab:
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    zb = max(0, lo - halo)
    ze = min(nz, hi + halo)
    return Slab(rank, len(cuts) - 1, lo, hi, zb, ze - zb, nxy)


def owned_ids(active: np.ndarray, s: Slab) -> np.ndarray:
    k = np.asarray(active, dtype=np.int64) // s.nxy
    return np.ascontiguousarray(active[(k >= s.lo) & (k < s.hi)], dtype=np.int64)


def exchange_halo(dist, out, s: Slab, halo: int) -> None:
    """Send the owned planes each neighbour reads as halo and receive theirs
    into the resident buffer `out` (a flat torch tensor of s.n_resident
    values). Requires every slab to be >= halo planes thick."""
    ops = []
    P = s.nxy
    if s.rank > 0:
        a, b = s.lo, min(s.hi, s.lo + halo)
        ops.append(dist.P2POp(dist.isend, out[s.local(a) * 1:s.local(b)], s.rank - 1))
        c = max(0, s.lo - halo)
        ops.append(dist.P2POp(dist.irecv, out[s.local(c):s.local(s.lo)], s.rank - 1))
    if s.rank < s.world - 1:
        a = max(s.lo, s.hi - halo)
        ops.append(dist.P2POp(dist.isend, out[s.local(a):s.local(s.hi)], s.rank + 1))
        e = min(s.z_base + s.z_planes, s.hi + halo)
        ops.append(dist.P2POp(dist.irecv, out[s.local(s.hi):s.local(e)], s.rank + 1))
    del P
    if ops and out.is_cuda and dist.get_backend() == "gloo":  # gloo moves host tensors: stage through host memory
        staged = [(op, op.tensor, op.tensor.cpu()) for op in ops]
        ops = [dist.P2POp(op.op, h, op.peer) for op, _, h in staged]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for op, dev_t, h in staged:
            if op.op == dist.irecv:
                dev_t.copy_(h)
        return
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def halo_planes(max_displacement: float, dx: float, interp: int) -> int:
    """H = ceil(max foot displacement / dx) + stencil radius (WENO 2 / Q1 1)
    + 1 for the centered gradient."""
    return int(np.ceil(max_displacement / dx)) + (2 if interp == 1 else 1) + 1


class FusedSlabStepper:
    """SURVEY §8(e) phase 2: one kernel per step computes the owned updates
    and stores those of the first/last `push` owned planes straight into the
    neighbours' resident out buffers (peer-mapped over NVLink). The only
    inter-rank operation left is ordering: `barrier()` (stream-ordered) after
    the kernel so a neighbour starts step n+1 only once our pushes landed.

    bufs: this rank's two resident buffers (device pointers; step n writes
    bufs[(n+1) % 2] from bufs[n % 2]); peer_lo / peer_hi: the lower / upper
    neighbour's two buffers (or None) and their first resident plane."""

    def __init__(self, slab: Slab, push: int, bufs, peer_lo, peer_hi, compute_fused, barrier=None):
        self.s, self.push, self.bufs = slab, push, bufs
        self.peer_lo, self.peer_hi = peer_lo, peer_hi
        self.compute = compute_fused
        self.barrier = barrier
        self.n = 0

    def pointers(self):
        src, dst = self.bufs[self.n % 2], self.bufs[(self.n + 1) % 2]
        lo = (self.peer_lo[0][(self.n + 1) % 2], self.peer_lo[1]) if self.peer_lo else (None, 0)
        hi = (self.peer_hi[0][(self.n + 1) % 2], self.peer_hi[1]) if self.peer_hi else (None, 0)
        return src, dst, lo, hi

    def step(self) -> None:
        src, dst, lo, hi = self.pointers()
        self.compute(src, dst, lo, hi, self.s, self.push)
        if self.barrier is not None:
            self.barrier()
        self.n += 1

    @property
    def current(self):
        return self.bufs[self.n % 2]


class SlabStepper:
    """Drives one rank's slab through K steps: compute(phi, dist, out, slab,
    ids) updates the owned ids (returns the halo-miss count), then the halo
    exchange, then the buffer swap."""

    def __init__(self, dist, slab: Slab, halo: int, phi, dfield, out, ids, compute):
        self.dist, self.s, self.halo = dist, slab, halo
        self.phi, self.d, self.out, self.ids = phi, dfield, out, ids
        self.compute = compute

    def step(self) -> int:
        miss = self.compute(self.phi, self.d, self.out, self.s, self.ids)
        if miss:
            return miss
        if self.s.world > 1:
            exchange_halo(self.dist, self.out, self.s, self.halo)
        self.phi, self.out = self.out, self.phi
        return 0


# ---------------------------------------------------------------------------
# The whole loop over z-slabs (driver.cpp:185-203 on each rank's owned
# planes). One iteration is written once, as a generator over one rank's
# SlabContext that yields its collective requests:
#   ("allgather", obj) -> list of every rank's obj
#   ("allreduce_max", x) -> max over ranks
#   ("exchange", field, h) -> h halo planes of `field` swapped with both neighbours
# A runner serves the requests: DistRunner over torch.distributed (one rank
# per process, NCCL between GPUs or gloo), or InProcessRunner, which steps
# several ranks' generators in lockstep in one process (one GPU, ranks run
# one after another, the exchanges are device copies) — the same per-rank
# code either way. Every phase gives the owned nodes the bits the
# whole-grid loop gives them (band, E_2 via the ranks' blocked_sum pieces,
# SL, one-step, the Jacobi sweeps with a global stop rule, clamp).

FIELD_PHI, FIELD_DIST, FIELD_OUT, FIELD_SCRATCH = 0, 1, 2, 3
BLOCK = 4096  # blocked_sum's block (parallel.hpp:28)


class HaloTooSmall(Exception):
    """The feet of some rank reach beyond the resident planes: widen and redo."""

    def __init__(self, need: int):
        super().__init__(f"halo too small: need {need} planes")
        self.need = need


def blocked_sum_pieces(pieces) -> float:
    """blocked_sum (parallel.hpp:26-42) of the concatenation of the ranks'
    contribution lists, from each rank's (full-block sums, head, tail): raw
    contributions are added serially inside their block, block partials in
    block order — the reference's exact operation sequence."""
    total, acc, pos = 0.0, 0.0, 0

    def raw(vals):
        nonlocal total, acc, pos
        for v in vals:
            acc += float(v)
            pos += 1
            if pos % BLOCK == 0:
                total += acc
                acc = 0.0

    for blocks, head, tail in pieces:
        raw(head)
        for b in blocks:
            assert pos % BLOCK == 0
            total += float(b)
            pos += BLOCK
        raw(tail)
    if pos % BLOCK:
        total += acc
    return total


def loop_iteration(ctx, rank: int, cfg, rcfg, gamma: float, refine: int, halo: int, energy_override=None):
    """One driver iteration on one rank's SlabContext (a generator yielding
    collective requests; returns the iteration's statistics). Raises
    HaloTooSmall (on every rank alike) before anything is committed when the
    feet may leave the resident planes."""
    import math

    na, nt = ctx.band(gamma, FIELD_PHI)  # driver.cpp:187
    if energy_override is None:  # driver.cpp:188, metrics.cpp:186-189
        nc = ctx.energy_cells(FIELD_PHI, 2, refine)
        counts = yield ("allgather", nc)
        pieces = ctx.energy_pieces(sum(counts[:rank]))
        e2 = math.pow(blocked_sum_pieces((yield ("allgather", pieces))), 1.0 / 2)
    else:
        e2 = float(energy_override)
    skip_sl = cfg.p > 1 and e2 == 0.0  # driver.cpp:191-195
    if not skip_sl:
        reach = yield ("allreduce_max", ctx.max_reach(cfg, e2) if na else 0.0)
        need = halo_planes(reach * ctx.grid.dx, ctx.grid.dx, int(cfg.interp))
        if need > halo:
            raise HaloTooSmall(need)
    miss = ctx.sl_step(cfg, e2)
    if (yield ("allreduce_max", miss)):
        raise HaloTooSmall(halo + 2)
    yield ("exchange", FIELD_OUT, 1)
    # reinitialize (reinit.cpp:133-145) of phi^{n+1} on the band of phi^n
    frozen, zero = ctx.one_step()
    had = bool((yield ("allreduce_max", int(frozen or zero))))
    it = 0
    result = FIELD_OUT  # NoInterfaceError: phi^{n+1} unchanged, then clamped
    if had:
        yield ("exchange", FIELD_SCRATCH, 1)
        ctx.reinit_begin(rcfg)
        tol = rcfg.residual_tol * ctx.grid.dx
        for k in range(rcfg.max_iters):  # reinit.cpp:110-130
            r = yield ("allreduce_max", ctx.reinit_sweep(rcfg, k))
            it = k + 1
            if r < tol:
                break
            yield ("exchange", FIELD_SCRATCH if it % 2 == 0 else FIELD_OUT, 1)
        result = FIELD_SCRATCH if it % 2 == 0 else FIELD_OUT
    ctx.reinit_end(result, gamma)
    yield ("exchange", FIELD_OUT, halo)
    ctx.swap()  # driver.cpp:203
    return dict(energy=e2, n_active=na, n_tube=nt, reinit_iterations=it, had_interface=had)


def _exchange_pairs(ranks, h):
    """(src rank, dst rank, first plane, planes) of a halo exchange of h planes."""
    for r in range(len(ranks) - 1):
        lo, hi = ranks[r], ranks[r + 1]
        yield r + 1, r, hi.own_lo, min(h, hi.own_hi - hi.own_lo)      # upper's bottom planes -> lower's top halo
        yield r, r + 1, lo.own_hi - min(h, lo.own_hi - lo.own_lo), min(h, lo.own_hi - lo.own_lo)


class InProcessRunner:
    """Runs the ranks of one job in this process (one GPU): every rank's
    generator is advanced to its next collective request, the request is
    served for all ranks together, and the results are sent back."""

    def __init__(self, ctxs):
        self.ctxs = ctxs

    def exchange(self, field, h):
        for src, dst, p0, n in _exchange_pairs(self.ctxs, h):
            if n > 0:
                s, d = self.ctxs[src], self.ctxs[dst]
                d.copy_planes(field, p0, n, s.plane_ptr(field, p0), to_field=True)

    def run(self, gens):
        vals = [None] * len(gens)
        done = [None] * len(gens)
        while True:
            reqs = []
            for r, g in enumerate(gens):
                try:
                    reqs.append(g.send(vals[r]))
                except StopIteration as e:
                    done[r] = e.value
                    reqs.append(None)
            if all(q is None for q in reqs):
                return done
            if any(q is None for q in reqs) or len({q[0] for q in reqs}) != 1:
                raise RuntimeError(f"ranks out of step: {[q and q[0] for q in reqs]}")
            kind = reqs[0][0]
            if kind == "allgather":
                allv = [q[1] for q in reqs]
                vals = [allv] * len(gens)
            elif kind == "allreduce_max":
                m = max(q[1] for q in reqs)
                vals = [m] * len(gens)
            elif kind == "exchange":
                self.exchange(reqs[0][1], reqs[0][2])
                vals = [None] * len(gens)
            else:
                raise RuntimeError(kind)


class DistRunner:
    """Serves one rank's requests over torch.distributed (NCCL between GPUs,
    or gloo): plane exchanges through device staging buffers and
    send/recv, reductions and gathers as collectives."""

    def __init__(self, dist, ctx, cuts):
        import torch

        self.dist, self.ctx, self.torch = dist, ctx, torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.cuts = cuts
        nccl = dist.get_backend() == "nccl"
        self.dev = torch.device("cuda", torch.cuda.current_device()) if nccl else None
        # staging buffers of the plane exchange: device memory for a device
        # context (it copies planes device to device); gloo moves host
        # tensors, so under gloo they are copied through host memory
        self.staging = "cuda" if getattr(ctx, "device_memory", False) else "cpu"
        self.wire_host = not nccl

    def exchange(self, field, h):
        torch, dist, c = self.torch, self.dist, self.ctx
        nxy = c.nxy
        ops, recvs = [], []
        for nb, mine0, theirs0, n in self._neighbours(h):
            send = torch.empty(n * nxy, dtype=torch.float64, device=self.staging)
            c.copy_planes(field, mine0, n, send.data_ptr(), to_field=False)
            recv = torch.empty(n * nxy, dtype=torch.float64, device=self.staging)
            if self.wire_host and send.is_cuda:
                ops += [dist.P2POp(dist.isend, send.cpu(), nb)]
                host_recv = torch.empty(n * nxy, dtype=torch.float64)
                ops += [dist.P2POp(dist.irecv, host_recv, nb)]
                recvs.append((theirs0, n, recv, host_recv))
            else:
                ops += [dist.P2POp(dist.isend, send, nb), dist.P2POp(dist.irecv, recv, nb)]
                recvs.append((theirs0, n, recv, None))
        if ops:
            if self.staging == "cuda":
                torch.cuda.synchronize()
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        for p0, n, buf, host in recvs:
            if host is not None:
                buf.copy_(host)
                torch.cuda.synchronize()
            c.copy_planes(field, p0, n, buf.data_ptr(), to_field=True)

    def _neighbours(self, h):
        """(neighbour rank, my first plane to send, first halo plane to receive, planes)"""
        r, cuts = self.rank, self.cuts
        out = []
        if r > 0:
            n = min(h, cuts[r + 1] - cuts[r], cuts[r] - cuts[r - 1])
            out.append((r - 1, cuts[r], cuts[r] - n, n))
        if r < self.world - 1:
            n = min(h, cuts[r + 1] - cuts[r], cuts[r + 2] - cuts[r + 1])
            out.append((r + 1, cuts[r + 1] - n, cuts[r + 1], n))
        return out

    def run(self, gen):
        torch, dist = self.torch, self.dist
        val = None
        while True:
            try:
                q = gen.send(val)
            except StopIteration as e:
                return e.value
            if q[0] == "allgather":
                out = [None] * self.world
                dist.all_gather_object(out, q[1])
                val = out
            elif q[0] == "allreduce_max":
                t = torch.tensor([float(q[1])], dtype=torch.float64, device=self.dev or "cpu")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                val = float(t.item())
            elif q[0] == "exchange":
                self.exchange(q[1], q[2])
                val = None
            else:
                raise RuntimeError(q[0])


class SlabLoop:
    """The loop over all ranks of one process (InProcessRunner) or this
    process's rank (DistRunner). make_ctx(win_lo, win_hi, own_lo, own_hi)
    creates a SlabContext; fill(ctx) uploads phi^0 and d for its window. On
    HaloTooSmall every rank widens its window (phi carried over, d
    refilled) and redoes the iteration."""

    def __init__(self, grid, cuts, ranks, halo, make_ctx, fill_dist, runner_factory):
        self.grid, self.cuts, self.ranks, self.halo = grid, list(int(c) for c in cuts), list(ranks), int(halo)
        self.make_ctx, self.fill_dist, self.runner_factory = make_ctx, fill_dist, runner_factory
        self._check_halo()
        self.ctxs = [self._new_ctx(r) for r in self.ranks]
        self.runner = runner_factory(self.ctxs)
        self.regrows = 0

    def _check_halo(self):
        thin = min(b - a for a, b in zip(self.cuts[:-1], self.cuts[1:]))
        if len(self.cuts) > 2 and thin < self.halo:
            raise ValueError(f"slabs of {thin} planes cannot feed halos of {self.halo} planes (one hop only)")

    def window(self, r):
        nz = self.grid.dims[2]
        return max(0, self.cuts[r] - self.halo), min(nz, self.cuts[r + 1] + self.halo), self.cuts[r], self.cuts[r + 1]

    def _new_ctx(self, r):
        c = self.make_ctx(*self.window(r))
        self.fill_dist(c)
        return c

    def upload_phi(self, phi_window_of):
        for r, c in zip(self.ranks, self.ctxs):
            c.upload(FIELD_PHI, phi_window_of(c))

    def widen(self, need):
        old = self.ctxs
        self.halo = max(need, self.halo + 1)
        self._check_halo()
        self.ctxs = [self._new_ctx(r) for r in self.ranks]
        for o, c in zip(old, self.ctxs):  # the owned planes of phi^n carry over, the halo comes by exchange
            c.copy_planes(FIELD_PHI, o.own_lo, o.own_hi - o.own_lo, o.plane_ptr(FIELD_PHI, o.own_lo), to_field=True)
            o.close()
        self.runner = self.runner_factory(self.ctxs)
        self._exchange_phi()
        self.regrows += 1

    def _exchange_phi(self):
        def g(c):
            yield ("exchange", FIELD_PHI, self.halo)
        self._run([g(c) for c in self.ctxs])

    def _run(self, gens):
        if isinstance(self.runner, InProcessRunner):
            return self.runner.run(gens)
        return [self.runner.run(gens[0])]

    def step(self, cfg, rcfg, gamma, refine=5, energy_override=None):
        while True:
            gens = [loop_iteration(c, r, cfg, rcfg, gamma, refine, self.halo, energy_override)
                    for r, c in zip(self.ranks, self.ctxs)]
            try:
                return self._run(gens)
            except HaloTooSmall as e:
                self.widen(e.need)
