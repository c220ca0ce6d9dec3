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
