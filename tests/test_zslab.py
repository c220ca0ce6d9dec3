"""z-slab decomposition: the partition + halo exchange logic
of paper_2410_22205_b200.zslab, run with world_size 2 over gloo on CPU (the
per-slab compute is the oracle restatement), must reproduce the single-domain
evolution bit for bit; on the GPU the slab-mode kernel must agree with the
whole-grid kernel and count stencils that leave the resident planes."""
import os
import socket

import numpy as np
import pytest

from conftest import bits

N = 40
STEPS = 3


def _inputs():
    dx = 2.0 / (N - 1)
    ax = -1.0 + np.arange(N) * dx
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    r = np.sqrt(x * x + y * y + z * z)
    phi = (r - 0.55 + 0.1 * x * y).ravel()
    dist = (np.abs(np.sqrt((x - 0.05) ** 2 + y * y + z * z) - 0.3) + 0.01).ravel()
    g = dict(dim=3, dims=[N, N, N], origin=[-1.0, -1.0, -1.0], dx=dx)
    gam = 6 * dx
    active = np.flatnonzero(np.abs(phi) < gam).astype(np.int64)
    cfg = dict(p=2, interp=1, delta=1.0, dt=0.25 * dx, fallback_c=1e-3, fallback_alpha=1.0, gamma=gam, beta=gam / 2)
    return g, phi, dist, active, cfg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle.bindings import Restatement
    from paper_2410_22205_b200 import zslab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, phi, dfield, active, cfg = _inputs()
    nxy = N * N
    halo = 5
    cuts = zslab.plan_cuts(active, nxy, N, world, min_planes=halo)
    s = zslab.make_slab(cuts, rank, halo, nxy, N)
    ids = zslab.owned_ids(active, s)
    sl = slice(s.z_base * nxy, (s.z_base + s.z_planes) * nxy)
    phi_t = torch.from_numpy(phi[sl].copy())
    out_t = phi_t.clone()
    d_t = torch.from_numpy(dfield[sl].copy())
    O = Restatement()

    def compute(p, d, o, slab, own):
        # embed the resident planes in a NaN field: a stencil that leaves them
        # would turn an owned update into NaN
        full_p = np.full(N ** 3, np.nan)
        full_d = np.full(N ** 3, np.nan)
        full_p[sl] = p.numpy()
        full_d[sl] = d.numpy()
        res, st, bad = O.sl_step(g, full_p, full_d, own, cfg, 0.8)
        vals = res[own]
        o.numpy()[own - s.z_base * nxy] = vals
        return int(np.count_nonzero(~np.isfinite(vals)))

    stepper = zslab.SlabStepper(dist, s, halo, phi_t, d_t, out_t, ids, compute)
    for _ in range(STEPS):
        assert stepper.step() == 0
    owned = stepper.phi.numpy()[(s.lo - s.z_base) * nxy:(s.hi - s.z_base) * nxy]
    np.save(os.path.join(outdir, f"rank{rank}.npy"), owned)
    np.save(os.path.join(outdir, f"cuts.npy"), cuts)
    dist.barrier()
    dist.destroy_process_group()


def test_zslab_two_ranks_gloo_bit_exact(built, tmp_path):
    import torch.multiprocessing as mp

    from oracle.bindings import Restatement

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g, phi, dfield, active, cfg = _inputs()
    O = Restatement()
    ref = phi.copy()
    for _ in range(STEPS):
        ref, st, _ = O.sl_step(g, ref, dfield, active, cfg, 0.8)
        assert st == 0
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    assert np.array_equal(bits(got), bits(ref))
    cuts = np.load(tmp_path / "cuts.npy")
    nxy = N * N
    k = active // nxy
    counts = [np.count_nonzero((k >= cuts[r]) & (k < cuts[r + 1])) for r in range(world)]
    assert abs(counts[0] - counts[1]) <= 0.25 * max(counts)  # band-balanced


def test_plan_cuts_balance_and_thickness():
    from paper_2410_22205_b200 import zslab

    _, phi, _, active, _ = _inputs()
    for world in (2, 3, 4):
        cuts = zslab.plan_cuts(active, N * N, N, world, min_planes=3)
        assert cuts[0] == 0 and cuts[-1] == N and np.all(np.diff(cuts) >= 3)
    with pytest.raises(ValueError):
        zslab.plan_cuts(active, N * N, N, 20, min_planes=5)


def test_plan_cuts_edge_cases_and_ownership():
    """Empty bands, a band in one plane, and 8 ranks: the cuts tile [0, nz)
    with slabs of at least min_planes, every active id is owned by exactly
    one rank, and the resident planes of a slab cover its owned planes plus
    the halo (clipped to the grid)."""
    from paper_2410_22205_b200 import zslab

    nxy, nz = 16 * 16, 64
    rng = np.random.default_rng(3)
    cases = [np.zeros(0, np.int64),
             np.sort(rng.choice(nxy, 50, replace=False)).astype(np.int64) + 30 * nxy,
             np.sort(rng.choice(nxy * nz, 5000, replace=False)).astype(np.int64)]
    for active in cases:
        for world in (1, 2, 8):
            cuts = zslab.plan_cuts(active, nxy, nz, world, min_planes=4)
            assert cuts[0] == 0 and cuts[-1] == nz and np.all(np.diff(cuts) >= 4)
            owned = [zslab.owned_ids(active, zslab.make_slab(cuts, r, 4, nxy, nz)) for r in range(world)]
            allown = np.concatenate(owned) if owned else np.zeros(0, np.int64)
            assert np.array_equal(np.sort(allown), active)
            for r in range(world):
                sl = zslab.make_slab(cuts, r, 4, nxy, nz)
                assert sl.lo == cuts[r] and sl.hi == cuts[r + 1]
                assert sl.z_base == max(0, sl.lo - 4) and sl.z_base + sl.z_planes == min(nz, sl.hi + 4)
                assert np.all((owned[r] // nxy >= sl.lo) & (owned[r] // nxy < sl.hi))


@pytest.mark.gpu
def test_fused_peer_push_two_slabs_one_gpu(gpu):
    """The fused SL + halo-push kernel, two slabs emulated on one GPU: the
    'peer' pointers are the other slab's buffers, the slabs' kernels run one
    after the other (neither waits on the other). K steps must reproduce the
    whole-grid evolution bit for bit with no plane exchange at all."""
    import ctypes as C

    import torch

    lsr = gpu
    from paper_2410_22205_b200 import zslab

    _, phi, dfield, active, cfgd = _inputs()
    g = lsr._api.cube_grid(N, 3)
    bp = lsr.BandParams(cfgd["gamma"], cfgd["beta"])
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=cfgd["dt"], band=bp)
    nxy = N * N
    halo = 5
    K = 4
    # whole grid, K ping-pong steps on the same band
    ctx = lsr.Context(g)
    ctx.upload(0, phi)
    ctx.upload(1, dfield)
    ctx.set_active(active)
    for _ in range(K):
        ctx.sl_step(cfg, 0.8)
        ctx.swap()
    whole = ctx.download(0)

    cuts = zslab.plan_cuts(active, nxy, N, 2, min_planes=halo)
    slabs = [zslab.make_slab(cuts, r, halo, nxy, N) for r in range(2)]
    bufs, dbuf, ids, miss, bad = [], [], [], [], []
    for s in slabs:
        sl = slice(s.z_base * nxy, (s.z_base + s.z_planes) * nxy)
        t = torch.from_numpy(phi[sl].copy()).cuda()
        bufs.append((t, t.clone()))
        dbuf.append(torch.from_numpy(dfield[sl].copy()).cuda())
        ids.append(torch.from_numpy(zslab.owned_ids(active, s)).cuda())
        miss.append(torch.zeros(1, dtype=torch.int64, device="cuda"))
        bad.append(torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda"))
    L = lsr.lib()
    cg, cc = g.c(), cfg.c()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def make_compute(r):
        def compute(src, dst, lo, hi, s, push):
            st = L.lsr_cuda_sl_step_device_fused(
                C.byref(cg), s.z_base, s.z_planes, s.lo, s.hi, C.c_void_p(src.data_ptr()),
                C.c_void_p(dbuf[r].data_ptr()), C.c_void_p(ids[r].data_ptr()), ids[r].numel(), C.byref(cc), 0.8,
                C.c_void_p(dst.data_ptr()), C.c_void_p(lo[0].data_ptr() if lo[0] is not None else None), lo[1],
                push if lo[0] is not None else 0, C.c_void_p(hi[0].data_ptr() if hi[0] is not None else None), hi[1],
                push if hi[0] is not None else 0, C.c_void_p(bad[r].data_ptr()), C.c_void_p(miss[r].data_ptr()),
                stream)
            assert st == 0, L.lsr_cuda_last_error_string()
        return compute

    steppers = [
        zslab.FusedSlabStepper(slabs[0], halo, bufs[0], None, (bufs[1], slabs[1].z_base), make_compute(0)),
        zslab.FusedSlabStepper(slabs[1], halo, bufs[1], (bufs[0], slabs[0].z_base), None, make_compute(1)),
    ]
    for _ in range(K):
        for st in steppers:
            st.step()
    torch.cuda.synchronize()
    assert int(miss[0].item()) == 0 and int(miss[1].item()) == 0
    got = np.empty_like(phi)
    for st, s in zip(steppers, slabs):
        cur = st.current.cpu().numpy()
        got[s.lo * nxy:s.hi * nxy] = cur[(s.lo - s.z_base) * nxy:(s.hi - s.z_base) * nxy]
    # planes outside every slab's ownership do not exist (cuts cover [0, N))
    assert np.array_equal(bits(got), bits(whole))
    # the buffers can be exported for peer mapping (CUDA IPC)
    h = C.create_string_buffer(64)
    p = C.c_void_p()
    assert L.lsr_cuda_malloc(1 << 20, C.byref(p)) == 0
    assert L.lsr_cuda_ipc_handle(p, h) == 0 and any(h.raw)
    assert L.lsr_cuda_free(p) == 0


@pytest.mark.gpu
def test_slab_kernel_matches_whole_grid_and_counts_misses(gpu):
    """Two slabs computed one after the other on one GPU (no kernel waits on
    another) reproduce the whole-grid step; a too-thin halo is reported."""
    import ctypes as C

    import torch

    lsr = gpu
    from paper_2410_22205_b200 import zslab

    g0, phi, dfield, active, cfgd = _inputs()
    g = lsr._api.cube_grid(N, 3)
    bp = lsr.BandParams(cfgd["gamma"], cfgd["beta"])
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=cfgd["dt"], band=bp)
    whole = lsr.ScalarField(g)
    lsr.sl_step(lsr.ScalarField(g, phi), lsr.DistanceField(lsr.ScalarField(g, dfield)), lsr.BandMask(g, active=active),
                cfg, 0.8, whole)
    nxy = N * N
    L = lsr.lib()
    for halo, expect_miss in ((5, False), (1, True)):
        cuts = zslab.plan_cuts(active, nxy, N, 2, min_planes=halo)
        got = phi.copy()
        misses = 0
        for rank in range(2):
            s = zslab.make_slab(cuts, rank, halo, nxy, N)
            sl = slice(s.z_base * nxy, (s.z_base + s.z_planes) * nxy)
            ids = torch.from_numpy(zslab.owned_ids(active, s)).cuda()
            p = torch.from_numpy(phi[sl].copy()).cuda()
            d = torch.from_numpy(dfield[sl].copy()).cuda()
            o = p.clone()
            bad = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
            miss = torch.zeros(1, dtype=torch.int64, device="cuda")
            st = L.lsr_cuda_sl_step_device(C.byref(g.c()), s.z_base, s.z_planes, C.c_void_p(p.data_ptr()),
                                           C.c_void_p(d.data_ptr()), C.c_void_p(ids.data_ptr()), ids.numel(),
                                           C.byref(cfg.c()), 0.8, C.c_void_p(o.data_ptr()), C.c_void_p(bad.data_ptr()),
                                           C.c_void_p(miss.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert st == 0, lsr.lib().lsr_cuda_last_error_string()
            torch.cuda.synchronize()
            misses += int(miss.item())
            own = slice(s.lo * nxy, s.hi * nxy)
            got[own] = o.cpu().numpy()[(s.lo - s.z_base) * nxy:(s.hi - s.z_base) * nxy]
        if expect_miss:
            assert misses > 0
        else:
            assert misses == 0
            assert np.array_equal(bits(got), bits(whole.values))


# ---------------------------------------------------------------------------
# The whole-loop driver (zslab.SlabLoop): blocked_sum from the ranks' pieces,
# and the rank protocol over gloo with a numpy stand-in for the slab context
# (the bit-exactness of the real phases against the single-GPU loop is
# test_zslab_loop_gpu.py).

def _pieces(vals, offset):
    """This rank's blocked_sum pieces as lsr_cuda_slab_energy_pieces forms them."""
    s0 = (4096 - offset % 4096) % 4096
    head = vals[:min(s0, vals.size)]
    full = (vals.size - s0) // 4096 if vals.size > s0 else 0
    blocks = [0.0] * full
    for b in range(full):
        acc = 0.0
        for v in vals[s0 + 4096 * b:s0 + 4096 * (b + 1)]:
            acc += float(v)
        blocks[b] = acc
    return np.array(blocks), head, vals[s0 + 4096 * full:] if vals.size > s0 else vals[:0]


def _blocked_sum(vals):  # parallel.hpp:26-42
    total = 0.0
    for b in range(0, vals.size, 4096):
        acc = 0.0
        for v in vals[b:b + 4096]:
            acc += float(v)
        total += acc
    return total


@pytest.mark.parametrize("sizes", [[0], [5], [4096], [9000, 0, 3, 12000], [100, 100, 100], [4095, 1, 8193, 4096]])
def test_blocked_sum_from_rank_pieces(sizes):
    from paper_2410_22205_b200 import zslab

    rng = np.random.default_rng(len(sizes) + sum(sizes))
    allv = rng.standard_normal(sum(sizes)) * np.exp(rng.uniform(-20, 20, sum(sizes)))
    pieces, off = [], 0
    for n in sizes:
        pieces.append(_pieces(allv[off:off + n], off))
        off += n
    assert zslab.blocked_sum_pieces(pieces) == _blocked_sum(allv)


class _MockSlab:
    """numpy stand-in for SlabContext with z-coupled toy phases: every phase
    reads the planes next to the owned ones, so a wrong or missing halo
    exchange changes the result."""

    def __init__(self, nxy, nz, wl, wh, ol, oh):
        import types

        self.grid = types.SimpleNamespace(dims=(nxy, 1, nz), dx=0.1)
        self.nxy, self.win_lo, self.win_hi, self.own_lo, self.own_hi = nxy, wl, wh, ol, oh
        self.f = {k: np.zeros((wh - wl) * nxy) for k in (0, 1, 2, 3)}

    def _pl(self, f, k):
        k = min(max(k, 0), self.grid.dims[2] - 1)
        return self.f[f][(k - self.win_lo) * self.nxy:(k - self.win_lo + 1) * self.nxy]

    def upload(self, which, v):
        self.f[which][:] = v

    def close(self):
        pass

    def plane_ptr(self, which, plane):
        return self.f[which].ctypes.data + 8 * (plane - self.win_lo) * self.nxy

    def copy_planes(self, which, p0, n, ptr, to_field):
        import ctypes

        a = self.plane_ptr(which, p0)
        if to_field:
            ctypes.memmove(a, ptr, 8 * n * self.nxy)
        else:
            ctypes.memmove(ptr, a, 8 * n * self.nxy)

    def _owned(self, f):
        return self.f[f][(self.own_lo - self.win_lo) * self.nxy:(self.own_hi - self.win_lo) * self.nxy]

    def _stencil(self, src, dst, a, b):
        for k in range(self.own_lo, self.own_hi):
            self._pl(dst, k)[:] = a * self._pl(src, k) + b * (self._pl(src, k - 1) + self._pl(src, k + 1))

    def band(self, gamma, which=0):
        na = int(np.count_nonzero(np.abs(self._owned(which)) < gamma))
        return na, na + 1

    def energy_cells(self, which=0, p=2, refine=5):
        self._contrib = np.abs(self._owned(which))
        self.n_cells = self._contrib.size
        return self.n_cells

    def energy_pieces(self, offset):
        return _pieces(self._contrib, offset)

    def max_reach(self, cfg, e2):
        return 0.5

    def sl_step(self, cfg, e2):
        self.f[2][:] = self.f[0]
        self._stencil(0, 2, 0.5 + 0.01 * e2, 0.25)
        return 0

    def one_step(self):
        self._stencil(2, 3, 0.9, 0.05)
        return True, False

    def reinit_begin(self, rcfg):
        self.f[2][:] = self.f[3]
        return 1

    def reinit_sweep(self, rcfg, k):
        cur, nxt = (3, 2) if k % 2 == 0 else (2, 3)
        self._stencil(cur, nxt, 0.5, 0.25)
        return float(np.max(np.abs(self._owned(nxt) - self._owned(cur))))

    def reinit_end(self, which, gamma):
        if which == 3:
            self.f[2], self.f[3] = self.f[3], self.f[2]
        o = self._owned(2)
        o[:] = np.minimum(np.maximum(o, -gamma), gamma)

    def swap(self):
        self.f[0], self.f[2] = self.f[2], self.f[0]


_LOOP_NZ, _LOOP_NXY, _LOOP_ITERS = 24, 6, 3


def _loop_cfg():
    import types

    cfg = types.SimpleNamespace(p=2, interp=1)
    rcfg = types.SimpleNamespace(max_iters=9, residual_tol=1e-3)
    phi = np.sin(np.arange(_LOOP_NZ * _LOOP_NXY) * 0.37) * 0.8
    return cfg, rcfg, phi


def _run_mock_loop(runner_factory, ranks, cuts, halo):
    from paper_2410_22205_b200 import zslab

    cfg, rcfg, phi = _loop_cfg()
    nxy = _LOOP_NXY

    def make(wl, wh, ol, oh):
        return _MockSlab(nxy, _LOOP_NZ, wl, wh, ol, oh)

    loop = zslab.SlabLoop(types_grid(), cuts, ranks, halo, make, lambda c: None, runner_factory)
    loop.upload_phi(lambda c: phi[c.win_lo * nxy:c.win_hi * nxy])
    stats = [loop.step(cfg, rcfg, 0.7) for _ in range(_LOOP_ITERS)]
    owned = [c._owned(0).copy() for c in loop.ctxs]
    return stats, owned


def types_grid():
    import types

    return types.SimpleNamespace(dims=(_LOOP_NXY, 1, _LOOP_NZ), dx=0.1)


def _loop_worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2410_22205_b200 import zslab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cuts = [0, 10, _LOOP_NZ] if world == 2 else [0, 8, 16, _LOOP_NZ]
    stats, owned = _run_mock_loop(lambda ctxs: zslab.DistRunner(dist, ctxs[0], cuts), [rank], cuts, 3)
    np.save(os.path.join(outdir, f"loop{rank}.npy"), owned[0])
    np.save(os.path.join(outdir, f"stats{rank}.npy"), np.array([[s[0]["energy"], s[0]["reinit_iterations"],
                                                                 s[0]["n_active"]] for s in stats]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_loop_protocol_gloo_matches_one_rank(tmp_path, world):
    """SlabLoop over torch.distributed (gloo, world 2 and 3, DistRunner) gives
    the one-rank loop's fields and statistics; so does the in-process runner."""
    import torch.multiprocessing as mp

    from paper_2410_22205_b200 import zslab

    ref_stats, ref_owned = _run_mock_loop(zslab.InProcessRunner, [0], [0, _LOOP_NZ], 3)
    mp.spawn(_loop_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"loop{r}.npy") for r in range(world)])
    assert np.array_equal(bits(got), bits(ref_owned[0]))
    for r in range(world):
        st = np.load(tmp_path / f"stats{r}.npy")
        assert np.array_equal(st[:, :2], np.array([[s[0]["energy"], s[0]["reinit_iterations"]] for s in ref_stats]))
    cuts = [0, 10, _LOOP_NZ] if world == 2 else [0, 8, 16, _LOOP_NZ]
    in_stats, in_owned = _run_mock_loop(zslab.InProcessRunner, list(range(world)), cuts, 3)
    assert np.array_equal(bits(np.concatenate(in_owned)), bits(ref_owned[0]))


@pytest.mark.parametrize("win,own", [((0, 20), (10, 30)),   # owned beyond the window
                                     ((5, 40), (5, 20)),    # window must start at own_lo - 1
                                     ((0, 20), (0, 20)),    # window must end at own_hi + 1
                                     ((0, 40), (20, 20)),   # empty ownership
                                     ((-1, 40), (0, 10))])
def test_slab_create_rejects_bad_windows_before_device_work(built, win, own):
    import paper_2410_22205_b200 as lsr

    g = lsr._api.cube_grid(N, 3)
    with pytest.raises(lsr.ConfigError):
        lsr.SlabContext(g, win[0], win[1], own[0], own[1])


def test_slab_create_needs_3d_and_aligned_planes(built):
    import paper_2410_22205_b200 as lsr

    with pytest.raises(lsr.ConfigError):
        lsr.SlabContext(lsr._api.cube_grid(16, 2), 0, 1, 0, 1)
    g = lsr.Grid(3, (-1.0, -1.0, -1.0), 0.1, (9, 7, 20))  # 63 nodes per plane
    with pytest.raises(lsr.ConfigError, match="multiple of 16"):
        lsr.SlabContext(g, 0, 11, 0, 10)


@pytest.mark.gpu
def test_whole_grid_entry_points_reject_slab_contexts(gpu):
    import ctypes as C

    lsr = gpu
    g = lsr._api.cube_grid(32, 3)
    c = lsr.SlabContext(g, 0, 17, 0, 16)
    L = lsr.lib()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1 * g.dx, band=lsr.default_band_params(3, g.dx))
    bad = C.c_int64(-1)
    assert L.lsr_cuda_sl_step(c.h, C.byref(cfg.c()), 1.0, C.byref(bad)) == 1  # LSR_ERR_CONFIG
    assert b"slab" in L.lsr_cuda_last_error_string()
    na, nt = C.c_int64(), C.c_int64()
    assert L.lsr_cuda_narrow_band(c.h, 0, 0.1, C.byref(na), C.byref(nt)) == 1
    c.close()
