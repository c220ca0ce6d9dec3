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
