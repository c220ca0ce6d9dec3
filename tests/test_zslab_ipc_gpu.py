"""The fused SL + halo-push step across two PROCESSES on one GPU (SURVEY
§8(e) phase 2): each rank maps its neighbour's resident buffers through CUDA
IPC handles (lsr_cuda_ipc_handle / lsr_cuda_ipc_open, exchanged over gloo)
and its SL kernel's epilogue stores the updates of its boundary planes
straight into them. Ranks are ordered by host barriers between steps only —
no kernel waits on another process. K steps must reproduce the whole-grid
evolution bit for bit."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

K = 4
HALO = 5


def _worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2410_22205_b200 as lsr
    from paper_2410_22205_b200 import zslab
    from test_zslab import N, _inputs

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, phi, dfield, active, cfgd = _inputs()
    g = lsr._api.cube_grid(N, 3)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=cfgd["dt"], band=lsr.BandParams(cfgd["gamma"], cfgd["beta"]))
    nxy = N * N
    cuts = zslab.plan_cuts(active, nxy, N, world, min_planes=HALO)
    s = zslab.make_slab(cuts, rank, HALO, nxy, N)
    L = lsr.lib()

    def raw(n):  # whole cudaMalloc allocations: what CUDA IPC exports
        p = C.c_void_p()
        assert L.lsr_cuda_malloc(8 * n, C.byref(p)) == 0
        return p.value

    class _View:  # a torch view of a raw allocation
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    sl = slice(s.z_base * nxy, (s.z_base + s.z_planes) * nxy)
    bufs = [raw(s.n_resident), raw(s.n_resident)]
    views = [torch.as_tensor(_View(b, s.n_resident), device="cuda") for b in bufs]
    for v in views:
        v.copy_(torch.from_numpy(np.ascontiguousarray(phi[sl])))
    torch.cuda.synchronize()
    d_t = torch.from_numpy(dfield[sl].copy()).cuda()
    ids = torch.from_numpy(zslab.owned_ids(active, s)).cuda()
    miss = torch.zeros(1, dtype=torch.int64, device="cuda")
    bad = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    handles = []
    for b in bufs:
        h = C.create_string_buffer(64)
        assert L.lsr_cuda_ipc_handle(C.c_void_p(b), h) == 0
        handles.append(h.raw)
    info = [None] * world
    dist.all_gather_object(info, {"handles": handles, "z_base": s.z_base})

    def peer(r):
        ptrs = []
        for hb in info[r]["handles"]:
            p = C.c_void_p()
            assert L.lsr_cuda_ipc_open(hb, C.byref(p)) == 0, L.lsr_cuda_last_error_string()
            ptrs.append(p.value)
        return ptrs, info[r]["z_base"]

    lo = peer(rank - 1) if rank > 0 else None
    hi = peer(rank + 1) if rank < world - 1 else None
    cg, cc = g.c(), cfg.c()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for n in range(K):
        src, dst = bufs[n % 2], bufs[(n + 1) % 2]
        lo_p = lo[0][(n + 1) % 2] if lo else None
        hi_p = hi[0][(n + 1) % 2] if hi else None
        st = L.lsr_cuda_sl_step_device_fused(
            C.byref(cg), s.z_base, s.z_planes, s.lo, s.hi, C.c_void_p(src), C.c_void_p(d_t.data_ptr()),
            C.c_void_p(ids.data_ptr()), ids.numel(), C.byref(cc), 0.8, C.c_void_p(dst), C.c_void_p(lo_p),
            lo[1] if lo else 0, HALO if lo else 0, C.c_void_p(hi_p), hi[1] if hi else 0, HALO if hi else 0,
            C.c_void_p(bad.data_ptr()), C.c_void_p(miss.data_ptr()), stream)
        assert st == 0, L.lsr_cuda_last_error_string()
        torch.cuda.synchronize()
        dist.barrier()  # the neighbours' pushes into our buffer have landed
    out = views[K % 2].cpu().numpy()
    np.save(os.path.join(outdir, f"r{rank}.npy"), out[(s.lo - s.z_base) * nxy:(s.hi - s.z_base) * nxy])
    np.save(os.path.join(outdir, f"m{rank}.npy"), np.array([int(miss.item()), int(bad.item())]))
    dist.barrier()
    for p in (lo, hi):
        if p:
            for q in p[0]:
                L.lsr_cuda_ipc_close(C.c_void_p(q))
    dist.destroy_process_group()


def test_fused_push_two_processes_cuda_ipc(gpu, tmp_path):
    import socket

    import torch.multiprocessing as mp

    from test_zslab import N, _inputs

    lsr = gpu
    _, phi, dfield, active, cfgd = _inputs()
    g = lsr._api.cube_grid(N, 3)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=cfgd["dt"], band=lsr.BandParams(cfgd["gamma"], cfgd["beta"]))
    ctx = lsr.Context(g)
    ctx.upload(0, phi)
    ctx.upload(1, dfield)
    ctx.set_active(active)
    for _ in range(K):
        ctx.sl_step(cfg, 0.8)
        ctx.swap()
    whole = ctx.download(0)
    ctx.close()

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    pc = mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=False)
    import time

    t0 = time.time()
    while not pc.join(timeout=5):
        if time.time() - t0 > 180:
            for p in pc.processes:
                p.kill()
            pytest.fail("two-process fused push timed out")
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(2)])
    for r in range(2):
        m = np.load(tmp_path / f"m{r}.npy")
        assert m[0] == 0 and m[1] == np.iinfo(np.int64).max, m
    assert np.array_equal(bits(got), bits(whole))
