"""The slab loop across PROCESSES (zslab.DistRunner over torch.distributed):
two ranks, each its own process with a SlabContext on cuda:0 (one GPU here;
the halo planes travel through host staging over gloo, ranks meet only at
the collectives — no kernel waits on the other process). After each of 3
iterations phi on the owned planes, E_2, |active| and the sweep count must
equal the single-GPU loop's (the same code as bench.py --gpus N runs over
NCCL)."""
import os
import sys

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

DIMS = (64, 64, 64)
ITERS = 3


def _setup(lsr):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_zslab_loop_gpu import _case

    g, phi0, dist = _case(lsr, DIMS)
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=bp, interp=lsr.InterpolatorKind(1))
    rcfg = lsr.ReinitConfig.defaults(g.dx, bp.gamma)
    return g, phi0, dist, cfg, rcfg


def _worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2410_22205_b200 as lsr
    from paper_2410_22205_b200 import zslab

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, phi0, dist_f, cfg, rcfg = _setup(lsr)
    nxy, nz = g.dims[0] * g.dims[1], g.dims[2]
    cuts = [int(c) for c in zslab.plan_cuts(np.flatnonzero(np.abs(phi0) < cfg.band.gamma), nxy, nz, world,
                                            min_planes=8)]
    loop = zslab.SlabLoop(g, cuts, [rank], 6, lambda wl, wh, ol, oh: lsr.SlabContext(g, wl, wh, ol, oh),
                          lambda c: c.upload(1, dist_f[c.win_lo * nxy:c.win_hi * nxy]),
                          lambda ctxs: zslab.DistRunner(dist, ctxs[0], cuts))
    loop.upload_phi(lambda c: phi0[c.win_lo * nxy:c.win_hi * nxy])
    stats = []
    for it in range(ITERS):
        st = loop.step(cfg, rcfg, cfg.band.gamma)[0]
        c = loop.ctxs[0]
        w = c.download(0)
        np.save(os.path.join(outdir, f"phi{rank}_{it}.npy"), w[(c.own_lo - c.win_lo) * nxy:(c.own_hi - c.win_lo) * nxy])
        stats.append([st["energy"], st["n_active"], st["reinit_iterations"]])
    np.save(os.path.join(outdir, f"stats{rank}.npy"), np.array(stats))
    dist.barrier()
    for c in loop.ctxs:
        c.close()
    dist.destroy_process_group()


def test_slab_loop_two_processes_gloo(gpu, tmp_path):
    import socket
    import time

    import torch.multiprocessing as mp

    lsr = gpu
    g, phi0, dist_f, cfg, rcfg = _setup(lsr)
    ctx = lsr.Context(g)
    ctx.upload(0, phi0)
    ctx.upload(1, dist_f)
    ref_fields, ref_stats = [], []
    for _ in range(ITERS):
        s = ctx.loop_step(cfg, rcfg, 5)
        ref_stats.append(s)
        ref_fields.append(ctx.download(0).copy())
    ctx.close()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    pc = mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=False)
    t0 = time.time()
    while not pc.join(timeout=5):
        if time.time() - t0 > 300:
            for p in pc.processes:
                p.kill()
            pytest.fail("two-process slab loop timed out")
    st = [np.load(tmp_path / f"stats{r}.npy") for r in range(2)]
    for it in range(ITERS):
        got = np.concatenate([np.load(tmp_path / f"phi{r}_{it}.npy") for r in range(2)])
        assert np.count_nonzero(bits(got) != bits(ref_fields[it])) == 0, f"iteration {it + 1}"
        assert st[0][it][0] == st[1][it][0] == ref_stats[it]["energy"]
        assert st[0][it][1] + st[1][it][1] == ref_stats[it]["n_active"]
        assert st[0][it][2] == st[1][it][2] == ref_stats[it]["reinit_iterations"]
