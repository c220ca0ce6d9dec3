import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
os.environ["LSR_PIPE_TRACE"] = "1"
import numpy as np
import paper_2410_22205_b200 as lsr
from test_sl_step_gpu import _run
from conftest import bits
from oracle.bindings import Restatement
oracle = Restatement()
for case in ["sorted", "scattered", "edge_planes"]:
  for pinned in [False, True]:
    rng = np.random.default_rng(5)
    g = lsr._api.cube_grid(96, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.6 + 0.2 * g.dx * rng.standard_normal(x.size)
    dist = np.abs(np.sqrt(x * x + y * y + z * z) - 0.3) + 0.01 * rng.random(x.size)
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    if case == "scattered":
        active = np.sort(rng.choice(active, active.size // 9, replace=False)).astype(np.int64)
    if case == "edge_planes":
        n = g.dims[0]
        kk, jj, ii = np.unravel_index(np.arange(x.size), (n, n, n))
        face = (ii == 0) | (jj == 0) | (kk == 0) | (ii == n - 1) | (jj == n - 1) | (kk == n - 1)
        active = np.union1d(active, np.flatnonzero(face & (rng.random(x.size) < 0.3))).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=bp)
    got = _run(lsr, g, phi, dist, active, cfg, 0.7, pinned)
    print(case, pinned, lsr._api.last_transfer_bytes(), flush=True)
    ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=bp.gamma, beta=bp.beta), 0.7)
    print("  mismatches", np.count_nonzero(bits(got) != bits(ref)), flush=True)
