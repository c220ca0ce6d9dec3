"""Kernel-only microbenchmark of the SL step at 512^3 on analytic inputs
(phi = |x| - 0.9, d = ||x| - 0.5| + ripple). Development aid; the contract
benchmark is bench.py."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_22205_b200 as lsr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--interp", type=int, default=1)
    ap.add_argument("--radius", type=float, default=0.9)
    ap.add_argument("--delta", type=float, default=1.0)
    ap.add_argument("--zslab", type=int, nargs=2, default=None, help="only band nodes with k in [lo, hi)")
    ap.add_argument("--order", default="id", help="thread order of the active ids: id or bXYZ (brick extents)")
    ap.add_argument("--mode", type=int, default=0, help="3d WENO step form: 0 z-line table, 1 TMA bricks")
    a = ap.parse_args()
    g = lsr._api.cube_grid(a.n, 3)
    ax = g.axes()
    r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2).ravel()
    phi = r - a.radius
    dist = np.abs(r - 0.5) + 1e-3 * np.cos(40 * r)
    bp = lsr.default_band_params(3, g.dx)
    band = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    if a.zslab:
        kk = band // (a.n * a.n)
        band = band[(kk >= a.zslab[0]) & (kk < a.zslab[1])]
    if a.order != "id":  # process the ids brick by brick (the step does not depend on the order)
        bx, by, bz = (int(c) for c in a.order[1:4])
        i, j, k = band % a.n, (band // a.n) % a.n, band // (a.n * a.n)
        key = (((k // bz) * (a.n // by + 1) + j // by) * (a.n // bx + 1) + i // bx)
        band = band[np.lexsort((band, key))]
    cfg = lsr.StepConfig(p=2, delta=a.delta, dt=0.25 * g.dx, band=bp, interp=lsr.InterpolatorKind(a.interp))
    ctx = lsr.Context(g)
    ctx.set_sl_mode(a.mode)
    ctx.upload(0, phi)
    ctx.upload(1, dist)
    ctx.set_active(band)
    ks, ss = [], []
    for s in range(a.steps + 3):
        ctx.sl_step(cfg, 1.3)
        k, st = ctx.last_times()
        if s >= 3:
            ks.append(k)
            ss.append(st)
    kmed = float(np.median(ks))
    print(json.dumps(dict(n=a.n, interp=a.interp, mode=a.mode, active=int(band.size), kernel_ms=kmed, step_ms=float(np.median(ss)),
                          node_updates_per_s=band.size / (kmed * 1e-3),
                          kernel_ms_all=[round(x, 4) for x in ks])))


if __name__ == "__main__":
    main()
