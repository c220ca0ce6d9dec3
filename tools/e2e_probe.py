"""Where the one-shot host entry's time goes at 512^3: PCIe bandwidth of the
box (H2D, D2H, both at once), host threads, and the pipelined call itself
with LSR_PIPE_TRACE timings. Usage: python tools/e2e_probe.py [--n 512]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LSR_PIPE_TRACE", "1")
import paper_2410_22205_b200 as lsr  # noqa: E402


def bw(label, fn, nbytes, reps=5):
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{label:28s} {dt * 1e3:8.2f} ms  {nbytes / dt / 1e9:7.1f} GB/s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    a = ap.parse_args()
    print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
    n = a.n
    N = n ** 3
    h = torch.empty(N, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(N, dtype=torch.float64, pin_memory=True)
    d = torch.empty(N, dtype=torch.float64, device="cuda")
    d2 = torch.empty(N, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    B = 8 * N
    bw("H2D", lambda: d.copy_(h, non_blocking=True), B)
    bw("D2H", lambda: h2.copy_(d2, non_blocking=True), B)

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    bw("H2D || D2H (each)", both, B)
    g = lsr.cube_grid(n, 3)
    ax = g.axes()
    r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2).reshape(-1)
    phi = h.numpy()
    phi[:] = r - 0.9
    bp = lsr.default_band_params(3, g.dx)
    act = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    active = torch.empty(act.size, dtype=torch.int64, pin_memory=True).numpy()
    active[:] = act
    dist = h2.numpy()
    dist[:] = np.abs(r - 0.5)
    field = np.empty(N)
    t0 = time.perf_counter()
    nv, nr, pv, pr = lsr._api.pack_host(lsr.DistanceField(lsr.ScalarField(g, dist)), active, field, 5, phi, np.empty(N))
    print(f"pack_distance_host (plan+gather+host scatter) {1e3 * (time.perf_counter() - t0):.1f} ms, "
          f"d {nv} values {nr} runs, phi {pv} values {pr} runs, active {active.size}")
    out = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
    from concurrent.futures import ThreadPoolExecutor

    for T in (1, 4, 8, 16):
        with ThreadPoolExecutor(T) as ex:
            parts = np.array_split(np.arange(N), T)
            list(ex.map(lambda p: np.copyto(out[p[0]:p[-1] + 1], phi[p[0]:p[-1] + 1]), parts))
            t0 = time.perf_counter()
            list(ex.map(lambda p: np.copyto(out[p[0]:p[-1] + 1], phi[p[0]:p[-1] + 1]), parts))
            dt = time.perf_counter() - t0
        print(f"host memcpy {T:2d} threads {dt * 1e3:7.2f} ms {B / dt / 1e9:6.1f} GB/s", flush=True)
    step = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=bp)
    sphi, sd = lsr.ScalarField(g, phi), lsr.DistanceField(lsr.ScalarField(g, dist))
    mask, so = lsr.BandMask(g, active=active), lsr.ScalarField(g, out)
    for _ in range(6):
        t0 = time.perf_counter()
        lsr.sl_step(sphi, sd, mask, step, 1.6, so)
        print(f"sl_step one-shot {1e3 * (time.perf_counter() - t0):.2f} ms  bytes {lsr._api.last_transfer_bytes()}",
              flush=True)


if __name__ == "__main__":
    main()
