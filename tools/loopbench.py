"""Per-phase device times of the full loop body (band, E2, SL, reinit) at a
config size; development aid. --run K: also time K iterations of the
device-controlled loop (lsr_cuda_loop_run, one host sync, graph replays)."""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_22205_b200 as lsr  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--run", type=int, default=0)
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
g, w, step = bench.make_inputs(lsr, cfg)
pts, phi = w["pts"], w["phi"]
ctx = lsr.Context(g)
t0 = time.perf_counter(); ctx.build_distance(pts); tdist = time.perf_counter() - t0
ctx.upload(0, phi)
rc = lsr.ReinitConfig.defaults(g.dx, step.band.gamma)
for s in range(a.steps):
    t0 = time.perf_counter()
    st = ctx.loop_step(step, rc, 5)
    st["wall_ms"] = 1e3 * (time.perf_counter() - t0)
    print(json.dumps(st))
if a.run:
    for rep in range(2):
        t0 = time.perf_counter()
        recs = ctx.loop_run(step, rc, a.run, 5, use_graph=not a.no_graph)
        wall = 1e3 * (time.perf_counter() - t0)
        ms = np.array([r["ms"] for r in recs])
        print(json.dumps({"loop_run": a.run, "graph": not a.no_graph, "wall_ms_per_iter": wall / a.run,
                          "device_ms_per_iter": float(ms[1:].sum(axis=1).mean()) if a.run > 1 else float(ms.sum()),
                          "phase_ms": [float(x) for x in ms[1:].mean(axis=0)] if a.run > 1 else ms[0].tolist(),
                          "iters": [r["reinit_iterations"] for r in recs][:8],
                          "n_active": recs[-1]["n_active"]}))
print(json.dumps({"build_distance_s": tdist}))
