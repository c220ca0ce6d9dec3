"""Per-phase device times of the full loop body (band, E2, SL, reinit) at a
config size; development aid."""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_22205_b200 as lsr  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--steps", type=int, default=5)
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
print(json.dumps({"build_distance_s": tdist}))
