"""bench.py — SL narrow-band node-updates/s (WENO, 512^3, fp64) on B200.

Workload (BASELINE.json config 4, the headline): bumpy sphere
r(t,p) = 0.5(1 + 0.1 sin 5t cos 4p), 1,000,000 seeded points, 10x denser at
the poles; grid 512^3 on [-1,1]^3 (dx = 2/511); d = lsr::build_distance_field
of the cloud (computed on the GPU, bit-identical to the reference's);
phi^0 = |x| - 0.9; band = |phi| < gamma = 6dx; E_2 = lsr::surface_energy
(GPU); p = 2, delta = 1 (Table 1 run r >= 3), WENO, dt = dx/4. `--config N`
runs BASELINE config N (1: 257^2 circle, Q1; 2: 128^3 sphere, Q1; 3: 256^3
torus, WENO; 5: 1024^3 three tori, WENO) with the same recipe.

One step = one lsr::sl_step over the whole band (resync of the double
buffer + the z-line table fill + the SL kernel), inputs resident in HBM;
successive steps ping-pong phi <-> out on the same band. L2 (126 MB) is
flushed by a 256 MB write between timed steps. Units = active node-updates.
`moving_band` reports the same metric inside the real loop, where the band
is rebuilt every iteration (so the covered-brick list is rebuilt too).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

N > 1: one rank per GPU (bench.py relaunches itself under torch.distributed.run
when WORLD_SIZE is unset); z-slab decomposition — each rank owns a
band-balanced range of z-planes, updates only its active nodes, and the halo
planes reach the neighbours through the fused peer push (or NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "node-updates/s"
BYTES_PER_UPDATE = {("weno", 3): 2176, ("q1", 3): 384, ("weno", 2): 352, ("q1", 2): 160}
COMPULSORY_BYTES = 32  # phi_j, d_j, out, id (SURVEY §8(d) "A")
SEED = 2410

CONFIGS = {
    # id: grid nodes per axis, dim, cloud generator id, points, noise (in dx), interp (0 Q1, 1 WENO),
    #     phi^0 sphere radius, p, delta
    1: dict(n=257, dim=2, cloud=1, points=200, sigma=0.0, interp=0, r0=0.9, p=1, delta=0.0,
            name="circle-257", shape="circle cloud"),
    2: dict(n=128, dim=3, cloud=2, points=20_000, sigma=0.0, interp=0, r0=0.9, p=2, delta=1.0,
            name="sphere-128", shape="sphere cloud"),
    3: dict(n=256, dim=3, cloud=3, points=100_000, sigma=0.5, interp=1, r0=0.9, p=2, delta=1.0,
            name="torus-256", shape="noisy torus cloud"),
    4: dict(n=512, dim=3, cloud=4, points=1_000_000, sigma=0.0, interp=1, r0=0.9, p=2, delta=1.0,
            name="bumpy-sphere-512", shape="bumpy-sphere cloud"),
    5: dict(n=1024, dim=3, cloud=5, points=4_000_000, sigma=0.25, interp=1, r0=0.95, p=2, delta=1.0,
            name="three-tori-1024", shape="three-tori cloud with two holes"),
}


def metric_name(cfg) -> str:
    grid = f"{cfg['n']}^{cfg['dim']}"
    return f"SL narrow-band node-updates/s ({'WENO' if cfg['interp'] == 1 else 'Q1'}, {grid}, fp64)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _json(path):
    try:
        with open(os.path.join(ROOT, path)) as f:
            return json.load(f)
    except Exception:
        return None


def peaks():
    p = _json("MEASURED_PEAKS.json")
    if p and "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Measured DFMA thread-instruction rate of this B200 model
    (tools/fp64_peak.cu, profiles/fp64_peak.json)."""
    p = _json(os.path.join("profiles", "fp64_peak.json"))
    if p and p.get("dfma_per_s"):
        return float(p["dfma_per_s"]), p.get("source")
    return None, None


def traffic_per_update():
    """DRAM bytes and fp64 instructions per node-update of the SL kernel from
    the committed ncu capture (profiles/sl_step_traffic.json), or None."""
    t = _json(os.path.join("profiles", "sl_step_traffic.json"))
    if not t:
        return None, None
    return float(t["dram_bytes_per_update"]), t


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (host time of arrival, fields)
        self.proc = None
        self.t0 = self.t1 = None

    # the sampler is started before the warm-up (nvidia-smi takes ~0.1 s to
    # come up); only rows that arrive inside [begin, end] describe the timed
    # region
    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        time.sleep(0.03)  # one more sampling period covers the region's tail
        self.t1 = time.perf_counter()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [c.strip() for c in line.split(",")]))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is None or (self.t0 <= t <= (self.t1 or t))]
        if not rows and self.t0 is not None:  # a region shorter than one period: the next sample
            rows = [r for t, r in self.rows if t >= self.t0][:1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}



# ---------------------------------------------------------------------------
# workload construction


def workload(cfg, cloud_fn, seed=SEED):
    """The config's inputs, shared by both arms (numpy only, no product code):
    the grid (n nodes per axis on [-1, 1]^dim, dx = 2/(n-1)), the seeded
    cloud (cloud_fn = the generator of include/lsr_workloads.h, linked into
    the product library for our arm and into oracle/_ref for the reference
    arm), phi^0 = |x| - r0, narrow_band's ACTIVE set |phi| < gamma
    (grid.cpp:85-88) and the step parameters (dt = dx/4, driver.hpp:27;
    default_band_params, grid.cpp:49-51)."""
    n, dim = cfg["n"], cfg["dim"]
    dx = 2.0 / (n - 1)
    gd = dict(dim=dim, dims=(n, n, n) if dim == 3 else (n, n, 1), origin=(-1.0, -1.0, -1.0 if dim == 3 else 0.0),
              dx=dx)
    pts = cloud_fn(cfg["cloud"], cfg["points"], seed=seed, sigma=cfg["sigma"] * dx)
    ax = [gd["origin"][d] + np.arange(gd["dims"][d], dtype=np.float64) * dx for d in range(3)]  # Grid::node
    if dim == 3:
        r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2)
    else:
        r = np.sqrt(ax[0][None, :] ** 2 + ax[1][:, None] ** 2)
    phi = (r - cfg["r0"]).reshape(-1)
    gamma, beta = (6.0 * dx, 3.0 * dx) if dim == 3 else (4.0 * dx, 2.0 * dx)
    active = np.flatnonzero(np.abs(phi) < gamma).astype(np.int64)
    step = dict(p=cfg["p"], interp=cfg["interp"], delta=cfg["delta"], dt=0.25 * dx, fallback_c=1e-3,
                fallback_alpha=1.0, gamma=gamma, beta=beta)
    return dict(grid=gd, pts=pts, phi=phi, active=active, step=step)


def config_block(cfg, w):
    """The JSON line's `config`: the workload only, identical in both arms."""
    st = w["step"]
    return {"workload": cfg["name"], "grid": list(w["grid"]["dims"]), "cloud_points": cfg["points"],
            "cloud_seed": SEED, "phi0": f"|x| - {cfg['r0']}", "active_nodes": int(w["active"].size),
            "interp": "weno" if cfg["interp"] == 1 else "q1", "p": st["p"], "delta": st["delta"], "dt": st["dt"],
            "gamma": st["gamma"], "beta": st["beta"],
            "l2": "the GPU arm flushes L2 (256 MB write) between timed steps"}


def make_inputs(lsr, cfg):
    """workload() in the product's host types."""
    w = workload(cfg, lsr.cloud_generate)
    gd = w["grid"]
    g = lsr.Grid(gd["dim"], tuple(gd["origin"]), gd["dx"], tuple(gd["dims"]))
    st = w["step"]
    step = lsr.StepConfig(p=st["p"], delta=st["delta"], dt=st["dt"], interp=lsr.InterpolatorKind(st["interp"]),
                          band=lsr.BandParams(st["gamma"], st["beta"]))
    return g, w, step


# ---------------------------------------------------------------------------


def run_ours(args):
    import torch

    import paper_2410_22205_b200 as lsr

    world, rank, local = dist_env()
    if args.debug_same_device:  # N ranks on cuda:0 over gloo: a 1-GPU smoke of the N > 1 code path
        local = 0
        args.exchange = "nccl"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.debug_same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if args.debug_same_device else "cuda"  # where reductions' tensors live
    cfg = CONFIGS[args.config]
    g, w, step = make_inputs(lsr, cfg)
    pts, phi, active = w["pts"], w["phi"], w["active"]
    nxy = g.dims[0] * g.dims[1]
    # one explicit (non-legacy) stream for everything: the context's kernels,
    # the L2 flush and the timing events are then ordered on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = lsr.Context(g, device=local)
    ctx.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    sentinel, rounds = ctx.build_distance(pts)
    t_dist = time.perf_counter() - t0
    ctx.upload(lsr._api.FIELD_PHI, phi)
    t0 = time.perf_counter()
    e2 = ctx.surface_energy(lsr._api.FIELD_PHI, 2, 5)
    t_energy = time.perf_counter() - t0

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    halo = 0
    table_ms = []  # z-line table fill per step (3d WENO, inside the step, outside the SL kernel)
    if world == 1:
        mine = active
        ctx.set_active(mine)

        # steps are enqueued back to back (lsr_cuda_sl_step_async, no host
        # sync per step); per-step device times come from the context's
        # events at the sync after the timed loop
        def one_step(i):
            ctx.sl_step_async(step, e2)
            ctx.swap()
            return None
    else:
        # z-slabs (paper_2410_22205_b200/zslab.py): slab-sized resident buffers,
        # the slab-mode kernel on owned ids, NCCL halo exchange, buffer swap
        import ctypes as C

        from paper_2410_22205_b200 import zslab

        h_d = ctx.download(lsr._api.FIELD_DIST)
        halo = zslab.halo_planes(max_displacement(g, h_d, active, step, e2), g.dx, cfg["interp"])
        cuts = zslab.plan_cuts(active, nxy, g.dims[2], world, min_planes=halo)
        s = zslab.make_slab(cuts, rank, halo, nxy, g.dims[2])
        mine = zslab.owned_ids(active, s)
        sl = slice(s.z_base * nxy, (s.z_base + s.z_planes) * nxy)
        # the two resident phi buffers are whole cudaMalloc allocations so that
        # their CUDA IPC handles map them on the neighbours (fused path)
        phi_t = raw_device_tensor(lsr, s.n_resident, torch)
        out_t = raw_device_tensor(lsr, s.n_resident, torch)
        phi_t.copy_(torch.from_numpy(phi[sl]))
        out_t.copy_(phi_t)
        d_t = torch.from_numpy(h_d[sl].copy()).cuda()
        ids_t = torch.from_numpy(mine).cuda()
        # (the whole-grid context stays: d for the slab loop, the e2e slabs and the CPU baseline)
        bad_t = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
        miss_t = torch.zeros(1, dtype=torch.int64, device="cuda")
        L = lsr.lib()
        cg, cc = g.c(), step.c()
        kev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

        def compute(p, d, o, slab, ids):
            kev[0].record(stream)
            st = L.lsr_cuda_sl_step_device(C.byref(cg), slab.z_base, slab.z_planes, C.c_void_p(p.data_ptr()),
                                           C.c_void_p(d.data_ptr()), C.c_void_p(ids_t.data_ptr()), ids_t.numel(),
                                           C.byref(cc), e2, C.c_void_p(o.data_ptr()), C.c_void_p(bad_t.data_ptr()),
                                           C.c_void_p(miss_t.data_ptr()), C.c_void_p(stream.cuda_stream))
            kev[1].record(stream)
            if st != 0:
                raise RuntimeError(L.lsr_cuda_last_error_string().decode())
            return 0

        fused = None
        if args.exchange == "fused":
            fused = setup_fused(L, C, dist, torch, s, halo, phi_t, out_t, world, rank)
        if fused is not None:
            peer_lo, peer_hi = fused
            tiny = torch.zeros(1, device="cuda")

            def compute_fused(src, dst, lo, hi, slab, push):
                kev[0].record(stream)
                st = L.lsr_cuda_sl_step_device_fused(
                    C.byref(cg), slab.z_base, slab.z_planes, slab.lo, slab.hi, C.c_void_p(src.data_ptr()),
                    C.c_void_p(d_t.data_ptr()), C.c_void_p(ids_t.data_ptr()), ids_t.numel(), C.byref(cc), e2,
                    C.c_void_p(dst.data_ptr()), C.c_void_p(lo[0]), lo[1], push if lo[0] else 0, C.c_void_p(hi[0]),
                    hi[1], push if hi[0] else 0, C.c_void_p(bad_t.data_ptr()), C.c_void_p(miss_t.data_ptr()),
                    C.c_void_p(stream.cuda_stream))
                kev[1].record(stream)
                if st != 0:
                    raise RuntimeError(L.lsr_cuda_last_error_string().decode())

            stepper = zslab.FusedSlabStepper(s, halo, (phi_t, out_t), peer_lo, peer_hi, compute_fused,
                                             barrier=lambda: dist.all_reduce(tiny))  # stream-ordered
        else:
            stepper = zslab.SlabStepper(dist, s, halo, phi_t, d_t, out_t, ids_t, compute)
        exchange_mode = "fused SL + peer halo push (CUDA IPC)" if fused is not None else "NCCL plane send/recv"

        def one_step(i):
            stepper.step()
            torch.cuda.current_stream().synchronize()
            return kev[0].elapsed_time(kev[1])

    clk = ClockSampler(local).__enter__()
    for i in range(args.warmup):
        one_step(i)
    if world == 1:
        ctx.sync()
    if world > 1:
        dist.barrier()
        if int(miss_t.item()) or int(bad_t.item()) != np.iinfo(np.int64).max:
            raise RuntimeError(f"rank {rank}: halo of {halo} planes too thin or non-finite update")
    torch.cuda.synchronize()
    kernel_ms, step_ms = [], []
    n0 = lsr.kernel_launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk.begin()
    try:
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 between timed steps (outside the step's events)
            evs[i][0].record(stream)
            km = one_step(i)  # resync + SL kernel (+ halo exchange when N > 1), all on `stream`
            evs[i][1].record(stream)
            kernel_ms.append(km)
        torch.cuda.synchronize()
        if world == 1:
            ctx.sync()  # raises NumericalError if any timed step went non-finite
            kernel_ms, _, table_ms = ctx.async_times()
        step_ms = [a.elapsed_time(b) for a, b in evs]
    finally:
        clk.end()
        clk.__exit__()
    torch.cuda.synchronize()
    launches = lsr.kernel_launches() - n0
    if world > 1:
        dist.barrier()
    tot = np.array([sum(step_ms), sum(kernel_ms), float(mine.size)], dtype=np.float64)
    if world > 1:
        t = torch.tensor(tot[:2], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot[:2] = t.cpu().numpy()
    ms_total = float(tot[0])
    units = float(active.size) * args.steps  # whole job: all ranks together cover the band
    value = units / (ms_total * 1e-3)
    kern_avg_ms = float(np.mean(kernel_ms))
    hbm_peak, peak_kind = peaks()
    bpu = BYTES_PER_UPDATE[("weno" if cfg["interp"] == 1 else "q1", cfg["dim"])]
    kernel_rate = mine.size / (kern_avg_ms * 1e-3)  # this rank's node-updates per second of SL kernel
    achieved = kernel_rate * bpu / 1e9
    traffic_pu, traffic_info = traffic_per_update()
    f64_peak, f64_src = fp64_peak()
    # the committed capture describes the headline kernel (config 4, WENO-3D table path) only
    capture_applies = bool(traffic_info) and traffic_info.get("config") == args.config
    f64_pu = traffic_info.get("fp64_inst_per_update") if capture_applies else None

    e2e = None
    cpu = None
    if world > 1 and (int(miss_t.item()) or int(bad_t.item()) != np.iinfo(np.int64).max):
        raise RuntimeError(f"rank {rank}: halo of {halo} planes too thin or non-finite update")
    if rank == 0 and world == 1 and not args.no_e2e:
        e2e = measure_e2e(lsr, g, phi, ctx, active, step, e2, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, phi, ctx, active, step, e2, lsr)
    loop = None
    if rank == 0 and world == 1 and not args.no_loop:
        loop = measure_loop(lsr, g, phi, ctx, step, cpu_too=not args.no_cpu_baseline)
    if world > 1:
        # the same metric end to end and the whole loop, both over z-slabs
        # (zslab.SlabLoop / SlabContext); guarded: a failure is reported in
        # the line, the SL measurement above stands
        def guarded(fn):
            try:
                return fn()
            except Exception as ex:  # noqa: BLE001
                return {"error": f"{type(ex).__name__}: {ex}"}

        if not args.no_e2e:
            e2e = guarded(lambda: measure_e2e_slabs(lsr, g, phi, ctx, active, step, e2, args, dist, world, rank,
                                                    red_dev))
        if not args.no_loop:
            loop = guarded(lambda: measure_loop_slabs(lsr, g, phi, ctx, step, dist, world, rank, red_dev))
        if rank == 0 and not args.no_cpu_baseline:
            cpu = guarded(lambda: cpu_baseline(g, phi, ctx, active, step, e2, lsr))

    if rank == 0:
        line = {
            "metric": metric_name(cfg),
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": f"synthetic (seeded {cfg['shape']}, BASELINE config {args.config} shapes/sizes)",
            "config": config_block(cfg, w),
            "run": {
                "energy_e2": e2, "dist_sweep_rounds": rounds,
                "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                "halo_exchange": exchange_mode if world > 1 else None,
                "halo_planes": halo,
                "step": "resync + z-line table fill + SL kernel" if (cfg["interp"] == 1 and cfg["dim"] == 3
                                                                      and cfg["delta"] > 0) else "resync + SL kernel",
            },
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": hbm_peak,
                "unit": "GB/s",
                "frac": achieved / hbm_peak,
                "traffic": (traffic_pu * mine.size) if (traffic_pu and capture_applies) else None,
                "peak_source": peak_kind,
                "algorithmic_bytes_per_update": bpu,
                "kernel_ms_avg": kern_avg_ms,
                "table_fill_ms_avg": float(np.mean(table_ms[-args.steps:])) if table_ms else None,
                # the compulsory-byte fraction and the measured fp64-peak fraction
                "compulsory_bytes_per_update": COMPULSORY_BYTES,
                "compulsory_frac": kernel_rate * COMPULSORY_BYTES / 1e9 / hbm_peak,
                "fp64_inst_per_update": f64_pu,
                "fp64_peak_inst_per_s": f64_peak,
                "fp64_peak_source": f64_src,
                "fp64_frac": (f64_pu * kernel_rate / f64_peak) if (f64_pu and f64_peak) else None,
                "ncu": ({k: traffic_info[k] for k in ("fp64_pipe_active", "l1_hit", "l2_hit", "source")
                         if k in traffic_info} if capture_applies else None),
                "note": "achieved = reference-access bytes per node-update (SURVEY 8(d)) over the SL kernel's "
                        "time; the kernel is bound by fp64 issue and load latency, not by DRAM: fp64_frac = fp64 "
                        "instructions per update (ncu capture) x kernel rate / measured DFMA rate; "
                        "compulsory_frac = 32 B per update at the kernel rate. The step (value, ms_per_step) "
                        "also holds the z-line table fill (table_fill_ms_avg) and the sparse resync",
            },
            "gpu_launches": int(launches),
            **({"debug_same_device": "N ranks on one GPU over gloo: a code-path smoke, not a multi-GPU number"}
               if args.debug_same_device else {}),
            "clocks": clk.summary(),
            "setup_s": {"build_distance": t_dist, "surface_energy": t_energy},
        }
        if loop and loop.get("moving_band"):
            # the band-changing rate of the faster loop form (device-controlled), the host-driven one beside it
            mb = dict(loop["moving_band"])
            dr = (loop.get("device_run") or {}).get("moving_band")
            if dr:
                mb = {**mb, "value": dr["value"], "sl_ms_per_step": dr["sl_ms_per_step"],
                      "host_driven_value": loop["moving_band"]["value"],
                      "what": "SL phase of the device-controlled loop (lsr_cuda_loop_run: band rebuilt every "
                              "iteration, covered bricks from the band's state bytes, z-line table fill, SL kernel), "
                              "globaltimer marks; host_driven_value: the same phase of lsr_cuda_loop_step"}
            line["moving_band"] = mb
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        if loop:
            line["loop"] = loop
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (torch.as_tensor shares it)."""

    def __init__(self, ptr, n, owner):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}
        self.owner = owner


class _RawAlloc:
    def __init__(self, lsr, nbytes):
        import ctypes as C

        self.lib = lsr.lib()
        p = C.c_void_p()
        if self.lib.lsr_cuda_malloc(nbytes, C.byref(p)) != 0:
            raise RuntimeError(self.lib.lsr_cuda_last_error_string().decode())
        self.ptr = p.value

    def __del__(self):
        try:
            import ctypes as C

            self.lib.lsr_cuda_free(C.c_void_p(self.ptr))
        except Exception:
            pass


_RAW_KEEP = []


def raw_device_tensor(lsr, n, torch):
    a = _RawAlloc(lsr, 8 * n)
    _RAW_KEEP.append(a)  # keep the allocation alive for the process
    return torch.as_tensor(_CudaArray(a.ptr, n, a), device="cuda")


def setup_fused(L, C, dist, torch, s, halo, phi_t, out_t, world, rank):
    """Map the neighbours' resident buffers into this process (CUDA IPC over
    NVLink/NVSwitch) for the fused SL + halo-push kernel. Every rank must
    succeed, else all fall back to the NCCL plane exchange."""
    handles, ok = [], True
    for t in (phi_t, out_t):
        h = C.create_string_buffer(64)
        ok = ok and L.lsr_cuda_ipc_handle(C.c_void_p(t.data_ptr()), h) == 0
        handles.append(h.raw)
    info = [None] * world
    dist.all_gather_object(info, {"handles": handles, "z_base": s.z_base, "ok": ok})

    def open_peer(r):
        if not info[r]["ok"]:
            return None
        ptrs = []
        for hb in info[r]["handles"]:
            p = C.c_void_p()
            if L.lsr_cuda_ipc_open(hb, C.byref(p)) != 0:
                return None
            ptrs.append(p.value)
        return tuple(ptrs), info[r]["z_base"]

    lo = open_peer(rank - 1) if rank > 0 else None
    hi = open_peer(rank + 1) if rank < world - 1 else None
    good = torch.tensor([1.0 if ok and (rank == 0 or lo) and (rank == world - 1 or hi) else 0.0], device="cuda")
    dist.all_reduce(good, op=dist.ReduceOp.MIN)
    if good.item() < 1.0:
        return None
    return lo, hi


def max_displacement(g, h_d, active, step, e2):
    """Upper bound of |foot - node| over the band (evolve.cpp:83-101):
    C dt |grad d| + spread * sqrt(2), C = d/E (p = 2) or 1."""
    nx, ny, nz = g.dims
    d3 = h_d.reshape(nz, ny, nx)
    k = active // (nx * ny)
    j = (active // nx) % ny
    i = active % nx
    gx = (d3[k, j, np.minimum(i + 1, nx - 1)] - d3[k, j, np.maximum(i - 1, 0)]) / g.dx
    gy = (d3[k, np.minimum(j + 1, ny - 1), i] - d3[k, np.maximum(j - 1, 0), i]) / g.dx
    gz = (d3[np.minimum(k + 1, nz - 1), j, i] - d3[np.maximum(k - 1, 0), j, i]) / g.dx
    dj = h_d[active]
    c = dj / e2 if step.p == 2 else np.ones_like(dj)
    spread = np.sqrt(np.maximum(0.0, c * step.delta * dj * step.dt / step.p))
    disp = c * step.dt * np.sqrt(gx * gx + gy * gy + gz * gz) + spread * np.sqrt(2.0)
    return float(disp.max()) if disp.size else 0.0


def measure_e2e(lsr, g, phi, ctx, active, step, e2, args):
    """The same metric through the public drop-in call lsr.sl_step (host
    buffers in pinned memory): H2D phi + d + active ids, the step, D2H out."""
    import torch

    n = g.num_nodes()
    h_phi = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    h_d = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    h_act = torch.empty(active.size, dtype=torch.int64, pin_memory=True).numpy()
    h_phi[:] = phi
    ctx.download(lsr._api.FIELD_DIST, h_d)
    h_act[:] = active
    sphi = lsr.ScalarField(g, h_phi)
    sd = lsr.DistanceField(lsr.ScalarField(g, h_d))
    mask = lsr.BandMask(g, active=h_act)
    out = lsr.ScalarField(g, h_out)
    for _ in range(2):
        lsr.sl_step(sphi, sd, mask, step, e2, out)
    ts = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        lsr.sl_step(sphi, sd, mask, step, e2, out)  # synchronous: returns after the D2H of out
        ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    import ctypes as C

    h2d, d2h = C.c_int64(), C.c_int64()
    lsr.lib().lsr_cuda_last_transfer_bytes(C.byref(h2d), C.byref(d2h))  # what the call actually copied
    return {"value": active.size / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d.value),
            "d2h_bytes_per_step": int(d2h.value), "ms_per_step": t * 1e3,
            "timing": "host clock around the synchronous call lsr.sl_step on pinned host buffers (phi, d, ids in, "
                      "out back): the GPU pulls the phi/d values the step reads (zero-copy) plus 1/8 of the planes "
                      "whole (DMA), returns the updated values, host threads copy phi to out and scatter them",
            "steps": args.e2e_steps}


def _max_over_ranks(dist, x, dev):
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(dist, x, dev):
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _slab_ctx(lsr, g, whole, wl, wh, ol, oh):
    """A SlabContext for resident planes [wl, wh), owned [ol, oh), with d
    copied from the whole-grid context."""
    nxy = g.dims[0] * g.dims[1]
    c = lsr.SlabContext(g, wl, wh, ol, oh)
    c.copy_planes(lsr._api.FIELD_DIST, wl, wh - wl, whole.field_ptr(lsr._api.FIELD_DIST) + 8 * wl * nxy, True)
    return c


def measure_e2e_slabs(lsr, g, phi, whole, active, step, e2, args, dist, world, rank, dev):
    """N > 1 end to end through the slab API: every step each rank uploads its
    resident planes of phi from pinned host memory, runs the SL step on its
    owned active nodes, and reads its window of out back; the time is the max
    over ranks (host clock, barrier before each step)."""
    import torch

    from paper_2410_22205_b200 import zslab

    nxy = g.dims[0] * g.dims[1]
    halo = zslab.halo_planes(max_displacement(g, whole.download(lsr._api.FIELD_DIST), active, step, e2), g.dx,
                             int(step.interp))
    cuts = zslab.plan_cuts(active, nxy, g.dims[2], world, min_planes=halo)
    nz = g.dims[2]
    c = _slab_ctx(lsr, g, whole, max(0, int(cuts[rank]) - halo), min(nz, int(cuts[rank + 1]) + halo),
                  int(cuts[rank]), int(cuts[rank + 1]))
    h_phi = torch.empty(c.n_resident, dtype=torch.float64, pin_memory=True).numpy()
    h_out = torch.empty(c.n_resident, dtype=torch.float64, pin_memory=True).numpy()
    h_phi[:] = phi[c.win_lo * nxy:c.win_hi * nxy]
    c.upload(lsr._api.FIELD_PHI, h_phi)
    c.band(step.band.gamma)
    ts = []
    for i in range(2 + args.e2e_steps):
        dist.barrier()
        t0 = time.perf_counter()
        c.upload(lsr._api.FIELD_PHI, h_phi)
        if c.sl_step(step, e2):
            raise RuntimeError("halo too small")
        lsr.lib().lsr_cuda_download_field(c.h, lsr._api.FIELD_OUT, h_out.ctypes.data)
        if i >= 2:
            ts.append(time.perf_counter() - t0)
    t = _max_over_ranks(dist, float(np.mean(ts)), dev)
    h2d = _sum_over_ranks(dist, 8 * c.n_resident, dev)
    c.close()
    return {"value": active.size / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(h2d),
            "ms_per_step": 1e3 * t, "steps": args.e2e_steps, "halo_planes": halo,
            "timing": "max over ranks of the host clock around: upload of the rank's resident planes of phi "
                      "(pinned), lsr_cuda_slab_sl_step, download of its window of out (pinned)"}


def measure_loop_slabs(lsr, g, phi, whole, step, dist, world, rank, dev, steps=5):
    """N > 1: the whole driver iteration over z-slabs (zslab.SlabLoop with the
    torch.distributed runner): band, E_2 (blocked_sum from the ranks'
    pieces), SL, the one-step and Jacobi sweeps with plane exchanges and a
    global stop rule, clamp. Wall time per iteration, max over ranks."""
    import torch

    from paper_2410_22205_b200 import zslab

    nxy = g.dims[0] * g.dims[1]
    band = np.flatnonzero(np.abs(phi) < step.band.gamma)
    halo = 6
    cuts = zslab.plan_cuts(band, nxy, g.dims[2], world, min_planes=3 * halo)
    rc = lsr.ReinitConfig.defaults(g.dx, step.band.gamma)
    loop = zslab.SlabLoop(g, cuts, [rank], halo, lambda wl, wh, ol, oh: _slab_ctx(lsr, g, whole, wl, wh, ol, oh),
                          lambda c: None, lambda ctxs: zslab.DistRunner(dist, ctxs[0], cuts))
    loop.upload_phi(lambda c: phi[c.win_lo * nxy:c.win_hi * nxy])
    ts, its = [], []
    for i in range(steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = loop.step(step, rc, step.band.gamma)
        torch.cuda.synchronize()
        if i >= 1:
            ts.append(time.perf_counter() - t0)
        its.append(st[0]["reinit_iterations"])
    t = _max_over_ranks(dist, float(np.mean(ts)), dev)
    for c in loop.ctxs:
        c.close()
    return {"gpu_total_ms_per_step": 1e3 * t, "steps": steps, "timed": steps - 1, "halo_planes": loop.halo,
            "regrows": loop.regrows, "reinit_iterations": its,
            "what": "driver.cpp:187-203 over z-slabs (zslab.SlabLoop, NCCL): wall time per iteration incl. the "
                    "per-sweep residual allreduce and plane exchanges, max over ranks, iterations 2..N from phi^0"}


def measure_loop(lsr, g, phi, ctx, step, steps=6, cpu_too=True):
    """The whole driver iteration (driver.cpp:187-203: band, E_2, SL,
    reinit, swap) from phi^0 on the device, per-phase device ms, next to one
    iteration of the reference's own loop body on the host cores. Its SL
    phase gives `moving_band`: the headline metric when the band (and so the
    z-line table's covered-brick list) is rebuilt every iteration."""
    ctx.upload(lsr._api.FIELD_PHI, phi)
    rc = lsr.ReinitConfig.defaults(g.dx, step.band.gamma)
    stats = [ctx.loop_step(step, rc, 5) for _ in range(steps)]
    ms = np.array([s["ms"] for s in stats[1:]])  # first iteration includes workspace allocation
    na = np.array([s["n_active"] for s in stats[1:]], dtype=np.float64)
    out = {"gpu_ms_per_step": dict(zip(("band", "energy", "sl", "reinit"), map(float, ms.mean(0)))),
           "gpu_total_ms_per_step": float(ms.sum(1).mean()), "steps": steps,
           "reinit_iterations": [s["reinit_iterations"] for s in stats]}
    out["moving_band"] = {
        "value": float(na.sum() / (ms[:, 2].sum() * 1e-3)), "unit": UNIT,
        "sl_ms_per_step": float(ms[:, 2].mean()), "active_nodes_mean": float(na.mean()), "iterations": steps - 1,
        "what": "SL phase of the device loop (band rebuilt every iteration: covered-brick list, z-line table "
                "fill, sparse resync, SL kernel), CUDA events; loop iterations 2..N from phi^0"}
    # the same iterations controlled on the device (lsr_cuda_loop_run: one host
    # sync per run, iterations 2..K replayed from a CUDA graph), again from
    # phi^0: device phase times from globaltimer marks, and the wall time of
    # the whole call per iteration
    run_iters = 2 * steps
    for _ in range(2):  # the first run captures the graphs
        ctx.upload(lsr._api.FIELD_PHI, phi)
        t0 = time.perf_counter()
        recs = ctx.loop_run(step, rc, run_iters, 5)
        wall = time.perf_counter() - t0
    rms = np.array([r["ms"] for r in recs[1:]])
    rna = np.array([r["n_active"] for r in recs[1:]], dtype=np.float64)
    out["device_run"] = {
        "gpu_ms_per_step": dict(zip(("band", "energy", "sl", "reinit"), map(float, rms.mean(0)))),
        "gpu_total_ms_per_step": float(rms.sum(1).mean()), "wall_ms_per_step": 1e3 * wall / run_iters,
        "iterations": run_iters, "host_syncs": 1,
        "reinit_iterations": [r["reinit_iterations"] for r in recs],
        "same_bands_as_host_loop": [r["n_active"] for r in recs[:steps]] == [s["n_active"] for s in stats],
        "moving_band": {"value": float(rna.sum() / (rms[:, 2].sum() * 1e-3)), "unit": UNIT,
                        "sl_ms_per_step": float(rms[:, 2].mean())},
        "what": "lsr_cuda_loop_run: band counts, E_2, the E_2 == 0 skip, NoInterface and the Jacobi stop rule "
                "decided on the device; iterations 2..K (graph replays) averaged"}
    if cpu_too:
        from oracle import bindings

        if bindings.reference_available():
            R = bindings.Reference()
            R.set_threads(os.cpu_count() or 1)
            d = ctx.download(lsr._api.FIELD_DIST)
            cc = dict(p=step.p, interp=int(step.interp), delta=step.delta, dt=step.dt, fallback_c=step.fallback_c,
                      fallback_alpha=step.fallback_alpha, gamma=step.band.gamma, beta=step.band.beta)
            _, _, _, _, sec = R.loop_step(dict(dim=g.dim, dims=g.dims, origin=g.origin, dx=g.dx), phi, d, cc)
            out["cpu_reference_ms_per_step"] = dict(zip(("band", "energy", "sl", "reinit"), map(lambda v: 1e3 * v, sec)))
            out["cpu_reference_total_ms_per_step"] = float(1e3 * sum(sec))
            out["cpu_cores"] = os.cpu_count()
            out["loop_speedup_vs_cpu_reference"] = out["cpu_reference_total_ms_per_step"] / out["gpu_total_ms_per_step"]
            out["device_run"]["speedup_vs_cpu_reference"] = (out["cpu_reference_total_ms_per_step"] /
                                                             out["device_run"]["gpu_total_ms_per_step"])
    return out


def cpu_model():
    """The host CPU's model name (/proc/cpuinfo), for the baseline's record."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(g, phi, ctx, active, step, e2, lsr, reps=3):
    """The reference's lsr::sl_step (OpenMP, all host threads) on the same
    inputs (oracle/_ref; the oracle restatement when _ref is absent)."""
    from oracle import bindings

    d = ctx.download(lsr._api.FIELD_DIST)
    gd = dict(dim=g.dim, dims=g.dims, origin=g.origin, dx=g.dx)
    cc = dict(p=step.p, interp=int(step.interp), delta=step.delta, dt=step.dt, fallback_c=step.fallback_c,
              fallback_alpha=step.fallback_alpha, gamma=step.band.gamma, beta=step.band.beta)
    threads = os.cpu_count() or 1
    serial = None
    if bindings.reference_available():
        R = bindings.Reference()
        R.set_threads(threads)
        h = R.ctx(gd, phi, d, active)
        secs = [R.ctx_sl_step(h, cc, e2, serial=False) for _ in range(reps)]
        R.ctx_free(h)
        kind = "reference"
        # lsr::ref::sl_step on 1 thread too, on a bounded
        # sample of the band (every k-th active node; its O(N) copy included)
        k = max(1, active.size // 400_000)
        sample = np.ascontiguousarray(active[::k])
        h = R.ctx(gd, phi, d, sample)
        ssec = min(R.ctx_sl_step(h, cc, e2, serial=True) for _ in range(2))
        R.ctx_free(h)
        serial = {"value": sample.size / ssec, "unit": UNIT, "cores": 1,
                  "sample": f"every {k}th active node ({sample.size} nodes), lsr::ref::sl_step incl. its O(N) copy, "
                            f"best of 2", "seconds": ssec}
    else:
        O = bindings.Restatement()
        secs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            O.sl_step(gd, phi, d, active, cc, e2, nthreads=threads)
            secs.append(time.perf_counter() - t0)
        kind = "port"
    best = min(secs)
    out = {"value": active.size / best, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": kind,
           "sample": f"full band ({active.size} active nodes) of the same workload, best of {reps} calls of "
                     f"lsr::sl_step incl. its internal O(N) copy", "seconds": secs}
    if serial:
        out["serial_reference"] = serial
    return out


# ---------------------------------------------------------------------------


def run_reference(args):
    """--impl reference: the reference's own CPU lsr::sl_step (oracle/_ref,
    built from the reference sources; OpenMP over all host cores) on the same
    workload, inputs produced by the reference's own functions. Nothing of
    the product is imported or loaded here: the cloud generator is linked
    into oracle/_ref as well."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import bindings

    cfg = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    if not bindings.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built on this machine"}))
        return
    R = bindings.Reference()
    R.set_threads(threads)
    kind = "reference"
    w = workload(cfg, R.cloud_generate)
    gd, phi, step = w["grid"], w["phi"], w["step"]
    t0 = time.perf_counter()
    d, _, _, rounds = R.build_distance(gd, w["pts"], cfg["dim"])  # lsr::build_distance_field
    t_dist = time.perf_counter() - t0
    e2 = R.surface_energy(gd, phi, d, 2, 5)
    _, act_ref, _ = R.narrow_band(gd, phi, step["gamma"])
    if not np.array_equal(act_ref, w["active"]):
        raise RuntimeError("the reference's narrow_band differs from the workload's active set")
    h = R.ctx(gd, phi, d, act_ref)
    # bound the run to a few minutes: sample a contiguous share of the band per step if needed
    probe = R.ctx_sl_step(h, step, e2)
    budget = 150.0
    frac = min(1.0, budget / max(1e-9, probe * (args.steps + args.warmup)))
    if frac < 1.0:
        R.ctx_free(h)
        m = max(1, int(act_ref.size * frac))
        h = R.ctx(gd, phi, d, act_ref[:m])
        units = m
    else:
        units = act_ref.size
    for _ in range(args.warmup):
        R.ctx_sl_step(h, step, e2)
    secs = [R.ctx_sl_step(h, step, e2) for _ in range(args.steps)]
    R.ctx_free(h)
    t = float(np.sum(secs))
    value = units * args.steps / t
    sample = (f"{units} of {act_ref.size} active nodes per step (lsr::sl_step incl. its O(N) copy), "
              f"OpenMP {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded {cfg['shape']}, BASELINE config {args.config} shapes/sizes)",
        "config": config_block(cfg, w),
        "run": {"energy_e2": e2, "dist_sweep_rounds": rounds, "setup_build_distance_s": t_dist,
                "parallelism": f"OpenMP, {threads} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without a torch.distributed launcher: start N ranks
    (one per GPU) on this node and pass their output through."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-loop", action="store_true")
    ap.add_argument("--exchange", choices=["fused", "nccl"], default="fused",
                    help="N > 1: fused SL + peer halo push (default) or NCCL plane exchange")
    ap.add_argument("--debug-same-device", action="store_true",
                    help="N > 1 on one GPU over gloo (host-staged exchanges): a smoke of the N > 1 code path")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
