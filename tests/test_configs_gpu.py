"""BASELINE configs end to end on the GPU (driver loop body on the device:
band, E_2, SL step, reinitialisation, swap) against the reference.

* config 1 (2d circle, 257^2, multilinear, 200 steps): bit-identical to the
  reference's 200-step run (golden fixture made by the reference itself);
* configs 2 and 3 (128^3 sphere / Q1, 256^3 noisy torus / WENO, p = 2,
  delta = 1) against the live reference loop (oracle/_ref), the GPU loop fed
  the reference's per-step E_2 (glibc pow) so the fields stay
  bit-identical; the GPU's own E_2 is checked to 16 ulp.
"""
import numpy as np
import pytest

from conftest import bits, golden_grid, load_golden

pytestmark = pytest.mark.gpu
ULP16 = 16 * np.finfo(np.float64).eps


def test_config1_circle_200_steps_bit_exact(gpu):
    lsr = gpu
    rec = load_golden("config1_circle_200.npz")
    gg = golden_grid(rec)
    g = lsr.Grid(2, tuple(gg["origin"]), gg["dx"], tuple(gg["dims"]))
    gam = float(rec["gamma"])
    d = lsr.build_distance_field(g, rec["pts"], 2)
    assert np.array_equal(bits(d.field.values), bits(rec["d"]))
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Q1,
                         band=lsr.BandParams(gam, gam / 2))
    rc = lsr.ReinitConfig.defaults(g.dx, gam)
    ctx = lsr.Context(g)
    ctx.upload(0, rec["phi0"])
    ctx.upload(1, rec["d"])
    for k in range(1, 201):
        s = ctx.loop_step(cfg, rc, 5)
        assert abs(s["energy"] - rec["e2"][k - 1]) <= ULP16 * rec["e2"][k - 1]
        if k in (50, 100, 200):
            got = ctx.download(0)
            assert np.array_equal(bits(got), bits(rec[f"phi{k}"])), f"step {k}"


@pytest.mark.parametrize("config,n,steps", [(2, 128, 8), (3, 256, 3)])
def test_configs_2_3_vs_live_reference(gpu, reference, config, n, steps):
    lsr = gpu
    g = lsr.cube_grid(n, 3)
    npts = {2: 20_000, 3: 100_000}[config]
    sigma = {2: 0.0, 3: 0.5 * g.dx}[config]
    interp = {2: lsr.InterpolatorKind.Q1, 3: lsr.InterpolatorKind.Weno}[config]
    pts = lsr.cloud_generate(config, npts, seed=2410, sigma=sigma)
    ax = g.axes()
    phi = (np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2) - 0.9).ravel()
    gd = dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx)
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=interp, band=bp)
    ccfg = dict(p=2, interp=int(interp), delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma,
                beta=bp.beta)
    ctx = lsr.Context(g)
    ctx.build_distance(pts)
    d = ctx.download(1)
    dref, _, _, _ = reference.build_distance(gd, pts, 3)
    assert np.array_equal(bits(d), bits(dref))
    ctx.upload(0, phi)
    rc = lsr.ReinitConfig.defaults(g.dx, bp.gamma)
    cur = phi
    for k in range(steps):
        cur, e2, na, it, _ = reference.loop_step(gd, cur, dref, ccfg)
        s = ctx.loop_step(cfg, rc, 5, energy_override=e2)
        assert s["n_active"] == na and s["reinit_iterations"] == it
        got = ctx.download(0)
        diff = np.count_nonzero(bits(got) != bits(cur))
        assert diff == 0, f"config {config} step {k}: {diff} nodes differ"
    own = lsr.surface_energy(lsr.ScalarField(g, cur), lsr.DistanceField(lsr.ScalarField(g, dref)), 2, 5)
    ref_e = reference.surface_energy(gd, cur, dref, 2, 5)
    assert abs(own - ref_e) <= ULP16 * ref_e


def test_config4_512_loop_step_and_one_shot_vs_reference(gpu, reference):
    """Config 4 at its full size (512^3, 1 M-point bumpy sphere, WENO, p = 2,
    delta = 1): three whole loop iterations (band, E_2, SL, reinit) against
    the reference's own loop body on the host, bit for bit, and the one-shot
    host entry on pinned buffers (the zero-copy pull path bench.py's e2e
    times) against the device-resident step."""
    import torch

    lsr = gpu
    g = lsr.cube_grid(512, 3)
    pts = lsr.cloud_generate(4, 1_000_000, seed=2410, sigma=0.0)
    ax = g.axes()
    phi = (np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2) - 0.9).ravel()
    gd = dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx)
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    ccfg = dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma,
                beta=bp.beta)
    ctx = lsr.Context(g)
    ctx.build_distance(pts)  # bit-identical to the reference's (tests/test_distance.py)
    d = ctx.download(1)
    # one-shot on pinned host buffers vs the device-resident step, same inputs
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    pin = lambda a: (lambda t: (t.__setitem__(slice(None), a), t)[1])(  # noqa: E731
        torch.empty(a.size, dtype=torch.float64 if a.dtype == np.float64 else torch.int64, pin_memory=True).numpy())
    hphi, hd, hact = pin(phi), pin(d), pin(active)
    hout = pin(np.zeros(phi.size))
    lsr.sl_step(lsr.ScalarField(g, hphi), lsr.DistanceField(lsr.ScalarField(g, hd)), lsr.BandMask(g, active=hact),
                cfg, 1.5, lsr.ScalarField(g, hout))
    ctx.upload(0, phi)
    ctx.set_active(active)
    ctx.sl_step(cfg, 1.5)
    dev = ctx.download(2)
    assert np.count_nonzero(bits(hout) != bits(dev)) == 0
    # three loop iterations vs the reference's loop body (band, E_2, SL with
    # the z-line table, reinit), the GPU fed the reference's E_2 (glibc pow)
    ctx.upload(0, phi)
    rc = lsr.ReinitConfig.defaults(g.dx, bp.gamma)
    ref_phi = phi
    for step in range(3):
        ref_phi, e2, na, it, _ = reference.loop_step(gd, ref_phi, d, ccfg)
        s = ctx.loop_step(cfg, rc, 5, energy_override=e2)
        assert s["n_active"] == na and s["reinit_iterations"] == it, step
        got = ctx.download(0)
        diff = np.count_nonzero(bits(got) != bits(ref_phi))
        assert diff == 0, f"iteration {step}: {diff} nodes differ"


def test_config5_1024_sampled_subset_vs_oracle(gpu, oracle):
    """Config 5 at its full size (1024^3, 4 M-point union of three tori with
    two holes, WENO, p = 2, delta = 1) through the device-resident context
    (z-line table path, where feet reach up to ~6 cells at the poles):
    a random subset of the band (sl_step reads only mask.active) against the
    oracle, bit for bit, plus whole-band properties."""
    lsr = gpu
    rng = np.random.default_rng(55)
    g = lsr.cube_grid(1024, 3)
    pts = lsr.cloud_generate(5, 4_000_000, seed=2410, sigma=0.25 * g.dx)
    ax = g.axes()
    phi = (np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2) - 0.95).ravel()
    bp = lsr.default_band_params(3, g.dx)
    band = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    sub = np.sort(rng.choice(band, 30000, replace=False)).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    ctx = lsr.Context(g)
    try:
        ctx.build_distance(pts)
        d = ctx.download(1)
        ctx.upload(0, phi)
        ctx.set_active(sub)
        ctx.sl_step(cfg, 2.4)
        assert ctx.last_table_ms() > 0.0
        got = ctx.download(2)
        ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, d, sub,
                                    dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                         gamma=bp.gamma, beta=bp.beta), 2.4, nthreads=0)
        assert st == 0
        assert np.array_equal(bits(got[sub]), bits(ref[sub]))
        del got, ref
        # whole band: finite, off-band untouched, bounded update
        ctx.set_active(band)
        ctx.sl_step(cfg, 2.4)
        out = ctx.download(2)
        assert np.all(np.isfinite(out[band]))
        changed = np.flatnonzero(out.view(np.int64) != phi.view(np.int64))
        assert np.all(np.isin(changed, band, assume_unique=True))  # off-band nodes carry phi over
        assert np.max(np.abs(out[band] - phi[band])) < 4 * g.dx
    finally:
        ctx.close()


def test_config5_1024_loop_iteration_vs_reference(gpu, reference):
    """Config 5 at its full size (1024^3, 4 M points): one whole loop
    iteration (band, E_2, SL with the z-line table, reinit) on the GPU
    against the reference's own loop body on the host, bit for bit (the GPU
    fed the reference's E_2)."""
    lsr = gpu
    g = lsr.cube_grid(1024, 3)
    pts = lsr.cloud_generate(5, 4_000_000, seed=2410, sigma=0.25 * g.dx)
    ax = g.axes()
    phi = (np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2) - 0.95).ravel()
    gd = dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx)
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    ccfg = dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma,
                beta=bp.beta)
    ctx = lsr.Context(g)
    try:
        ctx.build_distance(pts)
        d = ctx.download(1)
        ctx.upload(0, phi)
        ref_phi, e2, na, it, _ = reference.loop_step(gd, phi, d, ccfg)
        del phi
        s = ctx.loop_step(cfg, lsr.ReinitConfig.defaults(g.dx, bp.gamma), 5, energy_override=e2)
        assert s["n_active"] == na and s["reinit_iterations"] == it
        got = ctx.download(0)
        diff = np.count_nonzero(got.view(np.int64) != ref_phi.view(np.int64))
        assert diff == 0, f"{diff} nodes differ"
    finally:
        ctx.close()


@pytest.mark.parametrize("config,n,steps", [(2, 128, 8), (3, 256, 3)])
def test_configs_own_energy_within_tolerance(gpu, reference, config, n, steps):
    """The GPU loop with its own E_2 (few-ulp from the reference's glibc-pow
    sum) against the reference loop: the north star's fp64
    tolerance, normwise — max |phi_gpu - phi_ref| <= 1e-12 * gamma (the
    field's scale) — and pointwise relative 1e-12 where |phi| >= dx."""
    lsr = gpu
    g = lsr.cube_grid(n, 3)
    npts = {2: 20_000, 3: 100_000}[config]
    sigma = {2: 0.0, 3: 0.5 * g.dx}[config]
    interp = {2: lsr.InterpolatorKind.Q1, 3: lsr.InterpolatorKind.Weno}[config]
    pts = lsr.cloud_generate(config, npts, seed=2410, sigma=sigma)
    ax = g.axes()
    phi = (np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2) - 0.9).ravel()
    gd = dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx)
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=interp, band=bp)
    ccfg = dict(p=2, interp=int(interp), delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma,
                beta=bp.beta)
    ctx = lsr.Context(g)
    try:
        ctx.build_distance(pts)
        d = ctx.download(1)
        ctx.upload(0, phi)
        rc = lsr.ReinitConfig.defaults(g.dx, bp.gamma)
        cur = phi
        for _ in range(steps):
            cur, _, _, _, _ = reference.loop_step(gd, cur, d, ccfg)
            ctx.loop_step(cfg, rc, 5)  # the GPU's own E_2
        got = ctx.download(0)
        err = np.abs(got - cur)
        assert np.max(err) <= 1e-12 * bp.gamma, np.max(err) / bp.gamma
        big = np.abs(cur) >= g.dx
        assert np.all(err[big] <= 1e-12 * np.abs(cur[big]))
    finally:
        ctx.close()
