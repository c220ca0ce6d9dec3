"""GPU parity tests of the sm_100a SL step (through the C ABI).

Bar: bit-exact (0 differing bits) against the reference's outputs (golden
fixtures produced by the reference itself) and against the oracle
restatement on fresh seeded inputs; plus the reference's own known-answer
tests (test_evolve.cpp) and size-independent properties at full size.
"""
import numpy as np
import pytest

from conftest import SL_CASES, bits, golden_grid, load_golden

pytestmark = pytest.mark.gpu


def _grid_obj(lsr, g):
    return lsr.Grid(g["dim"], tuple(g["origin"]), g["dx"], tuple(g["dims"]))


def _cfg(lsr, rec, c):
    bp = lsr.BandParams(float(rec["gamma"]), float(rec["beta"]))
    return lsr.StepConfig(p=int(rec["case_p"][c]), delta=float(rec["case_delta"][c]), dt=0.25 * float(rec["dx"]),
                          interp=lsr.InterpolatorKind(int(rec["case_interp"][c])), band=bp)


def _pinned(a):
    import torch

    t = torch.empty(a.size, dtype=torch.float64 if a.dtype == np.float64 else torch.int64, pin_memory=True).numpy()
    t[:] = a
    return t


def _run(lsr, g, phi, dist, active, cfg, e, pinned=False):
    """One one-shot step; pinned=True hands over page-locked host buffers (the
    zero-copy pull path of lsr_cuda_sl_step_host), else pageable ones."""
    if pinned:
        phi, dist, active = _pinned(phi), _pinned(dist), _pinned(active)
    out = lsr.ScalarField(g, _pinned(np.zeros(g.num_nodes())) if pinned else None)
    lsr.sl_step(lsr.ScalarField(g, phi), lsr.DistanceField(lsr.ScalarField(g, dist)), lsr.BandMask(g, active=active),
                cfg, e, out)
    return out.values


@pytest.mark.parametrize("case", SL_CASES)
def test_sl_step_bit_exact_vs_reference_golden(gpu, case):
    lsr = gpu
    rec = load_golden(f"sl_{case}.npz")
    g = _grid_obj(lsr, golden_grid(rec))
    n0 = lsr.kernel_launches()
    for c in range(len(rec["case_p"])):
        out = _run(lsr, g, rec["phi"], rec["dist"], rec["active"], _cfg(lsr, rec, c), float(rec["e2"]))
        diff = np.count_nonzero(bits(out[rec["active"]]) != bits(rec["case_out"][c]))
        assert diff == 0, f"{case}[{c}]: {diff} active nodes differ"
        mask = np.ones(out.size, bool)
        mask[rec["active"]] = False
        assert np.array_equal(bits(out[mask]), bits(rec["phi"][mask]))
    assert lsr.kernel_launches() > n0


@pytest.mark.parametrize("dim,n,interp,p,delta,seed", [
    (2, 257, 0, 1, 0.0, 1), (2, 257, 1, 2, 1.0, 2),
    (3, 64, 0, 1, 0.0, 3), (3, 64, 0, 2, 1.0, 4), (3, 64, 1, 1, 0.0, 5), (3, 64, 1, 2, 1.0, 6),
    (3, 80, 1, 2, 0.3, 7),
])
def test_sl_step_bit_exact_vs_oracle_seeded(gpu, oracle, dim, n, interp, p, delta, seed):
    lsr = gpu
    rng = np.random.default_rng(seed)
    g = lsr._api.cube_grid(n, dim)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.6 + 0.25 * g.dx * rng.standard_normal(x.size)
    dist = np.abs(np.sqrt((x - 0.07) ** 2 + (y + 0.03) ** 2 + z * z) - 0.35) + 0.01 * rng.random(x.size)
    bp = lsr.default_band_params(dim, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=p, delta=delta, dt=0.25 * g.dx, interp=lsr.InterpolatorKind(interp), band=bp)
    e = 0.7
    got = _run(lsr, g, phi, dist, active, cfg, e)
    ref, st, _ = oracle.sl_step(dict(dim=dim, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                dict(p=p, interp=interp, delta=delta, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=bp.gamma, beta=bp.beta), e)
    assert st == 0
    diff = np.count_nonzero(bits(got) != bits(ref))
    assert diff == 0, f"{diff} of {active.size} active nodes differ"


def test_identity_step_constant_distance(gpu):
    """test_evolve.cpp:78-92: d constant, delta = 0 -> identity on active nodes."""
    lsr = gpu
    g = lsr.Grid(2, (-1.3, -1.3, 0.0), 0.1, (27, 27, 1))
    x, y, _ = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y) - 0.7
    bp = lsr.default_band_params(2, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.025, band=bp)
    out = _run(lsr, g, phi, np.full(x.size, 0.5), active, cfg, 1.0)
    assert np.max(np.abs(out - phi)) < 1e-12


def test_pure_advection_shifts_by_dt(gpu):
    """test_evolve.cpp:94-112: phi = x, d = x + 10, dt = 0.1 -> x + 0.1 where c = 1."""
    lsr = gpu
    for interp in (lsr.InterpolatorKind.Q1, lsr.InterpolatorKind.Weno):
        g = lsr.Grid(2, (-1.15, -1.15, 0.0), 0.05, (47, 47, 1))
        x, y, _ = (a.ravel() for a in g.mesh())
        bp = lsr.default_band_params(2, g.dx)
        active = np.flatnonzero(np.abs(x) < bp.gamma).astype(np.int64)
        cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=bp, interp=interp)
        out = _run(lsr, g, x.copy(), x + 10.0, active, cfg, 1.0)
        i, j, _ = g.unflatten(active)
        sel = (i >= 2) & (i <= 44) & (j >= 2) & (j <= 44) & (np.abs(x[active]) <= bp.beta)
        assert sel.sum() > 20
        np.testing.assert_allclose(out[active][sel], x[active][sel] + 0.1, rtol=1e-12, atol=1e-12)


def test_zero_field_fallback_stays_zero(gpu):
    """test_evolve.cpp:114-123."""
    lsr = gpu
    g = lsr.Grid(2, (-1.3, -1.3, 0.0), 0.1, (27, 27, 1))
    x, y, _ = (a.ravel() for a in g.mesh())
    bp = lsr.default_band_params(2, g.dx)
    active = np.arange(x.size, dtype=np.int64)
    out = _run(lsr, g, np.zeros(x.size), 1.0 + y, active, lsr.StepConfig(p=1, dt=0.05, band=bp), 1.0)
    assert np.all(out == 0.0)


def test_affine_diffusion_cancels_3d(gpu):
    """test_evolve.cpp:151-176: p=2, delta=1, d = 0.25, E = 0.5, affine phi."""
    lsr = gpu
    g = lsr.Grid(3, (-1.375, -1.375, -1.375), 0.125, (23, 23, 23))
    x, y, z = (a.ravel() for a in g.mesh())
    phi = 0.3 * x + 0.2 * y - 0.5 * z
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.05, band=bp)
    out = _run(lsr, g, phi, np.full(x.size, 0.25), active, cfg, 0.5)
    i, j, k = g.unflatten(active)
    inner = (i >= 2) & (i <= 20) & (j >= 2) & (j <= 20) & (k >= 2) & (k <= 20)
    assert np.max(np.abs(out[active][inner] - phi[active][inner])) < 1e-10


def test_nan_distance_raises_numerical_error(gpu, oracle):
    """test_evolve.cpp:195-210; out fully written, smallest bad id reported."""
    lsr = gpu
    g = lsr._api.cube_grid(41, 2)
    x, y, _ = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y) - 0.6
    dist = np.full(x.size, 0.5)
    bp = lsr.default_band_params(2, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    dist[active[len(active) // 2]] = np.nan
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.02, band=bp)
    out = lsr.ScalarField(g)
    with pytest.raises(lsr.NumericalError, match="non-finite update at node"):
        lsr.sl_step(lsr.ScalarField(g, phi), lsr.DistanceField(lsr.ScalarField(g, dist)),
                    lsr.BandMask(g, active=active), cfg, 1.0, out)
    ref, st, bad = oracle.sl_step(dict(dim=2, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                  dict(p=2, interp=1, delta=1.0, dt=0.02, fallback_c=1e-3, fallback_alpha=1.0,
                                       gamma=bp.gamma, beta=bp.beta), 1.0)
    assert st == 3
    assert np.array_equal(bits(out.values), bits(ref))
    c = lsr.Context(g)
    c.upload(0, phi)
    c.upload(1, dist)
    c.set_active(active)
    with pytest.raises(lsr.NumericalError):
        c.sl_step(cfg, 1.0)
    assert c.bad_node == bad


@pytest.mark.parametrize("c", [None, 3.0])
def test_constant_divisor_division_is_ieee(gpu, c):
    """div_const (sl_device.cuh) == hardware IEEE division, bit for bit."""
    lsr = gpu
    g = lsr._api.cube_grid(513, 3)
    divisors = [c] if c else [g.dx, g.dx * g.dx, lsr._api.cube_grid(1025, 3).dx ** 2, 2.0 / 127, 0.1, 1e-5]
    for d in divisors:
        assert lsr._api.selftest_div_const(d, 1 << 26, seed=int(d * 1e9) + 1) == 0, d


@pytest.mark.parametrize("dx", [2.0 / 511, 2.0 / 1023, 2.0 / 127, 2.0 / 255, 2.0 ** -7, 1.0, 2.0 ** -30])
def test_weno_fast_forms_selftest(gpu, dx):
    """weno1_fast and weno1_zt (the exact fast divisions the SL kernels use)
    against weno_1d with the plain IEEE operators on the GPU, 2^26 samples per
    dx: smooth lines, raw bit patterns, lines at the range guards (squared
    second differences at 2^-700 and 2^200, differences at 2^-1021), tiny and
    subnormal differences; theta uniform in [-0.7, 1.7] and at the guards
    (-1/2, 0, -0, 3/2, +-2^-510, +-2^-511 and neighbours). Whenever a fast
    form's guards pass, its bits must equal weno_1d's."""
    lsr = gpu
    c = lsr._api.selftest_weno(dx, 1 << 26, seed=int(1e6 * dx) + 7)
    assert c["fast_mismatch"] == 0 and c["table_mismatch"] == 0, c
    # the guards must not reject the common case: most samples take the fast path
    assert c["fast_taken"] > (1 << 26) // 10 and c["table_taken"] > (1 << 26) // 10, c


def test_context_multistep_swap_matches_oracle(gpu, oracle):
    """Device-resident loop: K ping-pong steps with changing active sets; the
    sparse resync must reproduce the reference's full copy (evolve.cpp:50)."""
    lsr = gpu
    g = lsr._api.cube_grid(48, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.55
    dist = np.abs(np.sqrt(x * x + y * y + z * z) - 0.3) + 1e-3
    bp = lsr.default_band_params(3, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=bp)
    ccfg = dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma,
                beta=bp.beta)
    gd = dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx)
    ctx = lsr.Context(g)
    ctx.upload(0, phi)
    ctx.upload(1, dist)
    ref = phi.copy()
    for step in range(4):
        active = np.flatnonzero(np.abs(ref) < bp.gamma * (1.0 - 0.15 * step)).astype(np.int64)
        ctx.set_active(active)
        ctx.sl_step(cfg, 0.9)
        ref, st, _ = oracle.sl_step(gd, ref, dist, active, ccfg, 0.9)
        assert st == 0
        got = ctx.download(2)
        assert np.array_equal(bits(got), bits(ref)), step
        ctx.swap()
        assert np.array_equal(bits(ctx.download(0)), bits(ref))


def test_full_size_sampled_subset_512(gpu, oracle):
    """Config-4 size (512^3): GPU vs oracle on a random subset of the band
    (sl_step reads only mask.active, SURVEY §7 'sampled oracle')."""
    lsr = gpu
    rng = np.random.default_rng(11)
    g = lsr._api.cube_grid(512, 3)
    ax = g.axes()
    r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2).ravel()
    phi = r - 0.9
    dist = np.abs(r - 0.5) + 1e-3 * np.cos(7 * r)
    bp = lsr.default_band_params(3, g.dx)
    band = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    sub = np.sort(rng.choice(band, 20000, replace=False)).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=bp)
    got = _run(lsr, g, phi, dist, sub, cfg, 1.3)
    ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, sub,
                                dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=bp.gamma, beta=bp.beta), 1.3, nthreads=0)
    assert st == 0
    assert np.array_equal(bits(got[sub]), bits(ref[sub]))
    # whole band: property checks (finite, unchanged off-band, bounded update)
    out = _run(lsr, g, phi, dist, band, cfg, 1.3)
    assert np.all(np.isfinite(out[band]))
    assert np.array_equal(bits(np.delete(out, band)), bits(np.delete(phi, band)))
    assert np.max(np.abs(out[band] - phi[band])) < 2 * g.dx


@pytest.mark.parametrize("pinned", [False, True], ids=["pageable", "pinned"])
@pytest.mark.parametrize("case", ["sorted", "unsorted", "far_feet", "scattered", "edge_planes"])
def test_pipelined_host_entry_exact(gpu, oracle, case, pinned):
    """The one-shot host entry pipelines 3d grids over z-chunks (slab-mode
    kernels, three streams) and uploads only the d values the gradients read
    (packed row runs); unsorted ids or feet beyond the upload lead must fall
    back to the unpipelined step and stay exact."""
    lsr = gpu
    rng = np.random.default_rng(5)
    g = lsr._api.cube_grid(96, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.6 + 0.2 * g.dx * rng.standard_normal(x.size)
    dist = np.abs(np.sqrt(x * x + y * y + z * z) - 0.3) + 0.01 * rng.random(x.size)
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    e = 0.7
    dt = 0.25 * g.dx
    if case == "unsorted":
        active = active.copy()
        rng.shuffle(active)
    if case == "far_feet":
        dt = 6.0 * g.dx  # displacements of several planes: beyond the pipeline's upload lead
    if case == "scattered":  # isolated ids: one-node runs, neighbours in other rows/planes
        active = np.sort(rng.choice(active, active.size // 9, replace=False)).astype(np.int64)
    if case == "edge_planes":  # the band plus the grid's outer faces (one-sided gradients)
        n = g.dims[0]
        kk, jj, ii = np.unravel_index(np.arange(x.size), (n, n, n))
        face = (ii == 0) | (jj == 0) | (kk == 0) | (ii == n - 1) | (jj == n - 1) | (kk == n - 1)
        active = np.union1d(active, np.flatnonzero(face & (rng.random(x.size) < 0.3))).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=dt, band=bp)
    got = _run(lsr, g, phi, dist, active, cfg, e, pinned)
    if case in ("sorted", "scattered"):  # packed transfers: phi around the band in, the band's values out
        h2d, d2h = lsr._api.last_transfer_bytes()
        assert d2h >= 8 * active.size
        assert case != "sorted" or (h2d < 8 * x.size and d2h < 8 * x.size)
    ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                dict(p=2, interp=1, delta=1.0, dt=dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=bp.gamma, beta=bp.beta), e)
    assert st == 0
    assert np.count_nonzero(bits(got) != bits(ref)) == 0


# ---- z-line table of the 3d WENO path (sl_step.cu: zt_fill_kernel) ----------

def _ctx_step(lsr, g, phi, dist, active, cfg, e):
    ctx = lsr.Context(g)
    try:
        ctx.upload(0, phi)
        ctx.upload(1, dist)
        ctx.set_active(active)
        ctx.sl_step(cfg, e)
        return ctx.download(2), ctx.last_table_ms()
    finally:
        ctx.close()


def _oracle_step(oracle, g, phi, dist, active, cfg, p, delta, e):
    ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                dict(p=p, interp=1, delta=delta, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=cfg.band.gamma, beta=cfg.band.beta), e, nthreads=0)
    assert st == 0
    return ref


@pytest.mark.parametrize("dt_dx,delta", [(0.25, 1.0), (3.0, 1.0), (12.0, 1.0)])
def test_ztab_context_far_feet_exact(gpu, oracle, dt_dx, delta):
    """Device-resident step with the z-line table: feet within the table's
    brick coverage read it, farther feet (large dt) take the per-line
    arithmetic; every node bit-identical to the reference either way."""
    lsr = gpu
    rng = np.random.default_rng(21)
    g = lsr._api.cube_grid(72, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    r = np.sqrt(x * x + y * y + z * z)
    phi = r - 0.55 + 0.2 * g.dx * rng.standard_normal(x.size)
    dist = np.abs(r - 0.3) + 0.02 * rng.random(x.size)
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=delta, dt=dt_dx * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    got, tms = _ctx_step(lsr, g, phi, dist, active, cfg, 0.4)
    assert tms > 0.0  # the table was built
    ref = _oracle_step(oracle, g, phi, dist, active, cfg, 2, delta, 0.4)
    assert np.count_nonzero(bits(got) != bits(ref)) == 0


def test_ztab_out_of_range_data_falls_back_exact(gpu, oracle):
    """Second differences whose squares fall below weno1_fast's range
    (nonzero, < 2^-700) flag the table; the step takes the guarded per-line
    path and stays bit-identical."""
    lsr = gpu
    rng = np.random.default_rng(5)
    g = lsr._api.cube_grid(40, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    r = np.sqrt(x * x + y * y + z * z)
    phi = r - 0.5
    tiny = np.flatnonzero(np.abs(z) < 0.3)
    phi[tiny] = 1e-140 * (1.0 + rng.random(tiny.size))  # a slab of near-zero values
    dist = np.abs(r - 0.3) + 0.01
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    got, _ = _ctx_step(lsr, g, phi, dist, active, cfg, 0.6)
    ref = _oracle_step(oracle, g, phi, dist, active, cfg, 2, 1.0, 0.6)
    assert np.count_nonzero(bits(got) != bits(ref)) == 0


def test_ztab_context_full_size_sampled_512(gpu, oracle):
    """Config-4 size through the device-resident context (table path): a
    random subset of the band vs the oracle, then the whole band against the
    one-shot host path (which does not use the table), bit for bit."""
    lsr = gpu
    rng = np.random.default_rng(17)
    g = lsr._api.cube_grid(512, 3)
    ax = g.axes()
    r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2).ravel()
    phi = r - 0.9
    dist = np.abs(r - 0.5) + 1e-3 * np.cos(9 * r)
    bp = lsr.default_band_params(3, g.dx)
    band = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    sub = np.sort(rng.choice(band, 20000, replace=False)).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    got, _ = _ctx_step(lsr, g, phi, dist, sub, cfg, 1.3)
    ref = _oracle_step(oracle, g, phi, dist, sub, cfg, 2, 1.0, 1.3)
    assert np.array_equal(bits(got[sub]), bits(ref[sub]))
    whole, _ = _ctx_step(lsr, g, phi, dist, band, cfg, 1.3)
    host = _run(lsr, g, phi, dist, band, cfg, 1.3)
    assert np.array_equal(bits(whole), bits(host))


def test_async_steps_match_sync_steps_and_report_nan(gpu):
    """lsr_cuda_sl_step_async x K + lsr_cuda_sync == K synchronous steps, bit
    for bit; a non-finite update surfaces at the sync with the node's id."""
    lsr = gpu
    g = lsr._api.cube_grid(56, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    r = np.sqrt(x * x + y * y + z * z)
    phi = r - 0.55
    dist = np.abs(r - 0.3) + 1e-3
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    res = []
    for mode in ("sync", "async"):
        ctx = lsr.Context(g)
        ctx.upload(0, phi)
        ctx.upload(1, dist)
        ctx.set_active(active)
        for _ in range(5):
            if mode == "sync":
                ctx.sl_step(cfg, 0.7)
            else:
                ctx.sl_step_async(cfg, 0.7)
            ctx.swap()
        if mode == "async":
            ctx.sync()
            k, s, t = ctx.async_times()
            assert len(k) == 5 and all(v > 0 for v in k) and all(a >= b for a, b in zip(s, k))
        res.append(ctx.download(0))
        ctx.close()
    assert np.array_equal(bits(res[0]), bits(res[1]))
    # NaN in d at one active node: reported by the sync, not by the enqueue
    bad_id = int(active[len(active) // 2])
    d2 = dist.copy()
    d2[bad_id] = np.nan
    ctx = lsr.Context(g)
    ctx.upload(0, phi)
    ctx.upload(1, d2)
    ctx.set_active(active)
    ctx.sl_step_async(cfg, 0.7)
    with pytest.raises(lsr.NumericalError):
        ctx.sync()
    assert ctx.bad_node >= 0
    ctx.close()


@pytest.mark.parametrize("dims,dt_dx", [((45, 37, 41), 0.25), ((33, 50, 29), 2.0)])
def test_ztab_ragged_grid_exact(gpu, oracle, dims, dt_dx):
    """Table path on non-cubic grids whose sizes are not multiples of the 4^3
    bricks (partial bricks at the high faces), vs the oracle bit for bit."""
    lsr = gpu
    rng = np.random.default_rng(sum(dims))
    dx = 2.0 / 48
    g = lsr.Grid(3, (-0.9, -0.8, -0.85), dx, dims)
    x, y, z = (a.ravel() for a in g.mesh())  # x fastest
    r = np.sqrt((x + 0.1) ** 2 + y ** 2 + (z + 0.05) ** 2)
    phi = r - 0.5 + 0.1 * dx * rng.standard_normal(x.size)
    dist = np.abs(r - 0.3) + 0.01 * rng.random(x.size)
    bp = lsr.default_band_params(3, dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=dt_dx * dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    got, tms = _ctx_step(lsr, g, phi, dist, active, cfg, 0.5)
    assert tms > 0.0
    ref, st, _ = oracle.sl_step(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, dist, active,
                                dict(p=2, interp=1, delta=1.0, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0,
                                     gamma=bp.gamma, beta=bp.beta), 0.5, nthreads=0)
    assert st == 0
    assert np.count_nonzero(bits(got) != bits(ref)) == 0


@pytest.mark.parametrize("dim,interp", [(2, 0), (3, 0), (3, 1)])
def test_empty_active_set_copies_phi(gpu, dim, interp):
    """An empty BandMask::active: out = phi everywhere (evolve.cpp:50), through
    the one-shot call, the synchronous context step and the async one."""
    lsr = gpu
    g = lsr._api.cube_grid(20 if dim == 3 else 64, dim)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.5
    dist = np.abs(phi) + 0.01
    bp = lsr.default_band_params(dim, g.dx)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, interp=lsr.InterpolatorKind(interp), band=bp)
    none = np.zeros(0, np.int64)
    assert np.array_equal(bits(_run(lsr, g, phi, dist, none, cfg, 0.5)), bits(phi))
    ctx = lsr.Context(g)
    try:
        ctx.upload(0, phi)
        ctx.upload(1, dist)
        ctx.set_active(none)
        ctx.sl_step(cfg, 0.5)
        assert np.array_equal(bits(ctx.download(2)), bits(phi))
        ctx.sl_step_async(cfg, 0.5)
        ctx.sync()
        assert np.array_equal(bits(ctx.download(2)), bits(phi))
    finally:
        ctx.close()


def test_async_rejects_bad_config_before_any_work(gpu):
    """sl_step_async validates like sl_step (evolve.hpp:25-30, evolve.cpp:45-46)
    and refuses a synchronous step while async steps are pending."""
    lsr = gpu
    g = lsr._api.cube_grid(16, 3)
    phi = np.zeros(g.num_nodes()) + 0.1
    ctx = lsr.Context(g)
    try:
        ctx.upload(0, phi)
        ctx.upload(1, phi)
        ctx.set_active(np.arange(10, dtype=np.int64))
        bp = lsr.default_band_params(3, g.dx)
        with pytest.raises(lsr.ConfigError):
            ctx.sl_step_async(lsr.StepConfig(p=2, delta=1.0, dt=0.0, band=bp), 0.5)
        with pytest.raises(lsr.Error):
            ctx.sl_step_async(lsr.StepConfig(p=2, delta=1.0, dt=0.1 * g.dx, band=bp), 0.0)  # E <= 0 with p > 1
        good = lsr.StepConfig(p=2, delta=1.0, dt=0.1 * g.dx, band=bp)
        ctx.sl_step_async(good, 0.5)
        with pytest.raises(lsr.ConfigError):
            ctx.sl_step(good, 0.5)
        ctx.sync()
        ctx.sl_step(good, 0.5)
    finally:
        ctx.close()


@pytest.mark.parametrize("n,p,delta,seed", [(64, 1, 0.0, 5), (64, 2, 1.0, 6), (80, 2, 0.3, 7), (96, 1, 1.0, 8)])
def test_ztab_context_seeded_vs_oracle(gpu, oracle, n, p, delta, seed):
    """The seeded WENO-3D cases through the device-resident context (z-line
    table path for delta > 0; the one-shot call takes the pipelined path at
    these sizes), including p = 1 and delta = 0 (coinciding feet, no table),
    vs the oracle."""
    lsr = gpu
    rng = np.random.default_rng(seed)
    g = lsr._api.cube_grid(n, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.6 + 0.25 * g.dx * rng.standard_normal(x.size)
    dist = np.abs(np.sqrt((x - 0.07) ** 2 + (y + 0.03) ** 2 + z * z) - 0.35) + 0.01 * rng.random(x.size)
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=p, delta=delta, dt=0.25 * g.dx, interp=lsr.InterpolatorKind.Weno, band=bp)
    got, tms = _ctx_step(lsr, g, phi, dist, active, cfg, 0.7)
    assert (tms > 0.0) == (delta > 0.0)  # delta = 0 (coinciding feet) runs without the table
    ref = _oracle_step(oracle, g, phi, dist, active, cfg, p, delta, 0.7)
    assert np.count_nonzero(bits(got) != bits(ref)) == 0


def test_context_rejects_out_of_grid_ids(gpu):
    """Active ids are node ids (grid.hpp:79-84): host and device id lists
    outside the grid are ConfigErrors before any kernel dereferences them."""
    import torch

    lsr = gpu
    g = lsr._api.cube_grid(12, 3)
    ctx = lsr.Context(g)
    with pytest.raises(lsr.ConfigError, match="node ids"):
        ctx.set_active(np.array([0, g.num_nodes()], dtype=np.int64))
    bad = torch.tensor([3, -2, 5], dtype=torch.int64, device="cuda")
    with pytest.raises(lsr.ConfigError, match="node ids"):
        ctx.set_active_device(bad.data_ptr(), bad.numel())
    ok = torch.arange(10, dtype=torch.int64, device="cuda")
    ctx.set_active_device(ok.data_ptr(), ok.numel())
    ctx.close()


@pytest.mark.parametrize("pinned", [False, True])
def test_one_shot_out_of_grid_ids_are_config_error(gpu, pinned):
    """The one-shot host call's pipelined path (3d, >= 64 planes; pinned =
    zero-copy pull, pageable = host packing) with an id past the grid: no
    kernel or host scatter dereferences it, the call raises ConfigError."""
    lsr = gpu
    g = lsr._api.cube_grid(64, 3)
    x, y, z = g.mesh()
    phi = (np.sqrt(x * x + y * y + z * z) - 0.6).ravel()
    dist = np.abs(phi) + 0.01
    active = np.flatnonzero(np.abs(phi) < 6 * g.dx).astype(np.int64)
    active = np.append(active, g.num_nodes() + 5)
    cfg = lsr.StepConfig(p=2, delta=1.0, dt=0.25 * g.dx, band=lsr.default_band_params(3, g.dx))
    with pytest.raises(lsr.ConfigError, match="node ids"):
        _run(lsr, g, phi, dist, active, cfg, 1.3, pinned=pinned)


@pytest.mark.parametrize("n,dt_dx,delta,dims", [(40, 0.25, 1.0, None), (48, 2.0, 0.5, None), (0, 0.25, 1.0, (36, 44, 52)),
                                               (64, 6.0, 1.0, None)])
def test_tma_brick_step_matches_table_step(gpu, oracle, n, dt_dx, delta, dims):
    """The TMA-brick form of the 3d WENO step (lsr_cuda_set_sl_mode 1: each
    8^3 brick's phi and halo staged by one tensor copy; feet beyond the box
    read global memory) gives the z-line-table step's bits and the oracle's,
    including far feet (dt = 6 dx) and a ragged grid."""
    lsr = gpu
    dims = dims or (n, n, n)
    g = lsr.Grid(3, (-1.0, -1.0, -1.0), 2.0 / (max(dims) - 1), dims)
    x, y, z = g.mesh()
    r = np.sqrt(x * x + y * y + z * z)
    phi = (r - 0.6 + 0.05 * np.sin(4 * x) * np.cos(3 * y)).ravel()
    dist = (np.abs(np.sqrt((x - 0.05) ** 2 + y * y + z * z) - 0.35) + 0.01).ravel()
    bp = lsr.default_band_params(3, g.dx)
    active = np.flatnonzero(np.abs(phi) < bp.gamma).astype(np.int64)
    cfg = lsr.StepConfig(p=2, delta=delta, dt=dt_dx * g.dx, band=bp, interp=lsr.InterpolatorKind(1))
    outs = []
    for mode in (0, 1):
        ctx = lsr.Context(g)
        ctx.set_sl_mode(mode)
        ctx.upload(0, phi)
        ctx.upload(1, dist)
        ctx.set_active(active)
        for _ in range(2):  # a second step exercises the cached brick grouping
            ctx.sl_step(cfg, 1.3)
        outs.append(ctx.download(2))
        ctx.close()
    assert np.array_equal(bits(outs[0]), bits(outs[1]))
    cc = dict(p=2, interp=1, delta=delta, dt=cfg.dt, fallback_c=1e-3, fallback_alpha=1.0, gamma=bp.gamma, beta=bp.beta)
    gd = dict(dim=3, dims=list(dims), origin=[-1.0, -1.0, -1.0], dx=g.dx)
    ref, st, _ = oracle.sl_step(gd, phi, dist, active, cc, 1.3)
    assert st == 0
    assert np.array_equal(bits(outs[1][active]), bits(ref[active]))
