"""The device-controlled loop (lsr_cuda_loop_run: K iterations of
driver.cpp:187-203 with every count, E_2, the E_2 == 0 skip, the
NoInterface case and the Jacobi stop rule decided on the device, one host
synchronisation per run, iterations after the first replayed from a captured
CUDA graph) against the host-driven loop (lsr_cuda_loop_step, itself pinned
to the reference loop in test_configs_gpu.py / test_endtoend_gpu.py).

The only value the two loops may compute differently is E_2's final
pow(total, 1/2): the host loop calls glibc pow, the device loop takes the
correctly rounded sqrt; glibc's pow returns that same value except in rare
hard cases. So: E_2 within 1 ulp every iteration, and while every E_2 is
bit-equal the fields must be bit-identical (and |active|, |tube|, the sweep
counts equal); after a differing E_2 the fields are held to the north star's
tolerance (1e-12 * gamma)."""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def _setup(lsr, config, n=None, interp=None, p=None, delta=None):
    """BASELINE config `config` (bench.CONFIGS, optionally on an n^dim grid or
    with another step config)."""
    import bench

    c = dict(bench.CONFIGS[config])
    for k, v in (("n", n), ("interp", interp), ("p", p), ("delta", delta)):
        if v is not None:
            c[k] = v
    g, w, step = bench.make_inputs(lsr, c)
    rc = lsr.ReinitConfig.defaults(g.dx, step.band.gamma)
    return g, w["pts"], w["phi"], step, rc


def _compare(lsr, g, pts, phi, cfg, rc, iters, use_graph=True, chunks=None):
    host, dev = lsr.Context(g), lsr.Context(g)
    try:
        for c in (host, dev):
            c.build_distance(pts)
            c.upload(0, phi)
        ref = [host.loop_step(cfg, rc, 5) for _ in range(iters)]
        recs = []
        for k in (chunks or [iters]):
            recs += dev.loop_run(cfg, rc, k, 5, use_graph=use_graph)
        assert len(recs) == iters
        same_e = True
        for it, (a, b) in enumerate(zip(ref, recs)):
            ea, eb = a["energy"], b["energy"]
            assert abs(ea - eb) <= np.spacing(max(abs(ea), abs(eb))), f"iteration {it}: E_2 {ea!r} vs {eb!r}"
            same_e = same_e and ea == eb
            if same_e:
                for key in ("n_active", "n_tube", "reinit_iterations", "had_interface"):
                    assert a[key] == b[key], f"iteration {it}: {key} {a[key]} vs {b[key]}"
        ph, pd = host.download(0), dev.download(0)
        if same_e:
            assert np.array_equal(bits(ph), bits(pd)), f"{np.count_nonzero(bits(ph) != bits(pd))} nodes differ"
        else:
            assert np.max(np.abs(ph - pd)) <= 1e-12 * cfg.band.gamma
        # the context continues like the host loop's: one more host step on both
        a, b = host.loop_step(cfg, rc, 5), dev.loop_step(cfg, rc, 5)
        assert a["n_active"] == b["n_active"] and a["n_tube"] == b["n_tube"]
        if same_e and a["energy"] == b["energy"]:
            assert np.array_equal(bits(host.download(0)), bits(dev.download(0)))
        return recs
    finally:
        host.close()
        dev.close()


@pytest.mark.parametrize("config,iters", [(2, 30), (3, 12), (4, 5)])
def test_loop_run_matches_host_loop(gpu, config, iters):
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, config)
    recs = _compare(lsr, g, pts, phi, cfg, rc, iters)
    assert all(r["reinit_iterations"] > 0 for r in recs)
    assert all(sum(r["ms"]) > 0 for r in recs)
    # the run's first one-step visits every node; the smooth fields after it
    # have no hard jump, so the rest visit the tube only
    assert recs[0]["dense_one_step"] and not any(r["dense_one_step"] for r in recs[1:])


def test_loop_run_2d_config1(gpu):
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 1)
    _compare(lsr, g, pts, phi, cfg, rc, 40)


def test_loop_run_without_graph_and_in_chunks(gpu):
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 3, n=96)
    _compare(lsr, g, pts, phi, cfg, rc, 9, use_graph=False)
    _compare(lsr, g, pts, phi, cfg, rc, 9, chunks=[1, 3, 5])


@pytest.mark.parametrize("p,delta", [(1, 0.0), (2, 0.0), (2, 0.5)])
def test_loop_run_step_configs(gpu, p, delta):
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 2, n=64, interp=1, p=p, delta=delta)
    _compare(lsr, g, pts, phi, cfg, rc, 8)


def test_loop_run_config_errors(gpu):
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 2, n=32)
    ctx = lsr.Context(g)
    try:
        ctx.build_distance(pts)
        ctx.upload(0, phi)
        with pytest.raises(lsr.ConfigError):
            ctx.loop_run(cfg, rc, 0)
        with pytest.raises(lsr.ConfigError):
            ctx.loop_run(cfg, rc, 2, energy_refine=0)
        assert len(ctx.loop_run(cfg, rc, 2)) == 2
    finally:
        ctx.close()


def test_loop_run_hard_jump_keeps_dense_one_step(gpu):
    """A field with opposite-sign neighbours that are both outside the band
    (a "hard jump", here a slab of the far corner flipped to -1): the one-step
    freezes nodes away from the tube, so the device loop must keep visiting
    every node while such pairs exist — and stay bit-identical to the host loop."""
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 2, n=64)
    ax = g.axes()
    x = np.broadcast_to(ax[0][None, None, :], (64, 64, 64)).ravel()
    y = np.broadcast_to(ax[1][None, :, None], (64, 64, 64)).ravel()
    phi = phi.copy()
    phi[(x > 0.9) & (y > 0.9)] = -1.0
    recs = _compare(lsr, g, pts, phi, cfg, rc, 6)
    assert recs[0]["dense_one_step"] and recs[1]["dense_one_step"]


@pytest.mark.parametrize("n", [36, 34, 48])
def test_loop_run_grid_shapes(gpu, n):
    """Row lengths that take the other forms of the band and table passes:
    36 (whole 4-node brick words but no 16-node groups: scalar band passes,
    covered bricks from the state bytes), 34 (neither: covered bricks from the
    active ids), 48 (both, the forms the configs run)."""
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 3, n=n)
    recs = _compare(lsr, g, pts, phi, cfg, rc, 7)
    assert not any(r["dense_one_step"] for r in recs[1:])


def test_loop_run_without_interface(gpu):
    """A field that never changes sign: no interface cell, so E_2 == 0 and the
    SL step is skipped (driver.cpp:191-195), and the one-step finds no
    interface, so only the clamp acts (reinit.cpp:140-144) — decided on the
    device, in the dense first iteration and in the sparse ones after it."""
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 2, n=32)
    ax = g.axes()
    r = np.sqrt(ax[0][None, None, :] ** 2 + ax[1][None, :, None] ** 2 + ax[2][:, None, None] ** 2).ravel()
    phi = r + 0.05  # positive everywhere, inside the band near the centre
    recs = _compare(lsr, g, pts, phi, cfg, rc, 4)
    assert all(r["energy"] == 0.0 and not r["had_interface"] and r["reinit_iterations"] == 0 for r in recs)
    assert all(r["n_active"] > 0 for r in recs)


def test_loop_run_after_distance_change(gpu):
    """The per-brick maxima of d behind the table's coverage are rebuilt when d
    changes: a run, a new cloud on the same context, another run — equal to a
    host-driven loop on a fresh context with the second cloud."""
    lsr = gpu
    g, pts, phi, cfg, rc = _setup(lsr, 3, n=64)
    pts2 = 0.8 * pts
    dev, host = lsr.Context(g), lsr.Context(g)
    try:
        dev.build_distance(pts)
        dev.upload(0, phi)
        dev.loop_run(cfg, rc, 3, 5)
        dev.build_distance(pts2)
        dev.upload(0, phi)
        recs = dev.loop_run(cfg, rc, 4, 5)
        host.build_distance(pts2)
        host.upload(0, phi)
        ref = [host.loop_step(cfg, rc, 5) for _ in range(4)]
        assert [r["n_active"] for r in recs] == [r["n_active"] for r in ref]
        if all(a["energy"] == b["energy"] for a, b in zip(ref, recs)):
            assert np.array_equal(bits(host.download(0)), bits(dev.download(0)))
        else:
            assert np.max(np.abs(host.download(0) - dev.download(0))) <= 1e-12 * cfg.band.gamma
    finally:
        dev.close()
        host.close()
