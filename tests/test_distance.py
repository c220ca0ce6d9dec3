"""Point-cloud preprocessing: the GPU
lsr::build_distance_field must equal the reference's bit for bit (golden
fixtures from the reference itself; the live reference where present), and
the seeded config clouds must be deterministic with the stated shapes."""
import numpy as np
import pytest

from conftest import bits, golden_grid, load_golden


# ---- CPU: the synthetic config clouds (include/lsr_workloads.h) -----------

@pytest.mark.parametrize("config,n", [(1, 200), (2, 20000), (3, 5000), (4, 200000), (5, 20000)])
def test_cloud_generators_are_seeded_and_shaped(built, config, n):
    import paper_2410_22205_b200 as lsr

    a = lsr.cloud_generate(config, n, seed=7, sigma=0.001)
    b = lsr.cloud_generate(config, n, seed=7, sigma=0.001)
    c = lsr.cloud_generate(config, n, seed=8, sigma=0.001)
    assert np.array_equal(bits(a), bits(b)) and not np.array_equal(a, c)
    assert np.all(np.abs(a) < 1.0)
    r = np.linalg.norm(a, axis=1)
    if config == 1:
        assert np.allclose(r, 0.3) and np.all(a[:, 2] == 0.0)
    if config == 2:
        assert np.allclose(r, 0.5)
    if config == 3:  # torus R = 0.5, r = 0.2 plus noise
        rho = np.hypot(a[:, 0], a[:, 1])
        tube = np.hypot(rho - 0.5, a[:, 2])
        assert np.all(np.abs(tube - 0.2) < 0.01)
    if config == 4:  # bumpy sphere, 10x denser at the poles
        assert np.all((r > 0.45 - 1e-12) & (r < 0.55 + 1e-12))
        z = a[:, 2] / r
        pole, eq = np.mean(np.abs(z) > 0.95), np.mean(np.abs(z) < 0.05)
        # band areas are equal on the sphere; density ratio ~ (1+9*0.975)/(1+9*0.025)
        assert 5.0 < pole / eq < 9.5
    if config == 5:  # three tori along x, all points within r + noise of a core circle
        core = np.min([np.hypot(np.hypot(a[:, 0] - cx, a[:, 1]) - 0.3, a[:, 2]) for cx in (-0.5, 0.0, 0.5)], axis=0)
        assert np.all(core < 0.1 + 0.01)


# ---- GPU: distance field parity ------------------------------------------

DIST_CASES = ["circle2d", "sphere3d", "torus3d", "seedonly3d"]


def _grid(lsr, rec):
    g = golden_grid(rec)
    return lsr.Grid(g["dim"], tuple(g["origin"]), g["dx"], tuple(g["dims"]))


@pytest.mark.gpu
@pytest.mark.parametrize("case", DIST_CASES)
def test_build_distance_bit_exact_vs_reference_golden(gpu, case):
    lsr = gpu
    rec = load_golden(f"dist_{case}.npz")
    g = _grid(lsr, rec)
    d = lsr.build_distance_field(g, rec["pts"], int(rec["dim"]), seed_only=bool(rec["seed_only"]))
    assert np.array_equal(d.exact, rec["exact"])
    assert d.sentinel == float(rec["sentinel"])
    assert d.rounds == int(rec["rounds"])
    diff = np.count_nonzero(bits(d.field.values) != bits(rec["d"]))
    assert diff == 0, f"{diff} nodes differ"


@pytest.mark.gpu
def test_build_distance_bit_exact_vs_live_reference(gpu, reference):
    lsr = gpu
    g = lsr._api.cube_grid(48, 3)
    pts = lsr.cloud_generate(3, 20000, seed=3, sigma=0.5 * g.dx)
    d = lsr.build_distance_field(g, pts)
    ref, ex, sent, rounds = reference.build_distance(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), pts, 3)
    assert d.rounds == rounds and np.array_equal(d.exact, ex)
    assert np.array_equal(bits(d.field.values), bits(ref))


@pytest.mark.gpu
def test_build_distance_errors(gpu):
    lsr = gpu
    g = lsr._api.cube_grid(17, 3)
    with pytest.raises(lsr.OutOfDomainError):
        lsr.build_distance_field(g, np.array([[0.0, 0.0, 1.5]]))
    with pytest.raises(lsr.ConfigError):
        lsr.build_distance_field(g, np.array([[0.0, 0.0, 0.0]]), dim=2)
    with pytest.raises(lsr.Error):
        lsr.build_distance_field(g, np.zeros((0, 3)))


@pytest.mark.gpu
def test_distance_512_properties(gpu):
    """Config-4 size: the swept field is an upper bound that is exact on
    seeded nodes; spot-check seeded nodes against brute force."""
    lsr = gpu
    g = lsr._api.cube_grid(512, 3)
    pts = lsr.cloud_generate(4, 200000, seed=1)
    d = lsr.build_distance_field(g, pts)
    assert 1 <= d.rounds <= 8
    seeded = np.flatnonzero(d.exact)
    rng = np.random.default_rng(0)
    for idx in rng.choice(seeded, 50, replace=False):
        i, j, k = g.unflatten(int(idx))
        q = np.array(g.node(i, j, k))
        assert d.field.values[idx] == pytest.approx(np.min(np.linalg.norm(pts - q, axis=1)), rel=1e-13)
    assert np.all(d.field.values[seeded] <= 3.5 * g.dx)  # 4^3 block around the point's cell
    assert np.all(d.field.values < d.sentinel)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["circle", "sphere", "torus"])
def test_compute_stats_vs_reference_golden(gpu, name):
    """lsr::compute_stats (cloud.cpp:480): the seeded sample, the exact NN
    distances and blocked_sum order are reproduced bit for bit."""
    lsr = gpu
    rec = load_golden("stats.npz")
    st = lsr.compute_stats(rec[f"{name}_pts"], int(rec[f"{name}_dim"]), float(rec[f"{name}_frac"]), 2.0,
                           int(rec[f"{name}_seed"]))
    assert st.h_s == float(rec[f"{name}_h"]) and st.gamma_s == float(rec[f"{name}_g"])
    assert np.array_equal(np.array(st.bbox_min + st.bbox_max), rec[f"{name}_bb"])


@pytest.mark.gpu
def test_compute_stats_known_answer_and_errors(gpu):
    """test_cloud.cpp: 64 lattice points on the unit circle -> h_S = 2 sin(pi/64)."""
    lsr = gpu
    th = 2 * np.pi * np.arange(64) / 64
    pts = np.stack([np.cos(th), np.sin(th), np.zeros(64)], 1)
    st = lsr.compute_stats(pts, 2, 1.0, 2.0, 3)
    assert st.h_s == pytest.approx(2 * np.sin(np.pi / 64), rel=1e-13)
    assert st.gamma_s == 2.0 * st.h_s
    with pytest.raises(lsr.ConfigError):
        lsr.compute_stats(pts, 2, 0.0)
    with pytest.raises(lsr.Error):
        lsr.compute_stats(pts[:1], 2, 1.0)
