"""CPU tests: the oracle restatement (oracle/lsr_oracle.c) is pinned against
(a) the golden fixtures produced by the reference itself and (b) the live
reference library (oracle/_ref) on fresh seeded inputs, including the
reference's own known-answer cases (test_evolve.cpp, test_interp.cpp,
test_grid.cpp)."""
import numpy as np
import pytest

from conftest import SL_CASES, bits, golden_grid, load_golden


def cfg_of(rec, c):
    return dict(p=int(rec["case_p"][c]), interp=int(rec["case_interp"][c]), delta=float(rec["case_delta"][c]),
                dt=0.25 * float(rec["dx"]), fallback_c=1e-3, fallback_alpha=1.0, gamma=float(rec["gamma"]),
                beta=float(rec["beta"]))


@pytest.mark.parametrize("case", SL_CASES)
def test_restatement_matches_golden_sl_step(oracle, case):
    rec = load_golden(f"sl_{case}.npz")
    g = golden_grid(rec)
    for c in range(len(rec["case_p"])):
        out, st, bad = oracle.sl_step(g, rec["phi"], rec["dist"], rec["active"], cfg_of(rec, c), float(rec["e2"]))
        assert st == 0
        assert np.array_equal(bits(out[rec["active"]]), bits(rec["case_out"][c])), (case, c)
        # non-active nodes copy phi exactly (test_evolve.cpp:178-193)
        mask = np.ones(out.size, bool)
        mask[rec["active"]] = False
        assert np.array_equal(bits(out[mask]), bits(rec["phi"][mask]))


def test_restatement_weno_1d_golden(oracle):
    rec = load_golden("weno_1d.npz")
    got = np.array([oracle.weno_1d(rec["v"][i], rec["dx"][i], rec["theta"][i]) for i in range(len(rec["dx"]))])
    assert np.array_equal(bits(got), bits(rec["out"]))


@pytest.mark.parametrize("dim", [2, 3])
def test_restatement_interp_golden(oracle, dim):
    rec = load_golden(f"interp_{dim}d.npz")
    g = golden_grid(rec)
    for kind, key in ((0, "q1"), (1, "weno")):
        got = np.array([oracle.interp(kind, g, rec["f"], p) for p in rec["pts"]])
        assert np.array_equal(bits(got), bits(rec[key])), key


def test_restatement_basis_golden(oracle):
    rec = load_golden("basis.npz")
    for i, gr in enumerate(rec["grad"]):
        v1, v2 = oracle.tangent_basis(3, gr)
        assert np.array_equal(bits(v1), bits(rec["v1_3"][i])) and np.array_equal(bits(v2), bits(rec["v2_3"][i]))
        w1, _ = oracle.tangent_basis(2, np.array([gr[0], gr[1], 0.0]))
        assert np.array_equal(bits(w1), bits(rec["v1_2"][i]))


@pytest.mark.parametrize("dim", [2, 3])
def test_restatement_band_golden(oracle, dim):
    rec = load_golden(f"band_{dim}d.npz")
    st, act, tube = oracle.narrow_band(golden_grid(rec), rec["phi"], float(rec["gamma"]))
    assert np.array_equal(st, rec["state"])
    assert np.array_equal(act, rec["active"]) and np.array_equal(tube, rec["tube"])


# ---- live comparison with the reference library (this container) ---------


def _mesh(g):
    ax = [g["origin"][d] + np.arange(g["dims"][d]) * g["dx"] for d in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return x.ravel(), y.ravel(), z.ravel()


def _grid(n, dim):
    dx = 2.0 / (n - 1)
    return dict(dim=dim, dims=[n, n, n if dim == 3 else 1], origin=[-1.0, -1.0, -1.0 if dim == 3 else 0.0], dx=dx)


@pytest.mark.parametrize("dim,n,seed", [(2, 97, 1), (3, 36, 2), (3, 41, 3)])
def test_restatement_equals_reference_random(reference, oracle, dim, n, seed):
    rng = np.random.default_rng(seed)
    g = _grid(n, dim)
    x, y, z = _mesh(g)
    phi = np.sqrt(x * x + y * y + z * z) - 0.55 + 0.3 * g["dx"] * rng.standard_normal(x.size)
    dist = np.abs(np.sqrt((x - 0.1) ** 2 + y * y + z * z) - 0.3) + 0.02 * rng.random(x.size)
    gam = (6.0 if dim == 3 else 4.0) * g["dx"]
    _, act, _ = reference.narrow_band(g, phi, gam)
    for interp in (0, 1):
        for p, delta in ((1, 0.0), (2, 1.0), (1, 0.7)):
            cfg = dict(p=p, interp=interp, delta=delta, dt=0.25 * g["dx"], fallback_c=1e-3, fallback_alpha=1.0,
                       gamma=gam, beta=gam / 2)
            ref, st, msg, _ = reference.sl_step(g, phi, dist, act, cfg, 0.61, serial=True)
            assert st == 0, msg
            got, st2, _ = oracle.sl_step(g, phi, dist, act, cfg, 0.61)
            assert st2 == 0
            assert np.array_equal(bits(ref), bits(got)), (interp, p, delta)


def test_reference_openmp_equals_serial_twin(reference):
    """lsr::sl_step (OpenMP) == lsr::ref::sl_step bit for bit."""
    g = _grid(40, 3)
    x, y, z = _mesh(g)
    phi = np.sqrt(x * x + y * y + z * z) - 0.7
    dist = np.abs(np.sqrt(x * x + y * y + z * z) - 0.3)
    gam = 6 * g["dx"]
    _, act, _ = reference.narrow_band(g, phi, gam)
    cfg = dict(p=2, interp=1, delta=1.0, dt=0.25 * g["dx"], fallback_c=1e-3, fallback_alpha=1.0, gamma=gam,
               beta=gam / 2)
    a = reference.sl_step(g, phi, dist, act, cfg, 0.9, serial=True)[0]
    b = reference.sl_step(g, phi, dist, act, cfg, 0.9, serial=False)[0]
    assert np.array_equal(bits(a), bits(b))


def test_oracle_nan_distance_reports_smallest_bad_node(oracle, reference):
    """test_evolve.cpp:195-210: a NaN in d surfaces as NumericalError."""
    g = _grid(41, 2)
    x, y, _ = _mesh(g)
    phi = np.sqrt(x * x + y * y) - 0.6
    dist = np.full(x.size, 0.5)
    gam = 4 * g["dx"]
    _, act, _ = oracle.narrow_band(g, phi, gam)
    poisoned = act[[len(act) // 2, len(act) // 3]]
    dist[poisoned] = np.nan
    cfg = dict(p=2, interp=1, delta=1.0, dt=0.02, fallback_c=1e-3, fallback_alpha=1.0, gamma=gam, beta=gam / 2)
    out, st, bad = oracle.sl_step(g, phi, dist, act, cfg, 1.0)
    ref, st_ref, msg, _ = reference.sl_step(g, phi, dist, act, cfg, 1.0, serial=False)
    assert st_ref == 3 and "non-finite update" in msg
    # out is fully written (evolve.cpp:110-117); NaN d also poisons the
    # neighbours' centered gradient of d, so the first bad id precedes `poisoned`
    assert np.array_equal(bits(out), bits(ref))
    assert st == 3 and bad == np.flatnonzero(~np.isfinite(ref)).min() <= poisoned.min()


def test_oracle_config_errors(oracle):
    g = _grid(9, 2)
    phi = np.zeros(81)
    base = dict(p=1, interp=1, delta=0.0, dt=0.1, fallback_c=1e-3, fallback_alpha=1.0, gamma=0.4, beta=0.2)
    for bad in (dict(dt=0.0), dict(p=3), dict(delta=1.5), dict(beta=0.5), dict(beta=0.0), dict(interp=7)):
        _, st, _ = oracle.sl_step(g, phi, phi, np.zeros(0, np.int64), {**base, **bad}, 1.0)
        assert st == 1, bad
    _, st, _ = oracle.sl_step(g, phi, phi, np.zeros(0, np.int64), {**base, "p": 2}, 0.0)
    assert st == 2  # energy must be positive for p > 1 (evolve.cpp:45-46)
