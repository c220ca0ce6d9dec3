"""CPU tests of the C-ABI library: it loads without a GPU, exports every
symbol include/lsr_cuda.h declares, and rejects bad configurations with the
reference's error classes *before* any device work (evolve.cpp:42-46), so
these run on a machine without CUDA."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_grid, load_golden

HEADER = os.path.join(ROOT, "include", "lsr_cuda.h")
HEADERS = [HEADER, os.path.join(ROOT, "include", "lsr_workloads.h")]


def declared_symbols():
    """Every function the C headers declare (lsr_cuda_* and lsr_cloud_*)."""
    out = set()
    for h in HEADERS:
        out |= set(re.findall(r"\b(lsr_(?:cuda|cloud)_\w+)\s*\(", open(h).read()))
    return sorted(out)


def test_library_exports_every_declared_symbol(built):
    import paper_2410_22205_b200 as lsr

    L = lsr.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s


def test_no_cpu_fallback_symbols_in_product(built):
    """The product library never links the oracle."""
    import paper_2410_22205_b200 as lsr

    L = lsr.lib()
    for s in ("lsro_sl_step", "lsrref_sl_step"):
        assert not hasattr(L, s)
    import sys

    assert "oracle" not in {m.split(".")[0] for m in sys.modules if m.startswith("paper_2410_22205_b200")}


def _args(g=None):
    import paper_2410_22205_b200 as lsr

    g = g or lsr._api.cube_grid(9, 2)
    return lsr, g, lsr.ScalarField(g), lsr.DistanceField(lsr.ScalarField(g)), lsr.BandMask(g)


@pytest.mark.parametrize("bad,exc", [
    (dict(dt=0.0), "ConfigError"),
    (dict(p=3), "ConfigError"),
    (dict(delta=1.5), "ConfigError"),
    (dict(delta=-0.1), "ConfigError"),
])
def test_config_errors_before_device_work(built, bad, exc):
    lsr, g, phi, d, m = _args()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    for k, v in bad.items():
        setattr(cfg, k, v)
    with pytest.raises(getattr(lsr, exc)):
        lsr.sl_step(phi, d, m, cfg, 1.0, lsr.ScalarField(g))


def test_band_and_energy_errors(built):
    lsr, g, phi, d, m = _args()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.5))
    with pytest.raises(lsr.ConfigError):
        lsr.sl_step(phi, d, m, cfg, 1.0, lsr.ScalarField(g))
    cfg = lsr.StepConfig(p=2, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    with pytest.raises(lsr.Error) as ei:
        lsr.sl_step(phi, d, m, cfg, 0.0, lsr.ScalarField(g))
    assert type(ei.value) is lsr.Error  # plain Error, as evolve.cpp:45-46


def test_grid_mismatch_is_config_error(built):
    lsr, g, phi, d, m = _args()
    g2 = lsr._api.cube_grid(11, 2)
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    with pytest.raises(lsr.ConfigError):
        lsr.sl_step(phi, lsr.DistanceField(lsr.ScalarField(g2)), m, cfg, 1.0, lsr.ScalarField(g))


def test_unknown_interpolator_is_config_error(built):
    lsr, g, phi, d, m = _args()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    cfg.interp = 7
    with pytest.raises(lsr.ConfigError):
        lsr.sl_step(phi, d, m, cfg, 1.0, lsr.ScalarField(g))


def test_golden_fixture_coverage():
    """The golden cases exercise the branches the kernel must get right:
    gradient fallback (evolve.cpp:65-78), boundary stencils (interp.cpp:46)."""
    rec = load_golden("sl_flat3d.npz")
    g = golden_grid(rec)
    nx, ny, nz = g["dims"]
    phi = rec["phi"].reshape(nz, ny, nx)
    gx = np.gradient(phi, axis=2) / g["dx"]
    gy = np.gradient(phi, axis=1) / g["dx"]
    gz = np.gradient(phi, axis=0) / g["dx"]
    gn = np.sqrt(gx * gx + gy * gy + gz * gz).ravel()[rec["active"]]
    assert np.count_nonzero(gn < 1e-3 * 0.25 * g["dx"]) > 50
    rec = load_golden("sl_hull3d.npz")
    g = golden_grid(rec)
    k = rec["active"] // (g["dims"][0] * g["dims"][1])
    assert np.count_nonzero((k <= 1) | (k >= g["dims"][2] - 2)) > 100


@pytest.mark.gpu
@pytest.mark.parametrize("ids", [[-1], [10**9], [0, 5, 1 << 40]])
def test_out_of_grid_ids_are_config_error(gpu, ids):
    """An id outside the grid is never dereferenced (device kernels and the
    host scatter skip it) and the step reports a ConfigError."""
    lsr, g, phi, d, m = _args()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    bad = lsr.BandMask(g, active=np.asarray(ids, dtype=np.int64))
    with pytest.raises(lsr.ConfigError, match="node ids"):
        lsr.sl_step(phi, d, bad, cfg, 1.0, lsr.ScalarField(g))


def test_short_host_arrays_are_config_error(built):
    lsr, g, phi, d, m = _args()
    cfg = lsr.StepConfig(p=1, delta=0.0, dt=0.1, band=lsr.BandParams(0.4, 0.2))
    short = lsr.ScalarField(g, np.zeros(g.num_nodes() - 1))
    with pytest.raises(lsr.ConfigError):
        lsr.sl_step(short, d, m, cfg, 1.0, lsr.ScalarField(g))
