"""Surface energy E_p: the GPU lsr::surface_energy
follows the reference's cells, quadrature and blocked_sum order; the only
difference is |d|^2 = |d|*|d| vs glibc pow, so the bar is a
few ulp (tolerance written below: 16 ulp relative, 3.6e-15)."""
import numpy as np
import pytest

from conftest import golden_grid, load_golden

pytestmark = pytest.mark.gpu
ULP_TOL = 16 * np.finfo(np.float64).eps

CASES = ["circle2d", "circle2d_p1", "sphere3d", "torus3d_r3", "sphere3d_p1"]


@pytest.mark.parametrize("case", CASES)
def test_surface_energy_vs_reference_golden(gpu, case):
    lsr = gpu
    rec = load_golden(f"energy_{case}.npz")
    gg = golden_grid(rec)
    g = lsr.Grid(gg["dim"], tuple(gg["origin"]), gg["dx"], tuple(gg["dims"]))
    e = lsr.surface_energy(lsr.ScalarField(g, rec["phi"]), lsr.DistanceField(lsr.ScalarField(g, rec["d"])),
                           int(rec["p"]), int(rec["refine"]))
    ref = float(rec["energy"])
    assert abs(e - ref) <= ULP_TOL * abs(ref), (e, ref, (e - ref) / ref)


def test_surface_energy_vs_live_reference_256(gpu, reference):
    lsr = gpu
    g = lsr._api.cube_grid(96, 3)
    pts = lsr.cloud_generate(4, 100000, seed=2)
    d = lsr.build_distance_field(g, pts)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.9
    e = lsr.surface_energy(lsr.ScalarField(g, phi), d, 2, 5)
    ref = reference.surface_energy(dict(dim=3, dims=g.dims, origin=g.origin, dx=g.dx), phi, d.field.values, 2, 5)
    assert abs(e - ref) <= ULP_TOL * abs(ref)


def test_energy_context_matches_host_entry(gpu):
    lsr = gpu
    g = lsr._api.cube_grid(40, 3)
    x, y, z = (a.ravel() for a in g.mesh())
    phi = np.sqrt(x * x + y * y + z * z) - 0.7
    d = np.abs(np.sqrt(x * x + y * y + z * z) - 0.4)
    ctx = lsr.Context(g)
    ctx.upload(0, phi)
    ctx.upload(1, d)
    a = ctx.surface_energy(0, 2, 5)
    b = lsr.surface_energy(lsr.ScalarField(g, phi), lsr.DistanceField(lsr.ScalarField(g, d)), 2, 5)
    assert a == b and a > 0
