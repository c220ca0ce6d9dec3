"""CPU tests of the one-shot step's packed uploads (csrc/host_pack.cpp): the
d values the pipelined lsr_cuda_sl_step_host uploads must be exactly the
active nodes and their in-grid axis neighbours — every value the centered
gradient of d reads (reference src/grid.cpp:53-74 via src/evolve.cpp:57-66)
and nothing else — and the phi values exactly the Chebyshev ball of radius R
around every active node, clipped to the grid. No GPU needed."""
import numpy as np
import pytest


def _needed(dims, ids):
    nx, ny, nz = dims
    m = np.zeros(nx * ny * nz, bool)
    m[ids] = True
    v = m.reshape(nz, ny, nx)
    need = v.copy()
    need[:, :, 1:] |= v[:, :, :-1]
    need[:, :, :-1] |= v[:, :, 1:]
    need[:, 1:, :] |= v[:, :-1, :]
    need[:, :-1, :] |= v[:, 1:, :]
    need[1:, :, :] |= v[:-1, :, :]
    need[:-1, :, :] |= v[1:, :, :]
    return need.ravel()


def _case(n, kind, seed=0):
    import paper_2410_22205_b200 as lsr

    g = lsr.Grid(dim=3, origin=(-1.0, -1.0, -1.0), dx=0.05, dims=tuple(n))
    rng = np.random.default_rng(seed)
    N = n[0] * n[1] * n[2]
    if kind == "shell":
        z, y, x = np.meshgrid(*[np.linspace(-1, 1, k) for k in (n[2], n[1], n[0])], indexing="ij")
        r = np.sqrt(x * x + y * y + z * z).ravel()
        ids = np.nonzero(np.abs(r - 0.6) < 0.15)[0]
    elif kind == "random":
        ids = np.unique(rng.integers(0, N, N // 7))
    elif kind == "faces":  # nodes on every face, edge and corner of the box
        z, y, x = np.unravel_index(np.arange(N), (n[2], n[1], n[0]))
        on = (x == 0) | (y == 0) | (z == 0) | (x == n[0] - 1) | (y == n[1] - 1) | (z == n[2] - 1)
        ids = np.nonzero(on & (rng.random(N) < 0.5))[0]
    elif kind == "dups":
        ids = np.sort(np.concatenate([rng.integers(0, N, 300)] * 2))
    else:
        ids = np.zeros(0, np.int64)
    d = rng.standard_normal(N)
    return g, lsr.DistanceField(field=lsr.ScalarField(g, d)), ids.astype(np.int64)


def _ball(dims, ids, R):
    from scipy.ndimage import binary_dilation

    nx, ny, nz = dims
    m = np.zeros(nx * ny * nz, bool)
    m[ids] = True
    return binary_dilation(m.reshape(nz, ny, nx), structure=np.ones((3, 3, 3), bool), iterations=R).ravel() \
        if ids.size else m


@pytest.mark.parametrize("kind", ["shell", "random", "faces", "dups", "empty"])
@pytest.mark.parametrize("n", [(24, 24, 24), (17, 9, 31), (2, 5, 7), (33, 2, 3)])
@pytest.mark.parametrize("reach", [0, 3, 5])
def test_packed_sets(built, n, kind, reach):
    import paper_2410_22205_b200 as lsr

    g, dist, ids = _case(n, kind)
    phi = np.random.default_rng(1).standard_normal(dist.field.values.size)
    dfield = np.full(phi.size, np.nan)
    pfield = np.full(phi.size, np.nan)
    nv, nr, pv, pr = lsr._api.pack_host(dist, ids, dfield, reach, phi, pfield)
    need = _needed(n, ids)
    assert np.array_equal(~np.isnan(dfield), need)
    assert nv == int(need.sum())
    assert np.array_equal(dfield[need], dist.field.values[need])
    assert (nr == 0) == (nv == 0)
    if reach == 0:
        assert pv == pr == 0 and np.all(np.isnan(pfield))
        return
    ball = _ball(n, ids, reach)
    assert np.array_equal(~np.isnan(pfield), ball)
    assert pv == int(ball.sum())
    assert np.array_equal(pfield[ball], phi[ball])


def test_unsorted_or_out_of_grid_ids_are_rejected(built):
    import paper_2410_22205_b200 as lsr

    g, dist, ids = _case((16, 16, 16), "random")
    field = np.zeros(dist.field.values.size)
    bad = ids.copy()
    bad[[3, 10]] = bad[[10, 3]]
    with pytest.raises(lsr.ConfigError):
        lsr._api.pack_host(dist, bad, field)
    for extra in ([-1], [16 ** 3]):
        with pytest.raises(lsr.ConfigError):
            lsr._api.pack_host(dist, np.sort(np.concatenate([ids, extra])), field)
