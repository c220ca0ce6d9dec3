"""CPU check of the identity behind band_reinit.cu:godunov_interior: per
axis, the reference's max(sqr(max(dm/dx, 0)), sqr(min(dp/dx, 0))) (reinit.cpp:
78-81, and the mirrored pair for sgn <= 0) equals sqr(c/dx) for c the
larger-magnitude one of max(dm, 0), min(dp, 0) — bit for bit, in IEEE fp64
(numpy divides and multiplies with round-to-nearest)."""
import numpy as np


def smax(a, b):  # std::max
    return np.where(a < b, b, a)


def smin(a, b):  # std::min
    return np.where(b < a, b, a)


def reference_term(dm, dp, dx, sgn):
    dminus, dplus = dm / dx, dp / dx
    if sgn > 0:
        a, b = smax(dminus, 0.0), smin(dplus, 0.0)
    else:
        a, b = smin(dminus, 0.0), smax(dplus, 0.0)
    return smax(a * a, b * b)


def selected_term(dm, dp, dx, sgn):
    if sgn > 0:
        u, v = smax(dm, 0.0), smin(dp, 0.0)
    else:
        u, v = smin(dm, 0.0), smax(dp, 0.0)
    c = np.where(np.abs(u) < np.abs(v), v, u)
    q = c / dx
    return q * q


def flipped_term(dm, dp, dx, sgn):
    """godunov_interior as shipped: for sgn <= 0 both differences are negated
    (a sign-bit flip) and the sgn > 0 pair max(., 0), min(., 0) is used."""
    if not sgn > 0:
        dm, dp = -dm, -dp
    u, v = smax(dm, 0.0), smin(dp, 0.0)
    c = np.where(np.abs(u) < np.abs(v), v, u)
    q = c / dx
    return q * q


def test_one_division_per_axis_is_bit_exact():
    rng = np.random.default_rng(7)
    n = 2_000_000
    dx = 2.0 / 511
    base = rng.standard_normal(n) * dx
    # values, exact ties, near-ties (1 ulp apart), signed zeros, tiny values
    dm = np.concatenate([base, base, base, np.zeros(1000), -np.zeros(1000), base[:1000] * 1e-300])
    dp = np.concatenate([rng.standard_normal(n) * dx, -base, np.nextafter(-base, 0.0), base[:1000],
                         -base[:1000], base[1000:2000] * 1e-300])
    with np.errstate(all="ignore"):
        for sgn in (1.0, -1.0):
            r = reference_term(dm, dp, dx, sgn)
            s = selected_term(dm, dp, dx, sgn)
            assert np.array_equal(r.view(np.int64), s.view(np.int64)), sgn
            f = flipped_term(dm, dp, dx, sgn)
            assert np.array_equal(r.view(np.int64), f.view(np.int64)), sgn


def test_nan_operands_pick_the_same_term():
    dx = 0.01
    vals = np.array([np.nan, 0.5, -0.5, 0.0])
    dm, dp = np.meshgrid(vals, vals)
    with np.errstate(all="ignore"):
        for sgn in (1.0, -1.0):
            r = reference_term(dm.ravel(), dp.ravel(), dx, sgn)
            s = selected_term(dm.ravel(), dp.ravel(), dx, sgn)
            assert np.array_equal(np.isnan(r), np.isnan(s))
            ok = ~np.isnan(r)
            assert np.array_equal(r[ok].view(np.int64), s[ok].view(np.int64))
            f = flipped_term(dm.ravel(), dp.ravel(), dx, sgn)
            assert np.array_equal(np.isnan(r), np.isnan(f))
            assert np.array_equal(r[ok].view(np.int64), f[ok].view(np.int64))
