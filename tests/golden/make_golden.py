"""Generate the golden fixtures under tests/golden/ from the REFERENCE ITSELF.

Run in the build container (where /root/reference exists and oracle/_ref is
built): ``python tests/golden/make_golden.py``. Every expected output in the
fixtures comes from the unmodified reference library (oracle/_ref/liblsr_ref.so,
built from /root/reference/proj/src by oracle/Makefile):

  sl_*.npz      lsr::ref::sl_step (reference.cpp:53) on seeded inputs; the
                distance field is lsr::build_distance_field (distance.cpp:144)
                of a seeded cloud, the band is lsr::narrow_band (grid.cpp:76)
                and E_2 is lsr::surface_energy (metrics.cpp:186) — i.e. the
                inputs the driver loop (driver.cpp:187-194) would feed.
  weno_1d.npz   lsr::weno_1d (interp.cpp:16) on random stencils.
  interp_*.npz  lsr::interp (interp.cpp:113) at random points.
  basis.npz     lsr::tangent_basis (evolve.cpp:10) on random gradients.
  band_*.npz    lsr::narrow_band state/active/tube.

The inputs are stored with the outputs, so the fixtures never need the
reference at test time (the GPU box has no /root/reference).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bindings import Reference, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def grid(n, dim, lo=-1.0, hi=1.0):
    dx = (hi - lo) / (n - 1)
    if dim == 2:
        return dict(dim=2, dims=[n, n, 1], origin=[lo, lo, 0.0], dx=dx)
    return dict(dim=3, dims=[n, n, n], origin=[lo, lo, lo], dx=dx)


def mesh(g):
    ax = [g["origin"][d] + np.arange(g["dims"][d]) * g["dx"] for d in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return x.ravel(), y.ravel(), z.ravel()


def cloud_circle(n, r, rng):
    th = 2 * np.pi * rng.random(n)
    return np.stack([r * np.cos(th), r * np.sin(th), np.zeros(n)], 1)


def cloud_sphere(n, r, rng, c=(0, 0, 0)):
    z = 2 * rng.random(n) - 1
    th = 2 * np.pi * rng.random(n)
    s = np.sqrt(1 - z * z)
    return np.stack([c[0] + r * s * np.cos(th), c[1] + r * s * np.sin(th), c[2] + r * z], 1)


def cloud_torus(n, R, r, sigma, rng):
    u = 2 * np.pi * rng.random(n)
    v = 2 * np.pi * rng.random(n)
    p = np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)], 1)
    return p + sigma * rng.standard_normal(p.shape)


def make_sl_case(R, name, g, phi, pts, perturb=0.0, seed=0, extra=None, energy=None):
    rng = np.random.default_rng(seed)
    d, exact, sent, rounds = R.build_distance(g, pts, g["dim"])
    if perturb:
        phi = phi + perturb * g["dx"] * rng.standard_normal(phi.shape)
    gam = (6.0 if g["dim"] == 3 else 4.0) * g["dx"]
    beta = gam / 2
    _, active, tube = R.narrow_band(g, phi, gam)
    # the reference energy aborts (OpenMP + OutOfDomainError) when the front
    # touches the hull, so the hull cases pass a fixed E_p instead
    e2 = R.surface_energy(g, phi, d, 2, 5) if energy is None else energy
    rec = dict(dims=np.array(g["dims"]), origin=np.array(g["origin"]), dx=g["dx"], dim=g["dim"], phi=phi, dist=d,
               active=active, gamma=gam, beta=beta, e2=e2)
    cases = []
    for interp in (0, 1):
        for p, delta in ((1, 0.0), (2, 1.0), (2, 0.5)):
            cfg = dict(p=p, interp=interp, delta=delta, dt=0.25 * g["dx"], fallback_c=1e-3, fallback_alpha=1.0,
                       gamma=gam, beta=beta)
            out, st, msg, _ = R.sl_step(g, phi, d, active, cfg, e2, serial=True)
            assert st == 0, msg
            out2, st2, _, _ = R.sl_step(g, phi, d, active, cfg, e2, serial=False)
            assert st2 == 0 and np.array_equal(out.view(np.int64), out2.view(np.int64))
            assert np.array_equal(np.delete(out, active), np.delete(phi, active))
            cases.append((interp, p, delta, out[active]))
    rec["case_interp"] = np.array([c[0] for c in cases])
    rec["case_p"] = np.array([c[1] for c in cases])
    rec["case_delta"] = np.array([c[2] for c in cases])
    rec["case_out"] = np.stack([c[3] for c in cases])
    if extra:
        rec.update(extra)
    np.savez_compressed(os.path.join(OUT, f"sl_{name}.npz"), **rec)
    print(name, "nodes", phi.size, "active", active.size, "E2", e2)


def main():
    build(ref=True)
    R = Reference()
    rng = np.random.default_rng(2410_22205)

    # 2d circle (config 1 shape at reduced size): cloud r=0.3, phi0 = |x|-0.9
    g = grid(65, 2)
    x, y, _ = mesh(g)
    make_sl_case(R, "circle2d", g, np.sqrt(x * x + y * y) - 0.9, cloud_circle(200, 0.3, rng))
    # 2d, band reaching the grid hull (stencil fallback + clamped feet)
    g = grid(41, 2)
    x, y, _ = mesh(g)
    make_sl_case(R, "hull2d", g, np.sqrt(x * x + y * y) - 1.0, cloud_circle(150, 0.6, rng), perturb=0.3, seed=3,
                 energy=0.75)
    # 3d sphere (config 2 shape): 20k -> 4k points at r = 0.5, phi0 = |x| - 0.9
    g = grid(28, 3)
    x, y, z = mesh(g)
    make_sl_case(R, "sphere3d", g, np.sqrt(x * x + y * y + z * z) - 0.9, cloud_sphere(4000, 0.5, rng))
    # 3d noisy torus (config 3 shape), perturbed phi for varied stencils
    g = grid(30, 3)
    x, y, z = mesh(g)
    make_sl_case(R, "torus3d", g, np.sqrt(x * x + y * y + z * z) - 0.6,
                 cloud_torus(6000, 0.5, 0.2, 0.5 * g["dx"], rng), perturb=0.2, seed=5)
    # 3d band touching the hull
    g = grid(22, 3)
    x, y, z = mesh(g)
    make_sl_case(R, "hull3d", g, np.sqrt(x * x + y * y + z * z) - 1.05, cloud_sphere(3000, 0.7, rng),
                 perturb=0.3, seed=7, energy=1.25)
    # 3d with flat patches: the gradient fallback (evolve.cpp:65-78) fires
    g = grid(24, 3)
    x, y, z = mesh(g)
    phi = np.sqrt(x * x + y * y + z * z) - 0.6
    phi = np.where(np.abs(x) < 0.25, np.round(phi / (0.5 * g["dx"])) * (0.5 * g["dx"]), phi)
    phi[(np.abs(x) < 0.3) & (z > 0)] = 0.01 * g["dx"]
    make_sl_case(R, "flat3d", g, phi, cloud_sphere(3000, 0.45, rng))

    # weno_1d on random stencils, including flat and kinked data
    n = 4000
    v = rng.standard_normal((n, 4)) * 10.0 ** rng.integers(-6, 3, (n, 1))
    v[:200] = v[:200, :1]  # constant stencils
    v[200:400, 1:] = v[200:400, 1:2] + np.arange(3) * 0.1  # linear right part
    dx = 10.0 ** rng.uniform(-3, -1, n)
    th = rng.random(n)
    th[:50] = 0.0
    th[50:100] = 1.0
    w = np.array([R.weno_1d(v[i], dx[i], th[i]) for i in range(n)])
    np.savez_compressed(os.path.join(OUT, "weno_1d.npz"), v=v, dx=dx, theta=th, out=w)

    # interp at random points (both kinds, 2d and 3d, including the hull and nodes)
    for dim, nn in ((2, 23), (3, 13)):
        g = grid(nn, dim)
        x, y, z = mesh(g)
        f = np.sin(3 * x) * np.cos(2 * y) + z * z - 0.3 * x * y
        m = 3000
        pts = rng.uniform(-1, 1, (m, 3))
        if dim == 2:
            pts[:, 2] = 0.0
        pts[:100] = np.stack(mesh(g), 1)[rng.integers(0, f.size, 100)]  # nodes
        pts[100:150, 0] = 1.0  # upper hull -> last cell
        pts[150:200, 1] = -1.0
        outs = {k: R.interp(k, g, f, pts) for k in (0, 1)}
        np.savez_compressed(os.path.join(OUT, f"interp_{dim}d.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=dim, f=f, pts=pts, q1=outs[0], weno=outs[1])

    # tangent bases
    gr = rng.standard_normal((2000, 3))
    gr[:20] = [0, 1, 0]
    gr[20:40, 0] = 0
    gr[20:40, 2] = 1e-16
    b3 = [R.tangent_basis(3, gr[i]) for i in range(len(gr))]
    b2 = [R.tangent_basis(2, np.array([gr[i, 0], gr[i, 1], 0.0])) for i in range(len(gr))]
    np.savez_compressed(os.path.join(OUT, "basis.npz"), grad=gr, v1_3=np.array([b[0] for b in b3]),
                        v2_3=np.array([b[1] for b in b3]), v1_2=np.array([b[0] for b in b2]))

    # narrow band classification
    for dim, nn in ((2, 57), (3, 26)):
        g = grid(nn, dim)
        x, y, z = mesh(g)
        phi = np.sqrt(x * x + y * y + z * z) - 0.55 + 0.05 * np.sin(7 * x)
        gam = (6.0 if dim == 3 else 4.0) * g["dx"]
        st, act, tube = R.narrow_band(g, phi, gam, serial=True)
        np.savez_compressed(os.path.join(OUT, f"band_{dim}d.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=dim, phi=phi, gamma=gam, state=st,
                            active=act, tube=tube)
    # distance fields: lsr::build_distance_field (distance.cpp:144) and
    # lsr::seed_exact_distance (distance.cpp:8)
    for name, g, pts, seed_only in (
        ("circle2d", grid(65, 2), cloud_circle(200, 0.3, rng), False),
        ("sphere3d", grid(33, 3), cloud_sphere(3000, 0.5, rng), False),
        ("torus3d", grid(37, 3), cloud_torus(5000, 0.5, 0.2, 0.01, rng), False),
        ("seedonly3d", grid(29, 3), cloud_sphere(800, 0.6, rng, c=(0.1, 0.0, -0.05)), True),
    ):
        d, ex, sent, rounds = R.build_distance(g, pts, g["dim"], seed_only=seed_only)
        np.savez_compressed(os.path.join(OUT, f"dist_{name}.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=g["dim"], pts=pts, d=d, exact=ex,
                            sentinel=sent, rounds=rounds, seed_only=int(seed_only))
        print("dist", name, "rounds", rounds, "exact", int(ex.sum()))
    # surface energy: lsr::surface_energy (metrics.cpp:186) with the reference's
    # interface_cells (metrics.cpp:35) — what the driver feeds to sl_step
    for name, g, shape, pts, p, refine in (
        ("circle2d", grid(129, 2), "circle", cloud_circle(300, 0.3, rng), 2, 5),
        ("circle2d_p1", grid(65, 2), "wavy", cloud_circle(200, 0.4, rng), 1, 5),
        ("sphere3d", grid(41, 3), "sphere", cloud_sphere(4000, 0.5, rng), 2, 5),
        ("torus3d_r3", grid(37, 3), "wavy", cloud_torus(5000, 0.5, 0.2, 0.01, rng), 2, 3),
        ("sphere3d_p1", grid(33, 3), "sphere", cloud_sphere(3000, 0.45, rng), 1, 5),
    ):
        x, y, z = mesh(g)
        r = np.sqrt(x * x + y * y + z * z)
        phi = r - 0.8 if shape != "wavy" else r - 0.6 + 0.05 * np.sin(9 * x) * np.cos(7 * y)
        if shape == "circle":
            phi = np.round(phi / (0.25 * g["dx"])) * (0.25 * g["dx"])  # exact zeros at corners
        d, _, _, _ = R.build_distance(g, pts, g["dim"])
        e = R.surface_energy(g, phi, d, p, refine)
        cells = R.interface_cells(g, phi)
        np.savez_compressed(os.path.join(OUT, f"energy_{name}.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=g["dim"], phi=phi, d=d, p=p, refine=refine,
                            energy=e, n_cells=cells.size)
        print("energy", name, e, cells.size)
    # reinitialisation: lsr::reinitialize (reinit.cpp:133) on the band of a
    # (possibly different) band field, as the driver does (driver.cpp:187,196)
    for name, g, kind in (("sphere3d", grid(30, 3), "scaled"), ("circle2d", grid(65, 2), "scaled"),
                          ("zeros3d", grid(26, 3), "zeros"), ("nointerface3d", grid(20, 3), "positive")):
        x, y, z = mesh(g)
        r = np.sqrt(x * x + y * y + z * z)
        band_phi = r - 0.55
        if kind == "scaled":
            phi = 0.6 * (r - 0.55) + 0.3 * g["dx"] * np.sin(11 * x) * np.cos(5 * y)
        elif kind == "zeros":
            phi = np.round((r - 0.5) / (0.5 * g["dx"])) * (0.5 * g["dx"]) * 0.7
        else:
            phi = r + 0.2
            band_phi = r - 0.55
        gam = (6.0 if g["dim"] == 3 else 4.0) * g["dx"]
        rc = R.reinit_defaults(g["dx"], gam)
        out, iters, had = R.reinitialize(g, phi, band_phi, gam, rc)
        np.savez_compressed(os.path.join(OUT, f"reinit_{name}.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=g["dim"], phi=phi, band_phi=band_phi,
                            gamma=gam, out=out, iterations=iters, had_interface=int(had), **{f"rc_{k}": v for k, v in rc.items()})
        print("reinit", name, iters, had)

    # whole loop iterations: driver.cpp:185-203 on a fixed grid (band, E_2,
    # sl_step, reinitialize, swap), K steps; per-step E_2 recorded so the GPU
    # loop can be fed the reference's energies (glibc pow)
    for name, g, pts, interp, p, delta, r0, steps in (
        ("circle2d_q1", grid(65, 2), cloud_circle(200, 0.3, rng), 0, 1, 0.0, 0.9, 6),
        ("sphere3d_weno_p2", grid(30, 3), cloud_sphere(4000, 0.5, rng), 1, 2, 1.0, 0.85, 4),
        ("torus3d_weno_p1", grid(28, 3), cloud_torus(4000, 0.5, 0.2, 0.01, rng), 1, 1, 0.0, 0.8, 4),
    ):
        x, y, z = mesh(g)
        phi = np.sqrt(x * x + y * y + z * z) - r0
        d, _, _, _ = R.build_distance(g, pts, g["dim"])
        gam = (6.0 if g["dim"] == 3 else 4.0) * g["dx"]
        cfg = dict(p=p, interp=interp, delta=delta, dt=0.25 * g["dx"], fallback_c=1e-3, fallback_alpha=1.0,
                   gamma=gam, beta=gam / 2)
        phis, e2s, nas, its = [phi], [], [], []
        cur = phi
        for _ in range(steps):
            cur, e2, na, it, _ = R.loop_step(g, cur, d, cfg)
            phis.append(cur)
            e2s.append(e2)
            nas.append(na)
            its.append(it)
        np.savez_compressed(os.path.join(OUT, f"loop_{name}.npz"), dims=np.array(g["dims"]),
                            origin=np.array(g["origin"]), dx=g["dx"], dim=g["dim"], phi0=phi, d=d, phis=np.stack(phis),
                            e2=np.array(e2s), n_active=np.array(nas), reinit_iters=np.array(its), p=p, interp=interp,
                            delta=delta, gamma=gam)
        print("loop", name, e2s, nas, its)
    # cloud statistics: lsr::compute_stats (cloud.cpp:480) — seeded
    # estimate_resolution (Fisher-Yates sample + exact NN + blocked_sum)
    stats = []
    for name, pts, dim, frac, seed in (("circle", cloud_circle(64, 1.0, rng), 2, 1.0, 0),
                                       ("sphere", cloud_sphere(20000, 0.5, rng), 3, 0.1, 7),
                                       ("torus", cloud_torus(50000, 0.5, 0.2, 0.002, rng), 3, 0.25, 11)):
        h, gm, bb = R.compute_stats(pts, dim, frac, 2.0, seed)
        stats.append(dict(name=name, pts=pts, dim=dim, frac=frac, seed=seed, h=h, g=gm, bb=bb))
    np.savez_compressed(os.path.join(OUT, "stats.npz"),
                        **{f"{s['name']}_{k}": v for s in stats for k, v in s.items() if k != "name"})
    print("stats", [(s["name"], s["h"]) for s in stats])

    # BASELINE config 1 end to end: 2d circle, 200 seeded points at r = 0.3,
    # 257^2 grid, phi0 = |x| - 0.9, multilinear, 200 loop iterations of the
    # reference driver body (Table 1 run 1: p = 1, delta = 0). Stores the
    # field after 50, 100 and 200 steps.
    g = grid(257, 2)
    x, y, _ = mesh(g)
    phi = np.sqrt(x * x + y * y) - 0.9
    th = 2 * np.pi * np.random.default_rng(1).random(200)
    pts = np.stack([0.3 * np.cos(th), 0.3 * np.sin(th), np.zeros(200)], 1)
    d, _, _, _ = R.build_distance(g, pts, 2)
    gam = 4.0 * g["dx"]
    cfg = dict(p=1, interp=0, delta=0.0, dt=0.25 * g["dx"], fallback_c=1e-3, fallback_alpha=1.0, gamma=gam,
               beta=gam / 2)
    cur, keep, e2s = phi, {}, []
    for k in range(1, 201):
        cur, e2, na, it, _ = R.loop_step(g, cur, d, cfg)
        e2s.append(e2)
        if k in (50, 100, 200):
            keep[f"phi{k}"] = cur
    np.savez_compressed(os.path.join(OUT, "config1_circle_200.npz"), dims=np.array(g["dims"]),
                        origin=np.array(g["origin"]), dx=g["dx"], dim=2, pts=pts, phi0=phi, d=d, gamma=gam,
                        e2=np.array(e2s), **keep)
    print("config1: E2 after 200 steps", e2s[-1])
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
