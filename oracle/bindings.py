"""TEST INFRASTRUCTURE ONLY — ctypes faces of the two CPU checkers.

* ``Restatement`` — ``oracle/liblsr_oracle.so``, our plain-C restatement of
  the reference path (oracle/lsr_oracle.c).
* ``Reference`` — ``oracle/_ref/liblsr_ref.so``, the unmodified reference
  library compiled from /root/reference/proj/src plus oracle/ref_shim.cpp.
  Present only where it was built (this container; it travels to the GPU box
  as a built artefact but /root/reference itself does not).

Arrays are numpy; the structs mirror include/lsr_cuda.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblsr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblsr_ref.so")
REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class CGrid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("dims", C.c_int32 * 3), ("origin", C.c_double * 3), ("dx", C.c_double)]


class CCfg(C.Structure):
    _fields_ = [
        ("p", C.c_int32),
        ("interp", C.c_int32),
        ("delta", C.c_double),
        ("dt", C.c_double),
        ("fallback_c", C.c_double),
        ("fallback_alpha", C.c_double),
        ("gamma", C.c_double),
        ("beta", C.c_double),
    ]


def cgrid(g) -> CGrid:
    """Accepts anything with dim/dims/origin/dx (paper_2410_22205_b200.Grid or a dict)."""
    get = (lambda k: g[k]) if isinstance(g, dict) else (lambda k: getattr(g, k))
    out = CGrid()
    out.dim = int(get("dim"))
    for d in range(3):
        out.dims[d] = int(get("dims")[d])
        out.origin[d] = float(get("origin")[d])
    out.dx = float(get("dx"))
    return out


def ccfg(c) -> CCfg:
    get = (lambda k: c[k]) if isinstance(c, dict) else (lambda k: getattr(c, k))
    out = CCfg()
    out.p = int(get("p"))
    out.interp = int(get("interp"))
    for k in ("delta", "dt", "fallback_c", "fallback_alpha", "gamma", "beta"):
        setattr(out, k, float(get(k)))
    return out


def build(ref: bool = True) -> None:
    """Compile the checkers (building the checker is not using it)."""
    subprocess.run(["make", "-s", "-C", HERE, "liblsr_oracle.so"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)
        # the reference's run_schedule built three ways; needs the product library
        if os.path.exists(os.path.join(HERE, "..", "paper_2410_22205_b200", "liblsr_b200.so")):
            subprocess.run(["make", "-s", "-C", HERE, "integration", f"REF={REF_SRC}"], check=True,
                           stdout=subprocess.DEVNULL)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.msg = msg


class Restatement:
    """oracle/lsr_oracle.c"""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.lsro_last_error.restype = C.c_char_p
        L.lsro_sl_step.argtypes = [C.POINTER(CGrid), _dp, _dp, _ip, C.c_int64, C.POINTER(CCfg), C.c_double, _dp,
                                   C.POINTER(C.c_int64), C.c_int]
        L.lsro_narrow_band.argtypes = [C.POINTER(CGrid), _dp, C.c_double, _u8p, _ip, C.POINTER(C.c_int64), _ip,
                                       C.POINTER(C.c_int64)]
        L.lsro_clamp_field.argtypes = [C.POINTER(CGrid), _dp, C.c_double]
        L.lsro_weno_1d.argtypes = [_dp, C.c_double, C.c_double]
        L.lsro_weno_1d.restype = C.c_double
        L.lsro_interp.argtypes = [C.c_int, C.POINTER(CGrid), _dp, _dp, C.POINTER(C.c_double)]
        L.lsro_tangent_basis.argtypes = [C.c_int, _dp, _dp, _dp]
        L.lsro_cutoff_weight.argtypes = [C.c_double, C.c_double, C.c_double]
        L.lsro_cutoff_weight.restype = C.c_double
        L.lsro_centered_gradient.argtypes = [C.POINTER(CGrid), _dp, C.c_int, C.c_int, C.c_int, _dp]
        L.lsro_locate_cell.argtypes = [C.POINTER(CGrid), _dp, _i32p]
        L.lsro_scale_factor.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]

    def _err(self, st):
        if st:
            raise OracleError(st, self.lib.lsro_last_error().decode())

    def sl_step(self, grid, phi, dist, active, cfg, energy_p, nthreads=0):
        """Returns (out, status, bad_node); never raises on numerical errors."""
        phi = np.ascontiguousarray(phi, dtype=np.float64).ravel()
        out = np.empty_like(phi)
        bad = C.c_int64(-1)
        st = self.lib.lsro_sl_step(C.byref(cgrid(grid)), phi, np.ascontiguousarray(dist, np.float64).ravel(),
                                   np.ascontiguousarray(active, np.int64), len(active), C.byref(ccfg(cfg)),
                                   float(energy_p), out, C.byref(bad), int(nthreads))
        return out, st, bad.value

    def narrow_band(self, grid, phi, gamma):
        phi = np.ascontiguousarray(phi, dtype=np.float64).ravel()
        n = phi.size
        state = np.zeros(n, np.uint8)
        act = np.zeros(n, np.int64)
        tube = np.zeros(n, np.int64)
        na, nt = C.c_int64(), C.c_int64()
        self._err(self.lib.lsro_narrow_band(C.byref(cgrid(grid)), phi, float(gamma), state, act, C.byref(na), tube,
                                            C.byref(nt)))
        return state, act[: na.value].copy(), tube[: nt.value].copy()

    def weno_1d(self, v, dx, theta):
        return self.lib.lsro_weno_1d(np.ascontiguousarray(v, np.float64), float(dx), float(theta))

    def interp(self, kind, grid, f, p):
        out = C.c_double()
        self._err(self.lib.lsro_interp(int(kind), C.byref(cgrid(grid)), np.ascontiguousarray(f, np.float64).ravel(),
                                       np.ascontiguousarray(p, np.float64), C.byref(out)))
        return out.value

    def tangent_basis(self, dim, grad):
        v1 = np.zeros(3)
        v2 = np.zeros(3)
        self.lib.lsro_tangent_basis(int(dim), np.ascontiguousarray(grad, np.float64), v1, v2)
        return v1, v2

    def cutoff_weight(self, phi, gamma, beta):
        return self.lib.lsro_cutoff_weight(float(phi), float(gamma), float(beta))


class Reference:
    """oracle/_ref/liblsr_ref.so — the reference library itself."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.lsrref_last_error.restype = C.c_char_p
        L.lsrref_sl_step.argtypes = [C.c_int, C.POINTER(CGrid), _dp, _dp, _ip, C.c_int64, C.POINTER(CCfg), C.c_double,
                                     _dp, C.POINTER(C.c_double)]
        L.lsrref_ctx_new.argtypes = [C.POINTER(CGrid), _dp, _dp, _ip, C.c_int64]
        L.lsrref_ctx_new.restype = C.c_void_p
        L.lsrref_ctx_free.argtypes = [C.c_void_p]
        L.lsrref_ctx_sl_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(CCfg), C.c_double, C.POINTER(C.c_double)]
        L.lsrref_ctx_out.argtypes = [C.c_void_p, _dp]
        L.lsrref_narrow_band.argtypes = [C.c_int, C.POINTER(CGrid), _dp, C.c_double, _u8p, _ip, C.POINTER(C.c_int64),
                                         _ip, C.POINTER(C.c_int64)]
        L.lsrref_clamp_field.argtypes = [C.POINTER(CGrid), _dp, C.c_double]
        L.lsrref_interp.argtypes = [C.c_int, C.POINTER(CGrid), _dp, _dp, C.c_int64, _dp]
        L.lsrref_weno_1d.argtypes = [_dp, C.c_double, C.c_double]
        L.lsrref_weno_1d.restype = C.c_double
        L.lsrref_weno_linear_weights.argtypes = [C.c_double, _dp]
        L.lsrref_weno_indicators.argtypes = [_dp, C.c_double, _dp]
        L.lsrref_locate_cell.argtypes = [C.POINTER(CGrid), _dp, _i32p]
        L.lsrref_centered_gradient.argtypes = [C.POINTER(CGrid), _dp, C.c_int, C.c_int, C.c_int, _dp]
        L.lsrref_tangent_basis.argtypes = [C.c_int, _dp, _dp, _dp]
        L.lsrref_scale_factor.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.lsrref_cutoff_weight.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.lsrref_surface_energy.argtypes = [C.POINTER(CGrid), _dp, _dp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.lsrref_interface_cells.argtypes = [C.POINTER(CGrid), _dp, _ip, C.POINTER(C.c_int64)]
        L.lsrref_reinitialize.argtypes = [C.POINTER(CGrid), _dp, _dp, C.c_double, C.c_double, C.c_int, C.c_double,
                                          C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lsrref_reinit_defaults.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                             C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.lsrref_build_distance.argtypes = [C.POINTER(CGrid), _dp, C.c_int64, C.c_int, C.c_int, _dp, _u8p,
                                            C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.lsrref_compute_stats.argtypes = [_dp, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double), _dp]
        L.lsrref_loop_step.argtypes = [C.POINTER(CGrid), _dp, _dp, C.POINTER(CCfg), C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int), _dp]
        L.lsrref_loop_run.argtypes = [C.POINTER(CGrid), _dp, _dp, C.POINTER(CCfg), C.c_int, C.c_int, _dp, _ip,
                                      _i32p]
        L.lsrref_set_threads.argtypes = [C.c_int]
        L.lsrref_max_threads.restype = C.c_int
        L.lsr_cloud_generate.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_double, _dp]

    def _err(self, st):
        if st:
            raise OracleError(st, self.lib.lsrref_last_error().decode())

    def set_threads(self, n):
        self.lib.lsrref_set_threads(int(n))

    def max_threads(self):
        return self.lib.lsrref_max_threads()

    def sl_step(self, grid, phi, dist, active, cfg, energy_p, serial=True):
        """Returns (out, status, message, seconds)."""
        phi = np.ascontiguousarray(phi, dtype=np.float64).ravel()
        out = np.zeros_like(phi)
        sec = C.c_double(0)
        st = self.lib.lsrref_sl_step(int(bool(serial)), C.byref(cgrid(grid)), phi,
                                     np.ascontiguousarray(dist, np.float64).ravel(),
                                     np.ascontiguousarray(active, np.int64), len(active), C.byref(ccfg(cfg)),
                                     float(energy_p), out, C.byref(sec))
        msg = self.lib.lsrref_last_error().decode() if st else ""
        return out, st, msg, sec.value

    def narrow_band(self, grid, phi, gamma, serial=False):
        phi = np.ascontiguousarray(phi, dtype=np.float64).ravel()
        n = phi.size
        state = np.zeros(n, np.uint8)
        act = np.zeros(n, np.int64)
        tube = np.zeros(n, np.int64)
        na, nt = C.c_int64(), C.c_int64()
        self._err(self.lib.lsrref_narrow_band(int(serial), C.byref(cgrid(grid)), phi, float(gamma), state, act,
                                              C.byref(na), tube, C.byref(nt)))
        return state, act[: na.value].copy(), tube[: nt.value].copy()

    def clamp_field(self, grid, phi, gamma):
        phi = np.array(phi, dtype=np.float64).ravel()
        self._err(self.lib.lsrref_clamp_field(C.byref(cgrid(grid)), phi, float(gamma)))
        return phi

    def interp(self, kind, grid, f, pts):
        pts = np.ascontiguousarray(np.atleast_2d(pts), np.float64)
        out = np.zeros(len(pts))
        self._err(self.lib.lsrref_interp(int(kind), C.byref(cgrid(grid)), np.ascontiguousarray(f, np.float64).ravel(),
                                         pts, len(pts), out))
        return out

    def weno_1d(self, v, dx, theta):
        return self.lib.lsrref_weno_1d(np.ascontiguousarray(v, np.float64), float(dx), float(theta))

    def weno_linear_weights(self, theta):
        o = np.zeros(2)
        self.lib.lsrref_weno_linear_weights(float(theta), o)
        return o

    def weno_indicators(self, v, dx):
        o = np.zeros(2)
        self.lib.lsrref_weno_indicators(np.ascontiguousarray(v, np.float64), float(dx), o)
        return o

    def locate_cell(self, grid, p):
        c = np.zeros(3, np.int32)
        self._err(self.lib.lsrref_locate_cell(C.byref(cgrid(grid)), np.ascontiguousarray(p, np.float64), c))
        return c

    def centered_gradient(self, grid, f, i, j, k):
        o = np.zeros(3)
        self.lib.lsrref_centered_gradient(C.byref(cgrid(grid)), np.ascontiguousarray(f, np.float64).ravel(), i, j, k,
                                          o)
        return o

    def tangent_basis(self, dim, grad):
        v1 = np.zeros(3)
        v2 = np.zeros(3)
        self.lib.lsrref_tangent_basis(int(dim), np.ascontiguousarray(grad, np.float64), v1, v2)
        return v1, v2

    def scale_factor(self, d, e, p):
        o = C.c_double()
        self._err(self.lib.lsrref_scale_factor(float(d), float(e), int(p), C.byref(o)))
        return o.value

    def cutoff_weight(self, phi, gamma, beta):
        o = C.c_double()
        self._err(self.lib.lsrref_cutoff_weight(float(phi), float(gamma), float(beta), C.byref(o)))
        return o.value

    def surface_energy(self, grid, phi, dist, p=2, refine=5):
        o = C.c_double()
        self._err(self.lib.lsrref_surface_energy(C.byref(cgrid(grid)), np.ascontiguousarray(phi, np.float64).ravel(),
                                                 np.ascontiguousarray(dist, np.float64).ravel(), int(p), int(refine),
                                                 C.byref(o)))
        return o.value

    def interface_cells(self, grid, phi):
        phi = np.ascontiguousarray(phi, np.float64).ravel()
        cells = np.zeros(phi.size, np.int64)
        n = C.c_int64()
        self._err(self.lib.lsrref_interface_cells(C.byref(cgrid(grid)), phi, cells, C.byref(n)))
        return cells[: n.value].copy()

    def reinit_defaults(self, dx, gamma):
        dtau, tol, eps = C.c_double(), C.c_double(), C.c_double()
        it = C.c_int()
        self.lib.lsrref_reinit_defaults(float(dx), float(gamma), C.byref(dtau), C.byref(it), C.byref(tol),
                                        C.byref(eps))
        return dict(dtau=dtau.value, max_iters=it.value, residual_tol=tol.value, sign_eps=eps.value)

    def reinitialize(self, grid, phi, band_phi, gamma, rcfg):
        phi = np.array(phi, dtype=np.float64).ravel()
        it, hi = C.c_int(), C.c_int()
        self._err(self.lib.lsrref_reinitialize(C.byref(cgrid(grid)), phi,
                                               np.ascontiguousarray(band_phi, np.float64).ravel(), float(gamma),
                                               rcfg["dtau"], int(rcfg["max_iters"]), rcfg["residual_tol"],
                                               rcfg["sign_eps"], C.byref(it), C.byref(hi)))
        return phi, it.value, bool(hi.value)

    def build_distance(self, grid, pts, dim, seed_only=False):
        n = int(np.prod(cgrid(grid).dims))
        d = np.zeros(n)
        ex = np.zeros(n, np.uint8)
        sent = C.c_double()
        rounds = C.c_int()
        pts = np.ascontiguousarray(pts, np.float64)
        self._err(self.lib.lsrref_build_distance(C.byref(cgrid(grid)), pts, len(pts), int(dim), int(seed_only), d, ex,
                                                 C.byref(sent), C.byref(rounds)))
        return d, ex, sent.value, rounds.value

    def compute_stats(self, pts, dim, fraction=0.1, k_s=2.0, seed=0):
        h, g = C.c_double(), C.c_double()
        bb = np.zeros(6)
        pts = np.ascontiguousarray(pts, np.float64)
        self._err(self.lib.lsrref_compute_stats(pts, len(pts), int(dim), float(fraction), float(k_s), int(seed),
                                                C.byref(h), C.byref(g), bb))
        return h.value, g.value, bb

    def loop_step(self, grid, phi, dist, cfg, refine=5):
        phi = np.array(phi, dtype=np.float64).ravel()
        e2 = C.c_double()
        na = C.c_int64()
        it = C.c_int()
        sec = np.zeros(4)
        self._err(self.lib.lsrref_loop_step(C.byref(cgrid(grid)), phi, np.ascontiguousarray(dist, np.float64).ravel(),
                                            C.byref(ccfg(cfg)), int(refine), C.byref(e2), C.byref(na), C.byref(it),
                                            sec))
        return phi, e2.value, na.value, it.value, sec

    def loop_run(self, grid, phi, dist, cfg, iters, refine=5, inplace=False):
        """iters loop iterations; returns (phi, e2 per iteration, |active| per
        iteration, reinit iterations per iteration). inplace: phi (contiguous
        float64) is overwritten instead of copied."""
        if not (inplace and isinstance(phi, np.ndarray) and phi.dtype == np.float64 and phi.flags.c_contiguous):
            phi = np.array(phi, dtype=np.float64)
        phi = phi.reshape(-1)
        e2 = np.zeros(iters)
        na = np.zeros(iters, np.int64)
        it = np.zeros(iters, np.int32)
        self._err(self.lib.lsrref_loop_run(C.byref(cgrid(grid)), phi, np.ascontiguousarray(dist, np.float64).ravel(),
                                           C.byref(ccfg(cfg)), int(refine), int(iters), e2, na, it))
        return phi, e2, na, it

    def cloud_generate(self, config, n, seed=0, sigma=0.0):
        """The seeded BASELINE cloud (paper_2410_22205_b200/csrc/workloads.cpp,
        compiled into this library), shape (n, 3)."""
        pts = np.zeros((int(n), 3))
        if self.lib.lsr_cloud_generate(int(config), int(n), int(seed), float(sigma), pts.reshape(-1)) != 0:
            raise OracleError(1, f"unknown cloud config {config}")
        return pts

    # bench helpers -------------------------------------------------------
    def ctx(self, grid, phi, dist, active):
        h = self.lib.lsrref_ctx_new(C.byref(cgrid(grid)), np.ascontiguousarray(phi, np.float64).ravel(),
                                    np.ascontiguousarray(dist, np.float64).ravel(),
                                    np.ascontiguousarray(active, np.int64), len(active))
        return h

    def ctx_sl_step(self, h, cfg, energy_p, serial=False):
        sec = C.c_double()
        self._err(self.lib.lsrref_ctx_sl_step(h, int(bool(serial)), C.byref(ccfg(cfg)), float(energy_p),
                                              C.byref(sec)))
        return sec.value

    def ctx_out(self, h, n):
        out = np.zeros(n)
        self.lib.lsrref_ctx_out(h, out)
        return out

    def ctx_free(self, h):
        self.lib.lsrref_ctx_free(h)


def reference_available() -> bool:
    return os.path.exists(REF_SO)
