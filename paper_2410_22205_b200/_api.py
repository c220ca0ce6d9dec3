"""ctypes binding of include/lsr_cuda.h plus the reference-shaped host types.

Reference interface mirrored here (file:line under /root/reference/proj):
  Grid            include/lsr/grid.hpp:10-52
  ScalarField     include/lsr/grid.hpp:63-75
  BandMask        include/lsr/grid.hpp:79-84 (NodeState :77)
  BandParams      include/lsr/grid.hpp:86-93, default_band_params grid.cpp:49-51
  DistanceField   include/lsr/distance.hpp:14-18
  StepConfig      include/lsr/evolve.hpp:16-31
  sl_step         include/lsr/evolve.hpp:42-43 -> lsr_cuda_sl_step_host
  exceptions      include/lsr/types.hpp:24-52
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("LSR_B200_LIB") or os.path.join(_HERE, "liblsr_b200.so")  # override: kernel experiments


# --------------------------------------------------------------------------
# exceptions (types.hpp:24-52)
class Error(RuntimeError):
    pass


class ParseError(Error):
    pass


class ConfigError(Error):
    pass


class OutOfDomainError(Error):
    pass


class NumericalError(Error):
    pass


class NoInterfaceError(Error):
    pass


class CudaError(Error):
    pass


LSR_OK, LSR_ERR_CONFIG, LSR_ERR, LSR_ERR_NUMERICAL, LSR_ERR_OUT_OF_DOMAIN, LSR_ERR_CUDA, LSR_ERR_NO_INTERFACE = range(7)
_EXC = {
    LSR_ERR_CONFIG: ConfigError,
    LSR_ERR: Error,
    LSR_ERR_NUMERICAL: NumericalError,
    LSR_ERR_OUT_OF_DOMAIN: OutOfDomainError,
    LSR_ERR_CUDA: CudaError,
    LSR_ERR_NO_INTERFACE: NoInterfaceError,
}
FIELD_PHI, FIELD_DIST, FIELD_OUT, FIELD_SCRATCH = 0, 1, 2, 3


class CGrid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("dims", C.c_int32 * 3), ("origin", C.c_double * 3), ("dx", C.c_double)]


class CStepCfg(C.Structure):
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


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_lib = None


def lib() -> C.CDLL:
    """The CUDA library. Raises (loudly) when it has not been built: there is
    no CPU fallback for any compute entry point."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(lib_path)
    P = C.POINTER
    L.lsr_cuda_last_error_string.restype = C.c_char_p
    L.lsr_cuda_kernel_launches.restype = C.c_int64
    L.lsr_cuda_sl_step_host.argtypes = [P(CGrid), _dp, _dp, C.c_void_p, C.c_int64, P(CStepCfg), C.c_double, _dp,
                                        P(C.c_int64)]
    L.lsr_cuda_create.argtypes = [C.c_int, P(CGrid), P(C.c_void_p)]
    L.lsr_cuda_destroy.argtypes = [C.c_void_p]
    L.lsr_cuda_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.lsr_cuda_upload_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.lsr_cuda_download_field.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.lsr_cuda_field_ptr.argtypes = [C.c_void_p, C.c_int, P(C.c_void_p)]
    L.lsr_cuda_mark_dirty.argtypes = [C.c_void_p, C.c_int]
    L.lsr_cuda_set_active.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.lsr_cuda_set_active_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.lsr_cuda_sl_step.argtypes = [C.c_void_p, P(CStepCfg), C.c_double, P(C.c_int64)]
    L.lsr_cuda_swap.argtypes = [C.c_void_p]
    L.lsr_cuda_set_sl_mode.argtypes = [C.c_void_p, C.c_int]
    L.lsr_cuda_sl_step_async.argtypes = [C.c_void_p, P(CStepCfg), C.c_double]
    L.lsr_cuda_sync.argtypes = [C.c_void_p, P(C.c_int64)]
    L.lsr_cuda_async_times.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float), P(C.c_float), C.c_int, P(C.c_int)]
    L.lsr_cuda_last_times.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float)]
    L.lsr_cuda_last_table_ms.argtypes = [C.c_void_p, P(C.c_float)]
    L.lsr_cuda_sl_step_device.argtypes = [P(CGrid), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_int64, P(CStepCfg), C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    L.lsr_cuda_selftest_div_const.argtypes = [C.c_double, C.c_int64, C.c_uint64, P(C.c_int64)]
    L.lsr_cuda_selftest_weno.argtypes = [C.c_double, C.c_int64, C.c_uint64, P(C.c_int64)]
    L.lsr_cuda_build_distance.argtypes = [P(CGrid), _dp, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          P(C.c_double), P(C.c_int)]
    L.lsr_cuda_ctx_build_distance.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int, C.c_int, P(C.c_double),
                                              P(C.c_int)]
    L.lsr_cloud_generate.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_double, _dp]
    L.lsr_cuda_surface_energy.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_double)]
    L.lsr_cuda_surface_energy_host.argtypes = [P(CGrid), _dp, _dp, C.c_int, C.c_int, P(C.c_double)]
    L.lsr_cuda_narrow_band.argtypes = [C.c_void_p, C.c_int, C.c_double, P(C.c_int64), P(C.c_int64)]
    L.lsr_cuda_band_download.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.lsr_cuda_clamp_field.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.lsr_cuda_reinitialize.argtypes = [C.c_void_p, C.c_int, C.c_double, P(CReinitCfg), P(C.c_int), P(C.c_int)]
    L.lsr_cuda_reinit_defaults.argtypes = [C.c_double, C.c_double, P(CReinitCfg)]
    L.lsr_cuda_reinit_defaults.restype = None
    L.lsr_cuda_loop_step.argtypes = [C.c_void_p, P(CStepCfg), P(CReinitCfg), C.c_int, C.c_double, P(CLoopStats)]
    L.lsr_cuda_loop_run.argtypes = [C.c_void_p, P(CStepCfg), P(CReinitCfg), C.c_int, C.c_int, C.c_int,
                                    P(CLoopStats), P(C.c_int)]
    L.lsr_cuda_sl_step_device_fused.argtypes = [P(CGrid), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_int64, P(CStepCfg), C.c_double,
                                                C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                                C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    L.lsr_cuda_last_transfer_bytes.argtypes = [P(C.c_int64), P(C.c_int64)]
    L.lsr_cuda_last_transfer_bytes.restype = None
    L.lsr_cuda_pack_host.argtypes = [P(CGrid), C.c_void_p, C.c_int64, C.c_int32, _dp, C.c_void_p, _dp, C.c_void_p,
                                     P(C.c_int64)]
    L.lsr_cuda_malloc.argtypes = [C.c_size_t, P(C.c_void_p)]
    L.lsr_cuda_free.argtypes = [C.c_void_p]
    L.lsr_cuda_ipc_handle.argtypes = [C.c_void_p, C.c_char_p]
    L.lsr_cuda_ipc_open.argtypes = [C.c_char_p, P(C.c_void_p)]
    L.lsr_cuda_ipc_close.argtypes = [C.c_void_p]
    L.lsr_cuda_compute_stats.argtypes = [_dp, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_uint64, P(C.c_double),
                                         P(C.c_double), _dp]
    L.lsr_cuda_slab_create.argtypes = [C.c_int, P(CGrid), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       P(C.c_void_p)]
    L.lsr_cuda_slab_copy_planes.argtypes = [C.c_void_p, C.c_int, C.c_int32, C.c_int32, C.c_void_p, C.c_int32]
    L.lsr_cuda_slab_band.argtypes = [C.c_void_p, C.c_int, C.c_double, P(C.c_int64), P(C.c_int64)]
    L.lsr_cuda_slab_energy_cells.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, P(C.c_int64)]
    L.lsr_cuda_slab_energy_pieces.argtypes = [C.c_void_p, C.c_int64, _dp, P(C.c_int64), _dp, P(C.c_int64), _dp,
                                              P(C.c_int64)]
    L.lsr_cuda_slab_max_reach.argtypes = [C.c_void_p, P(CStepCfg), C.c_double, P(C.c_double)]
    L.lsr_cuda_slab_sl_step.argtypes = [C.c_void_p, P(CStepCfg), C.c_double, P(C.c_int64), P(C.c_int64)]
    L.lsr_cuda_slab_one_step.argtypes = [C.c_void_p, P(C.c_int), P(C.c_int)]
    L.lsr_cuda_slab_reinit_begin.argtypes = [C.c_void_p, P(CReinitCfg), P(C.c_int64)]
    L.lsr_cuda_slab_reinit_sweep.argtypes = [C.c_void_p, P(CReinitCfg), C.c_int32, P(C.c_double)]
    L.lsr_cuda_slab_reinit_end.argtypes = [C.c_void_p, C.c_int, C.c_double]
    _lib = L
    return L


class CReinitCfg(C.Structure):  # ReinitConfig (reinit.hpp:7-18)
    _fields_ = [("dtau", C.c_double), ("max_iters", C.c_int32), ("residual_tol", C.c_double),
                ("sign_eps", C.c_double)]


class CLoopStats(C.Structure):
    _fields_ = [("energy", C.c_double), ("n_active", C.c_int64), ("n_tube", C.c_int64),
                ("reinit_iterations", C.c_int32), ("had_interface", C.c_int32), ("ms", C.c_float * 4),
                ("dense_one_step", C.c_int32), ("reserved", C.c_int32)]


@dataclass
class ReinitConfig:  # reinit.hpp:7-18
    dtau: float = 0.0
    max_iters: int = 0
    residual_tol: float = 1e-3
    sign_eps: float = 0.0

    @staticmethod
    def defaults(dx: float, gamma: float) -> "ReinitConfig":  # reinit.cpp:8-16
        c = CReinitCfg()
        lib().lsr_cuda_reinit_defaults(float(dx), float(gamma), C.byref(c))
        return ReinitConfig(c.dtau, c.max_iters, c.residual_tol, c.sign_eps)

    def c(self) -> CReinitCfg:
        return CReinitCfg(float(self.dtau), int(self.max_iters), float(self.residual_tol), float(self.sign_eps))


def surface_energy(phi: "ScalarField", dist: "DistanceField", p: int, subcell_refine: int = 5) -> float:
    """lsr::surface_energy (metrics.hpp:41-42) on the GPU."""
    if not (phi.grid == dist.field.grid):
        raise ConfigError("energy: grid mismatch")
    e = C.c_double()
    _check(lib().lsr_cuda_surface_energy_host(C.byref(phi.grid.c()), phi.values,
                                              np.ascontiguousarray(dist.field.values), int(p), int(subcell_refine),
                                              C.byref(e)))
    return e.value


def cloud_generate(config: int, n: int, seed: int = 0, sigma: float = 0.0) -> np.ndarray:
    """Seeded synthetic cloud of BASELINE config 1..5 (include/lsr_workloads.h), shape (n, 3)."""
    pts = np.zeros((int(n), 3), dtype=np.float64)
    if lib().lsr_cloud_generate(int(config), int(n), int(seed), float(sigma), pts.reshape(-1)) != 0:
        raise ConfigError(f"unknown cloud config {config}")
    return pts


@dataclass
class CloudStats:  # cloud.hpp:19-26
    h_s: float
    gamma_s: float
    k_s: float
    bbox_min: tuple
    bbox_max: tuple
    sample_seed: int


def compute_stats(points: np.ndarray, dim: int, sample_fraction: float = 0.1, k_s: float = 2.0,
                  seed: int = 0) -> CloudStats:
    """lsr::compute_stats (cloud.hpp:52-53): h_S from the exact NN distances
    of a seeded sample (computed on the GPU), gamma_S = k_s * h_S, bbox."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
    h, gm = C.c_double(), C.c_double()
    bb = np.zeros(6)
    _check(lib().lsr_cuda_compute_stats(pts, pts.size // 3, int(dim), float(sample_fraction), float(k_s), int(seed),
                                        C.byref(h), C.byref(gm), bb))
    return CloudStats(h.value, gm.value, float(k_s), tuple(bb[:3]), tuple(bb[3:]), int(seed))


def build_distance_field(grid: "Grid", points: np.ndarray, dim: int | None = None,
                         seed_only: bool = False) -> "DistanceField":
    """lsr::build_distance_field (distance.hpp:29) on the GPU; with
    seed_only, lsr::seed_exact_distance (distance.hpp:24). The sweep round
    count is returned as the attribute ``rounds``."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
    n = grid.num_nodes()
    d = np.empty(n, dtype=np.float64)
    ex = np.empty(n, dtype=np.uint8)
    sent, rounds = C.c_double(), C.c_int()
    _check(lib().lsr_cuda_build_distance(C.byref(grid.c()), pts, pts.size // 3, int(dim or grid.dim),
                                         int(bool(seed_only)), d.ctypes.data_as(C.c_void_p),
                                         ex.ctypes.data_as(C.c_void_p), C.byref(sent), C.byref(rounds)))
    out = DistanceField(ScalarField(grid, d), ex, sent.value)
    out.rounds = rounds.value
    return out


def last_transfer_bytes() -> tuple[int, int]:
    """(H2D, D2H) bytes the calling thread's last one-shot sl_step moved."""
    h2d, d2h = C.c_int64(), C.c_int64()
    lib().lsr_cuda_last_transfer_bytes(C.byref(h2d), C.byref(d2h))
    return int(h2d.value), int(d2h.value)


def pack_host(dist: "DistanceField", active: np.ndarray, dist_field: np.ndarray, reach: int = 0,
              phi: np.ndarray | None = None, phi_field: np.ndarray | None = None) -> tuple[int, int, int, int]:
    """Host-only view of the one-shot step's packed uploads: writes into
    dist_field the d values uploaded for these ascending active ids (active
    nodes and their axis neighbours) and, for reach > 0, into phi_field the
    phi values of the Chebyshev ball of radius `reach` around every active
    node. Returns (d values, d runs, phi values, phi runs)."""
    ids = np.ascontiguousarray(active, dtype=np.int64)
    d = np.ascontiguousarray(dist.field.values, dtype=np.float64)
    for f in (dist_field, phi_field) if reach > 0 else (dist_field,):
        if f is None or f.dtype != np.float64 or not f.flags.c_contiguous or f.size != d.size:
            raise ConfigError("pack_host: fields must be contiguous float64 arrays of the grid's size")
    ph = None
    if reach > 0:
        ph = np.ascontiguousarray(phi, dtype=np.float64)
    counts = (C.c_int64 * 4)()
    _check(lib().lsr_cuda_pack_host(C.byref(dist.field.grid.c()), _ids_ptr(ids), ids.size, int(reach), d,
                                    ph.ctypes.data_as(C.c_void_p) if ph is not None else None, dist_field,
                                    phi_field.ctypes.data_as(C.c_void_p) if reach > 0 else None, counts))
    return tuple(int(x) for x in counts)


def selftest_div_const(c: float, n: int, seed: int = 1) -> int:
    """Mismatching quotients of the kernels' constant-divisor division vs the
    hardware IEEE division over n pseudo-random numerators (must be 0)."""
    m = C.c_int64()
    _check(lib().lsr_cuda_selftest_div_const(float(c), int(n), int(seed), C.byref(m)))
    return int(m.value)


def selftest_weno(dx: float, n: int, seed: int = 1) -> dict:
    """GPU differential test of the fast exact WENO forms against the plain
    IEEE weno_1d (lsr_cuda_selftest_weno)."""
    c = (C.c_int64 * 4)()
    _check(lib().lsr_cuda_selftest_weno(float(dx), int(n), int(seed), c))
    return dict(fast_taken=int(c[0]), fast_mismatch=int(c[1]), table_taken=int(c[2]), table_mismatch=int(c[3]))


def _check(status: int) -> None:
    if status != LSR_OK:
        msg = lib().lsr_cuda_last_error_string().decode()
        raise _EXC.get(status, Error)(msg)


def kernel_launches() -> int:
    """Number of CUDA kernels this process launched through the library."""
    return int(lib().lsr_cuda_kernel_launches())


# --------------------------------------------------------------------------
# reference-shaped types
class InterpolatorKind(enum.IntEnum):  # interp.hpp:9
    Q1 = 0
    Weno = 1


class NodeState(enum.IntEnum):  # grid.hpp:77
    Inactive = 0
    Active = 1
    ReinitHalo = 2


@dataclass
class Grid:  # grid.hpp:10-52
    dim: int = 2
    origin: tuple = (0.0, 0.0, 0.0)
    dx: float = 1.0
    dims: tuple = (1, 1, 1)

    def num_nodes(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def index(self, i, j, k):
        return (k * self.dims[1] + j) * self.dims[0] + i

    def unflatten(self, idx):
        nx, ny = self.dims[0], self.dims[1]
        return idx % nx, (idx // nx) % ny, idx // (nx * ny)

    def node(self, i, j, k):
        return (self.origin[0] + i * self.dx, self.origin[1] + j * self.dx, self.origin[2] + k * self.dx)

    def upper(self):
        return tuple(self.origin[d] + (self.dims[d] - 1) * self.dx for d in range(3))

    def axes(self):
        """Node coordinates per axis, computed with Grid::node's expression."""
        return [self.origin[d] + np.arange(self.dims[d], dtype=np.float64) * self.dx for d in range(3)]

    def mesh(self):
        """(x, y, z) node coordinates, each shaped (nz, ny, nx)."""
        ax = self.axes()
        z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        return x, y, z

    def c(self) -> CGrid:
        g = CGrid()
        g.dim = int(self.dim)
        for d in range(3):
            g.dims[d] = int(self.dims[d])
            g.origin[d] = float(self.origin[d])
        g.dx = float(self.dx)
        return g

    def __eq__(self, o):
        return (self.dim == o.dim and tuple(map(float, self.origin)) == tuple(map(float, o.origin))
                and float(self.dx) == float(o.dx) and tuple(map(int, self.dims)) == tuple(map(int, o.dims)))


def cube_grid(n: int, dim: int = 3, lo: float = -1.0, hi: float = 1.0) -> Grid:
    """The benchmark grids: n nodes per axis on [lo, hi]^dim, dx = (hi-lo)/(n-1)."""
    dx = (hi - lo) / (n - 1)
    if dim == 2:
        return Grid(2, (lo, lo, 0.0), dx, (n, n, 1))
    return Grid(3, (lo, lo, lo), dx, (n, n, n))


@dataclass
class ScalarField:  # grid.hpp:63-75
    grid: Grid
    values: np.ndarray = None

    def __post_init__(self):
        if self.values is None:
            self.values = np.zeros(self.grid.num_nodes(), dtype=np.float64)
        else:
            self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)

    def at(self, i, j, k):
        return self.values[self.grid.index(i, j, k)]


@dataclass
class DistanceField:  # distance.hpp:14-18
    field: ScalarField
    exact: np.ndarray = None
    sentinel: float = 0.0


@dataclass
class BandMask:  # grid.hpp:79-84
    grid: Grid
    state: np.ndarray = None
    active: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    tube: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


@dataclass
class BandParams:  # grid.hpp:86-93
    gamma: float = 0.0
    beta: float = 0.0

    def validate(self):
        if not (self.beta > 0.0) or not (self.beta < self.gamma):
            raise ConfigError("band: need 0 < beta < gamma")


def default_band_params(dim: int, dx: float) -> BandParams:  # grid.cpp:49-51
    return BandParams(4.0 * dx, 2.0 * dx) if dim == 2 else BandParams(6.0 * dx, 3.0 * dx)


@dataclass
class StepConfig:  # evolve.hpp:16-31
    p: int = 1
    delta: float = 0.0
    dt: float = 0.0
    interp: InterpolatorKind = InterpolatorKind.Weno
    fallback_c: float = 1e-3
    fallback_alpha: float = 1.0
    band: BandParams = field(default_factory=BandParams)

    def validate(self):
        if self.p not in (1, 2):
            raise ConfigError("step: p must be 1 or 2")
        if not (self.dt > 0.0):
            raise ConfigError("step: dt must be positive")
        if self.delta < 0.0 or self.delta > 1.0:
            raise ConfigError("step: delta must be in [0, 1]")
        self.band.validate()

    def c(self) -> CStepCfg:
        s = CStepCfg()
        s.p = int(self.p)
        s.interp = int(self.interp)
        s.delta = float(self.delta)
        s.dt = float(self.dt)
        s.fallback_c = float(self.fallback_c)
        s.fallback_alpha = float(self.fallback_alpha)
        s.gamma = float(self.band.gamma)
        s.beta = float(self.band.beta)
        return s


def _ids_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


def sl_step(phi: ScalarField, dist: DistanceField, mask: BandMask, cfg: StepConfig, energy_p: float,
            out: ScalarField) -> None:
    """lsr::sl_step (evolve.hpp:42-43) on the B200. ``out`` is resized if its
    grid differs (evolve.cpp:48) and written in full; raises the reference's
    exception types."""
    if not (phi.grid == dist.field.grid) or not (phi.grid == mask.grid):
        raise ConfigError("sl_step: phi, dist and mask must share one grid")  # evolve.cpp:43-44
    g = phi.grid
    if not (out.grid == g) or out.values.size != g.num_nodes():
        out.grid = g
        out.values = np.zeros(g.num_nodes(), dtype=np.float64)
    n = g.num_nodes()
    if phi.values.size != n or dist.field.values.size != n:  # native code reads num_nodes() values of each
        raise ConfigError("sl_step: phi and dist must hold grid.num_nodes() values")
    if out.values.dtype != np.float64 or not out.values.flags.c_contiguous:
        out.values = np.ascontiguousarray(out.values, dtype=np.float64)
    active = np.ascontiguousarray(mask.active, dtype=np.int64)
    bad = C.c_int64(-1)
    st = lib().lsr_cuda_sl_step_host(C.byref(g.c()), phi.values, np.ascontiguousarray(dist.field.values), _ids_ptr(active),
                                     active.size, C.byref(cfg.c()), float(energy_p), out.values, C.byref(bad))
    _check(st)


class Context:
    """Device-resident context (lsr_cuda_create ...): phi, out and d live in
    HBM across steps; the per-step host traffic is the active-id list (or
    nothing, with set_active_device) and an 8-byte status."""

    def __init__(self, grid: Grid, device: int = 0):
        self.grid = grid
        self.h = C.c_void_p()
        _check(lib().lsr_cuda_create(int(device), C.byref(grid.c()), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().lsr_cuda_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        _check(lib().lsr_cuda_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def upload(self, which: int, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        assert v.size == self.grid.num_nodes()
        _check(lib().lsr_cuda_upload_field(self.h, which, v.ctypes.data_as(C.c_void_p)))

    def download(self, which: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.grid.num_nodes(), dtype=np.float64)
        assert out.flags.c_contiguous and out.dtype == np.float64 and out.size == self.grid.num_nodes()
        _check(lib().lsr_cuda_download_field(self.h, which, out.ctypes.data_as(C.c_void_p)))
        return out

    def field_ptr(self, which: int) -> int:
        p = C.c_void_p()
        _check(lib().lsr_cuda_field_ptr(self.h, which, C.byref(p)))
        return int(p.value)

    def mark_dirty(self, which: int):
        _check(lib().lsr_cuda_mark_dirty(self.h, which))

    def set_active(self, ids: np.ndarray):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        _check(lib().lsr_cuda_set_active(self.h, _ids_ptr(ids), ids.size))

    def set_active_device(self, ptr: int, n: int):
        _check(lib().lsr_cuda_set_active_device(self.h, C.c_void_p(ptr), int(n)))

    def sl_step(self, cfg: StepConfig, energy_p: float) -> None:
        bad = C.c_int64(-1)
        st = lib().lsr_cuda_sl_step(self.h, C.byref(cfg.c()), float(energy_p), C.byref(bad))
        self.bad_node = bad.value
        _check(st)

    def sl_step_async(self, cfg: StepConfig, energy_p: float) -> None:
        """Enqueue one step without host synchronisation (see sync())."""
        _check(lib().lsr_cuda_sl_step_async(self.h, C.byref(cfg.c()), float(energy_p)))

    def sync(self) -> None:
        """Wait for the pending async steps; raises NumericalError like sl_step."""
        bad = C.c_int64(-1)
        st = lib().lsr_cuda_sync(self.h, C.byref(bad))
        self.bad_node = bad.value
        _check(st)

    def async_times(self, cap: int = 4096):
        """(kernel_ms, step_ms, table_ms) lists of the steps the last sync() completed."""
        k, s, t = (C.c_float * cap)(), (C.c_float * cap)(), (C.c_float * cap)()
        n = C.c_int()
        _check(lib().lsr_cuda_async_times(self.h, k, s, t, cap, C.byref(n)))
        return list(k[:n.value]), list(s[:n.value]), list(t[:n.value])

    def swap(self):
        _check(lib().lsr_cuda_swap(self.h))

    def set_sl_mode(self, mode: int):
        """3d WENO step form: 0 = z-line table (default), 1 = TMA-staged bricks."""
        _check(lib().lsr_cuda_set_sl_mode(self.h, int(mode)))

    def build_distance(self, points: np.ndarray, dim: int | None = None, seed_only: bool = False):
        """Device-resident lsr::build_distance_field into the DIST field."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
        sent, rounds = C.c_double(), C.c_int()
        _check(lib().lsr_cuda_ctx_build_distance(self.h, pts, pts.size // 3, int(dim or self.grid.dim),
                                                 int(bool(seed_only)), C.byref(sent), C.byref(rounds)))
        return sent.value, rounds.value

    def surface_energy(self, which: int = FIELD_PHI, p: int = 2, subcell_refine: int = 5) -> float:
        e = C.c_double()
        _check(lib().lsr_cuda_surface_energy(self.h, int(which), int(p), int(subcell_refine), C.byref(e)))
        return e.value

    def narrow_band(self, gamma: float, which: int = FIELD_PHI):
        """lsr::narrow_band on the device; returns (n_active, n_tube). The
        ACTIVE list becomes this context's active set."""
        na, nt = C.c_int64(), C.c_int64()
        _check(lib().lsr_cuda_narrow_band(self.h, int(which), float(gamma), C.byref(na), C.byref(nt)))
        self.n_active, self.n_tube = na.value, nt.value
        return na.value, nt.value

    def band(self) -> "BandMask":
        """The last device-built band as a host BandMask (state, active, tube)."""
        n = self.grid.num_nodes()
        st = np.empty(n, np.uint8)
        act = np.empty(self.n_active, np.int64)
        tube = np.empty(self.n_tube, np.int64)
        _check(lib().lsr_cuda_band_download(self.h, st.ctypes.data_as(C.c_void_p), act.ctypes.data_as(C.c_void_p),
                                            tube.ctypes.data_as(C.c_void_p)))
        return BandMask(self.grid, st, act, tube)

    def clamp_field(self, gamma: float, which: int = FIELD_PHI):
        _check(lib().lsr_cuda_clamp_field(self.h, int(which), float(gamma)))

    def reinitialize(self, gamma: float, cfg: "ReinitConfig", which: int = FIELD_OUT):
        """lsr::reinitialize of `which` on the last built band; returns
        (iterations, had_interface)."""
        it, had = C.c_int(), C.c_int()
        _check(lib().lsr_cuda_reinitialize(self.h, int(which), float(gamma), C.byref(cfg.c()), C.byref(it),
                                           C.byref(had)))
        return it.value, bool(had.value)

    def loop_step(self, cfg: StepConfig, rcfg: "ReinitConfig", energy_refine: int = 5,
                  energy_override: float | None = None) -> dict:
        """One driver iteration (driver.cpp:187-203) on the device."""
        s = CLoopStats()
        _check(lib().lsr_cuda_loop_step(self.h, C.byref(cfg.c()), C.byref(rcfg.c()), int(energy_refine),
                                        -1.0 if energy_override is None else float(energy_override), C.byref(s)))
        return dict(energy=s.energy, n_active=s.n_active, n_tube=s.n_tube, reinit_iterations=s.reinit_iterations,
                    had_interface=bool(s.had_interface), ms=list(s.ms))

    def loop_run(self, cfg: StepConfig, rcfg: "ReinitConfig", iterations: int, energy_refine: int = 5,
                 use_graph: bool = True) -> list[dict]:
        """`iterations` driver iterations (driver.cpp:187-203) controlled on the
        device: one host synchronisation for all of them (lsr_cuda_loop_run);
        the GPU's own E_2 every iteration. Returns one record per iteration."""
        n = int(iterations)
        if n < 1:
            raise ConfigError("loop_run: iterations must be >= 1")
        recs = (CLoopStats * n)()
        done = C.c_int(0)
        _check(lib().lsr_cuda_loop_run(self.h, C.byref(cfg.c()), C.byref(rcfg.c()), int(energy_refine), n,
                                       1 if use_graph else 0, recs, C.byref(done)))
        return [dict(energy=r.energy, n_active=r.n_active, n_tube=r.n_tube, reinit_iterations=r.reinit_iterations,
                     had_interface=bool(r.had_interface), ms=list(r.ms), dense_one_step=bool(r.dense_one_step))
                for r in recs]

    def last_times(self):
        k, s = C.c_float(), C.c_float()
        _check(lib().lsr_cuda_last_times(self.h, C.byref(k), C.byref(s)))
        return k.value, s.value

    def last_table_ms(self) -> float:
        """Device time of the last step's z-line table fill (part of the step)."""
        t = C.c_float()
        _check(lib().lsr_cuda_last_table_ms(self.h, C.byref(t)))
        return t.value



class SlabContext:
    """One rank's z-slab of the loop (lsr_cuda_slab_*): fields hold the
    resident planes [win_lo, win_hi) of the global grid, the phases work on
    the owned planes [own_lo, own_hi). Node ids are global. See
    paper_2410_22205_b200.zslab.SlabLoop for the driver."""

    device_memory = True  # fields live on the device (zslab.DistRunner stages planes there)

    def __init__(self, grid: Grid, win_lo: int, win_hi: int, own_lo: int, own_hi: int, device: int = 0):
        self.grid = grid
        self.win_lo, self.win_hi, self.own_lo, self.own_hi = int(win_lo), int(win_hi), int(own_lo), int(own_hi)
        self.nxy = grid.dims[0] * grid.dims[1]
        self.h = C.c_void_p()
        _check(lib().lsr_cuda_slab_create(int(device), C.byref(grid.c()), self.win_lo, self.win_hi, self.own_lo,
                                          self.own_hi, C.byref(self.h)))

    @property
    def n_resident(self) -> int:
        return (self.win_hi - self.win_lo) * self.nxy

    def close(self):
        if self.h:
            lib().lsr_cuda_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, which: int, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if v.size != self.n_resident:
            raise ConfigError("slab upload: need the resident planes' values")
        _check(lib().lsr_cuda_upload_field(self.h, which, v.ctypes.data_as(C.c_void_p)))

    def download(self, which: int) -> np.ndarray:
        out = np.empty(self.n_resident, dtype=np.float64)
        _check(lib().lsr_cuda_download_field(self.h, which, out.ctypes.data_as(C.c_void_p)))
        return out

    def field_ptr(self, which: int) -> int:
        p = C.c_void_p()
        _check(lib().lsr_cuda_field_ptr(self.h, which, C.byref(p)))
        return int(p.value)

    def plane_ptr(self, which: int, plane: int) -> int:
        """Device address of global plane `plane` of field `which`."""
        assert self.win_lo <= plane <= self.win_hi
        return self.field_ptr(which) + 8 * (plane - self.win_lo) * self.nxy

    def copy_planes(self, which: int, plane0: int, nplanes: int, dev_ptr: int, to_field: bool):
        _check(lib().lsr_cuda_slab_copy_planes(self.h, int(which), int(plane0), int(nplanes), C.c_void_p(dev_ptr),
                                               int(bool(to_field))))

    def swap(self):
        _check(lib().lsr_cuda_swap(self.h))

    def band(self, gamma: float, which: int = FIELD_PHI):
        na, nt = C.c_int64(), C.c_int64()
        _check(lib().lsr_cuda_slab_band(self.h, int(which), float(gamma), C.byref(na), C.byref(nt)))
        self.n_active, self.n_tube = na.value, nt.value
        return na.value, nt.value

    def energy_cells(self, which: int = FIELD_PHI, p: int = 2, refine: int = 5) -> int:
        n = C.c_int64()
        _check(lib().lsr_cuda_slab_energy_cells(self.h, int(which), int(p), int(refine), C.byref(n)))
        self.n_cells = n.value
        return n.value

    def energy_pieces(self, offset: int):
        """(block sums, head, tail) of blocked_sum for this rank at global offset."""
        nb_cap = self.n_cells // 4096 + 1
        blocks, head, tail = np.empty(nb_cap), np.empty(4096), np.empty(4096)
        nb, nh, nt = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().lsr_cuda_slab_energy_pieces(self.h, int(offset), blocks, C.byref(nb), head, C.byref(nh), tail,
                                                 C.byref(nt)))
        return blocks[:nb.value].copy(), head[:nh.value].copy(), tail[:nt.value].copy()

    def max_reach(self, cfg: StepConfig, energy_p: float) -> float:
        c = C.c_double()
        _check(lib().lsr_cuda_slab_max_reach(self.h, C.byref(cfg.c()), float(energy_p), C.byref(c)))
        return c.value

    def sl_step(self, cfg: StepConfig, energy_p: float) -> int:
        """Returns the halo-miss count (0: the step is valid)."""
        bad, miss = C.c_int64(-1), C.c_int64(0)
        st = lib().lsr_cuda_slab_sl_step(self.h, C.byref(cfg.c()), float(energy_p), C.byref(bad), C.byref(miss))
        self.bad_node = bad.value
        _check(st)
        return miss.value

    def one_step(self):
        f, z = C.c_int(), C.c_int()
        _check(lib().lsr_cuda_slab_one_step(self.h, C.byref(f), C.byref(z)))
        return bool(f.value), bool(z.value)

    def reinit_begin(self, rcfg: "ReinitConfig") -> int:
        n = C.c_int64()
        _check(lib().lsr_cuda_slab_reinit_begin(self.h, C.byref(rcfg.c()), C.byref(n)))
        return n.value

    def reinit_sweep(self, rcfg: "ReinitConfig", k: int) -> float:
        r = C.c_double()
        _check(lib().lsr_cuda_slab_reinit_sweep(self.h, C.byref(rcfg.c()), int(k), C.byref(r)))
        return r.value

    def reinit_end(self, which: int, gamma: float):
        _check(lib().lsr_cuda_slab_reinit_end(self.h, int(which), float(gamma)))
