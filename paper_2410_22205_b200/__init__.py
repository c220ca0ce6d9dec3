"""paper_2410_22205_b200 — B200-native narrow-band semi-Lagrangian step.

Python face of ``liblsr_b200.so`` (C ABI: ``include/lsr_cuda.h``). It mirrors
the reference's C++ API for this path (``/root/reference/proj/include/lsr``):
the same type names (Grid, ScalarField, DistanceField, BandMask, StepConfig,
BandParams, InterpolatorKind), the same free functions (``sl_step``,
``default_band_params``, ...) and the same exception hierarchy
(types.hpp:24-52), so tests read like the reference's own tests.

The compute path is the CUDA library only. There is no CPU fallback: if the
extension is missing this module raises on import of any compute function.
"""
from __future__ import annotations

from ._api import (  # noqa: F401
    BandMask,
    BandParams,
    ConfigError,
    Context,
    DistanceField,
    Error,
    Grid,
    InterpolatorKind,
    NoInterfaceError,
    NodeState,
    NumericalError,
    OutOfDomainError,
    ReinitConfig,
    ScalarField,
    SlabContext,
    StepConfig,
    build_distance_field,
    compute_stats,
    cloud_generate,
    cube_grid,
    default_band_params,
    kernel_launches,
    lib,
    lib_path,
    sl_step,
    surface_energy,
)

__all__ = [
    "BandMask",
    "BandParams",
    "ConfigError",
    "Context",
    "DistanceField",
    "Error",
    "Grid",
    "InterpolatorKind",
    "NoInterfaceError",
    "NodeState",
    "NumericalError",
    "OutOfDomainError",
    "ScalarField",
    "StepConfig",
    "default_band_params",
    "kernel_launches",
    "lib",
    "lib_path",
    "sl_step",
]
