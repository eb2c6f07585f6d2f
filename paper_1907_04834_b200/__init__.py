"""paper_1907_04834_b200 -- B200-native Gaussian-kernel geodesic shooting.

The hot path of arXiv 1907.04834 (exact O(N^2) Hamiltonian flow, its adjoint,
and the Barnes-Hut octree build + traversal) as hand-written sm_100a CUDA
behind a C ABI (include/geoshoot_b200.h). ``geoshoot`` mirrors the
reference's API in Python; ``include/geoshoot/*.hpp`` does so in C++.
"""
from . import _lib  # noqa: F401
from .geoshoot import (  # noqa: F401
    BARNES_HUT, EULER, EXACT, F32, F64, RK4, ConfigError, ConfigMismatch, DegenerateConfiguration,
    DeviceError,
    DimensionMismatch, EmptyTree, Evaluation, Flow, Geoshoot, NonFiniteState, Octree,
    OutOfBounds, ParseError, ShootingConfig, Trajectory, UnsupportedFormat, VTK, XYZ,
    format_for_path, read_points, write_points)

__all__ = [
    "Geoshoot", "ShootingConfig", "Trajectory", "Octree", "Flow", "Evaluation",
    "EXACT", "BARNES_HUT", "EULER", "RK4", "F32", "F64",
    "ConfigError", "ConfigMismatch", "DimensionMismatch", "EmptyTree", "NonFiniteState",
    "OutOfBounds", "DeviceError",
]
