"""ctypes binding of the C ABI (include/geoshoot_b200.h).

The shared library is built in-tree (``paper_1907_04834_b200/libgeoshoot_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_1907_04834_b200/csrc``. There is
no fallback: if the library or a B200 is missing, every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GS_LIB_PATH: load a variant build instead (kernel experiments, tools/)
LIB_PATH = os.environ.get("GS_LIB_PATH") or os.path.join(HERE, "libgeoshoot_b200.so")

# gs_status (include/geoshoot_b200.h)
GS_OK = 0
GS_DIMENSION_MISMATCH = 1
GS_CONFIG_ERROR = 2
GS_NONFINITE = 3
GS_CONFIG_MISMATCH = 4
GS_EMPTY_TREE = 5
GS_OUT_OF_BOUNDS = 6
GS_INVALID_ARGUMENT = 7
GS_CUDA_ERROR = 8
GS_NO_DEVICE = 9
GS_PARSE_ERROR = 10
GS_UNSUPPORTED_FORMAT = 11
GS_IO_ERROR = 12
GS_DEGENERATE = 13

GS_F64, GS_F32 = 0, 1
GS_EXACT, GS_BARNES_HUT = 0, 1
GS_EULER, GS_RK4 = 0, 1
GS_FLAG_EXACT_CUTOFF, GS_FLAG_EXACT_MORTON = 1, 2


class gs_config(C.Structure):
    _fields_ = [
        ("sigma", C.c_double),
        ("lambda_", C.c_double),
        ("timesteps", C.c_int32),
        ("backend", C.c_int32),
        ("threshold_multiplier", C.c_double),
        ("integrator", C.c_int32),
        ("precision", C.c_int32),
        ("literal_mean_dot", C.c_int32),
        ("flags", C.c_uint32),
    ]


class gs_stats(C.Structure):
    _fields_ = [
        ("direct_interactions", C.c_uint64),
        ("approximated_interactions", C.c_uint64),
        ("nodes_visited", C.c_uint64),
        ("traversal_queries", C.c_uint64),
        ("tree_build_ms", C.c_double),
        ("forward_ms", C.c_double),
        ("backward_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class gs_opt_config(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int32),
        ("memory", C.c_int32),
        ("gradient_tolerance", C.c_double),
        ("relative_objective_tolerance", C.c_double),
        ("sufficient_decrease", C.c_double),
        ("curvature", C.c_double),
        ("max_trials", C.c_int32),
    ]


class gs_report(C.Structure):
    _fields_ = [
        ("energy", C.c_double),
        ("attachment", C.c_double),
        ("total", C.c_double),
        ("residual_sse", C.c_double),
    ]


_d = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p
_i64 = C.c_int64
_st = C.c_int

# (name, restype, argtypes) of every exported symbol of include/geoshoot_b200.h
SIGNATURES = [
    ("gs_default_config", gs_config, []),
    ("gs_abi_version", C.c_int, []),
    ("gs_create", _vp, [C.c_int, C.POINTER(C.c_int)]),
    ("gs_destroy", None, [_vp]),
    ("gs_last_error", C.c_char_p, [_vp]),
    ("gs_set_literal_mean_dot", _st, [_vp, C.c_int32]),
    ("gs_last_nonfinite_step", C.c_int, [_vp]),
    ("gs_last_config_violations", C.c_uint32, [_vp]),
    ("gs_validate_config", _st, [C.POINTER(gs_config), C.POINTER(C.c_uint32)]),
    ("gs_hamiltonian", _st, [_vp, C.c_int32, _i64, _d, _d, C.c_double, _d]),
    ("gs_exact_rhs", _st, [_vp, C.c_int32, _i64, _d, _d, C.c_double, _d, _d, _d]),
    ("gs_exact_velocity", _st, [_vp, C.c_int32, _i64, _d, _i64, _d, _d, C.c_double, _d]),
    ("gs_hessian_products", _st, [_vp, C.c_int32, _i64, _d, _d, _d, _d, C.c_double, _d, _d, _d, _d]),
    ("gs_tree_build", _st, [_vp, C.c_int32, _i64, _d, _d, C.POINTER(_vp)]),
    ("gs_tree_build_in_cell", _st, [_vp, C.c_int32, _i64, _d, _d, _d, _d, C.POINTER(_vp)]),
    ("gs_tree_free", None, [_vp]),
    ("gs_tree_node_count", _i64, [_vp]),
    ("gs_tree_point_count", _i64, [_vp]),
    ("gs_tree_accumulate_adjoints", _st, [_vp, _d, _d]),
    ("gs_tree_download", _st, [_vp, _i32p, _u64p, _u64p, _i32p, _i32p, _i32p, _i32p, _d, _d, _u32p]),
    ("gs_bh_velocity", _st, [_vp, _i64, _d, C.c_double, C.c_double, _d, C.POINTER(gs_stats)]),
    ("gs_bh_rhs", _st, [_vp, C.c_double, C.c_double, _d, _d, C.POINTER(gs_stats)]),
    ("gs_bh_query_stats", _st, [_vp, _u64p]),
    ("gs_bh_hamiltonian", _st, [_vp, C.c_double, C.c_double, _d, C.POINTER(gs_stats)]),
    ("gs_bh_hessian_products", _st, [_vp, _d, _d, C.c_double, C.c_double, _d, _d, _d, _d,
                                     C.POINTER(gs_stats)]),
    ("gs_bh_point_gradients", _st, [_vp, _i64, _d, _d, C.c_double, C.c_double, _d, _d,
                                    C.POINTER(gs_stats)]),
    ("gs_bh_point_hessian_products", _st, [_vp, _i64, _d, _d, _d, _d, _d, _d, C.c_double,
                                           C.c_double, _d, _d, _d, _d, C.POINTER(gs_stats)]),
    ("gs_set_bh_walk", _st, [C.c_int32, C.c_int32]),
    ("gs_set_exact_pairs", _st, [C.c_int32]),
    ("gs_exact_pairs_plan", _st, [C.c_int32, C.c_int64, C.POINTER(C.c_int32)]),
    ("gs_create_multi", _vp, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int)]),
    ("gs_ctx_device_count", C.c_int32, [_vp]),
    ("gs_ctx_peer_stores", C.c_int32, [_vp]),
    ("gs_profile", _st, [_vp, C.c_int32]),
    ("gs_profile_phases", _st, [_vp, _d, C.POINTER(_i64), C.c_int32]),
    ("gs_trace", _st, [_vp, C.c_int32]),
    ("gs_trace_read", _st, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _i64, C.POINTER(_i64)]),
    ("gs_shoot_forward", _st, [_vp, C.POINTER(gs_config), _i64, _d, _d, _d, _d, _d, _d, _d,
                               C.POINTER(gs_stats)]),
    ("gs_objective", _st, [_vp, C.POINTER(gs_config), _i64, _d, _d, _d, C.POINTER(gs_report)]),
    ("gs_backward_gradient", _st, [_vp, C.POINTER(gs_config), _i64, C.c_int32, _d, _d, _d, _d]),
    ("gs_warp_points", _st, [_vp, C.POINTER(gs_config), _i64, C.c_int32, _d, _d, _i64, _d, _d]),
    ("gs_evaluate", _st, [_vp, C.POINTER(gs_config), _i64, _d, _d, _d, C.POINTER(gs_report), _d,
                          C.POINTER(gs_stats)]),
    ("gs_flow_create", _st, [_vp, C.POINTER(gs_config), _i64, C.POINTER(_vp)]),
    ("gs_flow_destroy", None, [_vp]),
    ("gs_flow_upload", _st, [_vp, _d, _d]),
    ("gs_flow_advance", _st, [_vp, C.c_int32]),
    ("gs_flow_sync", _st, [_vp]),
    ("gs_flow_download", _st, [_vp, _d, _d]),
    ("gs_flow_last_launches", _i64, [_vp]),
    ("gs_flow_stats", _st, [_vp, C.POINTER(gs_stats)]),
    ("gs_flow_stream", _vp, [_vp]),
    ("gs_flow_profile", _st, [_vp, C.c_int32]),
    ("gs_flow_profile_read", _st, [_vp, _d, C.POINTER(_i64), _d, C.POINTER(_i64)]),
    ("gs_flow_profile_phases", _st, [_vp, _d, C.POINTER(_i64), C.c_int32]),
    ("gs_flow_set_shard", _st, [_vp, _i64, _i64]),
    ("gs_flow_source_buffer", _vp, [_vp]),
    ("gs_flow_record_bytes", _i64, [_vp]),
    ("gs_flow_stage", _st, [_vp, C.c_int32]),
    ("gs_flow_set_pair_rows", _st, [_vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
    ("gs_flow_stage_pairs", _st, [_vp, C.c_int32, C.POINTER(_vp)]),
    ("gs_flow_stage_apply", _st, [_vp, C.c_int32, _vp, C.c_int32]),
    ("gs_microbench", _st, [C.c_int, C.c_int32, _d]),
    ("gs_format_for_path", C.c_int32, [C.c_char_p]),
    ("gs_procrustes_align", _st, [_vp, _i64, _d, _d, _d, _d, _d]),
    ("gs_read_points", _st, [C.c_char_p, C.c_int32, _d, _i64, C.POINTER(_i64)]),
    ("gs_write_points", _st, [C.c_char_p, C.c_int32, _i64, _d, C.POINTER(C.c_char_p), C.c_int32]),
    ("gs_last_parse_line", C.c_longlong, []),
    ("gs_last_io_error", C.c_char_p, []),
    ("gs_default_opt_config", gs_opt_config, []),
    ("gs_evaluate_batch", _st, [C.c_int, C.POINTER(gs_config), C.c_int32, C.POINTER(_i64),
                                C.POINTER(_d), C.POINTER(_d), C.POINTER(_d), C.POINTER(gs_report),
                                C.POINTER(_d), C.POINTER(gs_stats)]),
    ("gs_optimize_batch", _st, [C.c_int, C.POINTER(gs_config), C.POINTER(gs_opt_config), C.c_int32,
                                C.POINTER(C.c_int64), C.POINTER(_d), C.POINTER(_d), C.POINTER(_d),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                _d]),
    ("gs_optimize", _st, [_vp, C.POINTER(gs_config), C.POINTER(gs_opt_config), _i64, _d, _d, _d,
                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32), _d,
                          C.POINTER(C.c_int32), C.POINTER(gs_stats)]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the product library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1907_04834_b200/csrc` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
