"""ctypes binding of include/loam_gpu.h (the C-ABI boundary).

This is the binding a Python maintainer of the reference would add (see
INTEGRATION.md): plain structures mirroring the descriptors and one prototype
per exported function.  It never falls back to CPU code -- loading fails
loudly if the in-tree CUDA library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libloam_gpu.so")

# loam::ErrorKind (common.hpp:10-33), same order
ERROR_KINDS = [
    "IndexOutOfRange", "ArityMismatch", "SourceMismatch", "AsymmetricAdjacency", "IllegalAccess",
    "MapSourceMismatch", "ShapeMismatch", "UnboundIdentifier", "NonDividingFactor",
    "OutsideSparsity", "EmptyPartials", "DimensionMismatch", "InvalidSubdivision", "ParseError",
    "NonManifold", "CellMismatch", "UnsupportedForm", "MissingDiagonal", "SpaceMismatch",
    "IndefiniteBreakdown", "InstabilityDetected", "InvalidArgument",
]
ERR_CUDA = 100
ERR_NO_DEVICE = 101

READ, WRITE, RW, INC, SUM, MIN, MAX = range(7)  # loam::Access (data.hpp:17)
ARG_DAT, ARG_MAT, ARG_GLOBAL = range(3)
ARG_ZERO = 1
OPT_INC_STRATEGY, OPT_CHECK_SPARSITY, OPT_LOCALITY, OPT_TEST_KERNELS, OPT_DETERMINISTIC = range(5)
STRATEGY = {"auto": 0, "atomic": 1, "owner": 2, "color": 3, "nbr": 4, "warpagg": 5, "patch": 6}


class LoamError(RuntimeError):
    """loam::Error (common.hpp:36-43): carries the machine-checkable kind."""

    def __init__(self, code: int, message: str):
        if 1 <= code <= len(ERROR_KINDS):
            kind = ERROR_KINDS[code - 1]
        elif code == ERR_CUDA:
            kind = "CudaError"
        elif code == ERR_NO_DEVICE:
            kind = "NoDevice"
        else:
            kind = f"Unknown({code})"
        super().__init__(f"{kind}: {message}")
        self.code = code
        self.kind = kind
        self.message = message


class MapDesc(C.Structure):
    _fields_ = [
        ("values", C.c_void_p), ("source_size", C.c_int32), ("target_size", C.c_int32),
        ("arity", C.c_int32), ("source_id", C.c_uint64), ("target_id", C.c_uint64),
        ("id", C.c_uint64), ("expand_dim", C.c_int32), ("node_values", C.c_void_p),
        ("node_arity", C.c_int32), ("node_target_size", C.c_int32), ("node_id", C.c_uint64),
    ]


class SparsityDesc(C.Structure):
    _fields_ = [
        ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("nrows", C.c_int32),
        ("ncols", C.c_int32), ("nnz", C.c_int64), ("row_dim", C.c_int32), ("col_dim", C.c_int32),
        ("id", C.c_uint64), ("pattern_row_map", C.c_uint64), ("pattern_col_map", C.c_uint64),
        ("pattern_row_dim", C.c_int32), ("pattern_col_dim", C.c_int32),
    ]


class ArgDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("access", C.c_int32), ("data", C.c_void_p), ("dim", C.c_int32),
        ("set_size", C.c_int32), ("set_id", C.c_uint64), ("obj_id", C.c_uint64),
        ("map", C.POINTER(MapDesc)), ("col_map", C.POINTER(MapDesc)),
        ("sparsity", C.POINTER(SparsityDesc)), ("flags", C.c_int32),
    ]


class KernelDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("params", C.POINTER(C.c_double)), ("nparams", C.c_int32)]


class LoopDesc(C.Structure):  # loam_loop_desc (one par_loop of fem::assemble_blocks, fem/assemble.hpp:439-448)
    _fields_ = [("kernel", C.POINTER(KernelDesc)), ("iterset_size", C.c_int32), ("iterset_id", C.c_uint64),
                ("args", C.POINTER(ArgDesc)), ("nargs", C.c_int32)]


class BlockMatDesc(C.Structure):  # loam_block_mat (solver.hpp:21-28 BlockMat)
    _fields_ = [("sparsity", (C.POINTER(SparsityDesc) * 2) * 2), ("values", (C.c_void_p * 2) * 2),
                ("row_sizes", C.c_int32 * 2), ("col_sizes", C.c_int32 * 2)]


class PwInstr(C.Structure):  # loam_pw_instr (pointwise program, fem/assemble.hpp:150-319)
    _fields_ = [("op", C.c_int32), ("field", C.c_int32), ("value", C.c_double)]


PW_CONST, PW_FIELD, PW_ADD, PW_SUB, PW_MUL, PW_DIV, PW_NEG = range(7)
PW_ASSIGN, PW_ADD_TO, PW_SUB_FROM = range(3)
REDUCE_SUM, REDUCE_MIN, REDUCE_MAX, REDUCE_MAX_ABS = range(4)


class SolveReportDesc(C.Structure):  # loam_solve_report (solver.hpp:13-18)
    _fields_ = [("iterations", C.c_int32), ("final_residual_norm", C.c_double), ("converged", C.c_int32),
                ("reason", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """The in-tree CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        i32, i64, u64, vp, dp = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        proto = {
            "loam_gpu_last_error": (C.c_char_p, []),
            "loam_gpu_version": (C.c_char_p, []),
            "loam_gpu_device_ok": (C.c_int, []),
            "loam_gpu_set_option": (C.c_int, [C.c_int, C.c_int]),
            "loam_gpu_get_option": (C.c_int, [C.c_int]),
            "loam_gpu_plan_cache_clear": (C.c_int, []),
            "loam_gpu_new_id": (u64, []),
            "loam_gpu_release_id": (C.c_int, [u64]),
            "loam_gpu_launch_count": (i64, []),
            "loam_gpu_kernel_signature": (C.c_int, [C.c_char_p, ip, C.c_int]),
            "loam_gpu_kernel_names": (C.c_char_p, []),
            "loam_gpu_validate": (C.c_int, [C.POINTER(KernelDesc), i32, u64, C.POINTER(ArgDesc), C.c_int]),
            "loam_gpu_execute": (C.c_int, [C.POINTER(KernelDesc), i32, u64, C.POINTER(ArgDesc), C.c_int, vp]),
            "loam_gpu_execute_host": (C.c_int, [C.POINTER(KernelDesc), i32, u64, C.POINTER(ArgDesc), C.c_int, vp]),
            "loam_gpu_execute_host_batch": (C.c_int, [C.POINTER(KernelDesc), i32, u64,
                                                      C.POINTER(C.POINTER(ArgDesc)), C.c_int, C.c_int, vp]),
            "loam_gpu_execute_blocks": (C.c_int, [C.POINTER(LoopDesc), C.c_int, vp]),
            "loam_gpu_execute_blocks_host": (C.c_int, [C.POINTER(LoopDesc), C.c_int, vp]),
            "loam_gpu_map_check": (C.c_int, [C.POINTER(MapDesc), vp]),
            "loam_gpu_build_sparsity": (C.c_int, [C.POINTER(MapDesc), C.POINTER(MapDesc), C.c_int, C.c_int,
                                                  C.POINTER(vp), C.POINTER(vp), C.POINTER(i64), vp]),
            "loam_gpu_color_iteration": (C.c_int, [i32, u64, C.POINTER(MapDesc), C.c_int, vp, ip, vp]),
            "loam_gpu_malloc": (C.c_int, [C.POINTER(vp), C.c_size_t]),
            "loam_gpu_free": (C.c_int, [vp]),
            "loam_gpu_host_alloc": (C.c_int, [C.POINTER(vp), C.c_size_t]),
            "loam_gpu_host_free": (C.c_int, [vp]),
            "loam_gpu_memcpy": (C.c_int, [vp, vp, C.c_size_t, vp]),
            "loam_gpu_memset": (C.c_int, [vp, C.c_int, C.c_size_t, vp]),
            "loam_gpu_stream_sync": (C.c_int, [vp]),
            "loam_gpu_unit_square_mesh": (C.c_int, [C.c_int, dp, ip]),
            "loam_gpu_unit_cube_mesh": (C.c_int, [C.c_int, dp, ip]),
            "loam_gpu_jitter": (C.c_int, [C.c_int, C.c_int, C.c_double, u64, dp]),
            "loam_gpu_permute_cells": (C.c_int, [C.c_int, C.c_int, u64, ip]),
            "loam_gpu_uniform": (C.c_int, [i64, u64, C.c_double, C.c_double, dp]),
            "loam_gpu_p2_cell_node_map": (C.c_int, [C.c_int, C.c_int, C.c_int, ip, ip]),
            "loam_gpu_expand_map": (C.c_int, [C.c_int, C.c_int, ip, C.c_int, ip]),
            "loam_gpu_spmv": (C.c_int, [C.POINTER(SparsityDesc), vp, vp, i64, vp, vp]),
            "loam_gpu_block_spmv": (C.c_int, [C.POINTER(BlockMatDesc), vp, i64, vp, vp]),
            "loam_gpu_cg_solve": (C.c_int, [C.POINTER(SparsityDesc), vp, vp, i64, vp, C.c_double, C.c_double,
                                            i32, i32, C.POINTER(SolveReportDesc), vp]),
            "loam_gpu_cg_solve_block": (C.c_int, [C.POINTER(BlockMatDesc), vp, i64, vp, C.c_double, C.c_double,
                                                  i32, i32, C.POINTER(SolveReportDesc), vp]),
            "loam_gpu_apply_dirichlet": (C.c_int, [C.POINTER(SparsityDesc), vp, vp, vp, i32, vp, C.c_double, vp]),
            "loam_gpu_bc_apply": (C.c_int, [vp, i32, vp, i32, vp, C.c_double, vp]),
            "loam_gpu_pointwise": (C.c_int, [vp, i64, i32, C.POINTER(PwInstr), i32, C.POINTER(vp), i32, vp]),
            "loam_gpu_reduce": (C.c_int, [vp, i64, i32, dp, vp]),
            "loam_gpu_reduce_dev": (C.c_int, [vp, i64, i32, vp, vp]),
            "loam_gpu_bc_apply_dev": (C.c_int, [vp, i32, vp, i32, vp, vp]),
            "loam_gpu_wave_clock": (C.c_int, [vp, C.c_double, C.c_double, i32, vp]),
            "loam_gpu_p2_cell_node_map_dev": (C.c_int, [i32, i32, i32, vp, vp, ip, vp]),
            "loam_gpu_exterior_facets": (C.c_int, [i32, i32, i32, vp, C.POINTER(vp), C.POINTER(vp), ip, vp]),
            "loam_gpu_rcm_order": (C.c_int, [i32, vp, vp, vp, vp]),
            "loam_gpu_wave_step": (C.c_int, [C.POINTER(KernelDesc), i32, u64, C.POINTER(ArgDesc), C.c_int, vp, vp, vp, vp, vp, vp, C.c_double, vp, vp]),
            "loam_gpu_vertex_adjacency": (C.c_int, [i32, i32, i32, vp, C.POINTER(vp), C.POINTER(vp),
                                                    C.POINTER(C.c_int64), vp]),
            "loam_gpu_renumber_vertices": (C.c_int, [i32, i32, vp, i32, vp, vp, vp, vp, vp]),
        }
        for name, (res, args) in proto.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


# Every symbol include/loam_gpu.h declares (checked by tests/test_capi_cpu.py).
EXPORTED = [
    "loam_gpu_last_error", "loam_gpu_version", "loam_gpu_device_ok", "loam_gpu_set_option",
    "loam_gpu_get_option", "loam_gpu_plan_cache_clear", "loam_gpu_new_id", "loam_gpu_release_id",
    "loam_gpu_launch_count",
    "loam_gpu_kernel_signature", "loam_gpu_kernel_names", "loam_gpu_validate", "loam_gpu_execute",
    "loam_gpu_execute_host", "loam_gpu_execute_host_batch", "loam_gpu_execute_blocks", "loam_gpu_execute_blocks_host", "loam_gpu_map_check", "loam_gpu_build_sparsity",
    "loam_gpu_color_iteration", "loam_gpu_malloc", "loam_gpu_free", "loam_gpu_host_alloc",
    "loam_gpu_host_free", "loam_gpu_memcpy", "loam_gpu_memset", "loam_gpu_stream_sync",
    "loam_gpu_unit_square_mesh", "loam_gpu_unit_cube_mesh", "loam_gpu_jitter",
    "loam_gpu_permute_cells", "loam_gpu_uniform", "loam_gpu_p2_cell_node_map",
    "loam_gpu_expand_map", "loam_gpu_spmv", "loam_gpu_block_spmv", "loam_gpu_cg_solve",
    "loam_gpu_cg_solve_block",
    "loam_gpu_apply_dirichlet", "loam_gpu_bc_apply", "loam_gpu_pointwise", "loam_gpu_reduce",
    "loam_gpu_p2_cell_node_map_dev", "loam_gpu_exterior_facets",
    "loam_gpu_reduce_dev", "loam_gpu_bc_apply_dev", "loam_gpu_wave_clock",
    "loam_gpu_rcm_order", "loam_gpu_vertex_adjacency", "loam_gpu_renumber_vertices", "loam_gpu_wave_step",
]


def new_id() -> int:
    """A process-unique object identity (shared with every other client of the library)."""
    return int(lib().loam_gpu_new_id())


def release_id(obj_id: int) -> None:
    """Evict the plans / resident copies keyed by obj_id (object destroyed)."""
    global _lib
    if _lib is not None:
        _lib.loam_gpu_release_id(obj_id)


def check(code: int) -> None:
    if code != 0:
        raise LoamError(code, lib().loam_gpu_last_error().decode())


def set_option(option: int, value: int) -> None:
    check(lib().loam_gpu_set_option(option, value))


def set_strategy(name: str) -> None:
    set_option(OPT_INC_STRATEGY, STRATEGY[name])


def launch_count() -> int:
    return int(lib().loam_gpu_launch_count())
