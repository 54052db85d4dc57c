"""ctypes binding of libtsgpu.so (include/tsgpu.h).

The library is the product: there is no Python/CPU fallback. Importing this
module loads the in-tree ``libtsgpu.so`` and raises if it is missing; compute
entry points return TS_ERR_CUDA (raised as ``TsError``) when no GPU exists.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtsgpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tsgpu.h")

TS_OK = 0
TS_ERR_VALIDATION = 1
TS_ERR_BREAKDOWN = 2
TS_ERR_NONFINITE = 3
TS_ERR_NO_CONVERGENCE = 4
TS_ERR_CUDA = 5
TS_ERR_NCCL = 6
TS_ERR_PARSE = 7


class SolverConfig(C.Structure):
    """ts_solver_config == tetsolve::SolverConfig (solver_config.hpp:21-48)."""

    _fields_ = [
        ("outer_tol", C.c_double),
        ("outer_max_iter", C.c_int32),
        ("level_tol", C.c_double * 3),
        ("level_max_iter", C.c_int32 * 3),
        ("batch_size", C.c_int32),
        ("aggregate_target", C.c_int32),
        ("residual_history_stride", C.c_int32),
    ]


class SolveReportC(C.Structure):
    """ts_solve_report == tetsolve::SolveReport (solver_config.hpp:50-63)."""

    _fields_ = [
        ("converged", C.c_int32),
        ("outer_iterations", C.c_int32),
        ("inner_iterations", C.c_int64 * 3),
        ("time_setup_s", C.c_double),
        ("time_outer_s", C.c_double),
        ("time_inner_s", C.c_double * 3),
        ("time_total_s", C.c_double),
        ("batch_size", C.c_int32),
        ("method", C.c_int32),
        ("inner_precision", C.c_int32),
        ("history_count", C.c_int32),
        ("history_capacity", C.c_int32),
        ("final_rel_residual", C.POINTER(C.c_double)),
        ("history_iter", C.POINTER(C.c_int32)),
        ("history", C.POINTER(C.c_double)),
    ]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtsgpu.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")

lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
i32 = C.c_int32
_sig = {
    "ts_last_error": (C.c_char_p, []),
    "ts_version": (C.c_char_p, []),
    "ts_config_default": (None, [vp]),
    "ts_config_validate": (C.c_int, [vp]),
    "ts_box_mesh": (C.c_int, [vp, vp, i32, vp, i32, vp]),
    "ts_mesh_from_arrays": (C.c_int, [i32, i32, vp, i32, vp, vp, i32, vp, vp, vp]),
    "ts_mesh_sizes": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_mesh_export": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "ts_mesh_dirichlet_mask": (C.c_int, [vp, vp]),
    "ts_mesh_destroy": (None, [vp]),
    "ts_mesh_write_tsmesh": (C.c_int, [vp, C.c_char_p]),
    "ts_mesh_read_tsmesh": (C.c_int, [C.c_char_p, vp]),
    "ts_mesh_write_dirichlet": (C.c_int, [vp, C.c_char_p]),
    "ts_mesh_read_dirichlet": (C.c_int, [vp, C.c_char_p]),
    "ts_mesh_write_tsbmesh": (C.c_int, [vp, C.c_char_p]),
    "ts_mesh_read_tsbmesh": (C.c_int, [C.c_char_p, vp]),
    "ts_tsvec_write": (C.c_int, [C.c_char_p, vp, C.c_int64, i32, i32]),
    "ts_tsvec_info": (C.c_int, [C.c_char_p, vp, vp]),
    "ts_tsvec_read": (C.c_int, [C.c_char_p, vp, C.c_int64, i32, i32]),
    "ts_fault_faces_write": (C.c_int, [C.c_char_p, vp, i32]),
    "ts_fault_faces_read": (C.c_int, [C.c_char_p, vp, vp]),
    "ts_observations_read": (C.c_int, [C.c_char_p, vp, vp, vp]),
    "ts_greens_bank_write": (C.c_int, [C.c_char_p, i32, i32, vp, vp, vp, vp, vp, vp]),
    "ts_greens_bank_read": (C.c_int, [C.c_char_p, vp, vp, vp, vp, vp, vp, vp, vp]),
    "ts_material_from_wavespeeds": (C.c_int, [C.c_double, C.c_double, C.c_double, vp, vp]),
    "ts_ebe_create": (C.c_int, [vp, i32, i32, vp, vp, vp, i32, vp]),
    "ts_ebe_destroy": (None, [vp]),
    "ts_ebe_info": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_ebe_apply": (C.c_int, [vp, vp, vp, i32, vp]),
    "ts_ebe_apply_host": (C.c_int, [vp, vp, vp, i32]),
    "ts_ebe_block_jacobi_host": (C.c_int, [vp, vp]),
    "ts_ebe_host_stream_chunks": (C.c_int, [vp, vp]),
    "ts_ebe_set_timing": (C.c_int, [vp, i32]),
    "ts_ebe_last_kernel_ms": (C.c_int, [vp, vp]),
    "ts_ebe_launches_per_apply": (C.c_int, [vp, i32, vp]),
    "ts_ebe_unit_stats": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "ts_ebe_set_deterministic": (C.c_int, [vp, i32]),
    "ts_levels_create": (C.c_int, [vp, i32, vp, vp, vp, vp, vp]),
    "ts_levels_destroy": (None, [vp]),
    "ts_levels_sizes": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_levels_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "ts_levels_operator": (C.c_int, [vp, i32, vp]),
    "ts_levels_apply": (C.c_int, [vp, i32, vp, vp, i32, vp]),
    "ts_levels_transfer": (C.c_int, [vp, i32, vp, vp, i32, vp]),
    "ts_levels_export_fine": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "ts_mesh_validate": (C.c_int, [vp]),
    "ts_ebe_element_matrix": (C.c_int, [vp, i32, vp]),
    "ts_ebe_assemble_bcsr": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_bcsr_create": (C.c_int, [i32, vp, vp, vp, i32, vp]),
    "ts_bcsr_destroy": (None, [vp]),
    "ts_bcsr_info": (C.c_int, [vp, vp, vp, vp]),
    "ts_bcsr_apply": (C.c_int, [vp, vp, vp, i32, vp]),
    "ts_bcsr_apply_host": (C.c_int, [vp, vp, vp, i32]),
    "ts_bcsr_block_jacobi_host": (C.c_int, [vp, vp]),
    "ts_bj_create": (C.c_int, [i32, vp, i32, vp]),
    "ts_bj_destroy": (None, [vp]),
    "ts_bj_apply": (C.c_int, [vp, vp, vp, i32, vp]),
    "ts_bj_apply_host": (C.c_int, [vp, vp, vp, i32]),
    "ts_prolong_create": (C.c_int, [i32, i32, vp, vp, vp, vp]),
    "ts_prolong_destroy": (None, [vp]),
    "ts_prolong_apply": (C.c_int, [vp, i32, vp, vp, i32, vp]),
    "ts_prolong_restrict": (C.c_int, [vp, i32, vp, vp, i32, vp]),
    "ts_prolong_apply_host": (C.c_int, [vp, i32, i32, vp, vp, i32]),
    "ts_geometric_prolongation": (C.c_int, [vp, vp, vp, vp]),
    "ts_inner_pcg": (C.c_int, [i32, vp, vp, vp, vp, i32, i32, C.c_double, i32, vp, vp, vp]),
    "ts_inner_pcg_host": (C.c_int, [i32, vp, vp, vp, vp, i32, i32, C.c_double, i32, vp, vp]),
    "ts_aggregate_p1": (C.c_int, [i32, vp, vp, i32, vp, vp, vp]),
    "ts_build_level2": (C.c_int, [i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]),
    "ts_dot_columns_host": (C.c_int, [i32, C.c_int64, i32, vp, vp, vp]),
    "ts_axpy_columns_host": (C.c_int, [i32, C.c_int64, i32, vp, vp, vp]),
    "ts_xpby_columns_host": (C.c_int, [i32, C.c_int64, i32, vp, vp, vp]),
    "ts_sub_columns_host": (C.c_int, [i32, C.c_int64, vp, vp, vp]),
    "ts_zero_masked_host": (C.c_int, [i32, C.c_int64, i32, vp, vp]),
    "ts_cast_batch_host": (C.c_int, [i32, i32, C.c_int64, vp, vp]),
    "ts_solve": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp]),
    "ts_solve_device": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp, vp]),
    "ts_solve_pcge": (C.c_int, [vp, vp, vp, vp, i32, i32, C.c_double, i32, vp]),
    "ts_comm_nccl_available": (C.c_int, [vp, i32]),
    "ts_comm_nccl_id": (C.c_int, [vp]),
    "ts_comm_create_nccl": (C.c_int, [i32, i32, vp, i32, vp]),
    "ts_thread_world_create": (C.c_int, [i32, vp]),
    "ts_thread_world_destroy": (None, [vp]),
    "ts_comm_create_thread": (C.c_int, [vp, i32, i32, vp]),
    "ts_comm_destroy": (None, [vp]),
    "ts_comm_info": (C.c_int, [vp, vp, vp, vp]),
    "ts_comm_allreduce_sum": (C.c_int, [vp, vp, C.c_int64, vp]),
    "ts_partition_rcb": (C.c_int, [vp, i32, vp]),
    "ts_dist_plan_sizes": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]),
    "ts_dist_plan_export": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]),
    "ts_dist_levels_create": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, vp]),
    "ts_level2_setup_host": (C.c_int, [vp, i32, vp, vp, vp, i32, vp, vp]),
    "ts_dist_levels_destroy": (None, [vp]),
    "ts_dist_levels_sizes": (C.c_int, [vp, vp, vp, vp]),
    "ts_dist_levels_info": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_dist_local_nodes": (C.c_int, [vp, vp]),
    "ts_dist_solve": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp]),
    "ts_dist_solve_device": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp, vp]),
    "ts_dist_ebe_apply": (C.c_int, [vp, i32, vp, vp, i32, vp]),
    "ts_dist_ebe_create": (C.c_int, [vp, i32, i32, vp, vp, vp, vp, i32, vp, vp]),
    "ts_dist_ebe_destroy": (None, [vp]),
    "ts_dist_ebe_info": (C.c_int, [vp, vp, vp, vp, vp]),
    "ts_dist_ebe_local_nodes": (C.c_int, [vp, vp]),
    "ts_dist_ebe_op_apply": (C.c_int, [vp, vp, vp, i32, vp]),
    "ts_dist_ebe_local_operator": (C.c_int, [vp, vp]),
    "ts_fault_plane_faces": (C.c_int, [vp, i32, C.c_double, vp, vp, vp, vp]),
    "ts_faulted_model_create": (C.c_int, [vp, i32, vp, vp, vp, i32, vp, vp]),
    "ts_faulted_model_destroy": (None, [vp]),
    "ts_faulted_info": (C.c_int, [vp, vp, vp, vp]),
    "ts_faulted_levels": (C.c_int, [vp, vp]),
    "ts_reconstruct_split_solution": (C.c_int, [vp, i32, vp, vp, vp, vp, vp]),
    "ts_slip_to_rhs": (C.c_int, [vp, i32, vp, vp, vp, vp]),
    "ts_greens_bank": (C.c_int, [vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]),
    "ts_dist_faulted_model_create": (C.c_int, [vp, i32, vp, vp, vp, i32, vp, vp, vp, vp]),
    "ts_dist_faulted_model_destroy": (None, [vp]),
    "ts_dist_faulted_levels": (C.c_int, [vp, vp]),
    "ts_dist_slip_to_rhs": (C.c_int, [vp, i32, vp, vp, vp, vp]),
    "ts_dist_greens_bank": (C.c_int, [vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(lib, _name, None)
    if _fn is not None:
        _fn.restype = _res
        _fn.argtypes = _args


class TsError(RuntimeError):
    """Raised for a non-OK ts_status; ``code`` is the status."""

    def __init__(self, code: int, msg: str, report=None):
        super().__init__(msg)
        self.code = code
        self.report = report


def check(rc: int):
    if rc != TS_OK:
        raise TsError(rc, lib.ts_last_error().decode())


def declared_symbols() -> list[str]:
    """Every function prototype declared in include/tsgpu.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", src)))
