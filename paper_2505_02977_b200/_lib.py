"""ctypes binding of the C ABI declared in include/parac_gpu.h.

The native library (lib/libparac_gpu.so, built by `make` / __graft_entry__.build)
is mandatory: there is no Python or CPU fallback, and importing this module
without it raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libparac_gpu.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"native library missing: {LIB_PATH} (run `make` or __graft_entry__.build()); "
        "this package has no CPU fallback"
    )

lib = C.CDLL(LIB_PATH)

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER


class parac_csr(C.Structure):
    _fields_ = [("n", i32), ("ptr", vp), ("adj", vp), ("w", vp)]


class parac_graph(C.Structure):
    _fields_ = [("n", i32), ("nnz", i64), ("ptr", P(i64)), ("adj", P(i32)), ("w", P(f64)),
                ("wdeg", P(f64))]


class parac_factor(C.Structure):
    _fields_ = [("n", i32), ("nnz", i64), ("col_ptr", P(i64)), ("rows", P(i32)), ("values", P(f64)),
                ("diag", P(f64)), ("perm", P(i32))]


class parac_gpu_options(C.Structure):
    _fields_ = [("fill_pool_entries", i64), ("column_arena_entries", i64),
                ("first_chunk", i32), ("watchdog_seconds", f64), ("record_stats", i32),
                ("verify", i32), ("grid_ctas", i32), ("delay_ns", i32),
                ("record_times", i32), ("trace_phases", i32), ("trace_position", i32)]


class parac_gpu_factor_info(C.Structure):
    _fields_ = [("n", i32), ("num_edges", i64), ("nnz_off_diagonal", i64), ("total_fills", i64),
                ("fill_pool_used", i64), ("arena_used", i64), ("max_raw", i32),
                ("large_columns", i32), ("setup_ms", f64), ("eliminate_ms", f64),
                ("assemble_ms", f64), ("device_ms", f64), ("upload_ms", f64), ("wall_ms", f64),
                ("attempts", i32)]


class parac_gpu_solve_report(C.Structure):
    _fields_ = [("iterations", i32), ("relative_residual", f64), ("recurrence_residual", f64),
                ("converged", i32), ("solve_ms", f64), ("wall_ms", f64), ("exact", i32)]


# name -> (restype, argtypes); mirrors include/parac_gpu.h one to one.
SIGNATURES = {
    "parac_errc_name": (C.c_char_p, [C.c_int]),
    "parac_gpu_last_error": (C.c_char_p, []),
    "parac_graph_free": (None, [P(parac_graph)]),
    "parac_graph_from_edges": (C.c_int, [i32, i64, vp, vp, vp, P(parac_graph)]),
    "parac_gen_poisson3d": (C.c_int, [i32, C.c_int, f64, f64, u64, P(parac_graph)]),
    "parac_gen_poisson2d": (C.c_int, [i32, P(parac_graph)]),
    "parac_gen_poisson27": (C.c_int, [i32, u64, P(parac_graph)]),
    "parac_gen_rmat": (C.c_int, [i32, i32, u64, P(parac_graph)]),
    "parac_gen_random_connected": (C.c_int, [i32, i64, u64, C.c_int, P(parac_graph)]),
    "parac_gen_random_components": (C.c_int, [i32, i32, i64, u64, P(parac_graph)]),
    "parac_ordering_random": (C.c_int, [i32, u64, vp]),
    "parac_ordering_nnz_sort": (C.c_int, [P(parac_csr), u64, vp]),
    "parac_ordering_check": (C.c_int, [i32, vp]),
    "parac_gpu_create": (C.c_int, [i32, P(vp)]),
    "parac_gpu_destroy": (None, [vp]),
    "parac_gpu_device_count": (C.c_int, []),
    "parac_gpu_default_options": (None, [P(parac_gpu_options)]),
    "parac_gpu_upload": (C.c_int, [vp, P(parac_csr), vp]),
    "parac_gpu_factor_resident": (C.c_int, [vp, u64, P(parac_gpu_options), P(parac_gpu_factor_info)]),
    "parac_gpu_factor": (C.c_int, [vp, P(parac_csr), vp, u64, P(parac_gpu_options),
                                   P(parac_gpu_factor_info)]),
    "parac_gpu_factor_begin": (C.c_int, [vp, u64, P(parac_gpu_options)]),
    "parac_gpu_factor_end": (C.c_int, [vp, P(parac_gpu_factor_info), vp, vp, vp, vp, i64]),
    "parac_gpu_factor_to_host": (C.c_int, [vp, P(parac_csr), vp, u64, P(parac_gpu_options),
                                           P(parac_gpu_factor_info), vp, vp, vp, vp, i64]),
    "parac_gpu_download": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "parac_gpu_download_times": (C.c_int, [vp, vp]),
    "parac_gpu_download_subtimes": (C.c_int, [vp, vp]),
    "parac_gpu_download_hub_trace": (C.c_int, [vp, vp, C.c_int32, vp]),
    "parac_gpu_download_phase_snapshots": (C.c_int, [vp, vp, vp]),
    "parac_gpu_upload_batch": (C.c_int, [vp, i32, P(parac_csr), vp, vp]),
    "parac_gpu_factor_batch": (C.c_int, [vp, i32, P(parac_csr), vp, vp, P(parac_gpu_options),
                                         P(parac_gpu_factor_info)]),
    "parac_gpu_factor_batch_end": (C.c_int, [vp, P(parac_gpu_factor_info), vp, vp, vp, vp, vp]),
    "parac_gpu_factor_batch_to_host": (C.c_int, [vp, i32, P(parac_csr), vp, vp, P(parac_gpu_options),
                                                 P(parac_gpu_factor_info), vp, vp, vp, vp, vp]),
    "parac_gpu_batch_nnz": (C.c_int, [vp, i32, P(i64)]),
    "parac_gpu_download_batch": (C.c_int, [vp, i32, vp, vp, vp, vp]),
    "parac_gpu_upload_factor": (C.c_int, [vp, i32, vp, vp, vp, vp, vp]),
    "parac_gpu_schedule_levels": (C.c_int, [vp, vp, P(i32)]),
    "parac_gpu_ordering_nnz_sort": (C.c_int, [vp, P(parac_csr), u64, vp]),
    "parac_read_laplacian": (C.c_int, [C.c_char_p, P(parac_graph)]),
    "parac_write_matrix_market": (C.c_int, [C.c_char_p, P(parac_csr)]),
    "parac_write_factor": (C.c_int, [C.c_char_p, i32, vp, vp, vp, vp]),
    "parac_factor_free": (None, [P(parac_factor)]),
    "parac_read_factor": (C.c_int, [C.c_char_p, C.c_char_p, P(parac_factor)]),
    "parac_write_vector": (C.c_int, [C.c_char_p, i64, vp]),
    "parac_read_vector": (C.c_int, [C.c_char_p, P(P(f64)), P(i64)]),
    "parac_free_array": (None, [vp]),
    "parac_write_permutation": (C.c_int, [C.c_char_p, i32, vp]),
    "parac_read_permutation": (C.c_int, [C.c_char_p, i32, vp]),
    "parac_gpu_pcg": (C.c_int, [vp, vp, f64, i32, vp, P(parac_gpu_solve_report)]),
    "parac_gpu_set_preconditioner_mode": (C.c_int, [vp, i32]),
    "parac_gpu_apply_preconditioner": (C.c_int, [vp, vp, vp]),
    "parac_gpu_laplacian_apply": (C.c_int, [vp, vp, vp]),
    "parac_make_rhs": (C.c_int, [P(parac_csr), C.c_int, u64, vp]),
    "parac_factor_checksum": (u64, [i32, vp, vp, vp, vp]),
    "parac_host_alloc": (vp, [C.c_size_t]),
    "parac_host_free": (None, [vp]),
    "parac_gpu_launch_count": (i64, []),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)  # AttributeError here = header/library mismatch
    _fn.restype = _res
    _fn.argtypes = _args
