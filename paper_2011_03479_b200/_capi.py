"""ctypes binding of include/gempe.h (libgempe_b200.so).

This is the only way Python reaches the device path: there is no Python or CPU implementation of the
round behind it.  Loading fails loudly when the library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

HIST_BINS = 512
OK, ERR_CONFIG, ERR_DATA, ERR_DIVERGENCE, ERR_CUDA = 0, 1, 2, 3, 4
NEG_PER_EDGE_2, NEG_PER_VERTEX_K = 0, 1
MATH_TABLES, MATH_EXACT = 0, 1
RNG_REFERENCE, RNG_PHILOX = 0, 1
INIT_REFERENCE, INIT_UNIFORM_PM1, INIT_NORMAL = 0, 1, 2

# every symbol include/gempe.h declares (tests/test_abi.py checks header == this list == exports)
SYMBOLS = [
    "gempe_default_options", "gempe_create", "gempe_destroy", "gempe_last_error", "gempe_is_degenerate",
    "gempe_hash_bits", "gempe_sample_slots", "gempe_pair_terms", "gempe_algorithmic_bytes",
    "gempe_get_work_graph", "gempe_set_coords", "gempe_get_coords", "gempe_init_coords", "gempe_relabel",
    "gempe_iterate", "gempe_step_host", "gempe_iterate_async", "gempe_graph_capture", "gempe_graph_launch", "gempe_pe_sampled", "gempe_sync", "gempe_set_sigma", "gempe_iterate_auto",
    "gempe_iterate_auto_async", "gempe_get_sigma_state", "gempe_sigma_update_async", "gempe_device_tallies", "gempe_run_begin", "gempe_run_enqueue", "gempe_run_poll", "gempe_run_best_snapshot", "gempe_run_rebase",
    "gempe_set_capture", "gempe_get_yz", "gempe_get_yz_rows", "gempe_get_coords_rows", "gempe_probe",
    "gempe_sample", "gempe_set_stream", "gempe_device_coords", "gempe_row_stride", "gempe_padded_rows",
    "gempe_block_rows", "gempe_begin_round", "gempe_begin_round_auto", "gempe_exchange_layout", "gempe_bucket_received", "gempe_gather_chunk", "gempe_coords_ipc_handles", "gempe_open_peer",
    "gempe_add_peer_pointers", "gempe_clear_peers", "gempe_exchange_ipc_handle", "gempe_open_peer_exchange",
    "gempe_add_peer_exchange_pointer", "gempe_exchange_recv_area", "gempe_device_coords_parity", "gempe_coords_parity", "gempe_end_round", "gempe_elapsed_ms",
    "gempe_kernel_launches", "gempe_bucket_spills", "gempe_trim_device_cache", "gempe_alloc_host", "gempe_free_host", "gempe_host_fastmath_table", "gempe_host_optimize_sigma",
    "gempe_host_histogram_objective", "gempe_host_histogram_objective_dsigma", "gempe_host_random_relabel",
    "gempe_host_mix_seed", "gempe_default_iteration_config", "gempe_engine_create", "gempe_engine_create_multi", "gempe_engine_destroy",
    "gempe_engine_last_error", "gempe_engine_context", "gempe_engine_degenerate", "gempe_engine_iteration",
    "gempe_engine_sigma", "gempe_engine_run_single_iteration", "gempe_engine_run", "gempe_parse_edge_list",
    "gempe_parse_graph_snapshot", "gempe_load_graph_file", "gempe_write_graph_snapshot", "gempe_graph_free",
    "gempe_write_embedding_tsv",
    "gempe_group_create", "gempe_group_destroy", "gempe_group_last_error", "gempe_group_world", "gempe_group_context",
    "gempe_group_exchange_path", "gempe_group_set_coords", "gempe_group_init_coords", "gempe_group_get_coords",
    "gempe_group_iterate", "gempe_group_set_sigma", "gempe_group_iterate_auto", "gempe_group_relabel",
    "gempe_group_replicas_agree",
]


class PeReportC(C.Structure):
    _fields_ = [("pe", C.c_double), ("mu_star", C.c_double), ("sigma_star", C.c_double), ("h_basic", C.c_double),
                ("compression_ratio", C.c_double), ("grid_pe", C.c_double), ("nonedge_samples", C.c_uint64)]


class RunStatusC(C.Structure):
    _fields_ = [("rounds_done", C.c_uint64), ("improved_at", C.c_uint64), ("draws", C.c_uint64), ("best_pe", C.c_double),
                ("sigma", C.c_double), ("pe_estimate", C.c_double), ("last_nonedge_weight", C.c_double),
                ("converged", C.c_int32), ("failed", C.c_int32)]


class Options(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("hash_bits", C.c_int32), ("seed", C.c_uint64), ("neg_mode", C.c_int32),
                ("negatives", C.c_uint32), ("math", C.c_int32), ("rng", C.c_int32), ("relabel", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("comm_chunks", C.c_int32),
                ("chunk_entries", C.c_uint32), ("deterministic", C.c_int32), ("precise_distance", C.c_int32),
                ("kernel_variant", C.c_int32), ("bucket_mode", C.c_int32), ("exchange", C.c_int32)]


class IterationConfigC(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("lane_width", C.c_uint32), ("workers", C.c_uint32),
                ("convergence_tol", C.c_double), ("convergence_window", C.c_int32), ("relabel_period", C.c_int32),
                ("fast_math", C.c_int32), ("hash_bits", C.c_int32), ("neg_mode", C.c_int32),
                ("negatives", C.c_uint32), ("device", C.c_int32), ("host_sigma", C.c_int32), ("deterministic", C.c_int32),
                ("batch_rounds", C.c_int32)]


class GraphC(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("src", C.POINTER(C.c_uint32)), ("dst", C.POINTER(C.c_uint32)),
                ("raw_labels", C.POINTER(C.c_uint64))]


class EmbedResultC(C.Structure):
    _fields_ = [("embedding", C.c_void_p), ("pe_trace", C.c_void_p), ("pe_trace_cap", C.c_int32),
                ("pe_trace_len", C.c_int32), ("final_sigma", C.c_double), ("converged", C.c_int32),
                ("degenerate", C.c_int32), ("iterations", C.c_int32), ("relabel_forward", C.c_void_p),
                ("last_hist_edge", C.c_void_p), ("last_hist_nonedge", C.c_void_p),
                ("last_nonedge_weight", C.c_double)]


_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_lib = None


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Loads libgempe_b200.so (building it in-tree first when sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and os.path.exists(_build.NVCC):
        _build.build()
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"{_build.LIB} is missing: run `python -m paper_2011_03479_b200.build` "
                           "(the GEMPE path has no CPU fallback)")
    L = C.CDLL(_build.LIB)
    vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sig = {
        "gempe_default_options": (None, [C.POINTER(Options)]),
        "gempe_create": (i32, [C.POINTER(vp), u32, u64, vp, vp, C.POINTER(Options)]),
        "gempe_destroy": (None, [vp]),
        "gempe_last_error": (C.c_char_p, [vp]),
        "gempe_is_degenerate": (i32, [vp]),
        "gempe_hash_bits": (i32, [vp]),
        "gempe_sample_slots": (u64, [vp]),
        "gempe_pair_terms": (u64, [vp]),
        "gempe_algorithmic_bytes": (u64, [vp]),
        "gempe_get_work_graph": (i32, [vp, vp, vp, vp]),
        "gempe_set_coords": (i32, [vp, vp]),
        "gempe_get_coords": (i32, [vp, vp]),
        "gempe_init_coords": (i32, [vp, i32, u64, dbl]),
        "gempe_relabel": (i32, [vp, u64]),
        "gempe_iterate": (i32, [vp, dbl, dbl, u64, vp, vp]),
        "gempe_step_host": (i32, [vp, vp, vp, dbl, dbl, u64, vp, vp]),
        "gempe_iterate_async": (i32, [vp, dbl, dbl, u64]),
        "gempe_sync": (i32, [vp, vp, vp]),
        "gempe_set_sigma": (i32, [vp, dbl, dbl]),
        "gempe_iterate_auto": (i32, [vp, u64, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(dbl), vp, vp]),
        "gempe_iterate_auto_async": (i32, [vp, u64]),
        "gempe_get_sigma_state": (i32, [vp, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(dbl)]),
        "gempe_sigma_update_async": (i32, [vp]),
        "gempe_device_tallies": (vp, [vp]),
        "gempe_run_begin": (i32, [vp, dbl, dbl, u64, i32, dbl, u32]),
        "gempe_run_enqueue": (i32, [vp, u32, u64, i32]),
        "gempe_run_poll": (i32, [vp, C.POINTER(RunStatusC), vp, vp, u32, vp, vp]),
        "gempe_run_best_snapshot": (vp, [vp]),
        "gempe_run_rebase": (i32, [vp]),
        "gempe_group_create": (i32, [C.POINTER(vp), u32, u64, vp, vp, C.POINTER(Options), vp, i32, i32]),
        "gempe_group_destroy": (None, [vp]),
        "gempe_group_last_error": (C.c_char_p, [vp]),
        "gempe_group_world": (i32, [vp]),
        "gempe_group_context": (vp, [vp, i32]),
        "gempe_group_exchange_path": (C.c_char_p, [vp]),
        "gempe_group_set_coords": (i32, [vp, vp]),
        "gempe_group_init_coords": (i32, [vp, i32, u64, dbl]),
        "gempe_group_get_coords": (i32, [vp, vp]),
        "gempe_group_iterate": (i32, [vp, dbl, dbl, u64, vp, vp]),
        "gempe_group_set_sigma": (i32, [vp, dbl, dbl]),
        "gempe_group_iterate_auto": (i32, [vp, u64, C.POINTER(dbl), C.POINTER(dbl), C.POINTER(dbl), vp, vp]),
        "gempe_group_relabel": (i32, [vp, u64]),
        "gempe_group_replicas_agree": (i32, [vp]),
        "gempe_bucket_spills": (C.c_int64, [vp]),
        "gempe_trim_device_cache": (None, []),
        "gempe_alloc_host": (vp, [u64]),
        "gempe_free_host": (None, [vp]),
        "gempe_set_capture": (i32, [vp, i32]),
        "gempe_get_yz": (i32, [vp, vp, vp]),
        "gempe_get_yz_rows": (i32, [vp, vp, u64, vp, vp]),
        "gempe_get_coords_rows": (i32, [vp, vp, u64, vp]),
        "gempe_probe": (i32, [vp, vp, vp, u64, vp]),
        "gempe_sample": (i32, [vp, u64, vp, C.POINTER(u64)]),
        "gempe_set_stream": (i32, [vp, vp]),
        "gempe_device_coords": (vp, [vp, i32]),
        "gempe_row_stride": (u32, [vp]),
        "gempe_padded_rows": (u32, [vp]),
        "gempe_block_rows": (u32, [vp]),
        "gempe_graph_capture": (i32, [vp, dbl, dbl, u64, i32]),
        "gempe_graph_launch": (i32, [vp]),
        "gempe_pe_sampled": (i32, [vp, i32, u64, C.POINTER(PeReportC)]),
        "gempe_begin_round": (i32, [vp, dbl, dbl, u64]),
        "gempe_begin_round_auto": (i32, [vp, u64]),
        "gempe_exchange_layout": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_uint32)]),
        "gempe_bucket_received": (i32, [vp]),
        "gempe_gather_chunk": (i32, [vp, i32]),
        "gempe_coords_ipc_handles": (i32, [vp, vp]),
        "gempe_open_peer": (i32, [vp, vp]),
        "gempe_add_peer_pointers": (i32, [vp, vp, vp]),
        "gempe_clear_peers": (i32, [vp]),
        "gempe_exchange_ipc_handle": (i32, [vp, vp]),
        "gempe_open_peer_exchange": (i32, [vp, i32, vp]),
        "gempe_add_peer_exchange_pointer": (i32, [vp, i32, vp]),
        "gempe_exchange_recv_area": (vp, [vp]),
        "gempe_device_coords_parity": (vp, [vp, i32]),
        "gempe_coords_parity": (i32, [vp]),
        "gempe_end_round": (i32, [vp]),
        "gempe_elapsed_ms": (i32, [vp, C.POINTER(C.c_float * 3)]),
        "gempe_kernel_launches": (u64, [vp]),
        "gempe_host_fastmath_table": (i32, [i32, _f64p]),
        "gempe_host_optimize_sigma": (dbl, [_u64p, _u64p, dbl, dbl, C.POINTER(i32)]),
        "gempe_host_histogram_objective": (dbl, [_u64p, _u64p, dbl, dbl, dbl]),
        "gempe_host_histogram_objective_dsigma": (dbl, [_u64p, _u64p, dbl, dbl, dbl]),
        "gempe_host_random_relabel": (i32, [u32, u64, _u32p]),
        "gempe_host_mix_seed": (u64, [u64, u64]),
        "gempe_default_iteration_config": (None, [C.POINTER(IterationConfigC)]),
        "gempe_engine_create": (i32, [C.POINTER(vp), u32, u64, vp, vp, u32, C.POINTER(IterationConfigC), u64]),
        "gempe_engine_create_multi": (i32, [C.POINTER(vp), u32, u64, vp, vp, u32, C.POINTER(IterationConfigC), u64, vp, i32]),
        "gempe_engine_destroy": (None, [vp]),
        "gempe_engine_last_error": (C.c_char_p, [vp]),
        "gempe_engine_context": (vp, [vp]),
        "gempe_engine_degenerate": (i32, [vp]),
        "gempe_engine_iteration": (i32, [vp]),
        "gempe_engine_sigma": (dbl, [vp]),
        "gempe_engine_run_single_iteration": (i32, [vp, C.POINTER(dbl), C.POINTER(dbl)]),
        "gempe_engine_run": (i32, [vp, C.POINTER(EmbedResultC)]),
        "gempe_parse_edge_list": (i32, [C.c_char_p, u64, C.POINTER(GraphC), C.POINTER(u64)]),
        "gempe_parse_graph_snapshot": (i32, [C.c_char_p, u64, C.POINTER(GraphC)]),
        "gempe_load_graph_file": (i32, [C.c_char_p, C.POINTER(GraphC), C.POINTER(u64)]),
        "gempe_write_graph_snapshot": (i32, [C.c_char_p, u32, u64, vp, vp]),
        "gempe_graph_free": (None, [C.POINTER(GraphC)]),
        "gempe_write_embedding_tsv": (i32, [C.c_char_p, u32, u32, vp, vp, vp]),
    }
    assert sorted(sig) == sorted(SYMBOLS)
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
