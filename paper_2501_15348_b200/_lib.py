"""ctypes binding of include/dgnn_b200.h -> paper_2501_15348_b200/_dgnn_b200.so.

The library is the product: there is no Python or CPU fallback. Importing
this module fails loudly when the shared library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# DGNN_LIB_PATH: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("DGNN_LIB_PATH") or os.path.join(_HERE, "_dgnn_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "dgnn_b200.h")

P, I32, I64, U64, D, F = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float


class RunCfg(C.Structure):
    """dgnn_run_cfg (include/dgnn_b200.h)."""
    _fields_ = [
        ("arch", I32), ("layers", I32), ("hidden", I32), ("seq_len", I32), ("horizon", I32),
        ("teacher_forcing", I32), ("aggr", I32), ("batch_size", I32), ("seed", U64),
        ("lr", D), ("optimizer", I32), ("stride", I32), ("fallback_threshold", D),
        ("rescratch_period", I32), ("incremental", I32), ("cache_policy", I32),
        ("cache_frac", D), ("workers", I32), ("epochs", I32), ("window_total", I32),
        ("record_events", I32), ("hbm_cache_budget_bytes", I64),
        ("n_fanouts", I32), ("fanouts", I32 * 8), ("iteration", I32),
    ]


class EpochReport(C.Structure):
    _fields_ = [("loss", D), ("seconds", D), ("samples", I64), ("hits", I64), ("misses", I64),
                ("evictions", I64), ("expirations", I64), ("invalidations", I64),
                ("rejected", I64), ("scratch_calls", I64), ("incremental_calls", I64),
                ("fallbacks", I64), ("skipped_steps", I64), ("spills", I64), ("refills", I64)]


PP = C.POINTER(P)

SIGNATURES = {
    "dgnn_last_error": (C.c_char_p, []),
    "dgnn_version": (C.c_char_p, []),
    "dgnn_launch_count": (I64, []),
    "dgnn_synchronize": (C.c_int, [P]),
    "dgnn_graph_create": (C.c_int, [I32, I32, P, PP]),
    "dgnn_graph_free": (None, [P]),
    "dgnn_graph_add_snapshot": (C.c_int, [P, P, P, I64, P]),
    "dgnn_graph_add_delta": (C.c_int, [P, P, P, I64, P, P, I64, P, I64, P]),
    "dgnn_graph_length": (I32, [P]),
    "dgnn_graph_num_edges": (I64, [P, I32]),
    "dgnn_graph_device_bytes": (I64, [P]),
    "dgnn_graph_feature_stats": (C.c_int, [P, C.POINTER(I32), C.POINTER(I64)]),
    "dgnn_graph_snapshot": (C.c_int, [P, I32, PP, PP, PP, PP, PP]),
    "dgnn_graph_delta_sizes": (C.c_int, [P, I32] + [C.POINTER(I64)] * 6),
    "dgnn_graph_delta_copy": (C.c_int, [P, I32, P, P, P, P, P]),
    "dgnn_graph_delta_layout": (C.c_int, [P, I32, PP, PP, PP]),
    "dgnn_graph_change_ratio": (D, [P, I32]),
    "dgnn_synth_create": (C.c_int, [I32, D, I32, I32, D, D, U64, PP]),
    "dgnn_synth_free": (None, [P]),
    "dgnn_synth_sizes": (C.c_int, [P, P]),
    "dgnn_synth_base": (C.c_int, [P, PP, PP, PP]),
    "dgnn_synth_step": (C.c_int, [P, I32, PP, PP, PP, PP, PP, PP]),
    "dgnn_synth_to_graph": (C.c_int, [P, P, PP]),
    "dgnn_dataset_open": (C.c_int, [C.c_char_p, I32, PP]),
    "dgnn_dataset_free": (None, [P]),
    "dgnn_dataset_info": (C.c_int, [P] + [C.POINTER(I32)] * 4),
    "dgnn_dataset_read_base": (C.c_int, [P, C.POINTER(I64), PP, PP, PP]),
    "dgnn_dataset_read_step": (C.c_int, [P, I32, P, PP, PP, PP, PP, PP, PP]),
    "dgnn_dataset_load": (C.c_int, [C.c_char_p, I32, P, PP]),
    "dgnn_dataset_save_graph": (C.c_int, [P, C.c_char_p, I32]),
    "dgnn_synth_save": (C.c_int, [P, C.c_char_p, I32]),
    "dgnn_khop": (C.c_int, [P, I32, P, I64, P, I32, U64, PP]),
    "dgnn_comm_ledger": (C.c_int, [P, I32, I32, I32, I32, I32, I32, I32, I64, I64, P]),
    "dgnn_cg_free": (None, [P]),
    "dgnn_cg_num_hops": (I32, [P]),
    "dgnn_cg_hop_sizes": (C.c_int, [P, I32, C.POINTER(I64), C.POINTER(I64)]),
    "dgnn_cg_hop_copy": (C.c_int, [P, I32, P, P, P]),
    "dgnn_cg_view": (C.c_int, [P, PP, PP, PP, PP, C.POINTER(I64)]),
    "dgnn_khop_delta": (C.c_int, [P, P, I32, PP]),
    "dgnn_cg_update_free": (None, [P]),
    "dgnn_cg_update_sizes": (C.c_int, [P, I32, C.POINTER(I64), C.POINTER(I64)]),
    "dgnn_cg_update_copy": (C.c_int, [P, I32, P, P, P, P]),
    "dgnn_cg_update_empty": (I32, [P]),
    "dgnn_apply_cg_update": (C.c_int, [P, P, PP]),
    "dgnn_agg_scratch": (C.c_int, [I32, I32, I32, P, P, P, P, P, P, P, P]),
    "dgnn_agg_delta": (C.c_int, [I32, I32, I32, P, P, P, P, P, P, P, P, P, P]),
    "dgnn_graph_apply_delta": (C.c_int, [P, I32, I32, P, P, P, P, P]),
    "dgnn_agg_backward": (C.c_int, [I32, I32, I32, P, P, P, P, P, P, P]),
    "dgnn_agg_incremental": (C.c_int, [P, I32, I32, P, P, P, P, I32, I64, D, I32, P, P, P, P, P]),
    "dgnn_pack_cell": (C.c_int, [I32, I32, I32, P, P, P, P]),
    "dgnn_cell_forward": (C.c_int, [I32, I32, I32, I32] + [P] * 10),
    "dgnn_cell_backward": (C.c_int, [I32, I32, I32, I32] + [P] * 14),
    "dgnn_session_create": (C.c_int, [P, C.POINTER(RunCfg), I32, P, PP]),
    "dgnn_session_free": (None, [P]),
    "dgnn_session_num_params": (I64, [P]),
    "dgnn_session_num_windows": (C.c_int, [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]),
    "dgnn_session_get_params": (C.c_int, [P, P]),
    "dgnn_session_set_params": (C.c_int, [P, P]),
    "dgnn_session_initial_params": (C.c_int, [P, P]),
    "dgnn_session_run_epoch": (C.c_int, [P, C.POINTER(EpochReport)]),
    "dgnn_session_begin_epoch": (C.c_int, [P, C.POINTER(I64)]),
    "dgnn_session_local_grads": (C.c_int, [P, I64, P]),
    "dgnn_session_apply": (C.c_int, [P, P, C.POINTER(I32)]),
    "dgnn_session_end_epoch": (C.c_int, [P]),
    "dgnn_set_device": (C.c_int, [I32]),
    "dgnn_graph_retain": (C.c_int, [P, I32, I32]),
    "dgnn_comm_unique_id": (C.c_int, [P]),
    "dgnn_comm_create": (C.c_int, [P, I32, I32, C.POINTER(P)]),
    "dgnn_comm_free": (None, [P]),
    "dgnn_grad_allreduce": (C.c_int, [P, P, I64, P]),
    "dgnn_session_run_dist_epoch": (C.c_int, [P, P, C.POINTER(EpochReport)]),
    "dgnn_session_losses": (C.c_int, [P, P, C.POINTER(I64)]),
    "dgnn_session_sample_grads": (C.c_int, [P, I32, C.POINTER(D), P, P]),
    "dgnn_session_invocations": (C.c_int, [P, P, C.POINTER(I64)]),
    "dgnn_session_cache_events": (C.c_int, [P, P, C.POINTER(I64)]),
    "dgnn_session_stats": (C.c_int, [P, P]),
    "dgnn_session_tier_stats": (C.c_int, [P, P]),
    "dgnn_sliding_windows": (I64, [I32, I32, I32, I32, P, I64]),
    "dgnn_plan": (C.c_int, [I32, I32, I32, I32, I32, P]),
    "dgnn_cache_scores": (C.c_int, [P, C.POINTER(I32), C.POINTER(I32)]),
    "dgnn_key_hash": (U64, [I32, I32, I32, I32, I64, I64]),
    "dgnn_make_batches": (I64, [I32, I32, U64, I64, P, I64]),
    "dgnn_init_params": (I64, [C.POINTER(RunCfg), I32, P]),
    "dgnn_mem_stats": (C.c_int, [C.POINTER(I64)] * 4),
    "dgnn_prof_get_max": (C.c_int, [I32, C.POINTER(D)]),
    "dgnn_prof_enable": (C.c_int, [I32]),
    "dgnn_prof_reset": (C.c_int, []),
    "dgnn_prof_get": (C.c_int, [I32, C.POINTER(I64), C.POINTER(D), C.POINTER(D), C.POINTER(D)]),
}

_lib = None


class DgnnError(RuntimeError):
    pass


def header_symbols() -> list[str]:
    """Function names declared in include/dgnn_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dgnn_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2501_15348_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int):
    if rc == 0:
        return
    msg = lib().dgnn_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise IndexError(msg)
    raise DgnnError(msg)
