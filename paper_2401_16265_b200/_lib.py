"""ctypes binding of the C ABI declared in include/co2_b200.h.

The shared library is built in-tree (``make`` at the repo root, or
``__graft_entry__.build()``).  There is no fallback: if the library is
missing or stale every entry point raises, loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libco2b200.so")

ABI_VERSION = 3
OK, ERR_VALIDATION, ERR_NUMERIC, ERR_CUDA, ERR_NCCL = 0, 2, 3, 4, 5
MODE_F64, MODE_F32, MODE_BF16_MIXED = 0, 1, 2
DTYPE_F64, DTYPE_F32, DTYPE_BF16 = 0, 1, 2
FLAG_GAP_NONFINITE, FLAG_GAP_BELOW_ONE, FLAG_M_NONFINITE = 1, 2, 4
FLAG_CLIP_NONFINITE, FLAG_X_NONFINITE, FLAG_AVG_NONFINITE = 8, 16, 32
FLAG_SLOWMO_M, FLAG_SLOWMO_X, FLAG_OVERLAP, FLAG_NORM_NONFINITE = 64, 128, 256, 512
CLIP_COORDINATE, CLIP_GLOBAL_NORM = 0, 1
FLAG_NONFINITE_INPUT = 1024
ALG_CO2, ALG_SLOWMO, ALG_LOCAL_SGD, ALG_OVERLAP_LOCAL_SGD, ALG_SYNC_SGD = 0, 1, 2, 3, 4
BUF_PARAMS, BUF_ANCHOR, BUF_XFIRST, BUF_PREV_X0, BUF_PREV_X1 = 0, 1, 2, 3, 4
BUF_MOMENTUM, BUF_GAP, BUF_XBAR, BUF_PARAMS_ALT, BUF_XFIRST_ALT = 5, 6, 7, 8, 9
IPC_HANDLE_BYTES = 72  # CUDA IPC handle (64) + int64 offset
NCCL_ID_BYTES = 128
NCCL_FIXED_ORDER, NCCL_SUM = 0, 1


class Hyper(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("phi", C.c_double),
                ("epsilon", C.c_double), ("tau", C.c_int32), ("penalty", C.c_uint8),
                ("clip", C.c_uint8), ("ghost_consistent", C.c_uint8), ("pad", C.c_uint8)]


class Diag(C.Structure):
    _fields_ = [("min_gap", C.c_double), ("max_outer_step", C.c_double),
                ("n_clipped", C.c_int64), ("n_floored", C.c_int64),
                ("flags", C.c_uint32), ("pad", C.c_uint32)]


class Cluster(C.Structure):
    _fields_ = [("workers", C.c_int32), ("gpus_per_node", C.c_int32), ("t_comp", C.c_double),
                ("t_outer", C.c_double), ("param_bytes", C.c_double),
                ("inter_bandwidth", C.c_double), ("latency", C.c_double),
                ("has_measured_override", C.c_int32), ("measured_override", C.c_double)]


class RoundTiming(C.Structure):
    _fields_ = [("t", C.c_int32), ("start", C.c_double), ("stall", C.c_double),
                ("end", C.c_double)]


class Timeline(C.Structure):
    _fields_ = [("workers", C.c_int32), ("tau", C.c_int32), ("rounds", C.c_int32),
                ("batch_size", C.c_int32), ("comm_time", C.c_double), ("wall_time", C.c_double),
                ("total_stall", C.c_double), ("overlap_ratio_achieved", C.c_double),
                ("throughput", C.c_double)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("handle", C.c_uint64),
                ("t", C.c_double), ("stall", C.c_double)]


class HandleInfo(C.Structure):
    _fields_ = [("id", C.c_uint64), ("launch_time", C.c_double), ("completion_time", C.c_double),
                ("stall", C.c_double), ("comm", C.c_double), ("completed", C.c_int32),
                ("consumed", C.c_int32), ("contributions", C.c_int32), ("polled", C.c_int32),
                ("last_poll", C.c_int32), ("completion_logged", C.c_int32)]


class RoundResult(C.Structure):
    _fields_ = [("stall_seconds", C.c_double), ("outer_applied", C.c_int32), ("pad", C.c_int32),
                ("min_gap", C.c_double), ("max_outer_step", C.c_double),
                ("n_clipped", C.c_int64), ("n_floored", C.c_int64)]


P, I32, I64, U64, D, U8P = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_char_p
ST = C.c_int32

# name -> (restype, argtypes); exactly the symbols of include/co2_b200.h
SIGNATURES = {
    "co2_last_error": (C.c_char_p, []),
    "co2_abi_version": (I32, []),
    "co2_hyper_validate": (ST, [C.POINTER(Hyper)]),
    "co2_workspace_bytes": (C.c_size_t, []),
    "co2_workspace_init": (ST, [P, P]),
    "co2_diag_fetch_async": (ST, [P, C.POINTER(Diag), P]),
    "co2_diag_fetch": (ST, [P, C.POINTER(Diag), P]),
    "co2_diag_status": (ST, [C.POINTER(Diag)]),
    "co2_outer_step": (ST, [I32, I64, P, P, P, P, I32, P, P, P, P, C.POINTER(Hyper), P, P]),
    "co2_outer_step_global_clip": (ST, [I32, I64, P, P, P, P, I32, P, P, P, P, C.POINTER(Hyper),
                                        P, P]),
    "co2_global_clip_norm_fetch": (ST, [P, C.POINTER(D), P]),
    "co2_global_clip_chunk": (I64, [I32, I64]),
    "co2_set_fused_variant": (ST, [I32]),
    "co2_set_grid_waves": (ST, [I32]),
    "co2_outer_step_host": (ST, [I32, I64, P, P, P, P, I32, P, P, P, C.POINTER(Hyper), I64, I32,
                                 C.POINTER(Diag)]),
    "co2_staleness_gap": (ST, [I32, I64, P, P, P, I32, D, P, P, P]),
    "co2_penalized_momentum": (ST, [I32, I64, P, D, P, P, I32, P, P, P]),
    "co2_outer_iterate": (ST, [I32, I64, P, D, P, D, I32, P, P, P]),
    "co2_clip_elementwise": (ST, [I32, I64, P, D, P, P, P]),
    "co2_ensure_finite": (ST, [I32, I64, P, C.c_char_p, P, P]),
    "co2_elementwise_abs_diff": (ST, [I32, I64, P, P, P, P, P]),
    "co2_l2_norm": (ST, [I32, I64, P, C.POINTER(D), P, P]),
    "co2_average": (ST, [I32, I32, C.POINTER(P), I64, P, P, P]),
    "co2_sub": (ST, [I32, I64, P, P, P, P]),
    "co2_divergence": (ST, [I32, I32, C.POINTER(P), I64, C.POINTER(D), C.POINTER(D), P, P]),
    "co2_convert": (ST, [I32, P, I32, P, I64, P]),
    "co2_synth": (ST, [I32, U64, I32, I64, I64, P, P, P, P, P, P]),
    "co2_synthetic_inner_step": (ST, [I32, I64, P, D, D, U64, I32, I64, I32, P]),
    "co2_synthetic_inner_step_snapshot": (ST, [I32, I64, P, D, D, U64, I32, I64, I32, P, P]),
    "co2_fill_u32": (ST, [P, C.c_uint32, I64, P]),
    "co2_cluster_validate": (ST, [C.POINTER(Cluster)]),
    "co2_allreduce_time": (ST, [C.POINTER(Cluster), C.POINTER(D)]),
    "co2_overlap_ratio": (ST, [I32, D, D, C.POINTER(D)]),
    "co2_simulate_timeline_co2": (ST, [C.POINTER(Cluster), I32, I32, I32, C.POINTER(Timeline),
                                       C.POINTER(RoundTiming)]),
    "co2_simulate_timeline": (ST, [I32, C.POINTER(Cluster), I32, I32, I32, C.POINTER(Timeline),
                                  C.POINTER(RoundTiming)]),
    "co2_scalability_ratio": (ST, [D, D, D, D, C.POINTER(D)]),
    "co2_nccl_unique_id": (ST, [C.POINTER(C.c_uint8)]),
    "co2_aar_create_nccl": (ST, [C.POINTER(P), C.POINTER(C.c_uint8), I32, I32, I32]),
    "co2_aar_create_local": (ST, [C.POINTER(P), I32]),
    "co2_ipc_export": (ST, [P, C.POINTER(C.c_uint8)]),
    "co2_aar_create_p2p": (ST, [C.POINTER(P), I32, I32, I32]),
    "co2_aar_signal_buffer": (P, [P]),
    "co2_aar_p2p_attach_signals": (ST, [P, C.POINTER(C.c_uint8)]),
    "co2_aar_p2p_attach": (ST, [P, P, C.POINTER(C.c_uint8)]),
    "co2_aar_p2p_detach": (ST, [P, P]),
    "co2_aar_set_fused": (ST, [P, I32]),
    "co2_aar_set_adaptive": (ST, [P, I32]),
    "co2_aar_ctas": (I32, [P]),
    "co2_aar_set_nccl_algo": (ST, [P, I32]),
    "co2_aar_order_after": (ST, [P, U64, P]),
    "co2_aar_destroy": (ST, [P]),
    "co2_aar_world": (I32, [P]),
    "co2_aar_launch": (ST, [P, I32, C.POINTER(P), P, I64, P, C.POINTER(U64)]),
    "co2_aar_poll": (ST, [P, U64, C.POINTER(I32)]),
    "co2_aar_wait": (ST, [P, U64, P]),
    "co2_aar_stall": (ST, [P, U64, C.POINTER(D), C.POINTER(D)]),
    "co2_aar_live": (ST, [P, C.POINTER(I32)]),
    "co2_aar_info": (ST, [P, U64, C.POINTER(HandleInfo)]),
    "co2_aar_totals": (ST, [P, C.POINTER(D), C.POINTER(U64)]),
    "co2_aar_allreduce_blocking": (ST, [P, I32, P, I64, P]),
    "co2_aar_events": (ST, [P, C.POINTER(Event), I64, C.POINTER(I64)]),
    "co2_worker_create": (ST, [C.POINTER(P), I32, I64, P, I32, P]),
    "co2_worker_destroy": (ST, [P]),
    "co2_worker_buffer": (P, [P, I32]),
    "co2_worker_set_clip_mode": (ST, [P, I32]),
    "co2_worker_round": (I32, [P]),
    "co2_worker_keep_average": (ST, [P, I32]),
    "co2_worker_snapshot_start": (ST, [P, P]),
    "co2_worker_snapshot_first": (ST, [P, P]),
    "co2_round": (ST, [C.POINTER(P), I32, P, C.POINTER(Hyper), P, I32, C.POINTER(RoundResult)]),
    "co2_round_finish": (ST, [C.POINTER(P), I32, P, C.POINTER(RoundResult)]),
    "co2_round_host": (ST, [C.POINTER(P), I32, P, C.POINTER(Hyper), C.POINTER(P), C.POINTER(P),
                            C.POINTER(P), P, I32, C.POINTER(RoundResult)]),
    "co2_round_drain": (ST, [C.POINTER(P), I32, P, P]),
    "co2_slowmo_step": (ST, [I32, I64, P, P, I32, P, P, P, D, D, P, P]),
    "co2_local_sgd_step": (ST, [I32, I64, P, P, I32, P, P, P, P]),
    "co2_overlap_correction": (ST, [I32, I64, P, P, P, I32, P, P]),
    "co2_slowmo_round": (ST, [C.POINTER(P), I32, P, D, D, P, I32, C.POINTER(RoundResult)]),
    "co2_local_sgd_round": (ST, [C.POINTER(P), I32, P, P, I32, C.POINTER(RoundResult)]),
    "co2_overlap_local_sgd_round": (ST, [C.POINTER(P), I32, P, I32, P, I32,
                                         C.POINTER(RoundResult)]),
    "co2_outer_step_ghost": (ST, [I32, I64, P, P, P, I32, P, I32, I32, P, P, P, P, P,
                                  C.POINTER(Hyper), P, P]),
    "co2_sharded_create": (ST, [C.POINTER(P), I32, I64, P, P, I32, P]),
    "co2_sharded_destroy": (ST, [P]),
    "co2_sharded_buffer": (P, [P, I32]),
    "co2_sharded_shard": (I64, [P, C.POINTER(I64), C.POINTER(I64)]),
    "co2_sharded_snapshot_start": (ST, [P, P]),
    "co2_sharded_snapshot_first": (ST, [P, P]),
    "co2_sharded_round": (ST, [P, P, C.POINTER(Hyper), P, I32, C.POINTER(RoundResult)]),
    "co2_sharded_drain": (ST, [P, P, P]),
    "co2_sharded_enable_timing": (ST, [P, I32]),
    "co2_sharded_step_times": (ST, [P, C.POINTER(D), I32, C.POINTER(I32)]),
    "co2_worker_enable_timing": (ST, [P, I32]),
    "co2_worker_step_times": (ST, [P, C.POINTER(D), I32, C.POINTER(I32)]),
}


class ValidationError(RuntimeError):
    """co2sim::validation_error (proj/include/co2sim/errors.hpp:8-13)."""


class NumericError(RuntimeError):
    """co2sim::numeric_error (proj/include/co2sim/errors.hpp:15-20)."""


class CudaError(RuntimeError):
    pass


_lib = None


def lib() -> C.CDLL:
    """Load libco2b200.so (no fallback: raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "the CO2 outer step has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.co2_abi_version() != ABI_VERSION:
            raise ImportError("libco2b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(code: int) -> None:
    """Map a co2_status_t to the reference's exception types."""
    if code == OK:
        return
    msg = lib().co2_last_error().decode()
    if code == ERR_VALIDATION:
        raise ValidationError(msg)
    if code == ERR_NUMERIC:
        raise NumericError(msg)
    raise CudaError(f"status {code}: {msg}")
