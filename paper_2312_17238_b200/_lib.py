"""ctypes binding of ``libmoeb200.so`` (include/moeb200.h).

The library is the product: there is no Python or CPU fallback.  Importing
this module does not need a GPU (symbols resolve lazily); any call that needs
the device fails with a CUDA error mapped to ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NonFiniteError, QuantFormatError, UnknownExpertError

HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_LIB_PATH: an A/B build of the same sources (tools/ab_build.sh), profiling only
LIB_PATH = os.environ.get("MOE_LIB_PATH") or os.path.join(HERE, "libmoeb200.so")

MOE_OK, MOE_ERR_VALUE, MOE_ERR_RUNTIME, MOE_ERR_NONFINITE = 0, 1, 2, 3
MOE_ERR_UNKNOWN_EXPERT, MOE_ERR_FORMAT, MOE_ERR_CUDA, MOE_ERR_TIMEOUT = 4, 5, 6, 7


class ModelDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ffn",
                                        "n_experts", "top_k", "max_seq_len")]


class CacheCfg(C.Structure):
    _fields_ = [("k", C.c_int32), ("b", C.c_int32), ("expert_bytes", C.c_int64)]


class SpecCfg(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("m", C.c_int32), ("lookahead", C.c_int32)]


class Matrix(C.Structure):
    _fields_ = [("bits", C.c_int32), ("group_size", C.c_int32), ("scale_group_size", C.c_int32),
                ("meta_bits", C.c_int32), ("rows", C.c_int32), ("cols", C.c_int32),
                ("pad_count", C.c_int32), ("codes", C.c_void_p), ("codes_len", C.c_int64),
                ("zeros", C.c_void_p), ("n_groups", C.c_int64), ("zero_scales", C.c_void_p),
                ("zero_offsets", C.c_void_p), ("n_zruns", C.c_int64), ("scales", C.c_void_p),
                ("n_scales", C.c_int64)]


class Event(C.Structure):
    _fields_ = [("seq", C.c_int64), ("kind", C.c_int32), ("layer", C.c_int32),
                ("expert", C.c_int32), ("token_pos", C.c_int32), ("bytes_moved", C.c_int64)]


class TraceRec(C.Structure):
    _fields_ = [("token_pos", C.c_int32), ("layer", C.c_int32), ("experts", C.c_int32 * 8),
                ("weights", C.c_float * 8)]


class Stats(C.Structure):
    _fields_ = [("h2d_copies", C.c_int64), ("h2d_bytes", C.c_int64), ("h2d_busy_ms", C.c_double),
                ("h2d_peak_gbs", C.c_double), ("n_buffers", C.c_int64), ("slot_bytes", C.c_int64),
                ("device_bytes", C.c_int64), ("arena_bytes", C.c_int64),
                ("kernel_launches", C.c_int64), ("last_call_ms", C.c_double)]


P = C.c_void_p
I32, I64, U64 = C.c_int32, C.c_int64, C.c_uint64
FP = C.POINTER(C.c_float)
IP = C.POINTER(C.c_int32)

# name -> (restype, argtypes); mirrors include/moeb200.h exactly
SIGNATURES = {
    "moe_create": (I32, [C.POINTER(ModelDesc), C.POINTER(CacheCfg), C.POINTER(SpecCfg), I32, I32,
                         C.POINTER(P)]),
    "moe_load_tensor": (I32, [P, C.c_char_p, C.POINTER(Matrix)]),
    "moe_load_expert": (I32, [P, I32, I32, C.POINTER(Matrix), C.POINTER(Matrix),
                              C.POINTER(Matrix)]),
    "moe_synth_model": (I32, [P, U64, I32, I32]),
    "moe_parse_block": (I32, [P, I64, C.POINTER(Matrix), P, I64, C.POINTER(C.c_int64)]),
    "moe_load_tensor_serialized": (I32, [P, C.c_char_p, P, I64]),
    "moe_load_expert_serialized": (I32, [P, I32, I32, P, I64, P, I64, P, I64]),
    "moe_finalize": (I32, [P]),
    "moe_set_device": (I32, [I32]),
    "moe_measure_h2d": (I32, [P, I32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "moe_prefill": (I32, [P, IP, I32, FP]),
    "moe_step": (I32, [P, I32, FP]),
    "moe_decode_greedy": (I32, [P, I32, IP, FP]),
    "moe_num_events": (I64, [P]),
    "moe_read_events": (I32, [P, I64, I64, C.POINTER(Event)]),
    "moe_num_trace": (I64, [P]),
    "moe_read_trace": (I32, [P, I64, I64, C.POINTER(TraceRec), FP]),
    "moe_reset_session": (I32, [P]),
    "moe_device_state": (I32, [P, IP, IP]),
    "moe_get_stats": (I32, [P, C.POINTER(Stats)]),
    "moe_ep_configure": (I32, [P, I32, I32]),
    "moe_ep_handle": (I32, [P, C.c_void_p]),
    "moe_ep_connect": (I32, [P, C.c_void_p]),
    "moe_nccl_unique_id": (I32, [C.c_void_p]),
    "moe_ep_connect_nccl": (I32, [P, C.c_void_p]),
    "moe_set_profiling": (I32, [P, I32]),
    "moe_kernel_times": (I32, [P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "moe_profiler_range": (I32, [I32]),
    "moe_timeline": (I32, [P, I32]),
    "moe_read_timeline": (I32, [P, C.POINTER(C.c_uint64), I32, C.POINTER(C.c_int32)]),
    "moe_last_error": (C.c_char_p, []),
    "moe_destroy": (I32, [P]),
    "moe_quantize_device": (I32, [FP, I32, I32, I32, I32, I32, P, P, P, P, P]),
    "moe_gemv_device": (I32, [C.POINTER(Matrix), FP, FP]),
    "moe_synth_tensor_device": (I32, [U64, U64, I64, C.c_float, FP]),
    "moe_bench_gemv": (I32, [I32, I32, I32, I32, I32, I32, C.POINTER(C.c_double),
                             C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "moe_store_sim_create": (I32, [I32, I32, I32, I32, I64, I32, I32, P, C.POINTER(P)]),
    "moe_store_sim_token": (I32, [P, I32, I32, IP, I32, IP, I32, I32, IP]),
    "moe_store_sim_prefill": (I32, [P, I32, IP, I32, I32, IP]),
    "moe_store_sim_num_events": (I64, [P]),
    "moe_store_sim_events": (I32, [P, C.POINTER(Event), I64]),
    "moe_store_sim_state": (I32, [P, IP, IP, IP, IP, IP, IP]),
    "moe_store_sim_copies": (I64, [P]),
    "moe_store_sim_copy_policy": (I32, [P, I64, I64, I32]),
    "moe_store_sim_chunks": (I64, [P]),
    "moe_store_sim_parked": (I64, [P]),
    "moe_store_sim_set_park": (I32, [P, I32]),
    "moe_store_sim_last_error": (C.c_char_p, []),
    "moe_store_sim_destroy": (I32, [P]),
}

_lib = None


def lib():
    """Load the C-ABI library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2312_17238_b200.build` "
                              "(the B200 engine has no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int):
    """Map a MOE_* status onto the reference's exception classes."""
    if rc == MOE_OK:
        return
    msg = (lib().moe_last_error() or b"").decode(errors="replace")
    if rc == MOE_ERR_VALUE:
        raise ValueError(msg)
    if rc == MOE_ERR_NONFINITE:
        raise NonFiniteError(msg)
    if rc == MOE_ERR_UNKNOWN_EXPERT:
        raise UnknownExpertError(msg)
    if rc == MOE_ERR_FORMAT:
        raise QuantFormatError(msg)
    raise RuntimeError(msg)
