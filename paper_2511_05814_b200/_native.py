"""ctypes binding of libmoeb200.so (the C ABI declared in include/moeb200.h).

The product path is CUDA-only: if the shared library is missing or no CUDA device is
visible, every entry point raises instead of falling back to a CPU implementation.
Device buffers are torch CUDA tensors; only their data pointers cross the ABI.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError

LIB_PATH = Path(__file__).resolve().parent / "libmoeb200.so"

MOE_OK, MOE_INVALID_CONFIG, MOE_NONFINITE, MOE_CUDA_ERROR, MOE_OOM = range(5)
P_LRU, P_LFU, P_LFU_AGED, P_OPT = range(4)
EXPERT_TOY_TANH_F32, EXPERT_SWIGLU_BF16 = 0, 1
PREFETCH_OFF, PREFETCH_EARLY = 0, 1
TRANSFER_AUTO, TRANSFER_COPY_ENGINE, TRANSFER_SM = 0, 1, 2

# Every exported symbol, as declared in include/moeb200.h (checked by the CPU test suite).
EXPORTED = (
    "moe_last_error", "moe_abi_version", "moe_kernel_launches",
    "moe_replay_policy", "moe_replay_policy_layers", "moe_policy_step",
    "moe_gate_topk_f64", "moe_toy_forward_f64",
    "moe_engine_create", "moe_engine_create_ex", "moe_engine_destroy", "moe_engine_set_dense_f32",
    "moe_engine_set_toy_expert_f32", "moe_engine_init_random", "moe_engine_expert_host_ptr",
    "moe_engine_dense_host", "moe_engine_reset", "moe_engine_decode", "moe_engine_prefill", "moe_engine_sync",
    "moe_engine_records", "moe_engine_record_gaps", "moe_engine_stats", "moe_engine_set_mode", "moe_engine_profile",
    "moe_engine_kernel_times", "moe_microbench_gemv",
    "moe_hash_weights_bf16", "moe_hash_weights_f32",
    "moe_tc_grouped_gemm_bf16", "moe_tc_grouped_swiglu_bf16",
    "moe_text_data", "moe_text_size", "moe_text_free", "moe_format_trace", "moe_format_event_log",
    "moe_sample_zipf", "moe_sample_markov", "moe_engine_decode_routed", "moe_engine_prefill_routed",
    "moe_xc_encode", "moe_xc_decode", "moe_engine_coded_size", "moe_engine_attach_coded",
    "moe_engine_attach_peer_tier",
)


class EngineConfigC(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32),
        ("top_k", ctypes.c_int32), ("hidden_dim", ctypes.c_int32), ("ffn_dim", ctypes.c_int32),
        ("expert_kind", ctypes.c_int32), ("cache_size", ctypes.c_int32),
        ("policy", ctypes.c_int32), ("decay_factor", ctypes.c_double),
        ("decay_period", ctypes.c_int64), ("mixing_scale", ctypes.c_float),
        ("prefetch", ctypes.c_int32), ("renormalize", ctypes.c_int32),
        ("record_speculation", ctypes.c_int32), ("max_tokens", ctypes.c_int32),
        ("chunk_bytes", ctypes.c_int64), ("prefetch_depth", ctypes.c_int32),
        ("device", ctypes.c_int32), ("rms_norm", ctypes.c_int32), ("rms_eps", ctypes.c_float),
        ("transfer", ctypes.c_int32), ("store_layers", ctypes.c_int32),
        ("prefetch_buffers", ctypes.c_int32), ("compress", ctypes.c_int32),
    ]


class StatsC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "tokens", "steps", "hits", "misses", "h2d_bytes", "demand_bytes", "prefetch_bytes",
        "prefetch_issued", "prefetch_used", "prefetch_wasted_bytes", "expert_bytes")] + [
        ("copy_busy_ms", ctypes.c_double), ("prefill_tokens", ctypes.c_int64),
        ("prefill_bytes", ctypes.c_int64), ("demand_link_bytes", ctypes.c_int64),
        ("compressed_store_bytes", ctypes.c_int64), ("peer_bytes", ctypes.c_int64)]


class KernelTimesC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("mix_ms", "gate_ms", "ffn_ms", "finalize_ms")] + [
        (n, ctypes.c_int64) for n in ("mix_launches", "gate_launches", "ffn_launches",
                                      "finalize_launches", "ffn_expert_runs")] + [
        ("ffn_active_ms", ctypes.c_double), ("ffn_active_bytes", ctypes.c_int64),
        ("ffn_active_launches", ctypes.c_int64), ("gemm_ms", ctypes.c_double),
        ("gemm_launches", ctypes.c_int64), ("gemm_flops", ctypes.c_double),
        ("gemm_bytes", ctypes.c_int64), ("prefill_ms", ctypes.c_double),
        ("ffn_kernel_ms", ctypes.c_double), ("gemm_kernel_ms", ctypes.c_double),
        ("xdec_ms", ctypes.c_double), ("xdec_kernel_ms", ctypes.c_double),
        ("xdec_bytes", ctypes.c_int64), ("xdec_launches", ctypes.c_int64)]


_P = ctypes.c_void_p
_I32, _I64, _U64, _F64, _F32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_float

_SIGNATURES = {
    "moe_last_error": ([], ctypes.c_char_p),
    "moe_abi_version": ([], _I32),
    "moe_kernel_launches": ([], _U64),
    "moe_replay_policy": ([_P, _I64, _I32, _I32, _I32, _I32, _F64, _I64, _P, _P, _P], _I32),
    "moe_replay_policy_layers": ([_P, _I32, _I64, _I32, _I32, _I32, _I32, _F64, _I64, _P, _P, _P], _I32),
    "moe_policy_step": ([_P, _P, _P, _I64, _I32, _I32, _I32, _F64, _I64, _P, _I32, _P, _P, _I64,
                         _P, _P, _P], _I32),
    "moe_gate_topk_f64": ([_P, _P, _P, _I32, _I32, _I32, _P, _P, _P], _I32),
    "moe_toy_forward_f64": ([_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _F64, _P, _P, _P, _P], _I32),
    "moe_engine_create": ([ctypes.POINTER(EngineConfigC), ctypes.POINTER(_P)], _I32),
    "moe_engine_destroy": ([_P], _I32),
    "moe_engine_set_dense_f32": ([_P, _I32, _P, _P, _P], _I32),
    "moe_engine_set_toy_expert_f32": ([_P, _I32, _I32, _P, _P], _I32),
    "moe_engine_init_random": ([_P, _U64, _F32, _I32], _I32),
    "moe_engine_create_ex": ([ctypes.POINTER(EngineConfigC), _P, _I64, ctypes.POINTER(_P)], _I32),
    "moe_engine_expert_host_ptr": ([_P, _I32, _I32, ctypes.POINTER(_P), ctypes.POINTER(_I64)], _I32),
    "moe_engine_dense_host": ([_P, _I32, _P, _P, _P], _I32),
    "moe_engine_reset": ([_P], _I32),
    "moe_engine_decode": ([_P, _P, _I64, _P, _P], _I32),
    "moe_engine_prefill": ([_P, _P, _I64, _P, _P], _I32),
    "moe_engine_sync": ([_P], _I32),
    "moe_engine_records": ([_P, _I64, _I64, _P, _P, _P, _P, _P], _I32),
    "moe_engine_record_gaps": ([_P, _I64, _I64, _P, _P, _P, _P], _I32),
    "moe_engine_attach_peer_tier": ([_P, _P, _I64], _I32),
    "moe_engine_stats": ([_P, ctypes.POINTER(StatsC)], _I32),
    "moe_engine_set_mode": ([_P, _I32, _F64, _I64, _I32, _I32], _I32),
    "moe_engine_profile": ([_P, _I32], _I32),
    "moe_engine_kernel_times": ([_P, ctypes.POINTER(KernelTimesC)], _I32),
    "moe_microbench_gemv": ([_I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                             ctypes.POINTER(_F32), ctypes.POINTER(_I64)], _I32),
    "moe_hash_weights_bf16": ([_U64, _U64, _F32, _I64, _P, _P], _I32),
    "moe_hash_weights_f32": ([_U64, _U64, _F32, _I64, _P, _P], _I32),
    "moe_tc_grouped_gemm_bf16": ([_P, _P, _P, _I32, _P, _I32, _I32, _I32, _I32, ctypes.POINTER(_F32), _P], _I32),
    "moe_engine_coded_size": ([_P, ctypes.POINTER(_I64)], _I32),
    "moe_engine_attach_coded": ([_P, _P, _I64, _I32], _I32),
    "moe_xc_encode": ([_P, _U64, _I32, _P, _U64, ctypes.POINTER(_U64)], _I32),
    "moe_xc_decode": ([_P, _P, _P, _P], _I32),
    "moe_sample_zipf": ([_P, _I32, _I32, _I64, _I32, _P, _P, _P], _I32),
    "moe_sample_markov": ([_P, _I32, _I32, _I64, _I32, _F64, _P, _P, _P, _P], _I32),
    "moe_engine_decode_routed": ([_P, _P, _I64, _P, _P, _P], _I32),
    "moe_engine_prefill_routed": ([_P, _P, _I64, _P, _P, _P], _I32),
    "moe_text_data": ([_P], ctypes.c_void_p),
    "moe_text_size": ([_P], _I64),
    "moe_text_free": ([_P], None),
    "moe_format_trace": ([_I32, _I32, _I32, _I32, _I64, _P, _P, ctypes.POINTER(_P)], _I32),
    "moe_format_event_log": ([ctypes.c_char_p, _I32, _I32, _I32, _I32, _I64, _I32, _P, _I64, _P, _P,
                              _P, ctypes.POINTER(_P)], _I32),
    "moe_tc_grouped_swiglu_bf16": ([_P, _P, _P, _I32, _P, _I32, _I32, _I32, ctypes.POINTER(_F32), _P], _I32),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA-side failure (MOE_CUDA_ERROR / MOE_OOM)."""


def load_library() -> ctypes.CDLL:
    """Load libmoeb200.so (no CUDA call is made). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (tools/build_native.sh). There is no CPU fallback."
        )
    # MOEB200_LIB: a variant build of the same library (tuning probes only)
    lib = ctypes.CDLL(os.environ.get("MOEB200_LIB") or str(LIB_PATH))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    """The library, after checking a CUDA device is present (the product path is GPU-only)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_05814_b200 needs a CUDA device (sm_100a); no CPU fallback")
    torch.cuda.init()
    return load_library()


def check(status: int) -> None:
    if status == MOE_OK:
        return
    msg = load_library().moe_last_error().decode("utf-8", "replace")
    if status == MOE_INVALID_CONFIG:
        raise ConfigError(msg)
    if status == MOE_NONFINITE:
        raise FloatingPointError(msg)
    if status == MOE_OOM:
        raise MemoryError(msg)
    raise NativeError(msg)


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def take_text(handle) -> bytes:
    """Copy a library-owned moe_text into Python bytes and free it."""
    lib_ = load_library()
    try:
        return ctypes.string_at(lib_.moe_text_data(handle), lib_.moe_text_size(handle))
    finally:
        lib_.moe_text_free(handle)


def kernel_launches() -> int:
    return int(load_library().moe_kernel_launches())


def library_loaded_path() -> str:
    return os.fspath(LIB_PATH)
