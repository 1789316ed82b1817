"""ORACLE (test infrastructure only): ctypes access to oracle/build/liboracle.so."""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"
_lib = None


def oracle_lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    lib = ctypes.CDLL(str(LIB))
    P = ctypes.c_void_p
    lib.oracle_replay_policy.argtypes = [P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                         ctypes.c_int64, P, P]
    lib.oracle_replay_policy.restype = ctypes.c_int
    lib.oracle_hash_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                     ctypes.c_int64, ctypes.c_int, P, ctypes.c_int]
    lib.oracle_hash_fill.restype = None
    lib.oracle_hash_fill_t.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P,
                                       ctypes.c_int]
    lib.oracle_hash_fill_t.restype = None
    _lib = lib
    return lib


def replay_policy(acts, num_experts, capacity, policy, decay_factor, decay_period):
    """kernels.replay_policy (kernels.py:60-147) restated in C: (T,K) -> two (T,E) uint8."""
    a = np.ascontiguousarray(acts, dtype=np.int64)
    T, K = a.shape
    rb = np.zeros((T, num_experts), np.uint8)
    ev = np.zeros((T, num_experts), np.uint8)
    status = oracle_lib().oracle_replay_policy(
        a.ctypes.data, T, K, num_experts, capacity, policy, float(decay_factor),
        int(decay_period), rb.ctypes.data, ev.ctypes.data)
    if status:
        raise ValueError("eviction without candidates (K > C)")
    return rb, ev


def hash_fill(seed: int, tensor_id: int, std: float, n: int, kind: str = "bf16",
              threads: int | None = None) -> np.ndarray:
    """Synthetic weights: kind 'bf16' (uint16 bits), 'f32', 'f64' / 'f32w' (bf16 widened)."""
    code, dtype = {"bf16": (0, np.uint16), "f32": (1, np.float32), "f64": (2, np.float64),
                   "f32w": (3, np.float32)}[kind]
    out = np.empty(n, dtype)
    oracle_lib().oracle_hash_fill(seed, tensor_id, std, n, code, out.ctypes.data,
                                  threads or os.cpu_count() or 1)
    return out


def hash_fill_t(seed: int, tensor_id: int, std: float, rows: int, cols: int, kind: str = "f64",
                threads: int | None = None) -> np.ndarray:
    """Transpose (cols, rows) of the logical (rows, cols) synthetic tensor; kind 'f64' / 'f32w'
    (bf16-rounded, widened) or 'f32'."""
    code, dtype = {"f32": (1, np.float32), "f64": (2, np.float64), "f32w": (3, np.float32)}[kind]
    out = np.empty((cols, rows), dtype)
    oracle_lib().oracle_hash_fill_t(seed, tensor_id, std, rows, cols, code, out.ctypes.data,
                                    threads or os.cpu_count() or 1)
    return out
