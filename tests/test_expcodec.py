"""Lossless bf16 exponent coding of expert parts (csrc/expcodec.cuh): host encoder (CPU tests:
sizes, ratio on the synthetic weights) and GPU decoder (bit-exact round trips on adversarial
inputs: zeros, denormals, inf/nan, wide exponent spreads, ragged lengths)."""
import ctypes
import math

import numpy as np
import pytest

from paper_2511_05814_b200 import _native


def encode(words: np.ndarray, kbits: int = 0) -> np.ndarray:
    lib = _native.load_library()
    w = np.ascontiguousarray(words, np.uint16)
    size = ctypes.c_uint64()
    _native.check(lib.moe_xc_encode(w.ctypes.data if w.size else None, w.size, kbits, None, 0,
                                    ctypes.byref(size)))
    out = np.zeros(size.value, np.uint8)
    _native.check(lib.moe_xc_encode(w.ctypes.data if w.size else None, w.size, kbits,
                                    out.ctypes.data, out.size, ctypes.byref(size)))
    assert size.value == out.size
    return out


def synthetic_expert_rows(n: int) -> np.ndarray:
    import oracle

    return np.asarray(oracle.hash_fill(42, (4 << 40) | 1, float(np.float32(1 / math.sqrt(4096))), n), np.uint16)


def test_ratio_on_synthetic_weights():
    w = synthetic_expert_rows(1 << 20)
    enc = encode(w)
    ratio = enc.size / (2 * w.size)
    assert ratio < 0.68, ratio            # two-level 2+3-bit codes: ~1.345 bytes / weight
    assert int.from_bytes(enc[4:8].tobytes(), "little") == 23
    assert encode(w, 3).size / (2 * w.size) < 0.71
    assert encode(w, 4).size / (2 * w.size) < 0.76


def _chunk_windows(enc):
    nch = int.from_bytes(enc[16:20].tobytes(), "little")
    return [int(enc[64 + 24 * c + 9]) for c in range(nch)]   # ChunkEntry: 24 bytes, win at 9


def _exponent_entropy_bound(w):
    _, cnt = np.unique((w >> 7) & 0xFF, return_counts=True)
    p = cnt / cnt.sum()
    return 1.0 + float(-(p * np.log2(p)).sum()) / 8.0


def test_level1_window_follows_the_exponent_mass():
    # bell-shaped weights: the most frequent offsets below the chunk maximum are 1..3
    w = synthetic_expert_rows(1 << 16)
    enc = encode(w, 23)
    assert set(_chunk_windows(enc)) == {1}
    # within 3 % of the order-0 exponent entropy bound (bytes / weight)
    assert enc.size / w.size < 1.03 * _exponent_entropy_bound(w)
    # a uniform draw keeps the window at the top
    rng = np.random.default_rng(1)
    u = (rng.uniform(-1, 1, 1 << 14).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    assert set(_chunk_windows(encode(u, 23))) == {0}
    # one large outlier per chunk pushes the window down
    z = synthetic_expert_rows(4096 * 3).copy()
    z[::4096] = 0x4780                                                      # 65536.0
    assert min(_chunk_windows(encode(z, 23))) >= 5


def test_sizes_are_deterministic_and_aligned():
    w = synthetic_expert_rows(12345)
    a, b = encode(w), encode(w)
    assert np.array_equal(a, b) and a.size % 16 == 0
    assert encode(np.zeros(0, np.uint16)).size % 16 == 0


def _cases():
    rng = np.random.default_rng(0)
    yield "synthetic", synthetic_expert_rows(4096 * 5)
    yield "normal", rng.standard_normal(10000).astype(np.float32).view(np.uint32).__rshift__(16).astype(np.uint16)
    yield "wide", rng.integers(0, 1 << 16, 9999, dtype=np.uint16)           # every exponent, nan/inf
    z = synthetic_expert_rows(8192)
    z[::3] = 0
    z[1::7] = 0x8000                                                        # -0
    z[2::11] = 0x0001                                                       # denormal
    yield "zeros", z
    yield "ragged", synthetic_expert_rows(4096 + 31)
    yield "tiny", synthetic_expert_rows(5)
    yield "const", np.full(4096 * 2, 0x3F80, np.uint16)
    o = synthetic_expert_rows(4096 * 4).copy()
    o[::4096] = 0x4780                                                      # windows 5..7
    o[4096 * 2 + 1::4096] = 0x7F00                                          # 2^127: window 7, escapes
    yield "outliers", o
    # exponents 253..255 dominate (Inf / NaN payloads, huge values) so the level-1 window is 0
    # and base + 1 - window = 256: byte-lane arithmetic must not carry across weights
    hi = rng.integers(0, 1 << 7, 4096 * 3, dtype=np.uint16) | (rng.integers(253, 256, 4096 * 3).astype(np.uint16) << 7)
    hi |= (rng.integers(0, 2, 4096 * 3).astype(np.uint16) << 15)
    hi[::5] = (hi[::5] & 0x807F) | (rng.integers(0, 250, hi[::5].size).astype(np.uint16) << 7)  # escapes
    yield "top_exponents", hi
    # escapes clustered in one lane (10 in lane 5 of chunk 1, 6 in lane 31 of chunk 2) with few
    # elsewhere: the chunk's escape window is used and a lane holds more than four escape bytes
    c = synthetic_expert_rows(4096 * 3).copy()
    c[4096 + 5 * 32 + np.arange(10) * 3] = 0x0100 | 0x8005                 # exponent 2
    c[2 * 4096 + 31 * 32 + np.arange(6) * 5] = 0x0180 | 0x0011              # exponent 3
    yield "clustered_escapes", c


@pytest.mark.gpu
@pytest.mark.parametrize("kbits", [0, 3, 4, 23])
def test_gpu_decode_round_trip_bit_exact(kbits):
    import torch

    lib = _native.lib()
    for name, w in _cases():
        enc = encode(w, kbits)
        dev = torch.from_numpy(enc).cuda()
        out = torch.full((w.size,), 0xABCD - 65536, dtype=torch.int16, device="cuda")
        _native.check(lib.moe_xc_decode(dev.data_ptr(), enc.ctypes.data, out.data_ptr(),
                                        _native.stream_ptr()))
        got = out.cpu().numpy().view(np.uint16)
        assert np.array_equal(got, w), name


@pytest.mark.gpu
def test_gpu_decode_rate():
    """One Mixtral-8x7B expert's w1|w3 part (117 M weights): decode must stay far below its
    PCIe time (235 MB compressed to ~162 MB; ~3 ms at 55 GB/s)."""
    import torch

    lib = _native.lib()
    w = synthetic_expert_rows(2 * 14336 * 4096)
    enc = encode(w)
    dev = torch.from_numpy(enc).cuda()
    out = torch.empty(w.size, dtype=torch.int16, device="cuda")
    args = (dev.data_ptr(), enc.ctypes.data, out.data_ptr(), _native.stream_ptr())
    _native.check(lib.moe_xc_decode(*args))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        _native.check(lib.moe_xc_decode(*args))
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    gbs = (enc.size + 2 * w.size) / ms / 1e6
    print(f"decode {ms:.3f} ms, {gbs:.0f} GB/s (read compressed + write bf16)")
    assert np.array_equal(out.cpu().numpy().view(np.uint16)[:1 << 20], w[:1 << 20])
    assert ms < 0.5
