"""K4 (tcgen05 grouped GEMM) against a plain PyTorch fp32 reference of the same op on the same
bf16 inputs.  Tolerance: fp32 accumulation of bf16 products in a different order, so
1e-3 relative to the output scale for the f32 outputs; the SwiGLU output is rounded to bf16,
so 1e-2 relative (the north star's bf16 bar)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2511_05814_b200 import _native

pytestmark = pytest.mark.gpu


def _gemm(A, B, G, gm, N, K, iters=1, splits=1):
    lib = _native.lib()
    C = torch.full((splits, A.shape[0], N), float("nan"), device="cuda", dtype=torch.float32)
    gm_c = (ctypes.c_int32 * G)(*gm)
    ms = ctypes.c_float(0)
    _native.check(lib.moe_tc_grouped_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), G, gm_c,
                                               N, K, splits, iters, ctypes.byref(ms),
                                               _native.stream_ptr()))
    torch.cuda.synchronize()
    return C.sum(0), ms.value


def _ref(A, B, gm, N):
    out, r = [], 0
    for g, m in enumerate(gm):
        out.append(A[r:r + m].float() @ B[g * N:(g + 1) * N].float().T)
        r += m
    return torch.cat(out)


@pytest.mark.parametrize("gm,N,K", [([128], 256, 64), ([128], 256, 512), ([300], 512, 1024),
                                    ([1, 77, 0, 130, 256], 256, 192), ([512], 4096, 4096)])
def test_grouped_gemm_matches_torch(gm, N, K):
    g = torch.Generator(device="cuda").manual_seed(sum(gm) + N + K)
    G = len(gm)
    A = torch.randn(sum(gm), K, device="cuda", generator=g).bfloat16()
    B = torch.randn(G * N, K, device="cuda", generator=g).bfloat16()
    C, _ = _gemm(A, B, G, gm, N, K)
    ref = _ref(A, B, gm, N)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-3, err


@pytest.mark.parametrize("splits", [2, 3, 9])
def test_split_k_planes_sum_to_the_product(splits):
    gm, N, K = [128, 5, 200], 512, 14 * 64
    g = torch.Generator(device="cuda").manual_seed(splits)
    A = torch.randn(sum(gm), K, device="cuda", generator=g).bfloat16()
    B = torch.randn(len(gm) * N, K, device="cuda", generator=g).bfloat16()
    C, _ = _gemm(A, B, len(gm), gm, N, K, splits=splits)
    ref = _ref(A, B, gm, N)
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-3


def test_grouped_swiglu_matches_torch():
    gm, f, d = [130, 0, 128, 255, 1], 256, 512
    G = len(gm)
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(sum(gm), d, device="cuda", generator=g).bfloat16()
    W = (torch.randn(G, 2 * f, d, device="cuda", generator=g) / d ** 0.5).bfloat16()
    act = torch.zeros(sum(gm), f, device="cuda", dtype=torch.bfloat16)
    lib = _native.lib()
    gm_c = (ctypes.c_int32 * G)(*gm)
    _native.check(lib.moe_tc_grouped_swiglu_bf16(X.data_ptr(), W.data_ptr(), act.data_ptr(), G, gm_c,
                                                 f, d, 1, None, _native.stream_ptr()))
    torch.cuda.synchronize()
    ref, r = [], 0
    for e, m in enumerate(gm):
        a1 = X[r:r + m].float() @ W[e, :f].float().T
        a3 = X[r:r + m].float() @ W[e, f:].float().T
        ref.append(torch.nn.functional.silu(a1) * a3)
        r += m
    ref = torch.cat(ref)
    err = (act.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err


def test_gemm_rate_mixtral_expert_shape():
    """Throughput on the prefill expert shape (512 tokens x top-2 over 8 experts): reported, and
    bounded below so a broken pipeline (e.g. serialised stages) fails loudly."""
    gm, N, K = [128] * 8, 4096, 14336
    A = torch.randn(sum(gm), K, device="cuda").bfloat16()
    B = torch.randn(8 * N, K, device="cuda").bfloat16()
    flops = 2.0 * sum(gm) * N * K
    for splits in (1, 2, 4):
        _, ms = _gemm(A, B, 8, gm, N, K, iters=5, splits=splits)
        bytes_ = B.numel() * 2 + A.numel() * 2 + splits * sum(gm) * N * 4
        print(f"grouped down-proj GEMM splits={splits}: {ms:.3f} ms, {flops / ms / 1e9:.1f} TFLOP/s, "
              f"{bytes_ / ms / 1e6:.1f} GB/s")
        assert flops / ms / 1e9 > 100
    # one expert (the prefill's per-expert launch): 16 tiles, split-K fills the SMs
    for splits in (1, 9):
        _, ms = _gemm(A[:128], B[:N], 1, [128], N, K, iters=5, splits=splits)
        bytes_ = N * K * 2 + 128 * K * 2 + splits * 128 * N * 4
        print(f"one-expert down-proj splits={splits}: {ms:.3f} ms, {bytes_ / ms / 1e6:.1f} GB/s")
