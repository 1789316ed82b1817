"""K4 in its tensor-bound regime: 8 experts x M rows (M = 128 .. 2048 token rows per expert, i.e.
prefills of 512 .. 8192 tokens), grouped SwiGLU up and down, CUDA-event timing per launch."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_05814_b200 import _native  # noqa: E402

lib = _native.lib()
D, F, G = 4096, 14336, 8
W13 = (torch.randn(G, 2 * F, D, device="cuda") / D ** 0.5).bfloat16()
W2 = (torch.randn(G * D, F, device="cuda") / F ** 0.5).bfloat16()
for m in [int(x) for x in (sys.argv[1:] or ["128", "256", "512", "1024", "2048"])]:
    gm = (ctypes.c_int32 * G)(*([m] * G))
    X = torch.randn(G * m, D, device="cuda").bfloat16()
    act = torch.empty(G * m, F, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(G * m, D, device="cuda", dtype=torch.float32)
    mu, md = ctypes.c_float(0), ctypes.c_float(0)
    _native.check(lib.moe_tc_grouped_swiglu_bf16(X.data_ptr(), W13.data_ptr(), act.data_ptr(), G, gm, F, D,
                                                 6, ctypes.byref(mu), _native.stream_ptr()))
    _native.check(lib.moe_tc_grouped_gemm_bf16(act.data_ptr(), W2.data_ptr(), out.data_ptr(), G, gm, D, F, 1,
                                               6, ctypes.byref(md), _native.stream_ptr()))
    torch.cuda.synchronize()
    fu, fd = 2.0 * G * m * 2 * F * D, 2.0 * G * m * F * D
    print(f"M={m:5d} rows/expert: up {mu.value:.3f} ms {fu / mu.value / 1e9:.0f} TFLOP/s | "
          f"down {md.value:.3f} ms {fd / md.value / 1e9:.0f} TFLOP/s", flush=True)
    del X, act, out
