"""Exponent decoder in isolation: one Mixtral-8x7B w1|w3 part (2 x 14336 x 4096 synthetic
bell-shaped bf16 weights) encoded on the host, decoded on the GPU.

python tools/xc_probe.py [--reps 20] [--once]
  prints coded bytes / weight, event-timed ms per decode and the HBM fraction of its
  algorithmic bytes (coded in + bf16 out) against MEASURED_PEAKS.json; --once decodes once
  after one warm-up (for `ncu --set full -k regex:decode`).
"""
import argparse
import ctypes
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2511_05814_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--n", type=int, default=2 * 14336 * 4096)
    a = ap.parse_args()
    import oracle

    lib = _native.lib()
    w = np.asarray(oracle.hash_fill(42, (4 << 40) | 1, float(np.float32(1 / math.sqrt(4096))), a.n),
                   np.uint16)
    size = ctypes.c_uint64()
    _native.check(lib.moe_xc_encode(w.ctypes.data, w.size, 0, None, 0, ctypes.byref(size)))
    enc = np.zeros(size.value, np.uint8)
    _native.check(lib.moe_xc_encode(w.ctypes.data, w.size, 0, enc.ctypes.data, enc.size,
                                    ctypes.byref(size)))
    dev = torch.from_numpy(enc).cuda()
    out = torch.empty(w.size, dtype=torch.int16, device="cuda")
    args = (dev.data_ptr(), enc.ctypes.data, out.data_ptr(), _native.stream_ptr())
    _native.check(lib.moe_xc_decode(*args))
    torch.cuda.synchronize()
    ok = bool(np.array_equal(out.cpu().numpy().view(np.uint16), w))
    if a.once:
        _native.check(lib.moe_xc_decode(*args))
        torch.cuda.synchronize()
        print(json.dumps({"bit_exact": ok}))
        return
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(a.reps):
        flush.zero_()   # L2 cold between decodes
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.moe_xc_decode(*args))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    algo = enc.size + 2 * w.size
    peaks = ROOT / "MEASURED_PEAKS.json"
    peak = 6552.6
    if peaks.exists():
        try:
            peak = float(json.loads(peaks.read_text()).get("hbm_gbs", peak))
        except Exception:
            pass
    gbs = algo / ms / 1e6
    print(json.dumps({"weights": w.size, "coded_bytes_per_weight": enc.size / w.size,
                      "bit_exact": ok, "ms_median": ms, "ms_min": float(min(ts)),
                      "algorithmic_MB": algo / 1e6, "GBps": gbs, "hbm_peak_GBps": peak,
                      "frac": gbs / peak}))


if __name__ == "__main__":
    main()
