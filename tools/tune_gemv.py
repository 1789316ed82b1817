"""Sweep the decode GEMV kernels in isolation (moe_microbench_gemv) and print GB/s.

python tools/tune_gemv.py [--quick]   -> JSON lines, one per configuration
"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2511_05814_b200 import _native  # noqa: E402

NAMES = ["stream-mix", "stream-up", "stream-down", "ldg-mix", "ldg-up", "ldg-down",
         "tma-only-mix", "tma-only-up", "tma-only-down"]


def run(kernel, d, f, experts, stage_kb=0, max_stages=6, grid=0, rpb=0, iters=20):
    lib = _native.lib()
    ms, nb = ctypes.c_float(), ctypes.c_int64()
    _native.check(lib.moe_microbench_gemv(kernel, d, f, experts, stage_kb, max_stages, grid, rpb,
                                          iters, ctypes.byref(ms), ctypes.byref(nb)))
    return {"kernel": NAMES[kernel], "d": d, "f": f, "experts": experts, "stage_kb": stage_kb,
            "max_stages": max_stages, "grid": grid, "rpb": rpb, "us": ms.value * 1e3,
            "GBps": nb.value / (ms.value / 1e3) / 1e9}


def main():
    d, f = 4096, 14336
    configs = []
    for k in (0, 1, 2):
        for ex in ((1, 2) if k else (1,)):
            configs.append(dict(kernel=k, d=d, f=f, experts=ex))          # engine defaults
            configs.append(dict(kernel=k + 6, d=d, f=f, experts=ex))      # same, no compute
            for rpb, skb in ((8, 64), (8, 96), (4, 64), (4, 32), (2, 64), (8, 32)):
                configs.append(dict(kernel=k + 6, d=d, f=f, experts=ex, stage_kb=skb, rpb=rpb))
    for c in configs:
        try:
            print(json.dumps(run(**c)), flush=True)
        except Exception as exc:  # noqa: BLE001
            print(json.dumps({"config": c, "error": str(exc)}), flush=True)


if __name__ == "__main__":
    main()
