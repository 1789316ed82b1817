"""Does the per-launch CUDA-event inflation under concurrent H2D depend on the copy chunk size?

Stream B streams 1 GiB host->device as back-to-back cudaMemcpyAsync chunks of S bytes; stream A
runs a 235 MB -> 235 MB elementwise SM kernel 20 times with an event pair around each launch.  If the event
timestamps are serialised behind the copy engine's current chunk, the inflation should track
S / link bandwidth.  Also reports the H2D throughput per chunk size (the link cost of chunking).
"""
import json
import os
import sys

import torch

# argv[1] == "hi": the kernel stream at the highest priority (CUDA_DEVICE_MAX_CONNECTIONS from
# the environment is reported too)
HI = len(sys.argv) > 1 and sys.argv[1] == "hi"

n = 235 * 2**20
src = torch.zeros(n // 2, dtype=torch.int16, device="cuda")
dst = torch.empty_like(src)
host = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
devh = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(priority=-5 if HI else 0), torch.cuda.Stream()


def h2d(chunk):
    for off in range(0, host.numel(), chunk):
        devh[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)


def spans(chunk, reps=20):
    torch.cuda.synchronize()
    if chunk:
        with torch.cuda.stream(sb):
            for _ in range(3):
                h2d(chunk)
    out = []
    with torch.cuda.stream(sa):
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(sa)
            torch.bitwise_not(src, out=dst)   # an SM kernel (a D2D memcpy may use a copy engine)
            b.record(sa)
            out.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) * 1e3 for a, b in out)
    return ms[len(ms) // 2], ms[0]


def link(chunk):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(sb):
        a.record(sb)
        h2d(chunk)
        b.record(sb)
    torch.cuda.synchronize()
    return host.numel() / (a.elapsed_time(b) * 1e-3) / 1e9


spans(0)
res = {"no_dma": spans(0)}
for c in [256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20]:
    med, mn = spans(c)
    res[f"{c >> 10}KB"] = {"median_us": round(med, 1), "min_us": round(mn, 1),
                            "h2d_GBps": round(link(c), 2)}
res["no_dma"] = {"median_us": round(res["no_dma"][0], 1), "min_us": round(res["no_dma"][1], 1)}
res["kernel_stream_high_priority"] = HI
res["CUDA_DEVICE_MAX_CONNECTIONS"] = os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS")
print(json.dumps(res))
