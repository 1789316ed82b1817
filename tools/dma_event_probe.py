"""Do busy H2D copies (another stream) inflate a kernel's CUDA-event span?  Times a D2D copy
(~235 MB, HBM-bound) with events on stream A, with and without a pinned H2D copy loop on stream
B, and the same copies back to back (event pairs around each).  Caveat (round 2): a contiguous
D2D `copy_` may run on a copy engine rather than the SMs; tools/event_chunk_probe.py repeats the
measurement with an SM kernel and per H2D chunk size (profiles/box_probe_r2.md)."""
import torch

n = 235 * 2**20
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
host = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
devh = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def run(dma: bool, reps=20):
    torch.cuda.synchronize()
    if dma:
        with torch.cuda.stream(sb):
            for _ in range(6):
                devh.copy_(host, non_blocking=True)
    spans = []
    with torch.cuda.stream(sa):
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(sa)
            dst.copy_(src, non_blocking=True)
            b.record(sa)
            spans.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in spans)
    return ms[len(ms) // 2], ms[0]


for dma in (False, True, False, True):
    med, mn = run(dma)
    print(f"dma={dma}: D2D 235 MB copy kernel event span median {med*1e3:.1f} us, min {mn*1e3:.1f} us")


def run_total(dma: bool, reps=20):
    torch.cuda.synchronize()
    if dma:
        with torch.cuda.stream(sb):
            for _ in range(6):
                devh.copy_(host, non_blocking=True)
    with torch.cuda.stream(sa):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sa)
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        b.record(sa)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for dma in (False, True):
    print(f"dma={dma}: one event pair over 20 copies: {run_total(dma)*1e3:.1f} us per copy")
# the same with a GEMM-free, read-only kernel: sum over 235 MB
x = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")


def run_sum(dma, reps=20):
    torch.cuda.synchronize()
    if dma:
        with torch.cuda.stream(sb):
            for _ in range(6):
                devh.copy_(host, non_blocking=True)
    with torch.cuda.stream(sa):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sa)
        for _ in range(reps):
            x.sum()
        b.record(sa)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for dma in (False, True):
    print(f"dma={dma}: read-only reduction over 235 MB: {run_sum(dma)*1e3:.1f} us")
