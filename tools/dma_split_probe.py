"""Does splitting a host->device transfer into parts with an event after each (as the coded
demand copies do: 5 parts per expert) cost link time?  Pinned host -> HBM, 240 MB per "expert",
24 experts back to back on one copy stream, parts per expert in {1, 2, 5, 10, 40}, with and
without an event record after each part; GB/s over the whole sequence.

python tools/dma_split_probe.py
"""
import json

import torch


def run(parts, events, experts=24, nbytes=240 << 20, reps=2):
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    cs = torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(parts * experts)]
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            a.record(cs)
            k = 0
            for _e in range(experts):
                step = nbytes // parts
                for p in range(parts):
                    lo = p * step
                    hi = nbytes if p == parts - 1 else lo + step
                    dev[lo:hi].copy_(host[lo:hi], non_blocking=True)
                    if events:
                        evs[k].record(cs)
                    k += 1
            b.record(cs)
        torch.cuda.synchronize()
        best = max(best, experts * nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def main():
    for parts in (1, 2, 5, 10, 40):
        for events in (False, True):
            print(json.dumps({"parts_per_expert": parts, "event_per_part": events,
                              "GBps": run(parts, events)}), flush=True)


if __name__ == "__main__":
    main()
