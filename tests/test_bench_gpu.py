"""bench.py end to end on a B200 at reduced size: one JSON line carrying the driver contract's
keys (value, e2e, roofline, cpu_baseline, clocks, gpu_launches) and every section."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


def test_bench_reduced_run_prints_contract_line():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--layers", "2", "--steps", "3", "--warmup", "3",
           "--variants", "lru,lfu+prefetch,lfu@2", "--e2e-steps", "3", "--cpu-sample-tokens", "2",
           "--cpu-sample-layers", "1", "--cpu-repeats", "1",
           "--prefill-tokens", "64", "--prefill-decode", "4", "--tiny-tokens", "64",
           "--trace-variants", "zipf:1.0", "--replay-streams", "64", "--replay-tokens", "256"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "roofline_ffn", "cpu_baseline", "cpu_baseline_fp32", "e2e", "gpu_launches", "clocks",
              "pcie", "variants", "prefill", "tiny", "trace_driven", "replay", "kernel_timing"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert set(d["variants"]) == {"lru", "lfu+prefetch", "lfu@2"}
    assert all(v["check_hits_from_records"] for v in d["variants"].values())
    assert d["tiny"]["trace_equals_oracle"] and d["replay"]["decisions_equal_oracle_sample"]
    assert d["prefill"]["prefill_tokens_per_s"] > 0
    # the line's tail: parity against the oracle, the comparison table, the 8x22B section
    p = d["parity"]
    assert p["traces_equal_oracle_replay_all_variants"] and p["prefetch_issued_used_equal_oracle"]
    assert p["fp64_selections_headline"]["layers"] == 1
    assert p["fp64_selections_headline"]["mismatches"] == p["fp64_selections_headline"]["mismatches_at_near_ties"]
    assert set(d["variants_summary"]) == {"lru", "lfu+prefetch", "lfu@2"}
    assert list(d)[-3:] == ["variants_summary", "parity", "mixtral_8x22b"]
    assert d["mixtral_8x22b"]["tok_s"] > 0 and d["mixtral_8x22b"]["parity"]["traces_equal_oracle_replay_all_variants"]
    # both arms print the same workload config (the driver compares them key for key)
    ref = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--cpu-sample-layers", "1", "--cpu-sample-tokens", "2",
                          "--cpu-repeats", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    r = json.loads([ln for ln in ref.stdout.splitlines() if ln.startswith("{")][-1])
    assert r["config"] == d["config"]


def test_bench_8x22b_shape_reduced():
    """configs[4]'s bench path (Mixtral-8x22B shape, LFU + prefetch default) on 2 layers."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--model", "mixtral_8x22b", "--layers", "2",
           "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--cpu-sample-tokens", "2",
           "--cpu-sample-layers", "1", "--cpu-repeats", "1",
           "--prefill-tokens", "0", "--tiny-tokens", "0", "--trace-variants", "", "--replay-streams", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["config"]["workload"].startswith("configs[4]") and d["value"] > 0
    assert list(d["variants"]) == ["lfu+prefetch"]
    assert d["variants"]["lfu+prefetch"]["prefetch_issued"] > 0


def test_two_replicas_on_one_gpu_through_bench():
    """The N>1 replica path end to end on the one GPU gpurun has: torch.distributed.run with 2
    ranks (gloo, MOEB200_REPLICA_DEVICE=0), a node-shared raw + coded expert store created by
    local rank 0 and page-locked by both, one engine per rank on disjoint token streams, and the
    peer-HBM tier (each rank's home half of the raw experts in HBM, the other rank's mapped
    through CUDA IPC).  Every replica's live cache traces equal the oracle replay of its own
    selections, and the line aggregates both ranks' tokens over the slowest rank's time."""
    import os
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, MOEB200_REPLICA_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", "2",
           "--layers", "4", "--steps", "6", "--warmup", "3", "--variants", "lru,lfu+prefetch",
           "--prefill-tokens", "0", "--tiny-tokens", "0", "--replay-streams", "0",
           "--trace-variants", "", "--no-cpu-baseline", "--peer-tier"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2
    assert d["engine"]["shared_store"] is True
    assert d["parity"]["replicas_with_oracle_equal_traces"] == "2/2"
    assert d["parity"]["traces_equal_oracle_replay_all_variants"]
    # the peer tier (rank 1's HBM mapped by rank 0 over CUDA IPC) served part of the misses
    assert d["engine"]["peer_tier"].startswith("NVLink")
    assert all(v["peer_tier_GBps"] > 0 for v in d["variants"].values())
    # value = both ranks' tokens / the slowest rank's time
    assert abs(d["value"] - 2 * d["steps"] / (d["ms_per_step"] * d["steps"] / 1e3)) < 1e-6 * d["value"]
