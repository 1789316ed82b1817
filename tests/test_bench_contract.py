"""bench.py's driver contract on the CPU: the reference arm (--impl reference, the oracle port of
the path on the host cores) prints one JSON line with the contract's keys; its GPU arm is
exercised by the round-end bench on a B200."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--cpu-sample-layers", "1", "--cpu-sample-tokens", "2",
                          "--cpu-repeats", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    assert d["cpu_baseline"]["layers_sampled"] == 1 and d["cpu_baseline"]["scale"] == 32
    # the config both arms print is one function of the workload (the driver's same_config)
    sys.path.insert(0, str(ROOT))
    import bench

    assert d["config"] == bench.workload_config("mixtral_8x7b", 1, 4, "lru")
