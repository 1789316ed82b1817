"""Summarise an ncu launch list (+ optional --set full report) into profiles/.

python tools/summarize_ncu.py <tag> [--rep gpurun_out/prof_<tag>.ncu-rep]
writes profiles/launches_<tag>.csv (compact), profiles/ncu_<tag>.md and, for the expert FFN
kernels, profiles/ncu_ffn_traffic.json (dram bytes per launch and per expert, read by bench.py).
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
EXPERT_UP = 2 * 14336 * 4096 * 2
EXPERT_DOWN = 14336 * 4096 * 2


def launches(tag):
    rows = list(csv.reader(open(ROOT / "gpurun_out" / f"launches_{tag}.csv")))
    hdr, per = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = per.setdefault(d["ID"], {"kernel": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(per.values())


def short(name):
    return name.replace("moe::", "").split("(")[0]


def main():
    tag = sys.argv[1]
    rep = sys.argv[sys.argv.index("--rep") + 1] if "--rep" in sys.argv else None
    ls = launches(tag)
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "grid", "time_us", "dram_read_MB", "dram_write_MB", "GBps"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in ls:
        t = e.get("gpu__time_duration.sum", 0.0) / 1e3
        rd = e.get("dram__bytes_read.sum", 0.0) / 1e6
        wr = e.get("dram__bytes_write.sum", 0.0) / 1e6
        w.writerow([short(e["kernel"]), e["grid"], f"{t:.2f}", f"{rd:.2f}", f"{wr:.2f}",
                    f"{(rd * 1e6) / (t * 1e3) if t else 0:.0f}"])
        a = agg[short(e["kernel"])]
        a[0] += 1
        a[1] += t
        a[2] += rd
    (ROOT / "profiles" / f"launches_{tag}.csv").write_text(out.getvalue())
    setup = {k: v for k, v in agg.items() if k.startswith(("hash_", "reset_states", "void at::"))}
    step = {k: v for k, v in agg.items() if k not in setup}
    total = sum(a[1] for a in step.values())
    md = [f"# ncu launch list `{tag}` (cold cache, serialised; compare shares, not absolutes)", "",
          "Decode kernels (share of the decode steps' kernel time; setup kernels listed below):", "",
          "| kernel | launches | total us | share | avg us | avg DRAM read MB | GB/s |",
          "|---|---|---|---|---|---|---|"]
    for k, (n, t, rd) in sorted(step.items(), key=lambda x: -x[1][1]):
        md.append(f"| `{k}` | {n} | {t:.1f} | {t / total:.1%} | {t / n:.2f} | {rd / n:.2f} | "
                  f"{rd * 1e3 / t if t else 0:.0f} |")
    md += ["", "Setup (weight synthesis, cold caches): " +
           ", ".join(f"`{k}` x{n} {t:.0f} us" for k, (n, t, rd) in setup.items())]
    # expert FFN traffic: launches that streamed a whole expert part
    ups = [e for e in ls if "stream_gemv_kernel<1" in e["kernel"] and e.get("dram__bytes_read.sum", 0) > 1e8]
    downs = [e for e in ls if "stream_gemv_kernel<2" in e["kernel"] and e.get("dram__bytes_read.sum", 0) > 5e7]
    if ups and downs:
        def per_expert(lst, unit):
            return sum((e["dram__bytes_read.sum"] + e.get("dram__bytes_write.sum", 0)) /
                       round(e["dram__bytes_read.sum"] / unit) for e in lst) / len(lst)
        up_b, dn_b = per_expert(ups, EXPERT_UP), per_expert(downs, EXPERT_DOWN)
        traffic = {"source": f"profiles/launches_{tag}.csv (ncu dram__bytes_read.sum + write.sum)",
                   "dram_bytes_per_expert": up_b + dn_b,
                   "algorithmic_bytes_per_expert": EXPERT_UP + EXPERT_DOWN,
                   "ratio": (up_b + dn_b) / (EXPERT_UP + EXPERT_DOWN),
                   "up_dram_bytes_per_expert": up_b, "down_dram_bytes_per_expert": dn_b}
        (ROOT / "profiles" / "ncu_ffn_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
        md += ["", f"Expert FFN DRAM traffic per expert: {(up_b + dn_b) / 1e6:.1f} MB vs "
                   f"{(EXPERT_UP + EXPERT_DOWN) / 1e6:.1f} MB algorithmic "
                   f"(ratio {(up_b + dn_b) / (EXPERT_UP + EXPERT_DOWN):.4f})."]
    if rep:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if rows:
            hdr = rows[0]
            want = ["gpu__time_duration.sum", "dram__bytes_read.sum",
                    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                    "launch__registers_per_thread", "launch__grid_size"]
            idx = [hdr.index(x) for x in want if x in hdr]
            md += ["", "## `--set full` captures", "",
                   "| kernel | " + " | ".join(hdr[i] for i in idx) + " |",
                   "|---" * (len(idx) + 1) + "|"]
            for r in rows[2:]:
                md.append(f"| `{short(r[hdr.index('Kernel Name')])}` | " +
                          " | ".join(r[i] for i in idx) + " |")
            stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled")
                     and not h.endswith("not_issued")]
            md += ["", "Top warp-stall samples:", ""]
            for r in rows[2:]:
                top = sorted(((float(r[i] or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                              for i in stall), reverse=True)[:4]
                md.append(f"* `{short(r[hdr.index('Kernel Name')])}`: " +
                          ", ".join(f"{n} {int(v)}" for v, n in top))
    (ROOT / "profiles" / f"ncu_{tag}.md").write_text("\n".join(md) + "\n")
    sys.stdout.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
