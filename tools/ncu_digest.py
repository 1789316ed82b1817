"""Digest of one ncu --set full report: headline section metrics, stall reasons, per-opcode
and per-source-line instruction counts.  python tools/ncu_digest.py report.ncu-rep [units]
(units: divide instruction counts by this, e.g. the number of warps launched)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ('Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput',
        'Issue Slots Busy', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Instructions', 'No Eligible',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction')


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, units=1.0):
    r = ncu(rep, "--page", "details", "--csv")
    h = r[0]
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in KEYS:
            print(f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
    r = ncu(rep, "--page", "raw", "--csv")
    raw = dict(zip(r[0], r[2] if len(r) > 2 else r[1]))
    st = {k.split("stalled_")[1]: float(v) for k, v in raw.items()
          if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and v.replace(".", "").isdigit()}
    print("stalls:", ", ".join(f"{k} {int(v)}" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in raw:
            print(k, raw[k])
    r = ncu(rep, "--page", "source", "--csv", "--print-source", "sass")
    hh = r[1]
    ops = collections.Counter()
    for x in r[2:]:
        d = dict(zip(hh, x))
        t = d["Source"].split()
        if not t:
            continue
        o = t[1] if t[0].startswith("@") else t[0]
        ops[o.split(".")[0]] += int(d["Instructions Executed"] or 0)
    print("opcodes / unit:", ", ".join(f"{o} {c / units:.1f}" for o, c in ops.most_common(24)))
    r = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    agg = {}
    for x in r:
        if len(x) < 8 or not x[0].isdigit():
            continue
        try:
            n, s = int(x[7] or 0), int(x[4] or 0)
        except ValueError:
            continue
        a = agg.setdefault((int(x[0]), x[1][:80]), [0, 0])
        a[0] += n
        a[1] += s
    print("line: instr / unit, stall samples, source")
    for k, v in sorted(agg.items()):
        if v[0] > 0:
            print(f"{k[0]}: {v[0] / units:.1f} {v[1]} {k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
