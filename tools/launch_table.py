"""Summarise an ncu --csv launch list: per-kernel count, total and mean gpu__time (us), and
any other metrics present (summed)."""
import csv
import sys
from collections import defaultdict, OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    data, names = defaultdict(dict), {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        i = int(r[ix["ID"]])
        names[i] = r[ix["Kernel Name"]]
        try:
            data[i][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    return names, data


def main(path, verbose=False):
    names, data = load(path)
    agg = OrderedDict()
    for i in sorted(data):
        n = names[i].split("(")[0]
        a = agg.setdefault(n, defaultdict(float))
        a["count"] += 1
        for k, v in data[i].items():
            a[k] += v
        if verbose:
            print(i, n, {k: v for k, v in data[i].items()})
    tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
    print(f"{'kernel':60s} {'n':>5s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for n, a in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
        t = a.get("gpu__time_duration.sum", 0) / 1e3
        print(f"{n[-60:]:60s} {int(a['count']):5d} {t:10.1f} {t / a['count']:9.1f} {t * 1e3 / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1], "-v" in sys.argv)
