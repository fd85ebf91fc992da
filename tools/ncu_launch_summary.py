"""Summarise an ncu --csv launch list (gpu__time_duration.sum + dram bytes per launch): per kernel
(name without template arguments) the launches, total time, share of the iteration, DRAM bytes
and achieved GB/s; and every launch of the fidelity / update passes individually.
    python tools/ncu_launch_summary.py launches.csv [title] > summary.txt"""
import csv
import re
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    launches = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = int(r[ix["ID"]])
        d = launches.setdefault(key, {"name": r[ix["Kernel Name"]]})
        try:
            d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    return launches


def short(name):
    n = re.sub(r"\(.*$", "", name)
    n = re.sub(r"^void\s+", "", n)
    return n


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    L = load(path)
    tot = sum(d.get("gpu__time_duration.sum", 0.0) for d in L.values())
    agg = OrderedDict()
    for d in L.values():
        k = re.sub(r"<.*", "", short(d["name"]))
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    print(f"ncu launch list: {title} (cold-cache, serialised: compare shares, not absolutes)")
    print(f"{'kernel':34s} {'launches':>8s} {'us':>10s} {'share':>7s} {'DRAM MB':>9s} {'GB/s':>7s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:34s} {n:8d} {t / 1e3:10.1f} {t / tot:7.3f} {b / 1e6:9.1f} {b / t if t else 0:7.0f}")
    print(f"{'total':34s} {len(L):8d} {tot / 1e3:10.1f}")
    print("\nfidelity / update launches:")
    for i, d in L.items():
        n = short(d["name"])
        if any(s in n for s in ("blur", "phase", "step", "mri")):
            t = d.get("gpu__time_duration.sum", 0.0)
            b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            print(f"  {i:4d} {n[:60]:60s} {t / 1e3:8.1f} us {b / 1e6:8.1f} MB {b / t if t else 0:7.0f} GB/s")


if __name__ == "__main__":
    main()
