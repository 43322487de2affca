"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.

python tools/launch_summary.py gpurun_out/launches_bench.csv [header line ...]
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        k = d["Kernel Name"][:70]
        agg[k][0] += 1
        agg[k][1] += v
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    for h in sys.argv[2:]:
        print("#", h)
    print("# cold-cache, serialised launches: compare shares, not absolutes")
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {v[0]:8d} {v[1]:10.2f} {100 * v[1] / tot:6.1f}%")
