"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total
device time per kernel, launch count and share (cold-cache, serialised times)."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def summarise(path):
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1e-6)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ms
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
        print(f"{ms:12.3f} ms {n:6d} {100 * ms / tot:6.1f}%  {k}")
    print(f"{tot:12.3f} ms total")
