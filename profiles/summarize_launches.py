"""Aggregates an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: share of device time, launches, mean duration."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if not r:
            continue
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"source: {path}")
    print(f"total {tot / 1e6:.2f} ms over {sum(v[0] for v in agg.values())} launches (ncu: serialized, cold caches)")
    print(f"{'share':>7} {'ms':>9} {'launches':>8} {'mean us':>9}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / tot * 100:6.1f}% {t / 1e6:9.3f} {c:8d} {t / c / 1e3:9.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
