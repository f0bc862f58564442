"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k:44s} n={v[0]:4d} total={v[1] / 1e3:9.1f}us avg={v[1] / v[0] / 1e3:8.2f}us "
              f"{100 * v[1] / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
