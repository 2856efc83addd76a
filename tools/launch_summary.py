"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").split("::")[-1]
        agg[name].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:24s} n={len(v):4d} {sum(v) / len(v) / 1e6:8.4f} ms/launch {sum(v) / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
