"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0]
            name = name.replace("void ", "").split("<")[0]
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d.get("Metric Unit"), 1e-3)
            v = float(d["Metric Value"].replace(",", "")) * scale
            per[name].append(v)
            order.append((d["ID"], name, v))
    for i, n, v in order:
        print(f"{i:>4} {n:<45} {v:10.2f} us")
    print("--- per kernel: launches, mean us, min us")
    for n, vs in per.items():
        print(f"{n:<45} {len(vs):4d} {sum(vs) / len(vs):10.2f} {min(vs):10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
