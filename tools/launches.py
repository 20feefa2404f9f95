"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel
time of the LAST build in the file (one_build.py runs N builds)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main(path, nbuilds=2):
    data = load(path)
    per = len(data) // nbuilds
    last = data[-per:]
    agg = collections.OrderedDict()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for d in last:
        name = d["Kernel Name"].split("(")[0][-48:]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1]:9.3f} ms {100 * v[1] / tot:5.1f}% x{v[0]:3d} {k}")
    print(f"total {tot:.3f} ms over {len(last)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
