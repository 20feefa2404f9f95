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
    if data and "Metric Name" in data[0]:   # several metrics per launch: durations only, DRAM bytes beside
        dram = collections.defaultdict(float)
        for d in data:
            if d["Metric Name"].startswith("dram__bytes"):
                dram[d.get("ID")] += float(d["Metric Value"].replace(",", "")) * (
                    1e9 if d["Metric Unit"] == "Gbyte" else 1e6 if d["Metric Unit"] == "Mbyte" else
                    1e3 if d["Metric Unit"] == "Kbyte" else 1.0)
        data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
        for d in data:
            d["_dram"] = dram.get(d.get("ID"), 0.0)
    per = len(data) // nbuilds
    last = data[-per:]
    agg = collections.OrderedDict()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for d in last:
        name = d["Kernel Name"].split("(")[0][-48:]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += v
        a[2] += d.get("_dram", 0.0)
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        extra = f"  DRAM {v[2] / 1e9:7.2f} GB ({v[2] / 1e6 / max(v[1], 1e-9):6.0f} GB/s)" if v[2] else ""
        print(f"{v[1]:9.3f} ms {100 * v[1] / tot:5.1f}% x{v[0]:3d} {k}{extra}")
    print(f"total {tot:.3f} ms over {len(last)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
