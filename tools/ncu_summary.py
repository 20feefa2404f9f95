"""Summarise an .ncu-rep: key metrics per kernel and the hottest SASS lines
with their dominant stall reasons.  Usage: python tools/ncu_summary.py rep [kernel-substr] [topN]"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Executed Instructions", "Avg. Active Threads Per Warp", "Grid Size", "Block Size")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, sub="", topn=25):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = hdr.index("ID")
    seen = {}
    for r in rows[1:]:
        if sub and sub not in r[ki]:
            continue
        if r[mi] in KEYS:
            seen.setdefault((r[idi], r[ki][:70]), []).append(f"{r[mi]}={r[vi]}{r[ui]}")
    for (i, k), v in seen.items():
        print(f"== [{i}] {k}")
        print("   " + "; ".join(v))
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h = raw[0]
    want = [c for c in h if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                                  "gpu__time_duration.sum")]
    for r in raw[2:]:
        d = dict(zip(h, r))
        if sub and sub not in d.get("Kernel Name", ""):
            continue
        print("   raw:", d.get("ID"), {c: d[c] for c in want})
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source=sass"))))
    cur, hdr2, out = None, None, {}
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = r[1]
            out[cur] = []
            hdr2 = None
            continue
        if r and r[0] == "Address":
            hdr2 = r
            continue
        if hdr2 and cur and len(r) == len(hdr2):
            out[cur].append(dict(zip(hdr2, r)))
    for k, lines in out.items():
        if sub and sub not in k:
            continue
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(float(l.get(key, 0) or 0) for l in lines) or 1.0
        stalls = [c for c in hdr2 if c.startswith("stall_") and "Not Issued" not in c]
        agg = {c: sum(float(l.get(c, 0) or 0) for l in lines) for c in stalls}
        print(f"-- {k[:80]}: {len(lines)} SASS, samples {tot:.0f}")
        print("   stall mix:", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in
                                        sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
        idx = sorted(range(len(lines)), key=lambda i: -float(lines[i].get(key, 0) or 0))[:topn]
        for i in sorted(idx):
            l = lines[i]
            v = float(l.get(key, 0) or 0)
            top = sorted(((float(l.get(c, 0) or 0), c[6:]) for c in stalls), reverse=True)[:2]
            print(f"   {i:5d} {100 * v / tot:5.1f}% {l['Source'].strip()[:60]:60s} {[(n, int(x)) for x, n in top if x > 0]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 25)
