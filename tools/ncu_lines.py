"""Per-source-line instruction and stall totals from an .ncu-rep (needs -lineinfo).
Usage: python tools/ncu_lines.py rep kernel-substr [topN]"""
import csv
import io
import subprocess
import sys


def main(rep, sub, topn=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fn, hdr, lines, path = None, None, {}, None
    for r in rows:
        if r and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r and r[0] == "Function Name":
            fn = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not (fn and sub in fn and hdr and len(r) == len(hdr) and r[0]):
            continue
        d = dict(zip(hdr, r))
        key = (path, int(r[0]))
        ex = float(d.get("Instructions Executed", 0) or 0)
        st = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        a = lines.setdefault(key, [0.0, 0.0, r[1]])
        a[0] += ex
        a[1] += st
    tex = sum(v[0] for v in lines.values()) or 1
    tst = sum(v[1] for v in lines.values()) or 1
    print(f"total instructions {tex / 1e9:.2f}e9, stall samples {tst:.0f}")
    for (f, ln), (ex, st, src) in sorted(lines.items(), key=lambda kv: -(kv[1][0] / tex + kv[1][1] / tst))[:topn]:
        print(f"{f}:{ln:<4d} inst {100 * ex / tex:5.1f}%  stall {100 * st / tst:5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
