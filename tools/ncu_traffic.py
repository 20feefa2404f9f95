"""Write profiles/fill_traffic.json from an ncu --set full report of the
triangle count + fill kernels: DRAM read/write bytes and duration of the fill
launch (k_triangles<1, ...>).  Usage: python tools/ncu_traffic.py rep workload [source-note]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, workload, note=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if "k_triangles<1" not in name and "k_triangles<(bool)1" not in name:
            continue

        def val(m):
            i = col[m]
            return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)

        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        d = {}
        path = os.path.join(ROOT, "profiles", "fill_traffic.json")
        if os.path.exists(path):
            d = json.load(open(path))
        d[workload] = {"kernel": name.split("(")[0], "dram_read_bytes_per_launch": rd,
                       "dram_write_bytes_per_launch": wr, "dram_bytes_per_launch": rd + wr,
                       "duration_ms_ncu": val("gpu__time_duration.sum"),
                       "source": note or f"{os.path.basename(rep)} (ncu --set full --clock-control none, 1 launch)"}
        json.dump(d, open(path, "w"), indent=1)
        print(json.dumps(d[workload]))
        return
    print("no fill kernel in", rep)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
