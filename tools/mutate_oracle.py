"""Mutation check of the oracle pins: apply plausible mistakes to a copy of
oracle/vr_oracle.c, rebuild, and confirm tests/test_oracle_pins.py fails for
each.  Usage: python tools/mutate_oracle.py   (CPU only, ~1 min)."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "vr_oracle.c")

MUTANTS = {
    "inclusive->strict": ("int keep = strict ? (len < radius) : (len <= radius);",
                          "int keep = strict ? (len < radius) : (len < radius);"),
    "ordinal ranks": ("if (p == 0 || er[p].len != er[p - 1].len) {\n            rank++;",
                      "if (1) {\n            rank++;"),
    "tie-break j before i": ("if (a->i != b->i) return a->i < b->i ? -1 : 1;\n    if (a->j != b->j) return a->j < b->j ? -1 : 1;",
                             "if (a->j != b->j) return a->j < b->j ? -1 : 1;\n    if (a->i != b->i) return a->i < b->i ? -1 : 1;"),
    "triangle filt drops jl": ("if (edge_filt(c, j, l) > f) f = edge_filt(c, j, l);", ""),
    "rows unsorted": ("for (int y = x; y > 0 && r[y - 1] > r[y]; --y) {\n                uint32_t tmp",
                      "for (int y = x; y > 0 && 0; --y) {\n                uint32_t tmp"),
    "fold drops last coord": ("for (int32_t c = 0; c < d; ++c) {\n        double t", "for (int32_t c = 0; c + 1 < d; ++c) {\n        double t"),
    "bar birth/death swapped": ("EMIT(k - 1, b, dth);", "EMIT(k - 1, dth, b);"),
    "essential ignores higher pivots": ("if (k + 1 <= K && piv[k + 1][q] >= 0) continue;", ""),
    "pHcol uses first low": ("while (R[j].n > 0 && pivot_row[R[j].a[R[j].n - 1]] >= 0)\n                gf2_add(&R[j], &R[pivot_row[R[j].a[R[j].n - 1]]], &tmp);",
                             "while (R[j].n > 0 && pivot_row[R[j].a[0]] >= 0)\n                gf2_add(&R[j], &R[pivot_row[R[j].a[0]]], &tmp);"),
    "sort by lex only": ("if (a->filt != b->filt) return a->filt < b->filt ? -1 : 1;\n    for (int t = 0; t < g_cmp_len",
                         "for (int t = 0; t < g_cmp_len"),
}


def main():
    orig = open(SRC).read()
    survived = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, (a, b) in MUTANTS.items():
            assert a in orig, name
            work = os.path.join(tmp, name.replace(" ", "_").replace(">", ""))
            shutil.copytree(ROOT, work, ignore=shutil.ignore_patterns(".git", "gpurun_out", "*.so", "build"))
            with open(os.path.join(work, "oracle", "vr_oracle.c"), "w") as f:
                f.write(orig.replace(a, b, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                "tests/test_oracle_pins.py"], cwd=work, capture_output=True, text=True)
            killed = r.returncode != 0
            print(f"{'killed ' if killed else 'SURVIVED'}  {name}")
            if not killed:
                survived.append(name)
    sys.exit(1 if survived else 0)


if __name__ == "__main__":
    main()
