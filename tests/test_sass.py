"""CPU check of the compiled distance kernels (reading A5, SURVEY 8(d)
"Evidence per kernel"): the fold acc = acc + t*t is written with
__dsub_rn / __dmul_rn / __dadd_rn, so the SASS of the mask kernel (no sqrt)
holds no DFMA at all, and the fill kernel's DFMAs are only those of its
__dsqrt_rn sequences (a few per MUFU.RSQ64H).  Read with cuobjdump from the
built library; profiles/r02/sass_distance.txt holds the census."""
import collections
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1809_04424_b200", "libvrb.so")


def _census():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or libvrb.so missing")
    txt = subprocess.run([exe, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    out = {}
    for f in re.split(r"\n\s+Function : ", txt)[1:]:
        name = f.split("\n", 1)[0].strip()
        ops = collections.Counter(m.split(".")[0] for m in re.findall(
            r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*(?:\.[A-Z0-9_]+)*)", f))
        out[name] = ops
    return out


def test_distance_fold_has_no_contraction():
    c = _census()
    mask = [v for k, v in c.items() if "k_dist_mask" in k]
    fill = [v for k, v in c.items() if "k_dist_fill" in k or "k_dist_full" in k]
    assert mask and len(fill) >= 2
    for ops in mask:
        assert ops["DFMA"] == 0 and ops["DADD"] > 0 and ops["DMUL"] > 0
    for ops in fill:
        assert ops["MUFU"] >= 1
        # the correctly rounded sqrt: ~5 DFMAs per MUFU.RSQ64H site, nothing
        # else (k_dist_full unrolls 16 folds and 16 sqrt sequences, whose own
        # DMULs outnumber the fold's)
        assert ops["DFMA"] <= 8 * ops["MUFU"]
        assert ops["DADD"] > 0 and ops["DMUL"] > 0


def test_bucket_rank_loads_by_tma():
    # the S3 chunk kernel takes its records by one cp.async.bulk (TMA) copy
    # completing on an mbarrier: UBLKCP plus the SYNCS barrier operations
    c = _census()
    rank = [v for k, v in c.items() if "k_bk_rank" in k]
    assert rank
    for ops in rank:
        assert ops["UBLKCP"] >= 1 and ops["SYNCS"] >= 2
