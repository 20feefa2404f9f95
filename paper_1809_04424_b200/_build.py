"""Build of libvrb.so (sm_100a) with nvcc: one object per .cu, compiled in
parallel, linked with -shared.  Used by __graft_entry__.build()."""
from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libvrb.so")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--fmad=false",            # belt and braces: the FP64 fold uses explicit _rn intrinsics anyway
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-O2",
    "-Xptxas", "-O3",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "vrb.h"))
    return hs


def build(verbose: bool = False, extra: list[str] | None = None, force: bool = False,
          out: str | None = None, objdir: str | None = None) -> str:
    """Compile every csrc/*.cu and link libvrb.so (or `out`, with objects in
    `objdir`: experiment variants built with extra -D flags)."""
    OUT_ = out or OUT
    OBJ_ = objdir or OBJ
    os.makedirs(OBJ_, exist_ok=True)
    srcs = _sources()
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    flags = NVCC_FLAGS + list(extra or [])

    def compile_one(src):
        obj = os.path.join(OBJ_, os.path.basename(src)[:-3] + ".o")
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src)
                and os.path.getmtime(obj) >= hdr_mtime):
            return obj
        cmd = [nvcc(), *flags, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr)
        return obj

    with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    if (force or not os.path.exists(OUT_)
            or os.path.getmtime(OUT_) < max(os.path.getmtime(o) for o in objs)):
        tmp = OUT_ + f".tmp{os.getpid()}"
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, OUT_)
    return OUT_


if __name__ == "__main__":
    import sys
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
