"""Build experiment variants of libvrb.so with extra -D flags (in-tree,
variants/<name>/libvrb.so, git-ignored; they travel with the gpurun snapshot).
    python tools/variants.py name:-DVRB_TRI_MODE=0,-DVRB_TRI_WIN=1024 name2:...
Select one at run time with VRB_LIB_PATH=variants/<name>/libvrb.so."""
import concurrent.futures
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_04424_b200 import _build  # noqa: E402


def one(spec):
    name, _, flags = spec.partition(":")
    os.makedirs(os.path.join(ROOT, "variants", name), exist_ok=True)
    out = _build.build(extra=[f for f in flags.split(",") if f],
                       out=os.path.join(ROOT, "variants", name, "libvrb.so"),
                       objdir=os.path.join(ROOT, "build", "variants", name), force=True)
    return out


if __name__ == "__main__":
    with concurrent.futures.ThreadPoolExecutor(4) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
