"""Build tuning variants of libpbng.so into build_variants/ (git-ignored; they travel to the GPU box).

    python tools/build_variants.py [--only float:MODEL_NH,common] NAME=DEF1,DEF2 [NAME=...]
e.g.  python tools/build_variants.py u2=PBNG_SWEEP_UNROLL=2 b256=PBNG_SWEEP_BLOCK=256
Time one with:  PBNG_LIB=build_variants/libpbng_u2.so python tools/tune_sweep.py --config 3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2306_09021_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "build_variants"), exist_ok=True)
    args = sys.argv[1:]
    only = None
    if args and args[0] == "--only":
        only = [None if u == "common" else tuple(u.split(":")) for u in args[1].split(",")]
        args = args[2:]
    for arg in args:
        name, defs = arg.split("=", 1)
        out = os.path.join(ROOT, "build_variants", f"libpbng_{name}.so")
        B.build(force=True, defines=[d for d in defs.split(",") if d], out=out, only=only)
        print(out)
