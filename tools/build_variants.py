"""Build tuning variants of the library (one element per lane only) in parallel.
usage: python tools/build_variants.py NAME=DEF1,DEF2 NAME2=DEF ...
Outputs paper_2108_11560_b200/variants/NAME.so (git-ignored; travels to the GPU box)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2108_11560_b200 import build as B  # noqa: E402

out_dir = os.path.join(ROOT, "paper_2108_11560_b200", "variants")
os.makedirs(out_dir, exist_ok=True)


def one(spec):
    name, _, defs = spec.partition("=")
    defines = ["BLK_MIN_INSTANCES", "BLK_DIAG"] + [d for d in defs.split(",") if d]
    path = os.path.join(out_dir, name + ".so")
    B.build(out=path, defines=defines)
    return path


if __name__ == "__main__":
    for f in os.listdir(out_dir):
        if f.endswith(".so"):
            os.remove(os.path.join(out_dir, f))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
