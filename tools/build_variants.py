"""Build tuning variants of the library: python tools/build_variants.py NAME "-DX=1 -DY=2" ...
-> variants/NAME/libmlbm_b200.so (select with MLBM_LIB=...)."""
import os, sys, shlex
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14982_b200 import _lib as L
args = sys.argv[1:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for name, flags in zip(args[::2], args[1::2]):
    out = os.path.join(root, "variants", name, "libmlbm_b200.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    L.build(force=True, extra=shlex.split(flags), out=out)
    print("built", out)
