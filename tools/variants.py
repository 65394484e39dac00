"""Build variant librs.so files (compile-time knobs) into build/var/ for A/B runs:
    python tools/variants.py NAME:DEF1,DEF2 ...   (DEF may be empty)"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1610_05141_b200 import build as B

os.makedirs(os.path.join(B.ROOT, "build", "var"), exist_ok=True)
def one(spec):
    name, _, defs = spec.partition(":")
    out = os.path.join(B.ROOT, "build", "var", f"librs_{name}.so")
    B.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out
with ThreadPoolExecutor(4) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
