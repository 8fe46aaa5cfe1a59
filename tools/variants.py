"""Build compile-time variants of libmpsm_b200.so for A/B timing on the GPU.

    python tools/variants.py name:DEF1=1,DEF2=3 name2:... 
Each variant lands in build/variants/<name>/libmpsm_b200.so; run
tools/sort_variants_run.py on the GPU box to time them.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1207_0145_b200 import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    defines = [d for d in defs.split(",") if d]
    out = os.path.join(ROOT, "build", "variants", name)
    lib = build.build(force=True, defines=defines, build_dir=os.path.join(out, "obj"), lib=os.path.join(out, "libmpsm_b200.so"))
    print(name, defines, lib)
