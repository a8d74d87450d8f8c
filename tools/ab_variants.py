#!/usr/bin/env python
"""Build compile-time variants of libctb200.so for A/B timing on the GPU box.

    python tools/ab_variants.py NAME=DEFINE[,DEFINE...] ...
    e.g. python tools/ab_variants.py ne0=CTB_F64Q_ENTRIES=0 ne1=CTB_F64Q_ENTRIES=1

Each variant lands in build/variants/NAME/libctb200.so (git-ignored, travels with gpurun);
run any script against it with CTB_LIB=build/variants/NAME/libctb200.so.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2409_16675_b200 import build as B  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = ROOT / "build" / "variants" / name
    lib = B.build(defines=[d for d in defs.split(",") if d], out=out / "libctb200.so", objdir=out / "obj")
    print(lib)
