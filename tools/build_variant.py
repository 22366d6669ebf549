"""Harness: build a variant of libnseries.so with extra -D flags into tools/variants/<name>.so
(for A/B timing of compile-time engine options; the binding loads it via NSERIES_LIB).
  python tools/build_variant.py NAME -DNSERIES_TF32_BK=32 -DNSERIES_TF32_STAGES=3 ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_11843_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
outdir = os.path.join(ROOT, "tools", "variants", name)
os.makedirs(outdir, exist_ok=True)
objs = []
for src in B.sources():
    obj = os.path.join(outdir, os.path.basename(src) + ".o")
    if src.endswith(".cc"):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-c", src, "-o", obj]
    else:
        cmd = [B.NVCC, *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], *defs, "-c", src, "-o", obj]
    subprocess.run(cmd, check=True)
    objs.append(obj)
out = os.path.join(ROOT, "tools", "variants", name + ".so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"], check=True)
print(out)
