"""Build an engine variant with extra nvcc defines into tools/libmk_<name>.so (dev A/B tool):
python tools/build_variant.py NAME -DFOO=1 ..."""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_00628_b200 import _build as b
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"libmk_{name}.so")
objs = []
for src in b.SOURCES:
    obj = f"/tmp/var_{name}_{src}.o"
    subprocess.run([b.NVCC, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-lcudart_static"], check=True)
print(out)
