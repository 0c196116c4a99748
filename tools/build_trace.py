"""Build tools/libmk_trace.so: the engine with per-CTA timeline stamps (-DMK_TRACE)."""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_00628_b200 import _build as b
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmk_trace.so")
objs = []
for src in b.SOURCES:
    obj = f"/tmp/trace_{src}.o"
    subprocess.run([b.NVCC, *b.FLAGS, "-DMK_TRACE", "-c", os.path.join(b.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs, "-lcudart_static"], check=True)
print(out)
