"""Build an A/B variant of libdyq.so with extra nvcc defines (tools only).
usage: python tools/build_variant.py NAME -DFOO=1 ...  -> tools/variants/libdyq_NAME.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_07904_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "variants")
os.makedirs(os.path.join(out, name), exist_ok=True)
objs, procs = [], []
for src in b.sources():
    obj = os.path.join(out, name, os.path.basename(src) + ".o")
    objs.append(obj)
    procs.append((src, subprocess.Popen([b.NVCC, *b.NVCC_FLAGS, *defs, "-c", src, "-o", obj])))
for src, p in procs:
    if p.wait():
        raise SystemExit(f"nvcc failed: {src}")
lib = os.path.join(out, f"libdyq_{name}.so")
subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs, "-ldl"])
print(lib)
