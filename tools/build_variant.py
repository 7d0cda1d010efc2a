"""Dev: build libedaa_cuda.so with extra nvcc defines into paper_2209_11002_b200/<name>.so
(for A/B timing via EDAA_CUDA_LIB).  usage: python tools/build_variant.py var_q32 -DEDAA_QMAX=32"""
import concurrent.futures as cf
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_11002_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join("/tmp", "var_" + name)
os.makedirs(out, exist_ok=True)
jobs = []
objs = []
for s in b.CUDA_SRCS:
    o = os.path.join(out, s + ".o")
    objs.append(o)
    jobs.append([b.NVCC] + b.NVFLAGS + defs + ["-c", os.path.join(b.CSRC, s), "-o", o])
with cf.ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
    for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
        if r.returncode:
            sys.exit(r.stderr[-3000:])
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-cudart", "static", "-o",
                os.path.join(b.PKG, name + ".so")] + objs, check=True)
print("built", name)
