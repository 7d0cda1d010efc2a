"""In-tree build of the native libraries (no JIT cache, no pip install).

* ``paper_2209_11002_b200/libedaa_cuda.so``  — sm_100a kernels + the C-ABI
  declared in ``include/edaa_b200.h``.
* ``paper_2209_11002_b200/libarchetype_b200.so`` — the C++ drop-in layer that
  implements the reference API of ``include/archetype/*.hpp`` on top of the
  C-ABI (linked against libedaa_cuda.so).

Both travel to the GPU box with the repo snapshot (``*.so`` is git-ignored but
not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                  "-I" + os.path.join(ROOT, "include")]
CUDA_SRCS = (["edaa_pass_%s_%s.cu" % (x, m) for x in ("f32", "f64") for m in ("alo", "ahi", "b", "init", "obj")]
             + ["edaa_pass_b64.cu", "edaa_kernels.cu", "edaa_prims.cu", "edaa_capi.cu"])
HOST_SRCS = ["matrix.cpp", "image.cpp", "types.cpp", "solver.cpp", "ensemble.cpp", "device.cpp",
             # the formats and the front end either side of the path
             "npy.cpp", "envi.cpp", "metrics.cpp", "outputs.cpp", "synth.cpp", "cli.cpp"]
# nlohmann/json (the reference's JSON dependency, vendor/json.hpp there) from the
# image's third-party copy; report.json byte-compatibility depends on it.
JSON_INC = os.path.join(__import__("sysconfig").get_paths()["purelib"],
                        "include", "cudnn_frontend", "thirdparty", "nlohmann")

CUDA_LIB = os.path.join(PKG, "libedaa_cuda.so")
HOST_LIB = os.path.join(PKG, "libarchetype_b200.so")
CLI_BIN = os.path.join(PKG, "archetype")  # the reference's tools/main.cpp equivalent


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: %s\n%s" % (" ".join(cmd), r.stdout))
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_cuda(force=False, verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in ("edaa_internal.cuh", "edaa_device.cuh", "edaa_pass.cuh")] + [os.path.join(ROOT, "include", "edaa_b200.h")]
    objs = []
    jobs = []
    for s in CUDA_SRCS:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC] + NVFLAGS + ["-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for out in ex.map(_run, jobs):
            if verbose and out:
                print(out)
    if force or _stale(CUDA_LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", CUDA_LIB] + objs)
    return CUDA_LIB


def build_host(force=False):
    hsrc = [os.path.join(CSRC, "host", s) for s in HOST_SRCS]
    hsrc = [s for s in hsrc if os.path.exists(s)]
    if not hsrc:
        return None
    hdr_dir = os.path.join(ROOT, "include", "archetype")
    deps = hsrc + [os.path.join(hdr_dir, h) for h in os.listdir(hdr_dir)] + [CUDA_LIB]
    if force or _stale(HOST_LIB, deps):
        objs = []
        jobs = []
        os.makedirs(BUILD, exist_ok=True)
        for src in hsrc:
            obj = os.path.join(BUILD, "host_" + os.path.basename(src) + ".o")
            objs.append(obj)
            jobs.append(["g++", "-std=c++20", "-O3", "-DNDEBUG", "-fPIC", "-Wall",
                         "-I" + os.path.join(ROOT, "include"), "-I" + JSON_INC, "-c", src, "-o", obj])
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            list(ex.map(_run, jobs))
        _run(["g++", "-shared", "-o", HOST_LIB] + objs +
             ["-L" + PKG, "-ledaa_cuda", "-Wl,-rpath,$ORIGIN", "-lpthread"])
    if force or _stale(CLI_BIN, [HOST_LIB]):
        main = os.path.join(BUILD, "archetype_main.cpp")
        with open(main, "w") as f:
            f.write('#include "archetype/cli.hpp"\n'
                    'int main(int argc, char** argv) { return archetype::cli_main(argc, argv); }\n')
        _run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), "-o", CLI_BIN, main,
              "-L" + PKG, "-larchetype_b200", "-ledaa_cuda", "-Wl,-rpath,$ORIGIN", "-lpthread"])
    return HOST_LIB


def build_all(force=False, verbose=False):
    build_cuda(force=force, verbose=verbose)
    build_host(force=force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", CUDA_LIB, HOST_LIB)
