"""Build liblouiskv.so (all CUDA kernels + the C ABI) in-tree for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "liblouiskv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
         "-Xptxas", "-v", "-cudart", "static"]
SOURCES = ["api.cu", "k_retrieve.cu", "k_append.cu", "k_attn.cu", "k_attn_tc.cu", "k_layer.cu", "k_kmeans.cu", "k_kmeans_tc.cu"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, prof: bool = False, variant: str = "", defines=()) -> str:
    """prof=True: a separate liblouiskv_prof.so with per-phase %globaltimer stamps (-DLKV_PROF) for
    tools/probe_phases.py; variant/defines: an experimental liblouiskv_<variant>.so. Neither is ever
    loaded by the tests or the bench."""
    tag = "prof" if prof else variant
    objdir = os.path.join(HERE, "build_" + tag if tag else "build")
    lib = LIB.replace(".so", "_" + tag + ".so") if tag else LIB
    flags = FLAGS + (["-DLKV_PROF"] if prof else []) + ["-D" + d for d in defines]
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in sorted(os.listdir(CSRC)) if h.endswith(".cuh")]
    headers.append(os.path.join(INCLUDE, "louiskv.h"))
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC] + ARCH + flags + ["-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {s}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib + ".tmp"] + objs
        subprocess.check_call(cmd)
        os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    var = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, prof="--prof" in sys.argv,
                variant=var[0] if var else "", defines=defs))
