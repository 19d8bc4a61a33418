"""In-tree build of libpf.so (the C-ABI of include/pf.h) for sm_100a."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpf.so")
SOURCES = ["pf_plan.cpp", "pf_eval.cu", "pf_reduce.cu", "pf_chol.cu", "pf_api.cu"]
NVCC_FLAGS = ["-shared", "-Xcompiler", "-fPIC", "-O3", "-lineinfo", "-std=c++17",
              "-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "pf.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose=False, force=False):
    if not force and not needs_build():
        return LIB
    cmd = [_nvcc()] + NVCC_FLAGS + ["-o", LIB + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    # compiler output to stderr: bench.py's stdout carries exactly one JSON line
    subprocess.run(cmd, check=True, stdout=sys.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force=True)
