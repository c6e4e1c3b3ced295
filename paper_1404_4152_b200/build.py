"""Build the in-tree native libraries (sm_100a CUDA library + host helpers)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1404_4152_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread",
           "-diag-suppress", "550"]
SOURCES = [os.path.join(PKG, "csrc", "sw_api.cu")]
DEPS = SOURCES + [os.path.join(PKG, "csrc", f) for f in sorted(os.listdir(os.path.join(PKG, "csrc")))
                  if f.endswith((".cuh", ".inc"))] + [os.path.join(ROOT, "include", "swsearch.h")]
OUT = os.path.join(PKG, "libswsearch.so")
# Same source with the f4 ablation kernels and tile/CTA-size instances
# (sw_tuning); the production library above carries only the shipped design.
OUT_ABLATION = os.path.join(PKG, "libswsearch_ablation.so")


def _stale(out, deps):
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps)


def build_cuda(force=False, verbose=False, ablation=True):
    jobs = []
    targets = [(OUT, [])] + ([(OUT_ABLATION, ["-DSW_ABLATION"])] if ablation else [])
    for out, extra in targets:
        if force or _stale(out, DEPS):
            cmd = [NVCC, *ARCH, *NVFLAGS, *extra, "-shared", "-o", out, *SOURCES]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            jobs.append((cmd, subprocess.Popen(cmd)))
    for cmd, p in jobs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    return OUT


def build_swgen(force=False):
    src = os.path.join(ROOT, "swdata", "swgen.c")
    out = os.path.join(ROOT, "swdata", "_libswgen.so")
    if force or _stale(out, [src]):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", "-o", out, src])
    return out


def build_all(force=False, verbose=False):
    build_swgen(force)
    return build_cuda(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
