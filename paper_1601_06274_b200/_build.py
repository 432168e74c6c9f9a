"""Build the sm_100a shared library libdmm_b200.so in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("DMM_B200_LIB_OUT") or os.path.join(HERE, "_lib", "libdmm_b200.so")
EXTRA = os.environ.get("DMM_NVCC_EXTRA", "").split()     # experiment variants (-D...)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",   # only the extern "C" API is exported
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


# Per-file extra flags.  refine.cu: no FMA contraction, so every float64
# operation of the refinement rounds exactly as the oracle's numpy operations
# (the iteration is chaotic at a few pixels: a 1e-12 perturbation moves them by
# up to ~1.6 labels, so parity needs the same rounding).
FILE_FLAGS = {"refine.cu": ["-fmad=false"]}


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "dmm.h"), __file__]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in _deps()):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tag = f"tmp{os.getpid()}"
    objs = [os.path.join(os.path.dirname(LIB), os.path.basename(src)[:-3] + f".{tag}.o") for src in sources()]
    comp = [f for f in FLAGS if f != "-shared"] + EXTRA
    # one nvcc per translation unit, in parallel (the chain-DP units dominate)
    procs = [subprocess.Popen([NVCC, *comp, *FILE_FLAGS.get(os.path.basename(src), []), "-c", "-o", o, src],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for src, o in zip(sources(), objs)]
    logs, failed = [], []
    for src, pr in zip(sources(), procs):
        out, _ = pr.communicate()
        logs.append(out)
        if pr.returncode != 0:
            failed.append(os.path.basename(src))
    tmp = LIB + "." + tag
    try:
        if failed:
            raise RuntimeError("nvcc failed (" + ", ".join(failed) + "):\n" + "".join(logs))
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    with open(os.path.join(os.path.dirname(LIB), "ptxas.log"), "w") as f:
        f.write("".join(logs))
    if verbose:
        print("".join(logs))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
