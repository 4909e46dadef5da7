"""Build the in-tree native artefacts.

    python build.py            # libscmwu.so (CUDA, sm_100a) + the oracle's C kernels
    python build.py --emu      # also the CPU emulator used by the CPU test-suite

The CUDA engine is compiled translation unit by translation unit in parallel
(nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo) and linked into
paper_2405_09157_b200/libscmwu.so, which travels with the repo snapshot to
the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2405_09157_b200")
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libscmwu.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "-diag-suppress", "177"] + ARCH

EMU_SRC = os.path.join(ROOT, "tests", "emu", "scmwu_emu.cpp")
EMU_LIB = os.path.join(ROOT, "tests", "emu", "_build", "libscmwu_emu.so")


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise SystemExit(f"build failed: {' '.join(cmd[:3])} ...")
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(jobs: int | None = None, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "scmwu.h")]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            todo.append((s, o))

    def compile_one(so):
        s, o = so
        _run([NVCC] + NVFLAGS + ["-c", s, "-o", o], log=o + ".log")

    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(compile_one, todo))
    if force or todo or _stale(LIB, objs):
        _run([NVCC, "-shared"] + ARCH + ["-o", LIB] + objs + ["-lcudart"])
    return LIB


def build_oracle() -> None:
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


def build_emu() -> str:
    os.makedirs(os.path.dirname(EMU_LIB), exist_ok=True)
    deps = [EMU_SRC, os.path.join(CSRC, "scmwu_control.h"), os.path.join(ROOT, "include",
                                                                          "scmwu.h")]
    if _stale(EMU_LIB, deps):
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", EMU_LIB, EMU_SRC])
    return EMU_LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--emu", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    build_oracle()
    if a.emu:
        build_emu()
    print(build_cuda(a.j, a.force))


if __name__ == "__main__":
    main()
