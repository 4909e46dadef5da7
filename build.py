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
CHECKED_LIB = os.path.join(PKG, "libscmwu_checked.so")   # test-only (-DSCMWU_CHECKED)
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


def build_cuda(jobs: int | None = None, force: bool = False, checked: bool = False) -> str:
    """Compile csrc/*.cu into libscmwu.so.  ``checked``: the same sources with
    -DSCMWU_CHECKED (device index invariants, SC_DCHECK) into libscmwu_checked.so, a
    test-only library (tests/test_gpu_checked.py)."""
    obj_dir = OBJ + "_checked" if checked else OBJ
    lib = CHECKED_LIB if checked else LIB
    flags = NVFLAGS + (["-DSCMWU_CHECKED"] if checked else [])
    os.makedirs(obj_dir, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "scmwu.h")]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            todo.append((s, o))

    def compile_one(so):
        s, o = so
        _run([NVCC] + flags + ["-c", s, "-o", o], log=o + ".log")

    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(compile_one, todo))
    if force or todo or _stale(lib, objs):
        _run([NVCC, "-shared"] + ARCH + ["-o", lib] + objs + ["-lcudart"])
    return lib


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
    ap.add_argument("--checked", action="store_true", help="also build libscmwu_checked.so")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    build_oracle()
    if a.emu:
        build_emu()
    print(build_cuda(a.j, a.force))
    if a.checked:
        print(build_cuda(a.j, a.force, checked=True))


if __name__ == "__main__":
    main()
