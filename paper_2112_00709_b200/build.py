"""Build libfb.so (C-ABI library: host graph compiler + sm_100a kernels) in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, static CUDA runtime
(so the library does not depend on which libcudart torch has loaded).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("FBX_LIB_OUT") or os.path.join(HERE, "libfb.so")  # FBX_LIB_OUT: experiment builds
EXTRA = os.environ.get("FBX_EXTRA_FLAGS", "").split()  # e.g. -DFBX_CTIMING (instrumented experiment builds)
OBJ_TAG = os.environ.get("FBX_OBJ_TAG", "")
SOURCES = ["fb_graph.cpp", "fb_kernels.cu", "fb_inst.cu", "fb_cluster.cu", "fb_literal.cu", "fb_semiring.cu"]
# fb_inst.cu is compiled once per (direction, mode): the k_fb instantiation sets
INST = [(bwd, mode) for bwd in (0, 1) for mode in (0, 1, 2, 4)] + [(1, 5)]
# fb_cluster.cu once per (direction, sequences per cluster)
CINST = [(bwd, s) for bwd in (0, 1) for s in (2, 4)]
HEADERS = ["fb_internal.h", "fb_device.cuh", os.path.join("..", "..", "include", "fb.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def _units():
    """(source, object, extra flags) of every translation unit."""
    units = [("fb_graph.cpp", "fb_graph.o", []), ("fb_kernels.cu", "fb_kernels.o", [])]
    units += [("fb_inst.cu", f"fb_inst_b{b}_m{m}.o", [f"-DFBX_BWD={b}", f"-DFBX_MODE={m}"]) for b, m in INST]
    units += [("fb_cluster.cu", f"fb_cluster_b{b}_s{s}.o", [f"-DFBX_BWD={b}", f"-DFBX_S={s}"]) for b, s in CINST]
    units += [("fb_literal.cu", "fb_literal.o", []), ("fb_semiring.cu", "fb_semiring.o", [])]
    return units


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmds, objs = [], []
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
    for src, obj, extra in _units():
        obj = os.path.join(CSRC, OBJ_TAG + obj)
        objs.append(obj)
        # an object newer than its source, the headers and this script (flags) is up to date
        if not force and not EXTRA and os.path.exists(obj) and os.path.getmtime(obj) > max(
                hdr_t, os.path.getmtime(os.path.join(CSRC, src)), os.path.getmtime(__file__)):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
               *extra, *EXTRA, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd[1:1] = ["-Xptxas", "-v"]
        cmds.append(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
