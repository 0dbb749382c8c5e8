"""Build libsttsv.so (in-tree) with nvcc for sm_100a.

One object per compiled rank (edge_inst.cu with -DSTTSV_INST_N=<N>, plus the
generic N=0 instantiation) so the slow unrolled instantiations compile in
parallel; kernels.cu holds the small kernels, plan.cpp the host planner and
the C ABI.  Objects are rebuilt only when a source is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsttsv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
           "-I" + os.path.join(ROOT, "include")] + ARCH


def compiled_ranks() -> list[int]:
    src = open(os.path.join(CSRC, "internal.h")).read()
    m = re.search(r"#define STTSV_COMPILED_RANKS\(X\)\s*\\\s*\n(.*)\n", src)
    return [int(v) for v in re.findall(r"X\((\d+)\)", m.group(1))]


def id16_ranks() -> list[int]:
    src = open(os.path.join(CSRC, "internal.h")).read()
    m = re.search(r"#define STTSV_ID16_RANKS\(X\)\s*\\\s*\n(.*)\n", src)
    return [int(v) for v in re.findall(r"X\((\d+)\)", m.group(1))]


def _newest(*names) -> float:
    deps = [os.path.join(CSRC, f) for f in names] + [os.path.join(ROOT, "include", "sttsv.h"),
                                                   os.path.join(CSRC, "internal.h")]
    return max(os.path.getmtime(d) for d in deps)


_DEVICE_HDRS = ("edge_kernel.cuh", "dp.cuh", "prefix.cuh")


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: %s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr))
    return r.stdout + r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    t_edge = _newest("edge_inst.cu", *_DEVICE_HDRS)
    t_kern = _newest("kernels.cu", *_DEVICE_HDRS)
    t_plan = _newest("plan.cpp")
    jobs = jobs or max(1, os.cpu_count() or 1)
    units = []
    for n in compiled_ranks() + [0]:
        units.append((os.path.join(OBJ, "edge_n%d.o" % n), t_edge,
                      [NVCC] + NVFLAGS + ["-DSTTSV_INST_N=%d" % n, "-c", os.path.join(CSRC, "edge_inst.cu")]))
    for n in id16_ranks():
        units.append((os.path.join(OBJ, "edge16_n%d.o" % n), t_edge,
                      [NVCC] + NVFLAGS + ["-DSTTSV_INST_N=%d" % n, "-DSTTSV_INST_ID16=1", "-c",
                                          os.path.join(CSRC, "edge_inst.cu")]))
    units.append((os.path.join(OBJ, "kernels.o"), t_kern,
                  [NVCC] + NVFLAGS + ["-c", os.path.join(CSRC, "kernels.cu")]))
    units.append((os.path.join(OBJ, "plan.o"), t_plan,
                  [NVCC] + NVFLAGS + ["-Xcompiler", "-fopenmp", "-c", os.path.join(CSRC, "plan.cpp")]))
    todo = [(o, c + ["-o", o]) for o, t, c in units
            if force or not os.path.exists(o) or os.path.getmtime(o) < t]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            for out in ex.map(lambda oc: _run(oc[1]), todo):
                if verbose and out.strip():
                    print(out, file=sys.stderr)
    objs = [o for o, _, _ in units]
    if force or todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lgomp"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
