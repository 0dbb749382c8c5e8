"""Build experimental variants of libsttsv.so that differ only in the rank-N
edge-kernel object (compile-time knobs), for A/B timing on one GPU call.

  python tools/variants.py N NAME:-DFLAG=1,-DOTHER=2 NAME2:...   -> build/variants/libsttsv_NAME.so
  STTSV_LIB_PATH=build/variants/libsttsv_NAME.so python tools/time_apply.py large
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_08595_b200 import build as B  # noqa: E402

N = int(sys.argv[1])
B.build()
out = os.path.join(ROOT, "build", "variants")
import shutil
if not os.environ.get("VARIANTS_KEEP"):
    shutil.rmtree(out, ignore_errors=True)  # keep the gpurun snapshot small: only this call's variants
os.makedirs(out, exist_ok=True)
objs = [os.path.join(B.OBJ, "edge_n%d.o" % n) for n in B.compiled_ranks() + [0] if n != N]
objs += [os.path.join(B.OBJ, "edge16_n%d.o" % n) for n in B.id16_ranks() if n != N]
objs += [os.path.join(B.OBJ, "kernels.o"), os.path.join(B.OBJ, "plan.o")]
for spec in sys.argv[2:]:
    name, _, flags = spec.partition(":")
    flags = [f for f in flags.split(",") if f]
    vobjs = []
    for id16 in ([0, 1] if N in B.id16_ranks() else [0]):
        o = os.path.join(out, "edge%s_n%d_%s.o" % ("16" if id16 else "", N, name))
        # "16:-DFLAG" applies to the 16-bit-id object only (e.g. STTSV_WAITPROF: one
        # object may define the debug counters)
        fl = [f[3:] for f in flags if f.startswith("16:") and id16] + [f for f in flags if not f.startswith("16:")]
        subprocess.check_call([B.NVCC] + B.NVFLAGS + fl + ["-DSTTSV_INST_N=%d" % N, "-DSTTSV_INST_ID16=%d" % id16,
                               "-c", os.path.join(B.CSRC, "edge_inst.cu"), "-o", o])
        vobjs.append(o)
    lib = os.path.join(out, "libsttsv_%s.so" % name)
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + vobjs + objs +
                          ["-ldl", "-lgomp"])
    print(lib)
