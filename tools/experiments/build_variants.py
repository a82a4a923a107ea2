"""Build libparse_gpu_<name>.so variants with extra -D flags for union_prog.cu
(experiments only; loaded with PG_LIB_VARIANT=<name>).
usage: python tools/experiments/build_variants.py name=-DA=1,-DB=2 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_08568_b200 import _build as B  # noqa: E402

B.build()
objs = [os.path.join(B.OBJDIR, f) for f in sorted(os.listdir(B.OBJDIR)) if f.endswith(".o") and f != "union_prog.o"]
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    os.makedirs(os.path.join(B.OBJDIR, "variants"), exist_ok=True)
    o = os.path.join(B.OBJDIR, "variants", f"union_prog_{name}.o")
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *defs.split(","), "-c", os.path.join(B.CSRC, "union_prog.cu"), "-o", o]
    subprocess.run(cmd, check=True)
    lib = B.LIB[:-3] + "_" + name + ".so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, o, "-cudart", "static", "-Xlinker", "--no-undefined"],
                   check=True)
    print("built", lib)
