"""Build libparse_gpu_<name>.so variants with extra -D flags for union_prog.cu
(experiments only; loaded with PG_LIB_VARIANT=<name>).
usage: python tools/experiments/build_variants.py name=-DA=1,-DB=2 ...  (union_prog.cu)
       python tools/experiments/build_variants.py name=umma.cu:-DA=1 ...  (another source)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_08568_b200 import _build as B  # noqa: E402

B.build()
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    src = "union_prog.cu"
    if ":" in defs:
        src, defs = defs.split(":", 1)
    objs = [os.path.join(B.OBJDIR, f) for f in sorted(os.listdir(B.OBJDIR))
            if f.endswith(".o") and f != src[:-3] + ".o"]
    os.makedirs(os.path.join(B.OBJDIR, "variants"), exist_ok=True)
    o = os.path.join(B.OBJDIR, "variants", f"{src[:-3]}_{name}.o")
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *[d for d in defs.split(",") if d], "-c", os.path.join(B.CSRC, src), "-o", o]
    subprocess.run(cmd, check=True)
    lib = B.LIB[:-3] + "_" + name + ".so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, o, "-cudart", "static", "-Xlinker", "--no-undefined"],
                   check=True)
    print("built", lib)
