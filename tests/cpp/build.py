"""Build tests/cpp/_bin/test_mirror: the C++ mirror (include/parse_gpu.hpp)
compiled against the reference headers where they lie (/root/reference) and
linked to libparse_gpu.so.  Built in this container by __graft_entry__.build();
the binary travels to the GPU box (git-ignored, not gpurun-ignored)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj/include"
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
OUT = os.path.join(HERE, "_bin", "test_mirror")


def build(verbose=False):
    if not os.path.isdir(REF):
        return OUT if os.path.exists(OUT) else None
    src = os.path.join(HERE, "test_mirror.cpp")
    lib = os.path.join(ROOT, "paper_2605_08568_b200", "lib")
    deps = [src, os.path.join(ROOT, "include", "parse_gpu.hpp"), os.path.join(ROOT, "include", "parse_gpu.h"),
            os.path.join(lib, "libparse_gpu.so")]
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{REF}", f"-I{JSON}", f"-I{ROOT}/include",
           "-I/usr/local/cuda/include", src, "-o", OUT, f"-L{lib}", "-lparse_gpu", "-Wl,-rpath,$ORIGIN/../../../paper_2605_08568_b200/lib",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
