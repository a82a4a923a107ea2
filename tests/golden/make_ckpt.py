"""Build tests/golden/make_ckpt.cpp against /root/reference and write the
checkpoint fixtures into tests/golden/ckpt (committed; run only here)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def main():
    exe = os.path.join("/tmp", "make_ckpt")
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I/root/reference/proj/include", f"-I{JSON}",
                    os.path.join(HERE, "make_ckpt.cpp"), "-o", exe], check=True)
    out = os.path.join(HERE, "ckpt")
    os.makedirs(out, exist_ok=True)
    subprocess.run([exe, out], check=True)
    print("wrote", out)


if __name__ == "__main__":
    sys.exit(main())
