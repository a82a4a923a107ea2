"""Build recipe for the parity CHECKERS (test infrastructure only).

* oracle/liboracle.so      -- the plain-C restatement (parse_oracle.c), gcc.
* oracle/_ref/libparse_ref.so -- the reference's own headers compiled where
  they lie under /root/reference (ref_shim.cpp marshals arrays into the
  reference types).  Built only when /root/reference is present (this
  container); the GPU box uses the prebuilt file that travels with the repo
  snapshot.  oracle/_ref/ is git-ignored.

Flags: -O2 -ffp-contract=off and no -march=native, so the reference's
sequential fp64 dots are never FMA-contracted.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_INCLUDE = "/root/reference/proj/include"
# nlohmann/json 3.11.3 (pattern_cache.hpp includes <json.hpp>); vendored by cudnn_frontend.
JSON_CANDIDATES = [
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
]

ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libparse_ref.so")
COMMON = ["-O2", "-ffp-contract=off", "-fPIC", "-shared"]


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs if os.path.exists(s))


def build_oracle(verbose: bool = False) -> str:
    src = os.path.join(HERE, "parse_oracle.c")
    hdr = os.path.join(HERE, "parse_oracle.h")
    if _stale(ORACLE_SO, [src, hdr, __file__]):
        cmd = ["gcc", "-std=c11", *COMMON, src, "-o", ORACLE_SO, "-lm"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return ORACLE_SO


def build_ref(verbose: bool = False) -> str | None:
    if not os.path.isdir(REF_INCLUDE):
        return REF_SO if os.path.exists(REF_SO) else None
    json_dir = next((d for d in JSON_CANDIDATES if os.path.exists(os.path.join(d, "json.hpp"))), None)
    if json_dir is None:
        print("oracle/build.py: nlohmann json.hpp not found; reference oracle not built", file=sys.stderr)
        return REF_SO if os.path.exists(REF_SO) else None
    src = os.path.join(HERE, "ref_shim.cpp")
    os.makedirs(os.path.dirname(REF_SO), exist_ok=True)
    if _stale(REF_SO, [src, __file__]):
        cmd = ["g++", "-std=c++20", *COMMON, f"-I{REF_INCLUDE}", f"-I{json_dir}", src, "-o", REF_SO]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return REF_SO


def build(verbose: bool = False) -> None:
    build_oracle(verbose)
    build_ref(verbose)


if __name__ == "__main__":
    build(verbose=True)
