"""Build recipe for the C restatement (test infrastructure).

    python oracle/build.py      ->  oracle/_build/libgg_oracle.so

gcc with -ffp-contract=off so every fp64 operation rounds like CPython's, and
glibc libm for log/exp (the functions CPython's math module calls).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libgg_oracle.so")
SRC = os.path.join(HERE, "gg_oracle.c")


def build(force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(
            os.path.getmtime(SRC),
            os.path.getmtime(os.path.join(HERE, "..", "include", "greengate_b200.h"))):
        return LIB
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-Wall", "-o", LIB, SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
