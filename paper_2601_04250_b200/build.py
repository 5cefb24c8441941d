"""In-tree nvcc build of the B200 library (sm_100a only).

    python -m paper_2601_04250_b200.build      ->  paper_2601_04250_b200/_lib/libgreengate_b200.so

Each translation unit under csrc/ is compiled with
`-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo` into an object, then
linked into one shared library exporting the C ABI of include/greengate_b200.h.
The controller TU adds -fmad=false (CPython rounding, no FMA contraction).
The CUDA runtime is linked statically, so the .so needs only the driver.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT, "libgreengate_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", *(["-DGG_GELU_TANH"] if os.environ.get("GG_GELU_TANH") else []),
          *os.environ.get("GG_EXTRA_NVCC", "").split(), "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
# per-translation-unit extra flags
UNITS = {
    "gg_controller.cu": ["-fmad=false"],
}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _sources() -> list[str]:
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    # objects built with other flags (e.g. GG_EXTRA_NVCC debug builds) are stale
    stamp = os.path.join(OUT, "obj", ".flags")
    flags = " ".join([*ARCH, *COMMON])
    prev = open(stamp).read() if os.path.exists(stamp) else None
    if prev != flags:
        force = True
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers += [os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))
                if h.endswith(".h")]
    objs = []
    for src in _sources():
        path = os.path.join(CSRC, src)
        obj = os.path.join(OUT, "obj", src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers + [__file__]):
            cmd = [nvcc(), *ARCH, *COMMON, *UNITS.get(src, []), "-c", path, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-ldl", "-lrt",
               "-lpthread"]
        subprocess.run(cmd, check=True)
    with open(stamp, "w") as f:
        f.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
