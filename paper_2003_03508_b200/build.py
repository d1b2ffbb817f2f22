"""Build the in-tree native artefacts with nvcc / gcc (no JIT cache).

* paper_2003_03508_b200/libthmm.so -- CUDA kernels + C-ABI, sm_100a
* oracle/liboracle.so              -- C restatement of the reference (tests only)
"""

from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2003_03508_b200")
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_native(force: bool = False, verbose: bool = False) -> str:
    target = os.path.join(PKG, "libthmm.so")
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))]
    srcs.append(os.path.join(ROOT, "include", "thmm.h"))
    if force or _stale(target, srcs):
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", target + ".tmp",
               os.path.join(CSRC, "thmm_capi.cu")]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        os.replace(target + ".tmp", target)
    return target


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "thmm_oracle.c")
    target = os.path.join(ROOT, "oracle", "liboracle.so")
    if os.path.exists(src) and (force or _stale(target, [src])):
        subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-fno-fast-math", "-fPIC",
                        "-shared", "-pthread", "-o", target + ".tmp", src, "-lm"], check=True)
        os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
    print(build_oracle(force=True))
