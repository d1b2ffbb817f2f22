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
    "-Xcompiler", "-fPIC",
]
OBJ_DIR = os.path.join(PKG, "csrc", "build")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_native(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every csrc/*.cu to an object in parallel, link libthmm.so."""
    target = os.path.join(PKG, "libthmm.so")
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "thmm.h"))
    units = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs, pending = [], []
    for u in units:
        obj = os.path.join(OBJ_DIR, os.path.basename(u)[:-3] + ".o")
        objs.append(obj)
        if force or _stale(obj, [u, *headers]):
            cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, u]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            pending.append(cmd)
    jobs = jobs or max(1, min(len(pending), os.cpu_count() or 1))
    running = []
    while pending or running:
        while pending and len(running) < jobs:
            running.append(subprocess.Popen(pending.pop(0)))
        proc = running.pop(0)
        if proc.wait() != 0:
            for p in running:
                p.wait()
            raise subprocess.CalledProcessError(proc.returncode, proc.args)
    if force or _stale(target, objs):
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target + ".tmp",
                        *objs], check=True)
        os.replace(target + ".tmp", target)
    return target


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "thmm_oracle.c")
    target = os.path.join(ROOT, "oracle", "liboracle.so")
    if os.path.exists(src) and (force or _stale(target, [src])):
        subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                        "-shared", "-pthread", "-o", target + ".tmp", src, "-lm"], check=True)
        os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
    print(build_oracle(force=True))
