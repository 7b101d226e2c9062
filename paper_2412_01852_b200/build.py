"""Build the in-tree CUDA library (sm_100a) with nvcc.

The .so is written next to this file so it travels with the repo snapshot to
the GPU box (a JIT cache under ~/.cache would not). Flags follow the B200
profiling recipe: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "rotseq_b200.cu")
HDR = os.path.join(ROOT, "include", "rotseq_b200.h")
OUT = os.path.join(HERE, "librotseq_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(OUT, [SRC, HDR, __file__]):
        return OUT
    fd, tmp = tempfile.mkstemp(suffix=".so", dir=HERE)
    os.close(fd)
    extra = os.environ.get("RS_NVCC_EXTRA", "").split()
    cmd = [nvcc_path(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", tmp, SRC]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        os.unlink(tmp)
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        print(proc.stderr)
    os.replace(tmp, OUT)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
        fh.write(proc.stderr)
    return OUT


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
