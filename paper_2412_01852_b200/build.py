"""Build the in-tree CUDA library (sm_100a) with nvcc.

The .so is written next to this file so it travels with the repo snapshot to
the GPU box (a JIT cache under ~/.cache would not). Flags follow the B200
profiling recipe: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.

Translation units (compiled in parallel, then linked with the static CUDA runtime):

* ``csrc/rotseq_b200.cu``       host side, C-ABI, pack / naive / peak kernels;
* ``csrc/pipeline_variant.cu``  compiled 8 times, once per pipeline-kernel family
  (fp64/fp32 x strict/fast x rotation/reflector);
* ``csrc/dmma_variant.cu``      the FP64 tensor-core accumulate-and-apply variant.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRC = os.path.join(CSRC, "rotseq_b200.cu")
VARIANT_SRC = os.path.join(CSRC, "pipeline_variant.cu")
DMMA_SRC = os.path.join(CSRC, "dmma_variant.cu")
DEVICE_HDR = os.path.join(CSRC, "rotseq_device.cuh")
HDR = os.path.join(ROOT, "include", "rotseq_b200.h")
OUT = os.path.join(HERE, "librotseq_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]

VARIANTS = [(t, s, r) for t in ("double", "float") for s in (0, 1) for r in (0, 1)]


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


def _run(cmd):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    return proc.stderr


OBJ_CACHE = os.path.join(ROOT, "build", "obj")  # git-ignored: per-TU objects keyed by content


def _key(cmd, sources) -> str:
    h = hashlib.sha1(" ".join(cmd).encode())
    for src in sources:
        with open(src, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def build_library(force: bool = False, verbose: bool = False, out: str | None = None, extra=None) -> str:
    """Compile (in parallel) and link the library. ``out``/``extra`` build developer
    variants (e.g. ``extra=["-DRS_TRACE"]``) without touching the product .so. Objects are
    cached per translation unit under build/obj, keyed by the compile command and the
    contents of the sources it includes, so an edit recompiles only what it touches
    (``force`` only forces the link)."""
    out = out or OUT
    deps = [SRC, VARIANT_SRC, DMMA_SRC, DEVICE_HDR, HDR, __file__]
    if not force and extra is None and not _stale(out, deps):
        return out
    extra = list(extra or []) + os.environ.get("RS_NVCC_EXTRA", "").split()
    nvcc = nvcc_path()
    only = [u for u in os.environ.get("RS_BUILD_ONLY", "").split(",") if u] if out != OUT else []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    os.makedirs(OBJ_CACHE, exist_ok=True)
    units = [("host", [], SRC, [SRC, DEVICE_HDR, HDR]), ("dmma", [], DMMA_SRC, [DMMA_SRC, DEVICE_HDR, HDR])]
    for t, s, r in VARIANTS:
        units.append((f"pipe_{t}_{s}_{r}", [f"-DRS_VARIANT_T={t}", f"-DRS_VARIANT_STRICT={s}", f"-DRS_VARIANT_REFL={r}",
                                             f"-DRS_VARIANT_F32={int(t == 'float')}"], VARIANT_SRC,
                      [VARIANT_SRC, DEVICE_HDR, HDR]))
    jobs = []
    for name, defs, src, srcdeps in units:
        base = [nvcc, *NVCC_FLAGS, *extra, *inc, *defs]
        obj = os.path.join(OBJ_CACHE, f"{name}-{_key(base + [src], srcdeps)}.o")
        if only and name not in only:
            # developer experiments (RS_BUILD_ONLY=host,pipe_double_0_0): every other unit
            # is compiled (or taken from the cache) without the extra flags
            base = [nvcc, *NVCC_FLAGS, *inc, *defs]
            obj = os.path.join(OBJ_CACHE, f"{name}-{_key(base + [src], srcdeps)}.o")
        jobs.append((obj, base + ["-c", "-o", obj + ".tmp", src]))
    todo = [j for j in jobs if not os.path.exists(j[0])]

    def compile_one(job):
        log = _run(job[1])
        os.replace(job[0] + ".tmp", job[0])
        with open(job[0] + ".log", "w") as fh:
            fh.write(log)
        return log

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo) or 1, os.cpu_count() or 1))) as pool:
        list(pool.map(compile_one, todo))
    logs = []
    for obj, _ in jobs:
        try:
            with open(obj + ".log") as fh:
                logs.append(fh.read())
        except OSError:
            pass
    fd, tmp = tempfile.mkstemp(suffix=".so", dir=os.path.dirname(out))
    os.close(fd)
    try:
        _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *[j[0] for j in jobs]])
        os.replace(tmp, out)
    finally:
        if os.path.exists(tmp):
            os.remove(tmp)
    info = "\n".join(logs)
    if verbose:
        print(info)
    if out == OUT:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
            fh.write(info)
    return out


if __name__ == "__main__":
    print(build_library(force=True, verbose=False))
