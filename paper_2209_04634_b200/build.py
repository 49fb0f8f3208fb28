"""Build the sm_100a CUDA library in-tree: paper_2209_04634_b200/libevsim_gpu.so.

nvcc -gencode arch=compute_100a,code=sm_100a, -fmad=false (the reference is
FMA-free; see csrc/evsim_device.cuh), -lineinfo for ncu source attribution.
The library exports exactly the C-ABI of include/evsim_gpu.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libevsim_gpu.so")
# bounds-checked variant (-DEVSIM_CHECKED: device-side checks of the kernels'
# global writes, evsim_device.cuh EVSIM_CHECK); loaded when EVSIM_GPU_LIB=checked
OUT_CHECKED = os.path.join(HERE, "libevsim_gpu_checked.so")
SOURCES = ["evsim_gpu.cu", "flow_kernels.cu", "event_kernels.cu", "io_kernels.cu", "wire_kernels.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-Xptxas", "-v",
    f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}",
]


def _stale(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "evsim_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile under an exclusive file lock (torchrun ranks may all call this)
    and publish the library with an atomic rename, so no process ever loads a
    half-written .so."""
    import fcntl
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    with open(os.path.join(HERE, "build", ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            out = OUT_CHECKED if checked else OUT
            if not force and not _stale(out):
                return out
            return _build(verbose, checked)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build(verbose: bool, checked: bool = False) -> str:
    objdir = os.path.join(HERE, "build_checked" if checked else "build")
    out = OUT_CHECKED if checked else OUT
    flags = FLAGS + (["-DEVSIM_CHECKED"] if checked else [])
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))  # (serialised by the build lock)
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = f"{out}.{os.getpid()}.tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
