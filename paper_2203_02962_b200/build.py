"""Build recipe of the native library (nvcc, sm_100a only).

Produces ``paper_2203_02962_b200/_lib/libhomfe_gpu.so`` in-tree so that it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(HERE, "_lib", "obj")
LIB = os.path.join(OUT_DIR, "libhomfe_gpu.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include")]
SOURCES = ["kernels.cu", "spectral.cu", "hexfast.cu", "fftfused.cu", "quad2d.cu", "j2.cu", "probe.cu", "slabfft.cu", "small2d.cu", "context.cu"]
HEADERS = ["common.cuh", "kernels.cuh", "tables.hpp", "hex_modes.inc", "spectral.cuh", "fft.cuh"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, verbose, obj_dir=None, defines=()):
    obj = os.path.join(obj_dir or OBJ_DIR, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(HERE, "..", "include", "homfe_gpu.h")]
    if not _stale(obj, deps):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def _nccl_link():
    """Link the NCCL that PyTorch bundles when it is installed (same soname
    libnccl.so.2 as the system one): whichever of torch and this library loads
    first, the process then holds one NCCL that satisfies both (torch needs
    symbols the older system NCCL lacks)."""
    import glob
    for base in sys.path:
        hits = glob.glob(os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so.2"))
        if hits:
            d = os.path.dirname(hits[0])
            return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{d}"]
    return ["-lnccl"]


def build(verbose=False, force=False, lib=None, defines=()):
    """Compile and link. `lib`/`defines` build a tuning variant elsewhere."""
    lib = lib or LIB
    obj_dir = OBJ_DIR if lib == LIB else os.path.join(os.path.dirname(lib), "obj")
    os.makedirs(obj_dir, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if force:
        for f in os.listdir(obj_dir):
            os.remove(os.path.join(obj_dir, f))
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, obj_dir, defines), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, srcs):
            if log:
                print(f"--- ptxas {s}\n{log}", file=sys.stderr)
    if _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcufft", *_nccl_link(),
               "-Xlinker", f"-rpath,{CUDA}/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
