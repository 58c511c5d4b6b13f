"""Build libdd.so in-tree with nvcc for sm_100a (no JIT caches: the .so travels with gpurun).

Links cudart statically; cuSOLVER (3D setup eigensolve only) from the CUDA toolkit and NCCL
(3D pole split) from the torch-bundled nvidia-nccl wheel, both found at run time by rpath.
Objects are rebuilt in parallel.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdd.so")
SOURCES = ["gemm_f64.cu", "gemm_pair.cu", "pcg_polesum.cu", "face3d.cu", "fx_sym.cu", "bulk2d.cu", "bulk3d.cu", "dd_api.cpp", "dd3d.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_LIB = "/usr/local/cuda/lib64"


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _nccl_dirs():
    for base in [os.path.dirname(os.path.dirname(p)) for p in sys.path if p.endswith("site-packages")] + \
            ["/opt/prime-rl/.venv/lib/python3.12/site-packages"]:
        inc = os.path.join(base, "nvidia", "nccl", "include")
        lib = os.path.join(base, "nvidia", "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
        inc = os.path.join(base, "site-packages", "nvidia", "nccl", "include")
        lib = os.path.join(base, "site-packages", "nvidia", "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "dd_api.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    nccl_inc, nccl_lib = _nccl_dirs()
    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", nccl_inc]

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        if src.endswith(".cu"):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", *inc,
                   "-c", os.path.join(CSRC, src), "-o", obj]
        else:
            cmd = [nvcc, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    nccl_so = sorted(glob.glob(os.path.join(nccl_lib, "libnccl.so*")))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl",
           "-L", CUDA_LIB, "-lcusolver", "-lcublas", "-lcublasLt",
           "-L", nccl_lib, f"-l:{os.path.basename(nccl_so[0])}" if nccl_so else "-lnccl",
           "-Xlinker", f"-rpath,{CUDA_LIB}", "-Xlinker", f"-rpath,{nccl_lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
