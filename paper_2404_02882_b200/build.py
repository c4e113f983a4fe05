"""Builds liblasp.so (the C-ABI library of include/lasp.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblasp.so")
SOURCES = ["lasp_api.cu", "kernels_simt.cu", "kernels_tc.cu", "kernels_gla.cu"]
HEADERS = ["lasp_common.cuh", "sm100.cuh", "gla.cuh"]


def _nccl_include() -> str:
    import nvidia.nccl  # torch's bundled NCCL (headers + libnccl.so.2)
    return os.path.join(list(nvidia.nccl.__path__)[0], "include")


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "lasp.h"), __file__]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    objs = []
    jobs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
               "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
               "-I", _nccl_include(), "-c", os.path.join(CSRC, src), "-o", obj]
        if os.environ.get("LASP_TRACE_BUILD"):
            cmd += ["-DLASP_TRACE_BUILD"]
        if os.environ.get("LASP_EXTRA_NVCC"):  # debug / experiment builds only (always with --out)
            cmd += os.environ["LASP_EXTRA_NVCC"].split()
        if os.environ.get("LASP_PTXAS_VERBOSE"):
            cmd += ["-Xptxas", "-v"]
        jobs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
        objs.append(obj)
    failed = False
    for j, src in zip(jobs, SOURCES):
        out, _ = j.communicate()
        if verbose or j.returncode:
            sys.stderr.write(out.decode())
        if j.returncode:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = lib + f".{os.getpid()}.tmp"
    subprocess.check_call([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs +
                          ["-ldl", "-lcudart"])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    out = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    print(build(force="--force" in sys.argv or out is not None, verbose=True, out=out))
