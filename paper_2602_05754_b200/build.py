"""In-tree build of the two native libraries (no JIT cache, no site-packages install).

  lib/libpf_host.so    C++20 host layer: schedule, DAG, timing, freeze-ratio LP,
                       freeze controller (namespace pipefreeze) + its C-ABI.
  lib/libpf_device.so  sm_100a kernels (nvcc -gencode arch=compute_100a,code=sm_100a)
                       + the per-stage step engine + its C-ABI.

Usage: python -m paper_2602_05754_b200.build [--force] [--host-only]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
INC = os.path.join(ROOT, "include")
HOST_SRC = os.path.join(PKG, "csrc", "host")
DEV_SRC = os.path.join(PKG, "csrc", "device")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")


def build_host(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    out = os.path.join(LIB, "libpf_host.so")
    srcs = sorted(glob.glob(os.path.join(HOST_SRC, "*.cpp")))
    deps = srcs + glob.glob(os.path.join(HOST_SRC, "*.hpp")) + glob.glob(os.path.join(INC, "*.h"))
    if force or _newer(out, deps):
        # -Bsymbolic: calls inside the library bind to its own definitions (the test oracle
        # defines the same pipefreeze:: names)
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-fopenmp", "-Wall", "-Wextra", "-Wl,-Bsymbolic",
               "-I", INC, "-I", HOST_SRC, *srcs, "-o", out]
        _run(cmd)
    return out


def _nccl_flags() -> list[str]:
    """Link NCCL: the system library when its headers and .so are installed (this image), else the
    nvidia-nccl wheel bundled with the Python environment."""
    import glob as _g

    if _g.glob("/usr/lib/x86_64-linux-gnu/libnccl.so*") or _g.glob("/usr/local/cuda/lib64/libnccl.so*"):
        return ["-lnccl"]
    for d in _g.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "lib")):
        return [f"-L{d}", "-Xlinker", f"-rpath={d}", "-l:libnccl.so.2"]
    return ["-lnccl"]


def build_device(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    out = os.path.join(LIB, "libpf_device.so")
    cu = sorted(glob.glob(os.path.join(DEV_SRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(DEV_SRC, "*.cpp")))
    headers = glob.glob(os.path.join(DEV_SRC, "*.cuh")) + glob.glob(os.path.join(DEV_SRC, "*.hpp")) + glob.glob(os.path.join(INC, "*.h"))
    common = ["-I", INC, "-I", DEV_SRC, "-I", HOST_SRC]
    jobs = []
    objs = []
    for src in cu + cpp:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if not (force or _newer(obj, [src] + headers)):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                   "-Xcompiler", "-fPIC", *common, "-c", src, "-o", obj]
        else:
            cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", *common, f"-I{CUDA_HOME}/include",
                   "-c", src, "-o", obj]
        jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
            list(ex.map(_run, jobs))
    if force or jobs or _newer(out, objs):
        # no libtorch: the device library needs only the CUDA runtime / driver, NCCL and libpf_host
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", out, "-lcudart",
               f"-L{LIB}", "-lpf_host", "-Xlinker", "-rpath=$ORIGIN", *_nccl_flags()]
        _run(cmd)
    return out


def build(force: bool = False, host_only: bool = False) -> list[str]:
    outs = [build_host(force)]
    if not host_only:
        outs.append(build_device(force or _newer(os.path.join(LIB, "libpf_device.so"), [outs[0]])))
    return outs


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--host-only", action="store_true")
    a = ap.parse_args()
    for o in build(a.force, a.host_only):
        print(o)
