"""Build libntt.so in-tree for sm_100a (nvcc; no JIT cache).

    python -m paper_2012_01968_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libntt.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include")]

SOURCES = ["ntt_kernels.cu", "ntt_kernels_p.cu", "ntt_kernels_d.cu", "ntt_k1.cu", "ntt_single.cu", "ntt_native.cu", "ntt_fused.cu", "ntt_request.cu", "ntt32.cu", "ntt_baselines.cu", "ntt_api.cu", "ntt32_api.cu", "params.cpp"]
HEADERS = ["ntt_kernels.cuh", "ntt_fused.cuh", "ntt_device.cuh", "ntt_launch.h", "params.h"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(BUILD, src + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "ntt.h")]
    if force or _newer(obj, deps):
        cmd = [NVCC, *ARCH, *COMMON, "-x", "cu" if src.endswith(".cu") else "c++", "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-warn-spills"]
        subprocess.check_call(cmd)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or _newer(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
                               "-Xcompiler", "-pthread"])
        os.replace(tmp, LIB)
    return LIB


def build_ceiling_probe(force: bool = False) -> str:
    """tools/libs/bf_roof: the register-only butterfly throughput probe (the
    practical ALU ceiling bench.py reports its roofline against)."""
    src = os.path.join(ROOT, "tools", "bf_roof.cu")
    out = os.path.join(ROOT, "tools", "libs", "bf_roof")
    deps = [src, os.path.join(CSRC, "ntt_device.cuh")]
    if force or _newer(out, deps):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        subprocess.check_call([NVCC, *ARCH, "-O3", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-o", out, src])
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
    print(build_ceiling_probe(force="--force" in sys.argv))
