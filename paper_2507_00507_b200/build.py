"""In-tree build of the native libraries (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

  paper_2507_00507_b200/libmesh_gpu.so   CUDA sm_100a data plane  (include/mesh_gpu.h)
  paper_2507_00507_b200/libllmmesh.so    C++20 control plane      (include/llmmesh.h)
  oracle/_build/libmesh_oracle.so        CPU numeric oracle (tests only)
  oracle/_ref/*                          the unmodified reference, built from its sources (tests/bench only)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2507_00507_b200")
CSRC = os.path.join(PKG, "csrc")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

GPU_LIB = os.path.join(PKG, "libmesh_gpu.so")
CTRL_LIB = os.path.join(PKG, "libllmmesh.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "libmesh_oracle.so")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd: list[str], cwd: str | None = None) -> None:
    r = subprocess.run(cmd, cwd=cwd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError(f"build step failed ({r.returncode}): {' '.join(cmd)}")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_gpu(force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "gpu", "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "gpu", "*.cuh")) + [os.path.join(ROOT, "include", "mesh_gpu.h")]
    if force or _stale(GPU_LIB, deps):
        tmp = GPU_LIB + ".tmp"
        _run([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-I", os.path.join(ROOT, "include"), "-o", tmp, *srcs])
        os.replace(tmp, GPU_LIB)
    return GPU_LIB


def build_control(force: bool = False) -> str | None:
    srcs = sorted(glob.glob(os.path.join(CSRC, "control", "*.cpp")))
    if not srcs:
        return None
    deps = srcs + glob.glob(os.path.join(CSRC, "control", "*.hpp")) + [os.path.join(ROOT, "include", "llmmesh.h")]
    if force or _stale(CTRL_LIB, deps):
        tmp = CTRL_LIB + ".tmp"
        # -ffp-contract=off: decisions compare doubles with ==
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-ffp-contract=off", "-fvisibility=hidden",
              "-I", os.path.join(ROOT, "include"), "-I", JSON_INC, "-o", tmp, *srcs])
        os.replace(tmp, CTRL_LIB)
    return CTRL_LIB


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "llama_ref.c")
    fast = os.path.join(ROOT, "oracle", "cpu_decode.c")  # batched CPU baseline (bench only)
    hdr = os.path.join(ROOT, "oracle", "llama_ref.h")
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    if force or _stale(ORACLE_LIB, [src, fast, hdr]):
        tmp = ORACLE_LIB + ".tmp"
        bdir = os.path.dirname(ORACLE_LIB)
        # the checker keeps plain -O2 numerics; the baseline may vectorise (AVX2 + FMA)
        _run(["gcc", "-O2", "-fopenmp", "-fPIC", "-c", "-o", os.path.join(bdir, "llama_ref.o"), src])
        _run(["gcc", "-O3", "-mavx2", "-mfma", "-fopenmp", "-fPIC", "-c", "-o", os.path.join(bdir, "cpu_decode.o"),
              fast])
        _run(["gcc", "-fopenmp", "-shared", "-o", tmp, os.path.join(bdir, "llama_ref.o"),
              os.path.join(bdir, "cpu_decode.o"), "-lm"])
        os.replace(tmp, ORACLE_LIB)
    return ORACLE_LIB


def build_reference() -> bool:
    """Builds the unmodified reference into oracle/_ref when its sources exist here."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_capture"))
    _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle")])
    return True


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_control(force)
    build_oracle(force)
    build_reference()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", GPU_LIB, CTRL_LIB, ORACLE_LIB)
