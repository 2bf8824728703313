"""In-tree build of the native libraries (sm_100a only).

* ``libmp_b200.so``   -- the CUDA kernels + C-ABI (include/mp_cuda.h).
* ``libmp_datagen.so`` -- seeded synthetic-input generator (harness).

Both are built IN-TREE next to this file so they travel with the repo
snapshot to the GPU box (``*.so`` is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libmp_b200.so")
DATAGEN = os.path.join(PKG, "libmp_datagen.so")
DROPIN = os.path.join(PKG, "libmultiproj_b200.so")  # the reference C++ API over the C-ABI

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-shared",
]
CU_SOURCES = ["mp_device.cu", "mp_host.cu"]
# MP_TUNING_SWITCHES=1 at build time compiles in the A/B route switches
# (MP_L1_PIPE, MP_L1_TMA, ... read from the environment; tuning builds only).
if os.environ.get("MP_TUNING_SWITCHES") == "1":
    NVCC_FLAGS = NVCC_FLAGS + ["-DMP_TUNING_SWITCHES"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cpp_test(out: str) -> str:
    """Compile tests/cpp/dropin_test.cpp against the drop-in library."""
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{INCLUDE}", src, f"-L{PKG}", "-lmultiproj_b200", "-lmp_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


DROPIN_BENCH = os.path.join(PKG, "dropin_bench")


def build_dropin_bench(out: str = DROPIN_BENCH) -> str:
    """Compile tests/cpp/dropin_bench.cpp (bench.py's C++ drop-in e2e leg)."""
    src = os.path.join(ROOT, "tests", "cpp", "dropin_bench.cpp")
    if _stale(out, [src, DROPIN]):
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{INCLUDE}", src, f"-L{PKG}", "-lmultiproj_b200", "-lmp_b200",
                        "-Wl,-rpath,$ORIGIN", "-o", out], check=True)
    return out


def build_io_test(out: str) -> str:
    """Compile tests/cpp/io_compat.cpp (host-side formats, no GPU calls)."""
    src = os.path.join(ROOT, "tests", "cpp", "io_compat.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{INCLUDE}", src, f"-L{PKG}", "-lmultiproj_b200", "-lmp_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def build(force: bool = False, verbose: bool = False) -> None:
    deps = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(INCLUDE, "mp_cuda.h")]
    if force or _stale(LIB, deps):
        cmd = [NVCC, *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}",
               *[os.path.join(CSRC, s) for s in CU_SOURCES], "-o", LIB + ".tmp"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    di = [os.path.join(CSRC, "dropin", f) for f in ("multiproj_dropin.cpp", "multiproj_io.cpp")]
    di_deps = di + [LIB] + glob.glob(os.path.join(INCLUDE, "multiproj", "*.hpp"))
    if force or _stale(DROPIN, di_deps):
        subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", f"-I{INCLUDE}", *di, f"-L{PKG}", "-lmp_b200",
                        "-Wl,-rpath,$ORIGIN", "-o", DROPIN], check=True)
    build_dropin_bench()
    dg = os.path.join(CSRC, "datagen.c")
    if force or _stale(DATAGEN, [dg]):
        subprocess.run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", dg,
                        "-o", DATAGEN, "-lm"], check=True)


if __name__ == "__main__":
    build(force=True, verbose=True)
