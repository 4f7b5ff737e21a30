"""In-tree build of the sm_100a CUDA library and the C++ host layer.

libeigenid_b200.so : kernels + the extern "C" boundary (include/eigenid_b200.h)
libeigenid.so      : the reference-shaped C++ API (include/eigenid/*.hpp)
                     implemented over the C-ABI (host/*.cpp)
Both land next to this file so gpurun ships them with the snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
LIB = os.path.join(PKG, "libeigenid_b200.so")
HOSTLIB = os.path.join(PKG, "libeigenid.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
REFERENCE = os.environ.get("EIGENID_REFERENCE", "/root/reference/proj")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = cu + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "eigenid_b200.h")]
    if force or _newer(LIB, deps):
        objs = []
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        for src in cu:
            obj = os.path.join(ROOT, "build", os.path.basename(src) + ".o")
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17",
                   "-Xcompiler", "-fPIC", "-c", src, "-o", obj]
            if verbose_ptxas:
                cmd.insert(4, "-Xptxas=-v")
            _run(cmd)
            objs.append(obj)
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs])
    hsrc = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    hdeps = hsrc + glob.glob(os.path.join(ROOT, "include", "eigenid", "*.hpp")) + [LIB]
    if hsrc and (force or _newer(HOSTLIB, hdeps)):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared",
              "-I" + os.path.join(ROOT, "include"), *hsrc, "-o", HOSTLIB,
              "-L" + PKG, "-leigenid_b200", "-Wl,-rpath,$ORIGIN", "-pthread"])
    # The reference's own acceptance suite against the drop-in headers
    # (tests/cpp/acceptance_shim.cpp supplies the reference's Jacobi oracle
    # from oracle/_ref).  Only where /root/reference exists; the binary ships
    # to the GPU box with the snapshot.
    acc_src = os.path.join(REFERENCE, "tests", "acceptance.cpp")
    acc_bin = os.path.join(ROOT, "tests", "cpp", "acceptance")
    shim = os.path.join(ROOT, "tests", "cpp", "acceptance_shim.cpp")
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libeigenid_ref.so")
    if os.path.exists(acc_src) and os.path.exists(ref_so) and (
            force or _newer(acc_bin, [acc_src, shim, HOSTLIB, ref_so])):
        _run(["g++", "-O2", "-std=gnu++20", "-I" + os.path.join(ROOT, "include"),
              "-I" + os.path.join(REFERENCE, "include"), acc_src, shim, "-o", acc_bin,
              "-L" + PKG, "-leigenid", "-leigenid_b200",
              "-L" + os.path.dirname(ref_so), "-leigenid_ref",
              "-Wl,-rpath," + PKG + ":" + os.path.dirname(ref_so), "-pthread"])
    test_src = os.path.join(ROOT, "tests", "cpp", "test_host.cpp")
    test_bin = os.path.join(ROOT, "tests", "cpp", "test_host")
    if os.path.exists(test_src) and (force or _newer(test_bin, [test_src, HOSTLIB])):
        _run(["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "include"),
              test_src, "-o", test_bin, "-L" + PKG, "-leigenid", "-leigenid_b200",
              "-Wl,-rpath," + PKG, "-pthread"])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
