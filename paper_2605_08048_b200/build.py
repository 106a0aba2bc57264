"""Build libhap.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhap.so")
# the checked build (device-side bounds / invariant checks and workspace guard bytes,
# DESIGN.md "Device checks"): tests only, loaded with HAP_LIB=checked
LIB_CHECKED = os.path.join(PKG, "libhap_checked.so")
SOURCES = ["hap_api.cu", "k_align.cu", "k_perm.cu", "k_maskgemm.cu", "k_gram.cu"]
HEADERS = ["hap_device.cuh", "hap_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
# experiments only (e.g. -DHAP_K3_STAGES=4); empty in normal builds
FLAGS += os.environ.get("HAP_EXTRA_NVCC_FLAGS", "").split()


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(os.path.dirname(PKG), "include", h) for h in ("hap.h", "hap_debug.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    flags = FLAGS + (["-DHAP_DEVICE_CHECKS"] if checked else [])
    tag = ".chk" if checked else ""
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", tag + ".o"))
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stdout.write(out.decode())
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *flags, "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
