"""Build libisycos.so in-tree with nvcc for sm_100a (B200).  No JIT cache, no torch extension."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libisycos.so")
SOURCES = ["ksg_small.cu", "ksg_tile.cu", "ksg_lat.cu", "ksg_sorted.cu", "ksg_fused.cu", "ksg_wsorted.cu", "ksg_misc.cu",
           "engine.cu", "search.cpp", "capi.cpp"]
HEADERS = ["engine.h", "ksg_device.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
         "--fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "isycos.h"))
    files.append(os.path.abspath(__file__))
    return files


STAMP = LIB + ".sha256"


def _digest() -> str:
    """Content hash of every input plus the compiler command line (an mtime can lie after a copy or checkout)."""
    h = hashlib.sha256()
    for f in _inputs():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join([NVCC, *ARCH, *FLAGS]).encode())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as fh:
        return fh.read().strip() != _digest()


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, defines=(), out: str = "") -> str:
    """Build libisycos.so.  `defines` + `out`: an alternative build (kernel A/B measurements, loaded through
    ISYCOS_LIB) into another file; it never replaces the product library."""
    if not out and not force and not needs_build():
        return LIB
    objs = []
    tmpdir = os.path.join(HERE, "build" + ("_" + os.path.basename(out).replace(".", "_") if out else ""))
    os.makedirs(tmpdir, exist_ok=True)
    procs = []
    for s in SOURCES:
        obj = os.path.join(tmpdir, s + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c",
               os.path.join(CSRC, s), "-o", obj]
        if ptxas_info and s.endswith(".cu"):
            cmd.insert(1, "-Xptxas=-v")
        if s.endswith(".cpp"):
            cmd[cmd.index("-c"):cmd.index("-c")] = ["-x", "cu"]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = []
    for s, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            failed.append((s, log))
        elif verbose and log:
            sys.stderr.write(log)
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    target = out or LIB
    tmp = target + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    os.replace(tmp, target)
    if out:
        return out
    with open(STAMP, "w") as fh:
        fh.write(_digest() + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
