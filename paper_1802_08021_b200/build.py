"""Build libsparcml.so (sm_100a) in-tree with nvcc.

Every kernel is compiled for `-gencode arch=compute_100a,code=sm_100a` with
-lineinfo; the library is a plain shared object with the C ABI of
include/sparcml.h (no torch, no Python in it)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsparcml.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
                              glob.glob(os.path.join(HERE, "csrc", "*.h")) +
                              [os.path.join(ROOT, "include", "sparcml.h"), __file__])


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return lib
    objdir = os.path.join(HERE, "build" if lib == LIB else "build_" + os.path.basename(lib).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    # an object is reused when it is newer than its source, every header and this
    # script, and was compiled with the same flags (stamp file)
    hdr_t = max(os.path.getmtime(d) for d in deps() if not d.endswith(".cu"))
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        objs.append(obj)
        stamp = obj + ".cmd"
        if (not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == " ".join(cmd)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t)):
            continue
        if os.path.exists(stamp):
            os.remove(stamp)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), stamp,
                      " ".join(cmd)))
    logs = []
    for src, p, stamp, cmdline in procs:
        out, _ = p.communicate()
        logs.append(out.decode())
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        with open(stamp, "w") as f:
            f.write(cmdline)
    with open(os.path.join(objdir, "ptxas.log"), "a" if not procs else "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    tmp = lib + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
           "-Xcompiler", "-fPIC"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
