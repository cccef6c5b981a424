"""Build an A/B variant of libsparcml.so: recompile the named sources with extra
-D macros and link them with the main build's other objects (diagnostics; the
product library is paper_1802_08021_b200/libsparcml.so from build.py).

  python tools/build_variant.py OUT.so kernels_topk.cu -D SPARCML_TOPK_ROLES=0 [-D ...]
"""
import argparse
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1802_08021_b200 import build as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("sources", nargs="+", help="csrc file names to recompile")
ap.add_argument("-D", dest="defines", action="append", default=[])
args = ap.parse_args()

B.build()   # the main objects are current
objdir = os.path.join(B.HERE, "build")
tmpdir = os.path.join(B.HERE, "build_var_" + os.path.basename(args.out).replace(".so", ""))
os.makedirs(tmpdir, exist_ok=True)
objs = []
for o in sorted(glob.glob(os.path.join(objdir, "*.o"))):
    name = os.path.basename(o)[:-2]
    if name in args.sources:
        src = os.path.join(B.HERE, "csrc", name)
        obj = os.path.join(tmpdir, name + ".o")
        cmd = [B.NVCC, *B.FLAGS, *[f"-D{d}" for d in args.defines], "-I", os.path.join(ROOT, "include"), "-c", src,
               "-o", obj]
        subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
        objs.append(obj)
    else:
        objs.append(o)
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", args.out, *objs,
                "-Xcompiler", "-fPIC"], check=True)
print(args.out)
