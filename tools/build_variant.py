"""Build an in-tree variant of libenkf_b200.so with extra -D flags (A/B timing).

    python tools/build_variant.py NAME -DFOO=1 -DBAR=0   -> paper_1302_3876_b200/libenkf_b200_NAME.so
Load it with ENKF_LIB_VARIANT=NAME.
"""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1302_3876_b200 import build as B

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, f"libenkf_b200_{name}.so")
cmd = [B.nvcc_path(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
       "-I", os.path.join(B.ROOT, "include"), *defs, "-o", out, *B.SOURCES]
subprocess.run(cmd, check=True)
print(out)
