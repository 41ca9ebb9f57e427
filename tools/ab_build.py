"""Build an A/B variant of libbfla.so: the attention2 unit recompiled with extra -D flags.

  python tools/ab_build.py NAME -DFOO=1 ...   ->  paper_2605_12193_b200/libbfla_NAME.so
Select it at run time with BFLA_LIB_VARIANT=NAME (experiments only; never used by tests)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12193_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
B.build()
obj = os.path.join(B.BUILD, f"attention2_{name}.o")
subprocess.check_call([B.nvcc(), *B.ARCH, *B.COMMON, *flags, "-c", os.path.join(B.CSRC, "attention2.cu"), "-o", obj])
objs = [os.path.join(B.BUILD, u.replace(".cu", ".o")) for u in B.UNITS if u != "attention2.cu"]
out = os.path.join(B.HERE, f"libbfla_{name}.so")
subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", out, *objs, obj])
print(out)
