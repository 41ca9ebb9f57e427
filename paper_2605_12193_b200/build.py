"""Build libbfla.so (the C-ABI library) in-tree with nvcc for sm_100a.

Each translation unit is compiled separately; stage1_select.cu and stage1_scores.cu are compiled
with -fmad=false so no multiply-add contraction can change the canonical fp32 sequence of the
mask; the attention kernel is compiled with the default contraction.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbfla.so")
BUILD = os.path.join(HERE, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
UNITS = {
    "api.cu": [],
    "stage1_scores.cu": ["-fmad=false"],
    "stage1_select.cu": ["-fmad=false"],
    "stage1_tc.cu": ["-fmad=false"],
    "stage2.cu": [],
    "attention.cu": [],
    "attention2.cu": [],
    "merge.cu": [],
}


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


# Library variants.  The product library (libbfla.so) has no switches.  The others are built on
# demand for tools only: debug (mbarrier-timeout traps, build.py --debug), exp (experiment switches
# read from the environment, tools/ab_build.py) and trace (attention timeline, tools/attn_trace.py).
VARIANTS = {"": [], "debug": ["-DBFLA_DEBUG"], "exp": ["-DBFLA_EXPERIMENTS"], "trace": ["-DBFLA_TRACE"]}


def lib_path(variant: str = "") -> str:
    return LIB if not variant else os.path.join(HERE, f"libbfla_{variant}.so")


def build(force: bool = False, verbose: bool = False, variant: str = "", extra=()) -> str:
    """Compile every unit for sm_100a and link libbfla[_variant].so; returns its path."""
    flags = list(VARIANTS.get(variant, ["-DBFLA_EXPERIMENTS"])) + list(extra)
    objdir = BUILD if not variant else BUILD + "_" + variant
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "bfla.h"))
    objs = []
    for unit, unit_flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or extra or _stale(obj, [src, *headers, __file__]):
            cmd = [nvcc(), *ARCH, *COMMON, *flags, *unit_flags, "-c", src, "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
    out = lib_path(variant)
    if force or extra or _stale(out, objs):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs])
        os.replace(tmp, out)
    return out


def build_trace() -> str:
    """libbfla_trace.so: the attention timeline instrumentation compiled in (-DBFLA_TRACE;
    tools/attn_trace.py).  Never loaded by the product path or the tests."""
    return build(variant="trace")


if __name__ == "__main__":
    var = "trace" if "--trace" in sys.argv else "debug" if "--debug" in sys.argv else ""
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var))
