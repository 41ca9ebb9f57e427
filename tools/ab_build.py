"""Build an A/B variant of the library: every unit recompiled with -DBFLA_EXPERIMENTS (the environment
switches of common.cuh experiment_knob) plus extra -D flags.

  python tools/ab_build.py NAME -DFOO=1 ...   ->  paper_2605_12193_b200/libbfla_NAME.so
Select it in a tool with paper_2605_12193_b200._lib.use_variant(NAME) (experiments only; never used by
the product path or the tests)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_12193_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
print(B.build(variant=name, extra=flags))
