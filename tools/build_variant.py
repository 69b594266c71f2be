"""Build a measurement variant of the engine library with extra -D defines.

    python tools/build_variant.py <name> DEF1=1 [DEF2 ...]   ->  abtest/<name>/libsamp_b200.so

Load it with SAMP_B200_LIB=abtest/<name>/libsamp_b200.so (tools/ab.sh compares two).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_09130_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "abtest", name)
print(_build.build(defines=defs, lib=os.path.join(out, "libsamp_b200.so"), objdir=os.path.join(out, "obj")))
