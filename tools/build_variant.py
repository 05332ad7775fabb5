"""Build libsvf.so (name 'main') or a tuning variant paper_2601_08528_b200/libsvf_<name>.so with extra nvcc flags,
for A/B runs selected with SVF_LIB (experiments only):  python tools/build_variant.py w4 -DSVF_GATHER_W_LP=4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08528_b200 import build_lib  # noqa: E402

name, *flags = sys.argv[1:]
out = build_lib.OUT if name == "main" else os.path.join(build_lib.HERE, f"libsvf_{name}.so")
print(build_lib.build(out=out, extra=tuple(flags)))
