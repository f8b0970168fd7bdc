"""Builds the library with extra nvcc defines into another path (A/B experiments):
python tools/build_variant.py exp/lib_t640.so -DPLAN_THREADS=640"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0911_2900_b200 import build as b  # noqa: E402

out = os.path.abspath(sys.argv[1])
os.makedirs(os.path.dirname(out), exist_ok=True)
b.FLAGS = b.FLAGS + sys.argv[2:]
b.OUT = out
b.build(force=True)
print(out)
