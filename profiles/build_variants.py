"""Measurement builds of the library with extra nvcc flags (occupancy / code-shape A/B),
each into its own object dir and .so under scratch/variants/; select one at run time with
FNLH_B200_LIB=<path>.  usage: python profiles/build_variants.py tag="-DFLAG=1 -DX=2" ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_01407_b200 import build as b  # noqa: E402

for arg in sys.argv[1:]:
    tag, flags = arg.split("=", 1)
    out = os.path.join(ROOT, "scratch", "variants")
    os.makedirs(out, exist_ok=True)
    lib = b.build(lib=os.path.join(out, f"libfnlh_{tag}.so"), obj_dir=os.path.join(out, f"obj_{tag}"),
                  extra=flags.split())
    print(tag, lib)
