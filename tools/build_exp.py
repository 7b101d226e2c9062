"""Developer tool: build experiment variants of the library into tools/exp/lib_<name>.so.
Usage: python tools/build_exp.py name=-DFLAG1,-DFLAG2 name2=... """
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_01852_b200.build import build_library
os.makedirs(os.path.join(ROOT, "tools", "exp"), exist_ok=True)
for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = os.path.join(ROOT, "tools", "exp", f"lib_{name}.so")
    build_library(force=True, out=out, extra=[f for f in flags.split(",") if f])
    print("built", out, flush=True)
