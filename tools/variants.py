"""Build experiment variants of libvoltana.so with extra -D defines into variants/<name>.so.

    python tools/variants.py name=DEF1,DEF2 name2=DEF3 ...
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04827_b200 import build as b
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for a in sys.argv[1:]:
    name, defs = a.split("=", 1)
    so = os.path.join(root, "variants", name + ".so")
    b.build(defines=[d for d in defs.split(",") if d], so=so)
    print(so)
