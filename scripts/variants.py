"""Build experiment variants of the library (never the product): python scripts/variants.py name DEF=V ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_11408_b200 import build
print(build.build_variant(sys.argv[1], sys.argv[2:]))
