"""Small asral solve for ncu: one engine launch on a 2000 x 100 instance."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import pyoracle as po
from paper_2304_06543_b200 import solver as S
inst = po.oracle().generate(42, int(sys.argv[1]) if len(sys.argv) > 1 else 2000, 20.0, 0.8, 1, 200)
rep = S.asral_solve(inst)
print("objective", rep.objective, rep.timings)
