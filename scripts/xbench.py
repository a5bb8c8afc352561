import sys, ctypes as C
sys.path.insert(0, '.')
from paper_2304_06543_b200 import solver as S
f = S._lib.lbdd_b200_debug_exchange_cycles
f.restype = C.c_longlong
for cs in [1, 2, 4, 8, 16]:
    print(cs, [f(cs, 20000, m) for m in range(4)], flush=True)
