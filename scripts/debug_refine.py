import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import pyoracle as po
from paper_2304_06543_b200 import solver as S
O, R = po.oracle(), po.reference()
rng = po.Mt19937_64(47)
for it in range(30):
    n, k = 5 + rng() % 30, 2 + rng() % 4
    inst = po.random_instance(rng, n=n, k=k)
    asg = np.array([rng() % k for _ in range(n)], np.int32)
    anchor = int(rng() % k)
    a = O.refine(inst, 0, anchor, asg)
    try:
        b = S.negative_cycle_refine(inst, asg, anchor)
    except Exception as e:
        b = repr(e)
    r = R.refine(inst, 0, anchor, asg) if R else None
    if isinstance(b, str) or a[0] != b[0] or a[1] != b[1] or (a[2] != b[2]).any():
        print("it", it, "n", n, "k", k, "anchor", anchor)
        print("oracle", a[:3]); print("ref", r[:3] if r else None); print("dev", b if isinstance(b, str) else b[:3])
        M = O.build_index(inst, asg)
        print("keys\n", np.where(M == po.NO_EDGE, 99999, M >> 32))
        print("gamma cycle (oracle):", O.gamma_has_negative_cycle(inst, asg))
        # dense anchored graph the reference would build
        w = np.full((k, k + 1), po.NO_EDGE, np.int64)
        for u in range(k):
            for v in range(k):
                if u != v and M[u, v] != po.NO_EDGE:
                    w[u, k if v == anchor else v] = M[u, v] >> 32
        try: print("dense oracle lcp:", O.lowest_cost_path(w, anchor))
        except Exception as e: print("dense oracle lcp:", repr(e))
        try: print("dense dev lcp:", S.lowest_cost_path(w, anchor))
        except Exception as e: print("dense dev lcp:", repr(e))
        break
    dm = np.array([rng() % 3 for _ in range(k)], np.int64)
    a = O.refine(inst, 0, anchor, asg, dm)
    b = S.negative_cycle_refine(inst, asg, anchor, dm)
print("done")
