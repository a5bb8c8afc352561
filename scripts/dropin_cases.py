"""The instances of oracle/drop_in_check.cpp (splitmix64 generator), in
Python, so a single case can be replayed through the Python API.
usage: python scripts/dropin_cases.py CASE [gpu] — prints the oracle's
objectives (and the GPU's, each solve in a child process with a timeout)."""
import os, sys, subprocess
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np

M64 = (1 << 64) - 1


class Rng:
    def __init__(self, s): self.s = s

    def next(self):
        self.s = (self.s + 0x9e3779b97f4a7c15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M64
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M64
        return z ^ (z >> 31)

    def inn(self, lo, hi): return lo + self.next() % (hi - lo + 1)


def make_instance(c):
    from paper_2304_06543_b200.instance import PenaltySpec, ProblemInstance, ServiceCenter
    n, k = 40 + 37 * c, 3 + c % 9
    theta = 1.2 if c % 3 == 0 else (0.8 if c % 3 == 1 else 1.0)
    r = Rng(1000 + c)
    total = int(theta * n)
    centers = []
    for s in range(k):
        cap = total // k + (1 if s < total % k else 0)
        f = r.next() % 3
        if f == 0:
            pen = PenaltySpec(0, [r.inn(1, 60)])
        elif f == 1:
            a = r.inn(1, 30); b = r.inn(0, 9); pen = PenaltySpec(1, [a, b])
        else:
            ln = r.inn(1, 4); v = r.inn(1, 20); t = []
            for _ in range(ln):
                t.append(v); v += r.inn(0, 15)
            pen = PenaltySpec(2, t)
        centers.append(ServiceCenter(s, cap, pen))
    costs = np.array([r.inn(1, 100) for _ in range(n * k)], dtype=np.int32).reshape(n, k)
    return ProblemInstance(centers, costs)


def run_one(c, mode, fix, par):
    from paper_2304_06543_b200 import solver as S, SolverOptions
    inst = make_instance(c)
    o = SolverOptions(refine_to_fixpoint=bool(fix), parallel=bool(par))
    r = S.solve(inst, mode, o)
    print(r.objective)


if __name__ == "__main__":
    if sys.argv[1] == "one":
        run_one(int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5]))
        sys.exit(0)
    import pyoracle
    c = int(sys.argv[1])
    O = pyoracle.reference() or pyoracle.oracle()
    from paper_2304_06543_b200.instance import SolverOptions
    inst = make_instance(c)
    for mode, fix, par in [("asral", 0, 0), ("strict", 0, 0), ("asral", 1, 0), ("strict", 1, 0),
                           ("greedy", 0, 0), ("asral", 0, 1)]:
        want = O.solve(inst, mode, SolverOptions(refine_to_fixpoint=bool(fix))).objective
        got = "-"
        if "gpu" in sys.argv:
            try:
                p = subprocess.run([sys.executable, __file__, "one", str(c), mode, str(fix), str(par)],
                                   capture_output=True, text=True, timeout=30)
                got = p.stdout.strip() or ("ERR " + p.stderr.strip().splitlines()[-1])
            except subprocess.TimeoutExpired:
                got = "TIMEOUT"
        print(f"case {c} {mode} fix {fix} par {par}: oracle {want} gpu {got}", flush=True)
