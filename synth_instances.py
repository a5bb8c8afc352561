"""Host-side synthetic instances of the BASELINE shapes ("lbdd-synth-v2").

Independent of the product library and of oracle/: bench.py generates the
instance both of its arms solve here, hashes it, and the repo arm uploads
exactly these bytes. The device generator (`lbdd_b200_instance_generate`,
csrc/scan.cu `generate_costs_kernel`) implements the same spec bit for bit,
so large GPU tests can generate in HBM and spot-check rows against this
module (tests/test_synth.py, tests/test_gpu_scale.py).

Spec (every step is integer arithmetic or one IEEE-754 double sqrt/div/add,
correctly rounded on every platform, so numpy, C++ and CUDA agree):

    mix(z)            splitmix64 finaliser
    stream(seed,t,i)  mix(mix(seed ^ t) + (i + 1) * 0x9E3779B97F4A7C15)
    demand d:  x = stream(seed, 1, d) % 10000,  y = stream(seed, 2, d) % 10000
    center s:  x = stream(seed, 3, s) % 10000,  y = stream(seed, 4, s) % 10000
    cost(d,s) = max(1, floor(sqrt(dx^2 + dy^2) / 10 + 0.5))   in [1, 1414]

Capacities: total = n * theta_num // theta_den, split over centers with
integer weights w_s = 1 + stream(seed, 5, s) % cap_spread (heterogeneous),
cap_s = total * w_s // sum(w); the remainder adds 1 to centers 0, 1, ...
Penalties (core.hpp:43-96 families): p = stream(seed, 6, s);
family = p % 3 when mixed else constant; base = lo + (p >> 8) % (hi-lo+1);
linear step = (p >> 24) % 6; table = 4 values, v_t = v_{t-1} + (p >> (32+3t)) % 8.

Configs (BASELINE.json):
  configs[1]  n=1M,  k=1000, theta 8/10, mixed penalties, spread 16, seed 20250
  configs[2]  n=4M,  k=2000, theta 1/1 (capacity = demand)
"""
from __future__ import annotations

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

GOLD = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK = (1 << 64) - 1
GRID = 10000
SPEC = "lbdd-synth-v2"


def mix_int(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * M1) & MASK
    z = ((z ^ (z >> 27)) * M2) & MASK
    return z ^ (z >> 31)


def stream_int(seed: int, tag: int, i: int) -> int:
    return mix_int((mix_int(seed ^ tag) + (i + 1) * GOLD) & MASK)


def _mix_np(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(M1)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def stream_np(seed: int, tag: int, i0: int, count: int) -> np.ndarray:
    base = np.uint64(mix_int(seed ^ tag))
    i = np.arange(i0 + 1, i0 + 1 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix_np(base + i * np.uint64(GOLD))


@dataclass(frozen=True)
class SynthSpec:
    n: int
    k: int
    seed: int = 20250
    theta_num: int = 8
    theta_den: int = 10
    pen_lo: int = 1
    pen_hi: int = 200
    mixed: bool = True
    cap_spread: int = 16

    def name(self) -> str:
        return (f"{SPEC}(n={self.n},k={self.k},seed={self.seed},theta={self.theta_num}/"
                f"{self.theta_den},pen=[{self.pen_lo},{self.pen_hi}],mixed={int(self.mixed)},"
                f"spread={self.cap_spread})")


# configs[0]: 10K x 100, capacity 80% of demand, constant penalties drawn uniformly
CONFIG0 = SynthSpec(10_000, 100, seed=7, mixed=False, cap_spread=1)
CONFIG1 = SynthSpec(1_000_000, 1000)
CONFIG2 = SynthSpec(4_000_000, 2000, theta_num=1, theta_den=1)


def coords(spec: SynthSpec, tag_x: int, tag_y: int, i0: int, count: int):
    x = (stream_np(spec.seed, tag_x, i0, count) % np.uint64(GRID)).astype(np.int64)
    y = (stream_np(spec.seed, tag_y, i0, count) % np.uint64(GRID)).astype(np.int64)
    return x, y


def cost_rows(spec: SynthSpec, row0: int, rows: int, out: np.ndarray | None = None) -> np.ndarray:
    """int32 costs of demands [row0, row0 + rows) x all k centers."""
    dx_, dy_ = coords(spec, 1, 2, row0, rows)
    cx, cy = coords(spec, 3, 4, 0, spec.k)
    dx = dx_[:, None] - cx[None, :]
    dy = dy_[:, None] - cy[None, :]
    q = (dx * dx + dy * dy).astype(np.float64)
    c = np.floor(np.sqrt(q) / 10.0 + 0.5)
    np.maximum(c, 1.0, out=c)
    if out is None:
        return c.astype(np.int32)
    out[...] = c
    return out


def costs(spec: SynthSpec, out: np.ndarray | None = None, threads: int | None = None,
          chunk: int = 8192) -> np.ndarray:
    """The full n x k int32 matrix, generated in row chunks on `threads`
    host threads (numpy releases the GIL). `out` may be a pinned buffer."""
    if out is None:
        out = np.empty((spec.n, spec.k), np.int32)
    threads = threads or min(16, os.cpu_count() or 1)
    starts = range(0, spec.n, chunk)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda r0: cost_rows(spec, r0, min(chunk, spec.n - r0),
                                         out[r0:r0 + min(chunk, spec.n - r0)]), starts))
    return out


def centers(spec: SynthSpec):
    """(capacity int64[k], family int32[k], offset int64[k+1], params int64[])."""
    k = spec.k
    total = spec.n * spec.theta_num // spec.theta_den
    w = [1 + stream_int(spec.seed, 5, s) % spec.cap_spread for s in range(k)]
    W = sum(w)
    cap = [total * ws // W for ws in w]
    rem = total - sum(cap)
    for s in range(rem):
        cap[s] += 1
    fam, off, par = [], [0], []
    span = spec.pen_hi - spec.pen_lo + 1
    for s in range(k):
        p = stream_int(spec.seed, 6, s)
        f = p % 3 if spec.mixed else 0
        base = spec.pen_lo + (p >> 8) % span
        fam.append(f)
        if f == 0:
            par.append(base)
        elif f == 1:
            par += [base, (p >> 24) % 6]
        else:
            v = base
            par.append(v)
            for t in range(1, 4):
                v += (p >> (32 + 3 * t)) % 8
                par.append(v)
        off.append(len(par))
    return (np.array(cap, np.int64), np.array(fam, np.int32), np.array(off, np.int64),
            np.array(par, np.int64))


def problem(spec: SynthSpec, cost_matrix: np.ndarray | None = None):
    """A paper_2304_06543_b200.instance.ProblemInstance (host mirror type)."""
    from paper_2304_06543_b200.instance import ProblemInstance  # pure-Python types, no .so
    cap, fam, off, par = centers(spec)
    params = [list(par[off[i]:off[i + 1]]) for i in range(spec.k)]
    cm = costs(spec) if cost_matrix is None else cost_matrix
    return ProblemInstance.from_arrays(cm, cap, fam, params)


def instance_sha256(cost_matrix: np.ndarray, spec: SynthSpec) -> str:
    """sha256 over the cost bytes (row-major int32) and the center arrays."""
    h = hashlib.sha256()
    mv = memoryview(np.ascontiguousarray(cost_matrix)).cast("B")
    step = 1 << 28
    for i in range(0, len(mv), step):
        h.update(mv[i:i + step])
    for a in centers(spec):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def assignment_sha256(assignment) -> str:
    return hashlib.sha256(np.ascontiguousarray(assignment, dtype=np.int32).tobytes()).hexdigest()
