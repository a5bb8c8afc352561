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


# ---------------------------------------------------------------------------
# configs[3]: road-network-like distances ("lbdd-road-v1")
# ---------------------------------------------------------------------------
#
# A road graph of V vertices: uniform random points in the unit square
# (numpy PCG64 seeded with `seed`), each joined to its 6 nearest neighbours,
# edge length = euclidean x a winding factor in [1, 1.5); components joined
# to the largest by their nearest pair. Centers sit on k distinct vertices;
# demand d sits on vertex stream(seed, 13, d) % V with an access length
# (stream(seed, 14, d) >> 11) * 2^-53 * 0.01. The float32 cost is the
# shortest-path length (scipy Dijkstra from every center) plus the access
# length; the solver's integer cost is max(1, rint(1000 * float32 cost)),
# the integerisation of the reference's own road-graph generator
# (instgen.hpp:87-90, scaled_cost) -- the reference's Cost is int64
# (core.hpp:16), so float costs reach it only integerised.
# Capacities: theta = 9/10, weights 1 + (h % 1000)^2 // 1000 (heavily skewed).

@dataclass(frozen=True)
class RoadSpec:
    n: int
    k: int
    seed: int = 20250
    vertices: int = 16384
    theta_num: int = 9
    theta_den: int = 10
    pen_lo: int = 1
    pen_hi: int = 200

    def name(self) -> str:
        return (f"lbdd-road-v1(n={self.n},k={self.k},seed={self.seed},V={self.vertices},"
                f"theta={self.theta_num}/{self.theta_den},pen=[{self.pen_lo},{self.pen_hi}])")


CONFIG3 = RoadSpec(2_000_000, 1000)
_ROAD_CACHE = {}


def road_distances(spec: RoadSpec) -> np.ndarray:
    """(V, k) float32 shortest-path lengths from every center vertex."""
    key = (spec.seed, spec.vertices, spec.k)
    if key in _ROAD_CACHE:
        return _ROAD_CACHE[key]
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components, dijkstra
    from scipy.spatial import cKDTree
    V = spec.vertices
    rng = np.random.default_rng(spec.seed)
    pts = rng.random((V, 2))
    tree = cKDTree(pts)
    dd, idx = tree.query(pts, k=7)
    rows = np.repeat(np.arange(V), 6)
    cols = idx[:, 1:].reshape(-1)
    w = dd[:, 1:].reshape(-1) * (1.0 + 0.5 * rng.random(V * 6))
    g = csr_matrix((w, (rows, cols)), shape=(V, V))
    g = g.maximum(g.T).tolil()
    ncomp, lab = connected_components(g, directed=False)
    if ncomp > 1:
        big = np.bincount(lab).argmax()
        main = np.nonzero(lab == big)[0]
        mtree = cKDTree(pts[main])
        for c in range(ncomp):
            if c == big:
                continue
            mem = np.nonzero(lab == c)[0]
            dist, j = mtree.query(pts[mem])
            i = int(np.argmin(dist))
            a, b = int(mem[i]), int(main[j[i]])
            g[a, b] = g[b, a] = float(dist[i]) * 1.25
    g = g.tocsr()
    centers = rng.choice(V, spec.k, replace=False)
    D = dijkstra(g, indices=centers).T.astype(np.float32)
    _ROAD_CACHE[key] = D
    return D


def road_float_rows(spec: RoadSpec, row0: int, rows: int) -> np.ndarray:
    D = road_distances(spec)
    v = (stream_np(spec.seed, 13, row0, rows) % np.uint64(spec.vertices)).astype(np.int64)
    acc = ((stream_np(spec.seed, 14, row0, rows) >> np.uint64(11)).astype(np.float64)
           * 2.0 ** -53 * 0.01).astype(np.float32)
    return D[v] + acc[:, None]


def road_cost_rows(spec: RoadSpec, row0: int, rows: int, out: np.ndarray | None = None):
    c = np.rint(road_float_rows(spec, row0, rows).astype(np.float64) * 1000.0)
    np.maximum(c, 1.0, out=c)
    if out is None:
        return c.astype(np.int32)
    out[...] = c
    return out


def road_costs(spec: RoadSpec, out: np.ndarray | None = None, chunk: int = 16384,
               threads: int | None = None) -> np.ndarray:
    if out is None:
        out = np.empty((spec.n, spec.k), np.int32)
    road_distances(spec)  # build once, outside the threads
    threads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda r0: road_cost_rows(spec, r0, min(chunk, spec.n - r0),
                                              out[r0:r0 + min(chunk, spec.n - r0)]),
                    range(0, spec.n, chunk)))
    return out


def road_centers(spec: RoadSpec):
    k = spec.k
    total = spec.n * spec.theta_num // spec.theta_den
    w = [1 + (stream_int(spec.seed, 15, s) % 1000) ** 2 // 1000 for s in range(k)]
    W = sum(w)
    cap = [total * ws // W for ws in w]
    for s in range(total - sum(cap)):
        cap[s] += 1
    span = spec.pen_hi - spec.pen_lo + 1
    fam, off, par = [], [0], []
    for s in range(k):
        p = stream_int(spec.seed, 16, s)
        f = p % 3
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


def road_problem(spec: RoadSpec):
    from paper_2304_06543_b200.instance import ProblemInstance
    cap, fam, off, par = road_centers(spec)
    params = [list(par[off[i]:off[i + 1]]) for i in range(spec.k)]
    return ProblemInstance.from_arrays(road_costs(spec), cap, fam, params)
