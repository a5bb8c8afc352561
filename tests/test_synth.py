"""The host generator (synth_instances.py, spec lbdd-synth-v2): the
vectorised numpy path against a scalar restatement of the spec, and the
properties the BASELINE configs state."""
import math

import numpy as np

import synth_instances as SI


def scalar_cost(spec, d, s):
    dx = SI.stream_int(spec.seed, 1, d) % SI.GRID - SI.stream_int(spec.seed, 3, s) % SI.GRID
    dy = SI.stream_int(spec.seed, 2, d) % SI.GRID - SI.stream_int(spec.seed, 4, s) % SI.GRID
    return max(1, math.floor(math.sqrt(dx * dx + dy * dy) / 10.0 + 0.5))


def test_numpy_matches_scalar_spec():
    spec = SI.SynthSpec(5000, 37, seed=3)
    m = SI.costs(spec, threads=3, chunk=777)
    rng = np.random.default_rng(0)
    for d, s in zip(rng.integers(0, spec.n, 300), rng.integers(0, spec.k, 300)):
        assert m[d, s] == scalar_cost(spec, int(d), int(s))
    assert m.min() >= 1 and m.max() <= 1414


def test_rows_independent_of_n_and_chunking():
    a = SI.costs(SI.SynthSpec(3000, 50, seed=9), threads=1, chunk=3000)
    b = SI.cost_rows(SI.SynthSpec(100000, 50, seed=9), 1000, 2000)
    assert np.array_equal(a[1000:3000], b)


def test_centers_match_config_statements():
    cap, fam, off, par = SI.centers(SI.CONFIG1)
    assert cap.sum() == SI.CONFIG1.n * 8 // 10          # total capacity 80% of demand
    assert len(set(cap.tolist())) > 10                  # heterogeneous capacities
    assert set(fam.tolist()) == {0, 1, 2}               # mixed penalty families
    assert off[-1] == len(par) and (par >= 0).all()
    cap2, _, _, _ = SI.centers(SI.SynthSpec(4000, 20, theta_num=1, theta_den=1))
    assert cap2.sum() == 4000                           # configs[2]: capacity = demand
    cap0, fam0, _, _ = SI.centers(SI.CONFIG0)
    assert cap0.sum() == 8000 and set(fam0.tolist()) == {0}


def test_instance_hash_is_stable():
    spec = SI.SynthSpec(200, 10, seed=1)
    h1 = SI.instance_sha256(SI.costs(spec), spec)
    h2 = SI.instance_sha256(SI.costs(spec, threads=2, chunk=7), spec)
    assert h1 == h2
