"""Full-size checks through size-independent properties (the oracle cannot
run these sizes in seconds)."""
import numpy as np
import pytest

import synth_instances as SI

import pyoracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big(dev):
    # configs[1] shape: |D| = 1M x |S| = 1000 int32, heterogeneous capacities
    inst = dev.DeviceInstance.generate(1_000_000, 1000, seed=11)
    yield inst
    inst.close()


def test_arrival_queue_sorted_and_minimal(dev, big):
    bc, cost, order = dev.arrival_queue(big)
    keys = cost[order] * (1 << 32) + order
    assert (np.diff(keys) > 0).all()                      # ascending (cost, demand)
    assert np.array_equal(np.sort(order), np.arange(big.n))
    rows = big.costs(0, 2000)                             # spot-check row minima
    assert (rows.min(axis=1) == cost[:2000]).all()
    assert (rows.argmin(axis=1) == bc[:2000]).all()       # first minimum = smallest id


def test_sharded_partials_min_combine_to_full_build(dev, big):
    bc, _, _ = dev.arrival_queue(big)
    full = dev.build_index(big, bc)
    parts = [dev.build_index(big, bc, row0=r0, rows=rows)
             for r0, rows in [(0, 333_333), (333_333, 333_333), (666_666, 333_334)]]
    assert (np.minimum.reduce(parts) == full).all()
    # spot-check one row against a direct host recount over its bucket
    counts = np.bincount(bc, minlength=big.k)
    u = int(np.argmin(np.where(counts > 0, counts, counts.max() + 1)))
    members = np.nonzero(bc == u)[0]
    rows = np.stack([big.costs(int(d), 1)[0] for d in members]).astype(np.int64)
    packed = ((rows - rows[:, [u]]) << 32) | members[:, None]
    expect = packed.min(axis=0)
    expect[u] = po.NO_EDGE
    assert (expect == full[u]).all()


def test_greedy_full_size_recount(dev, big):
    g = dev.greedy_solve(big)
    bc, cost, _ = dev.arrival_queue(big)
    assert (g.assignment == bc).all()
    assert g.objective >= int(cost.sum())


def test_asral_medium_properties(dev):
    inst = dev.DeviceInstance.generate(20_000, 500, seed=5, theta_num=7, theta_den=10)
    a = dev.asral_solve(inst)          # the engine recounts the objective itself
    g = dev.greedy_solve(inst)
    assert a.objective <= g.objective  # acceptance.cpp:182 dominance
    assert np.bincount(a.assignment, minlength=inst.k).tolist() == a.load.tolist()
    assert not dev.gamma_has_negative_cycle(inst, a.assignment)  # Lemma invariant
    assert dev.evaluate_objective(inst, a.assignment) == a.objective


def test_device_generator_matches_host_spec(dev, big):
    """lbdd_b200_instance_generate == synth_instances.py (spec lbdd-synth-v2)
    bit for bit: sampled row blocks and the center arrays."""
    spec = SI.SynthSpec(1_000_000, 1000, seed=11)
    for r0 in (0, 123_457, 999_000):
        assert np.array_equal(big.costs(r0, 1000), SI.cost_rows(spec, r0, 1000))
    cap, fam, off, par = big.centers()
    hc, hf, ho, hp = SI.centers(spec)
    assert np.array_equal(cap, hc) and np.array_equal(fam, hf)
    assert np.array_equal(off, ho) and np.array_equal(par[:len(hp)], hp)
