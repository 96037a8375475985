"""Host planners (libmb_planner.so behind the moebalance-shaped API) against golden vectors
produced by the reference itself (tests/golden/planners.json, oracle/gen_golden.py).

Everything is compared EXACTLY: integer plans, replica lists in insertion order, and float64
fractions / loads bit for bit (floats are stored as float.hex()).
"""

import json
import os

import numpy as np
import pytest

import paper_2605_08639_b200 as mb
from paper_2605_08639_b200 import _native
from paper_2605_08639_b200.policies import _eplb_replication, _uniform_matrices

GOLD = os.path.join(os.path.dirname(__file__), "golden", "planners.json")


@pytest.fixture(scope="module")
def cases():
    with open(GOLD) as f:
        return json.load(f)["cases"]


def unhex(v, shape=None):
    a = np.array([float.fromhex(s) for s in v], dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def hw_of(t):
    return mb.HardwareProfile(*[float.fromhex(s) for s in t])


def test_numpy_blas_bridge_active():
    # greedy/LP bit-exactness relies on issuing numpy's own BLAS calls
    assert _native.planner().mbp_numpy_blas_active() == 1


def test_kat_twelve_vs_four(cases):
    c = cases["kat_twelve_vs_four"]
    hw = mb.HardwareProfile(6.0, 1e18, 1e18, 1.0)
    topo = mb.build_topology(1, 2, hw)
    model = mb.ModelProfile(1, 2, 1, hidden_size=1, intermediate_size=1)
    x = np.array(c["x"])
    p, s = mb.greedy_replicate(x, mb.ReorderPlan(np.array([0, 1])), topo, model, hw, mb.ReplicaConfig(1))
    assert p.replicas == {0: [1]} == {int(k): v for k, v in c["replicas"].items()}
    assert np.array_equal(s.fractions[0], unhex(c["frac0"], (2, 2)))
    comp = mb.compute_loads(x, np.array([0, 1]), topo, s.to_split_map(p)).comp
    assert np.array_equal(comp, unhex(c["comp"]))
    np.testing.assert_allclose(comp, [8.0, 8.0], atol=1e-9)   # reference test_replicate.py:118-124


def test_kat_round_split(cases):
    pl = mb.ReplicaPlacement(home=np.array([0, 1]), replicas={0: [1]})
    x = np.array([[10.0, 0.0], [0.0, 4.0]])
    for c in cases["kat_round_split"]:
        got = mb.round_split(mb.SplitPlan({0: np.array(c["frac"])}), pl, x)[0]
        assert got.tolist() == c["counts"]
    assert [c["counts"][0] for c in cases["kat_round_split"]] == [[10, 0], [5, 5], [7, 3]]


def test_kat_topology_and_lpt(cases):
    t = mb.build_topology(2, 2, mb.HardwareProfile(1.0, 1.0, 1.0, 1.0))
    assert t.class_matrix.tolist() == cases["kat_relay"]["cls"]
    assert t.relay_matrix.tolist() == cases["kat_relay"]["relay"]
    c = cases["kat_lpt"]
    unit = mb.HardwareProfile(6.0, 1e18, 1e18, 1.0)
    assert mb.lpt_initial(np.array(c["x"]), mb.build_topology(1, 2, unit)).assignment.tolist() == c["assignment"]
    assert mb.skewness(cases["kat_skew"]["loads"]) == cases["kat_skew"]["skew"] == 1.5


def test_compute_loads_bit_exact(cases):
    for c in cases["compute_loads"]:
        topo = mb.build_topology(c["nodes"], c["gpn"], mb.HardwareProfile(1.0, 1.0, 1.0, 1.0))
        x = np.array(c["x"])
        splits = {ex: (np.array(gp), unhex(fr, (x.shape[0], len(gp)))) for ex, gp, fr in c["splits"]}
        lv = mb.compute_loads(x, np.array(c["home"]), topo, splits)
        for f, v in c["loads"].items():
            assert np.array_equal(getattr(lv, f), unhex(v)), f


def test_lpt_static_eplb_exact(cases):
    unit = mb.HardwareProfile(6.0, 1e18, 1e18, 1.0)
    for c in cases["lpt_static_eplb"]:
        topo = mb.build_topology(c["nodes"], c["gpn"], unit)
        x = np.array(c["x"])
        plan = mb.lpt_initial(x, topo)
        assert plan.assignment.tolist() == c["lpt"]
        assert mb.static_plan(x.shape[1], topo).assignment.tolist() == c["static"]
        ep = _eplb_replication(x.astype(np.float64).sum(axis=0), plan.assignment, topo, 2)
        assert [[k, v] for k, v in ep.replicas.items()] == c["eplb"]


def test_uniform_matrices(cases):
    c = cases["uniform"]
    mats = np.array(c["mats"], dtype=np.uint32)
    tr = mb.RoutingTrace(model=mb.ModelProfile(1, 16, 2), topo=mb.build_topology(1, 4, mb.HardwareProfile(1, 1, 1, 1)),
                         matrices=mats, tokens_per_gpu=0)
    assert _uniform_matrices(tr).tolist() == c["out"]


def test_anneal_small_exact(cases):
    for c in cases["anneal_small"]:
        hw = hw_of(c["hw"])
        topo = mb.build_topology(c["nodes"], c["gpn"], hw)
        x = np.array(c["x"])
        model = mb.ModelProfile(1, x.shape[1], 1, hidden_size=1, intermediate_size=1)
        cfg = mb.AnnealConfig(seeds=tuple(c["seeds"]), cooling_rate=c["cooling"])
        plan = mb.anneal_reorder(x, topo, model, hw, cfg, extra_initial_plans=[mb.static_plan(x.shape[1], topo)])
        assert plan.assignment.tolist() == c["assignment"]


def test_anneal_qwen3_default_config_exact(cases):
    """Production shape (E=128, 2 groups x 4, 16 chains, cooling 0.9995): same plan as the reference."""
    for c in cases["anneal_qwen3"]:
        hw = hw_of(c["hw"])
        topo = mb.build_topology(c["nodes"], c["gpn"], hw)
        x = np.array(c["x"])
        model = mb.ModelProfile(1, x.shape[1], 8, hidden_size=c["h"], intermediate_size=c["hp"])
        plan = mb.anneal_reorder(x, topo, model, hw, mb.AnnealConfig(),
                                 extra_initial_plans=[mb.static_plan(x.shape[1], topo)])
        assert plan.assignment.tolist() == c["assignment"]


def _check_greedy(c, model):
    hw = hw_of(c["hw"])
    topo = mb.build_topology(c["nodes"], c["gpn"], hw)
    x = np.array(c["x"])
    p, s = mb.greedy_replicate(x, mb.ReorderPlan(np.array(c["home"])), topo, model, hw, mb.ReplicaConfig(c["slots"]))
    assert [[k, v] for k, v in p.replicas.items()] == c["replicas"]
    assert [k for k in s.fractions] == [k for k, _, _ in c["fractions"]]
    for k, shape, v in c["fractions"]:
        assert np.array_equal(s.fractions[k], unhex(v, shape)), k
    counts = mb.round_split(s, p, x)
    assert [[k, v.tolist()] for k, v in counts.items()] == c["counts"]


def test_greedy_replicate_small_exact(cases):
    for c in cases["greedy_small"]:
        x = np.array(c["x"])
        _check_greedy(c, mb.ModelProfile(1, x.shape[1], 1, hidden_size=1, intermediate_size=1))


def test_greedy_replicate_qwen3_exact(cases):
    for c in cases["greedy_qwen3"]:
        x = np.array(c["x"])
        _check_greedy(c, mb.ModelProfile(1, x.shape[1], 8, hidden_size=c["h"], intermediate_size=c["hp"]))


def test_error_behaviour():
    hw = mb.HardwareProfile(6.0, 1e18, 1e18, 1.0)
    topo = mb.build_topology(1, 2, hw)
    model = mb.ModelProfile(1, 2, 1, hidden_size=1, intermediate_size=1)
    with pytest.raises(ValueError):
        mb.solve_token_split_lp(np.array([[12.0, 0.0], [0.0, 4.0]]),
                                mb.ReplicaPlacement(home=np.array([0, 1]), replicas={0: [0]}), topo, model, hw)
    with pytest.raises(ValueError):
        mb.static_plan(3, topo)
    with pytest.raises(ValueError):
        mb.HardwareProfile(0.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        mb.replica_memory(model, mb.ReplicaConfig(1), "global")
    assert mb.replica_memory(mb.ModelProfile(48, 8, 1, expert_param_bytes=1000), mb.ReplicaConfig(2),
                             "layer-shared") == 2000
