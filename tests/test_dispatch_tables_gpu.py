"""On-device dispatch tables (mb_dispatch_tables: round_split + receive layout + route table +
executed flow) against the host planner library (mbp_round_split + mbp_dispatch_plan) and the
oracle's executed flow: bit-identical, on synthetic ReLibra / EPLB plans and on plan files the
reference's own `solve` wrote (its LP fractions, tests/golden/io)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import moe_ref
from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs, planio
from paper_2605_08639_b200 import traces as rt
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile
from paper_2605_08639_b200.moe_layer import LayerShape, build_step_plan, step_plan_from_bundle
from paper_2605_08639_b200.workload import SHAPES, make_routing

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden" / "io"
FIELDS = ("route_tab", "ncopies", "slot_tab", "slot_w", "nslots", "total_rows", "flow")


def _same(host, dev):
    assert host.maxc == dev.maxc and host.max_slots == dev.max_slots and host.rows_cap == dev.rows_cap
    assert dev.tables == "device"
    for m, (a, b) in enumerate(zip(host.mbs, dev.mbs)):
        for f in FIELDS:
            assert np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(b, f))), (m, f)
        assert sorted(a.counts) == sorted(b.counts)
        for e in a.counts:
            assert np.array_equal(a.counts[e], b.counts[e]), (m, e)
        x = host.mats[m]
        assert np.array_equal(b.flow, moe_ref.executed_flow(x, host.home, b.placement.replicas, b.counts))


@pytest.mark.parametrize("name,world,group,zipf,policy", [
    ("tiny", 2, 2, 1.5, "relibra"), ("tiny", 4, 4, 2.0, "relibra"), ("qwen3-30b-a3b", 4, 4, 1.5, "relibra"),
    ("qwen3-30b-a3b", 8, 4, 1.0, "relibra"), ("qwen3-30b-a3b", 8, 8, 2.0, "relibra"),
    ("qwen3-30b-a3b", 8, 4, 1.5, "eplb_like"), ("mixtral-8x7b", 8, 4, 1.5, "relibra")])
def test_device_tables_match_host(name, world, group, zipf, policy):
    cfg = SHAPES[name]
    shape = cfg["shape"]
    r = make_routing(shape, 1024, 3, world, 0, zipf_s=zipf, shift=cfg["shift"])
    topo = b200_box_topology(world, group, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=(0, 1, 2)), replica=ReplicaConfig(cfg["slots"]))
    host = build_step_plan(policy, r.mats, topo, model, topo.profile, cfgs, shape, device_tables=False)
    dev = build_step_plan(policy, r.mats, topo, model, topo.profile, cfgs, shape, device_tables=True)
    _same(host, dev)


@pytest.mark.parametrize("case", ["qwen3_ep4", "qwen3_ep8", "small", "samples"])
def test_device_tables_on_reference_plan_files(case):
    """Fractions from the reference's own token-split LP (its replication.json): the device
    round_split and layout equal the host's for every (micro-batch, layer)."""
    trace = rt.load_trace(GOLD / case / "trace")
    bundle = planio.load_plan_bundle(GOLD / case / "plans", trace)
    tm = trace.model
    shape = LayerShape(tm.num_experts, tm.top_k, max(256, tm.hidden_size), max(256, tm.intermediate_size))
    mats_all = trace.matrices.astype(np.int64)
    for layer in range(min(2, tm.num_layers)):
        mats = mats_all[:, layer]
        host = step_plan_from_bundle("relibra", bundle, mats, shape, layer=layer, device_tables=False)
        dev = step_plan_from_bundle("relibra", bundle, mats, shape, layer=layer, device_tables=True)
        _same(host, dev)
