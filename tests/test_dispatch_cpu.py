"""Integer data-plane tables (libmb_planner.so mbp_dispatch_plan, used to drive K2/K3) against the
independent CPU oracle (oracle/moe_ref.py): receive layout, route table, executed flow and the
canonical permutation, bit-exact, on random placements with replicas and round_split counts."""

import numpy as np
import pytest
import torch

import paper_2605_08639_b200 as mb
from oracle import moe_ref
from paper_2605_08639_b200.moe_layer import LayerShape, build_step_plan
from paper_2605_08639_b200.workload import SHAPES, make_routing


def _route_perm(plan_mb, j, idx, E):
    """Apply the route table exactly as the K2 kernel does (host emulation)."""
    rt = plan_mb.route_tab[j]
    nc = plan_mb.ncopies
    seen = {}
    out = np.zeros(idx.shape + (2,), dtype=np.int32)
    for t in range(idx.shape[0]):
        for i in range(idx.shape[1]):
            e = int(idx[t, i])
            r = seen.get(e, 0)
            seen[e] = r + 1
            c, prev = 0, 0
            while c + 1 < nc[e] and r >= rt[e, c, 0]:
                prev = rt[e, c, 0]
                c += 1
            out[t, i] = (rt[e, c, 1], rt[e, c, 2] + r - prev)
    return out


@pytest.mark.parametrize("name,world,policy,zipf", [
    ("tiny", 2, "relibra", 1.5), ("tiny", 2, "eplb_like", 1.0), ("qwen3-30b-a3b", 4, "relibra", 1.2),
    ("qwen3-30b-a3b", 8, "relibra", 1.5), ("qwen3-30b-a3b", 8, "eplb_like", 2.0), ("qwen3-30b-a3b", 8, "static", 1.0),
])
def test_dispatch_tables_match_oracle(name, world, policy, zipf):
    cfg = SHAPES[name]
    shape = cfg["shape"]
    T = 256
    topo = mb.b200_box_topology(world, min(world, cfg["group"]), mb.b200_profile(shape.hidden))
    model = mb.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    r = make_routing(shape, T, 2, world, 0, zipf_s=zipf, shift=cfg["shift"])
    cfgs = mb.SimConfigs(anneal=mb.AnnealConfig(seeds=(0, 1)), replica=mb.ReplicaConfig(cfg["slots"]))
    plan = build_step_plan(policy, r.mats, topo, model, topo.profile, cfgs, shape)
    for m, mbp in enumerate(plan.mbs):
        reps, counts = mbp.placement.replicas, mbp.counts
        # integer counts conserve every (source, expert) routing entry
        for e, c in counts.items():
            assert np.array_equal(c.sum(axis=1), r.mats[m][:, e])
        slots, row_base = moe_ref.receive_layout(r.mats[m], plan.home, reps, counts, pad=128)
        for d in range(world):
            n = int(mbp.nslots[d])
            assert n == len(slots[d])
            got = mbp.slot_tab[d][:n]
            want = np.array([[b, real, padded, e] for e, c, b, real, padded in slots[d]], dtype=np.int32).reshape(-1, 4)
            assert np.array_equal(got, want)
        assert np.array_equal(mbp.flow, moe_ref.executed_flow(r.mats[m], plan.home, reps, counts))
        # pin the oracle's executed flow to the reference's flow_matrix semantics (costmodel.py:91-108):
        # the planner-level flow_matrix (bit-exact with the reference, tests/test_planners_golden.py)
        # with the split fractions count / x gives the same integer flow
        x = r.mats[m].astype(np.float64)
        splits = {}
        for e, c in counts.items():
            col = x[:, e][:, None]
            frac = np.divide(c, col, out=np.zeros(c.shape), where=col > 0)
            frac[x[:, e] == 0, 0] = 1.0
            splits[e] = (np.array(mbp.placement.copies(e)), frac)
        ref_flow = mb.flow_matrix(x, plan.home, topo, splits)
        assert np.array_equal(np.rint(ref_flow).astype(np.int64), mbp.flow)
        assert np.abs(ref_flow - mbp.flow).max() < 1e-6
        # executed GEMM rows per GPU equal the reference cost model's comp loads (integer splits)
        assert np.array_equal(mbp.flow.sum(axis=0), plan.executed_loads()[m])
        # canonical permutation from the route table (the kernel's rule) == oracle definition
        idx0 = make_routing(shape, T, 2, world, 0, zipf_s=zipf, shift=cfg["shift"]).idx[m]
        ref = moe_ref.canonical_permutation(idx0, 0, r.mats[m], plan.home, reps, counts, row_base)
        assert np.array_equal(_route_perm(mbp, 0, idx0, shape.num_experts), ref)
        assert np.array_equal(moe_ref.canonical_permutation_fast(idx0, 0, r.mats[m], plan.home, reps, counts, row_base),
                              ref)


def test_relibra_reduces_skew_at_ep8():
    cfg = SHAPES["qwen3-30b-a3b"]
    shape = cfg["shape"]
    topo = mb.b200_box_topology(8, 4, mb.b200_profile(shape.hidden))
    model = mb.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    r = make_routing(shape, 2048, 2, 8, 0, zipf_s=1.5, shift=cfg["shift"])
    cfgs = mb.SimConfigs(anneal=mb.AnnealConfig(seeds=(0, 1, 2, 3)), replica=mb.ReplicaConfig(2))
    skew = {p: build_step_plan(p, r.mats, topo, model, topo.profile, cfgs, shape).skew()
            for p in ("static", "eplb_like", "relibra")}
    assert skew["relibra"] < skew["eplb_like"] < skew["static"]
    assert skew["relibra"] < 1.3


def test_oracle_layer_math_matches_autograd():
    """The fp32 oracle's hand-written backward equals torch autograd of the same forward."""
    torch.manual_seed(0)
    E, k, h, hp, T = 4, 2, 16, 8, 32
    x = torch.randn(T, h, dtype=torch.float64)
    idx = torch.stack([torch.randperm(E)[:k] for _ in range(T)])
    gates = torch.rand(T, k, dtype=torch.float64)
    wg, wu = torch.randn(E, hp, h, dtype=torch.float64), torch.randn(E, hp, h, dtype=torch.float64)
    wd = torch.randn(E, h, hp, dtype=torch.float64)
    dout = torch.randn(T, h, dtype=torch.float64)
    ref = moe_ref.moe_layer_fp32(x, idx, gates, wg, wu, wd, dout)
    xs, gs = x.clone().requires_grad_(), gates.clone().requires_grad_()
    ws = [w.clone().requires_grad_() for w in (wg, wu, wd)]
    out = torch.zeros_like(xs)
    for t in range(T):
        for i in range(k):
            e = int(idx[t, i])
            hg, hu = ws[0][e] @ xs[t], ws[1][e] @ xs[t]
            out = out.index_add(0, torch.tensor([t]), (gs[t, i] * (ws[2][e] @ (torch.nn.functional.silu(hg) * hu)))[None])
    out.backward(dout)
    assert torch.allclose(ref["out"].double(), out.detach(), rtol=1e-4, atol=1e-4)
    assert torch.allclose(ref["dx"].double(), xs.grad, rtol=1e-4, atol=1e-4)
    assert torch.allclose(ref["dgate"].double(), gs.grad, rtol=1e-4, atol=1e-4)
    for a, b in zip((ref["dWg"], ref["dWu"], ref["dWd"]), ws):
        assert torch.allclose(a.double(), b.grad, rtol=1e-4, atol=1e-4)


def test_histogram_oracle_and_trace():
    shape = LayerShape(16, 4, 256, 256)
    r = make_routing(shape, 512, 3, 2, 1, zipf_s=1.0, shift=3)
    for m in range(3):
        assert np.array_equal(moe_ref.histogram(r.idx[m], 16), r.mats[m, 1])
        assert (r.mats[m].sum(axis=1) == 512 * 4).all()
        # distinct experts per token (top-k without replacement): x[j, e] <= T
        assert (r.mats[m] <= 512).all()
    tr = mb.build_trace(mb.ModelProfile(1, 16, 4), mb.build_topology(1, 2, mb.HardwareProfile(1, 1, 1, 1)),
                        r.mats[:, None], tokens_per_gpu=512)
    assert np.array_equal(mb.aggregate_batch(tr, 0), r.mats.sum(axis=0))
    assert len(tr.trace_id()) == 16
