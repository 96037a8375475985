"""End-to-end MoE-layer step on one B200 (world = 1) against the CPU oracle.

Integer outputs (device histogram, canonical permutation) must be bit-exact; layer outputs
and gradients must be within the documented bf16 tolerance rel 2e-2 of the fp32 oracle.
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import moe_ref
from paper_2605_08639_b200 import ModelProfile, SimConfigs, ReplicaConfig, build_topology
from paper_2605_08639_b200.cluster import b200_profile
from paper_2605_08639_b200.comm import Comm
from paper_2605_08639_b200.moe_layer import MoEDataPlane, build_step_plan, deinterleave_w1
from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _assert_close(got, ref, what=""):
    c = moe_ref.close(got, ref)
    assert c["ok"], f"{what}: {c}"


def _run(name, T, MB, zipf_s=1.0, balanced=False, **dp_kw):
    cfg = SHAPES[name]
    shape = cfg["shape"]
    routing = make_routing(shape, T, MB, 1, 0, zipf_s=zipf_s, shift=cfg["shift"], balanced=balanced)
    topo = build_topology(1, 1, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    plan = build_step_plan("static", routing.mats, topo, model, topo.profile, SimConfigs(replica=ReplicaConfig(0)),
                           shape)
    dp = MoEDataPlane(Comm(), shape, T, MB, plan, **dp_kw)
    wg, wu, wd = make_weights(shape)
    dp.set_weights(wg.cuda(), wu.cuda(), wd.cuda())
    dp.zero_grads()
    x, dout = make_activations(shape, T, MB, 0)
    x, dout = x.cuda(), dout.cuda()
    idx = torch.from_numpy(routing.idx).cuda()
    gates = torch.from_numpy(routing.gates).cuda()
    out = torch.empty_like(x)
    dx = torch.empty_like(x)
    dgate = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    dp.step(x, idx, gates, dout, out, dx, dgate)
    dp.check(sync=True)
    return shape, routing, plan, dp, (wg, wu, wd), (x, dout, idx, gates), (out, dx, dgate)


@pytest.mark.parametrize("name,T,MB,mode", [("tiny", 256, 2, "step"), ("qwen3-30b-a3b", 512, 2, "step"),
                                            ("mixtral-8x7b", 256, 1, "step"), ("qwen3-235b-a22b", 256, 1, "step"),
                                            ("qwen3-30b-a3b", 512, 5, "micro_batch"), ("tiny", 256, 4, "micro_batch")])
def test_layer_step_matches_oracle(name, T, MB, mode):
    shape, routing, plan, dp, (wg, wu, wd), (x, dout, idx, gates), (out, dx, dgate) = _run(name, T, MB,
                                                                                            wgrad_mode=mode)
    E = shape.num_experts
    home = plan.home
    gwg = torch.zeros(E, shape.ffn, shape.hidden, device="cuda")
    gwu = torch.zeros_like(gwg)
    gwd = torch.zeros(E, shape.hidden, shape.ffn, device="cuda")
    for m in range(MB):
        # K1: device histogram == np.bincount (bit-exact)
        assert np.array_equal(dp.counts[m].cpu().numpy(), moe_ref.histogram(routing.idx[m], E))
        # K2: device permutation == canonical permutation (bit-exact)
        _, row_base = moe_ref.receive_layout(routing.mats[m], home, {}, {}, pad=128)
        ref_perm = moe_ref.canonical_permutation_fast(routing.idx[m], 0, routing.mats[m], home, {}, {}, row_base)
        assert np.array_equal(dp.perm[m].cpu().numpy(), ref_perm)
        ref = moe_ref.moe_layer_fp32(x[m], idx[m], gates[m], wg.cuda(), wu.cuda(), wd.cuda(), dout[m])
        _assert_close(out[m], ref["out"], f"out mb{m}")
        _assert_close(dx[m], ref["dx"], f"dx mb{m}")
        _assert_close(dgate[m], ref["dgate"], f"dgate mb{m}")
        gwg += ref["dWg"]
        gwu += ref["dWu"]
        gwd += ref["dWd"]
    g_gate, g_up = deinterleave_w1(dp.gW1[:dp.M])
    for got, ref, what in ((g_gate, gwg, "dWg"), (g_up, gwu, "dWu"), (dp.gW2[:dp.M], gwd, "dWd")):
        c = moe_ref.expert_grads_close(got, ref)
        assert c["ok"], f"{what}: {c}"
    dp.close()


def test_balanced_routing_is_uniform():
    shape, routing, plan, dp, *_ = _run("tiny", 256, 1, balanced=True)
    counts = dp.counts[0].cpu().numpy()
    assert counts.max() - counts.min() <= 1
    dp.close()


def test_step_host_matches_device_step():
    """The user-facing host-buffer step (the e2e path) gives the same results as the device step."""
    shape, routing, plan, dp, (wg, wu, wd), (x, dout, idx, gates), (out, dx, dgate) = _run("qwen3-30b-a3b", 512, 3)
    g1, g2 = dp.gW1.clone(), dp.gW2.clone()
    dp.zero_grads()
    host = {"x": x.cpu().pin_memory(), "dout": dout.cpu().pin_memory(), "idx": idx.cpu().pin_memory(),
            "gates": gates.cpu().pin_memory(), "out": torch.empty_like(out, device="cpu").pin_memory(),
            "dx": torch.empty_like(dx, device="cpu").pin_memory(),
            "dgate": torch.empty_like(dgate, device="cpu").pin_memory()}
    dev = {k: torch.empty_like(v, device="cuda") for k, v in host.items()}
    dp.step_host(host, dev)
    assert torch.equal(host["out"], out.cpu())
    assert torch.equal(host["dx"], dx.cpu())
    assert torch.equal(host["dgate"], dgate.cpu())
    torch.cuda.synchronize()
    assert torch.equal(dp.gW1, g1) and torch.equal(dp.gW2, g2)
    dp.close()


def test_per_micro_batch_api_and_autograd_match_fused_step():
    """begin_step / forward_mb / backward_mb / end_step and the autograd Function run the same
    kernels as the fused schedule: identical out, dx, dgate and expert gradients."""
    from paper_2605_08639_b200.moe_layer import MoELayerFunction
    shape, routing, plan, dp, (wg, wu, wd), (x, dout, idx, gates), (out, dx, dgate) = _run("qwen3-30b-a3b", 512, 3)
    g1, g2 = dp.gW1[:dp.M].clone(), dp.gW2[:dp.M].clone()
    MB = x.shape[0]
    # explicit per-micro-batch calls
    dp.zero_grads()
    o2, dx2, dg2 = torch.empty_like(out), torch.empty_like(dx), torch.empty_like(dgate)
    dp.begin_step()
    for m in range(MB):
        dp.forward_mb(m, x[m], idx[m], gates[m], o2[m])
    for m in reversed(range(MB)):
        dp.backward_mb(m, dout[m], dx2[m], dg2[m])
    dp.end_step()
    torch.cuda.synchronize()
    assert torch.equal(o2, out) and torch.equal(dx2, dx) and torch.equal(dg2, dgate)
    assert torch.equal(dp.gW1[:dp.M], g1) and torch.equal(dp.gW2[:dp.M], g2)
    # autograd
    dp.zero_grads()
    xs = [x[m].clone().requires_grad_(True) for m in range(MB)]
    gs = [gates[m].clone().requires_grad_(True) for m in range(MB)]
    dp.begin_step()
    outs = [MoELayerFunction.apply(xs[m], gs[m], dp, idx[m], m) for m in range(MB)]
    torch.autograd.backward(outs, [dout[m] for m in range(MB)])
    dp.end_step()
    torch.cuda.synchronize()
    for m in range(MB):
        assert torch.equal(outs[m].detach(), out[m])
        assert torch.equal(xs[m].grad, dx[m]) and torch.equal(gs[m].grad, dgate[m])
    assert torch.equal(dp.gW1[:dp.M], g1) and torch.equal(dp.gW2[:dp.M], g2)
    dp.close()


def test_dropped_token_choices():
    """Choices with idx = -1 (capacity-dropped, or padding of a short micro-batch) are not
    counted, not dispatched and contribute nothing; the rest of the layer matches the oracle."""
    cfg = SHAPES["qwen3-30b-a3b"]
    shape = cfg["shape"]
    T, MB = 384, 1
    routing = make_routing(shape, T, MB, 1, 0, zipf_s=1.0, shift=cfg["shift"])
    rng = np.random.default_rng(3)
    drop = rng.random(routing.idx.shape) < 0.1
    drop[:, -32:, :] = True          # a fully dropped tail (padding tokens)
    routing.idx[drop] = -1
    routing.gates[drop] = 0.0
    routing.mats = np.stack([moe_ref.histogram(routing.idx[m], shape.num_experts) for m in range(MB)])[:, None]
    topo = build_topology(1, 1, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    # the planners' trace format needs row sums divisible by k: plan on the kept choices only
    plan = build_step_plan("static", routing.mats, topo, model, topo.profile, SimConfigs(replica=ReplicaConfig(0)),
                           shape) if routing.mats.sum() % shape.top_k == 0 else None
    if plan is None:
        keep = int(routing.mats.sum() % shape.top_k)
        flat = routing.idx.reshape(-1)
        nz = np.flatnonzero(flat >= 0)[-keep:]
        flat[nz] = -1
        routing.mats = np.stack([moe_ref.histogram(routing.idx[m], shape.num_experts) for m in range(MB)])[:, None]
        plan = build_step_plan("static", routing.mats, topo, model, topo.profile,
                               SimConfigs(replica=ReplicaConfig(0)), shape)
    dp = MoEDataPlane(Comm(), shape, T, MB, plan)
    wg, wu, wd = make_weights(shape)
    dp.set_weights(wg.cuda(), wu.cuda(), wd.cuda())
    dp.zero_grads()
    x, dout = make_activations(shape, T, MB, 0)
    x, dout = x.cuda(), dout.cuda()
    idx = torch.from_numpy(routing.idx).cuda()
    gates = torch.from_numpy(routing.gates).cuda()
    out, dx = torch.empty_like(x), torch.empty_like(x)
    dgate = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    dp.step(x, idx, gates, dout, out, dx, dgate)
    torch.cuda.synchronize()
    assert np.array_equal(dp.counts[0].cpu().numpy(), moe_ref.histogram(routing.idx[0], shape.num_experts))
    assert bool((dp.perm[0].cpu().numpy()[routing.idx[0] < 0] == -1).all())
    ref = moe_ref.moe_layer_fp32(x[0], idx[0], gates[0], wg.cuda(), wu.cuda(), wd.cuda(), dout[0])
    _assert_close(out[0], ref["out"], "out")
    _assert_close(dx[0], ref["dx"], "dx")
    _assert_close(dgate[0], ref["dgate"], "dgate")
    assert torch.all(out[0, -32:] == 0) and torch.all(dx[0, -32:] == 0)
    dp.check(sync=True)
    dp.close()


@pytest.mark.parametrize("name,T,MB", [("qwen3-30b-a3b", 512, 3), ("mixtral-8x7b", 256, 1), ("tiny", 256, 2)])
def test_tma_row_movers_bit_identical(name, T, MB):
    """The TMA bulk-copy row movers (mb_set_comm_blocks > 0: scatter, combine, dX un-permute with
    the dgate gather) give bit-identical step results to the register-copy kernels."""
    shape, routing, plan, dp, _, (x, dout, idx, gates), (out, dx, dgate) = _run(name, T, MB)
    g1, g2 = dp.gW1.clone(), dp.gW2.clone()
    assert dp.comm_blocks == 0           # world 1: register movers
    dp.comm_blocks = 12                  # per-plane engine: confined bulk-copy movers on 12 SMs
    dp.zero_grads()
    o2, dx2, dg2 = torch.empty_like(out), torch.empty_like(dx), torch.empty_like(dgate)
    dp.step(x, idx, gates, dout, o2, dx2, dg2)
    torch.cuda.synchronize()
    assert torch.equal(o2, out) and torch.equal(dx2, dx) and torch.equal(dg2, dgate)
    assert torch.equal(dp.gW1, g1) and torch.equal(dp.gW2, g2)
    dp.close()


def test_micro_batch_wgrad_mode_matches_step_mode():
    """wgrad_mode="micro_batch" (per-micro-batch weight gradients, a 3-set activation ring) runs
    the same forward / dgrad kernels: out / dx / dgate bit-identical, fp32 gradients equal up to
    the accumulation order, and far fewer activation bytes."""
    shape, routing, plan, dp, wts, (x, dout, idx, gates), (out, dx, dgate) = _run("qwen3-30b-a3b", 512, 6)
    shape2, _, _, dp2, _, _, (o2, dx2, dg2) = _run("qwen3-30b-a3b", 512, 6, wgrad_mode="micro_batch")
    assert torch.equal(o2, out) and torch.equal(dx2, dx) and torch.equal(dg2, dgate)
    for a, b in ((dp.gW1, dp2.gW1), (dp.gW2, dp2.gW2)):
        assert moe_ref.rel_l2(b, a) < 1e-5
    assert dp2.memory_report()["activations"] * 2 == dp.memory_report()["activations"]
    dp.close()
    dp2.close()


def test_bench_configuration_parity():
    """The benchmarked configuration itself (Qwen3-30B-A3B layer, T = 8192 tokens, MB = 8
    micro-batches, EP = 1, Zipf 1.0, 128 ragged expert groups, weight gradients contracted over
    every micro-batch): two micro-batches' out / dx / dgate and the gradients of 16 hot and cold
    experts against the fp32 oracle."""
    T, MB = 8192, 8
    shape, routing, plan, dp, (wg, wu, wd), (x, dout, idx, gates), (out, dx, dgate) = _run("qwen3-30b-a3b", T, MB)
    wgc, wuc, wdc = wg.cuda(), wu.cuda(), wd.cuda()
    for m in (0, MB - 1):
        ref = moe_ref.moe_layer_fp32(x[m], idx[m], gates[m], wgc, wuc, wdc, dout[m])
        for key, got in (("out", out[m]), ("dx", dx[m]), ("dgate", dgate[m])):
            _assert_close(got, ref[key], f"{key} mb{m}")
        del ref
    load = routing.mats.sum(axis=(0, 1))
    order = np.argsort(-load, kind="stable")
    experts = np.concatenate([order[:8], order[-8:]])          # 8 hottest + 8 coldest
    sel = torch.from_numpy(experts).cuda()
    gsum = None
    for m in range(MB):
        # oracle restricted to the sampled experts: drop every other expert's choices
        keep = torch.isin(idx[m], sel)
        idx_m = torch.where(keep, idx[m], torch.full_like(idx[m], -1))
        r = moe_ref.moe_layer_fp32(x[m], idx_m, gates[m], wgc, wuc, wdc, dout[m])
        g = (r["dWg"][sel], r["dWu"][sel], r["dWd"][sel])
        gsum = g if gsum is None else tuple(a + b for a, b in zip(gsum, g))
    g_gate, g_up = deinterleave_w1(dp.gW1[sel])
    for got, ref, what in ((g_gate, gsum[0], "dWg"), (g_up, gsum[1], "dWu"), (dp.gW2[sel], gsum[2], "dWd")):
        c = moe_ref.expert_grads_close(got, ref)
        assert c["ok"], f"{what}: {c}"
    dp.close()


def test_routing_plan_mismatch_is_caught():
    """Routing that differs from the counts the step plan was built for never writes past a
    receive slot: the permutation drops the excess choices and the host raises."""
    shape, routing, plan, dp, _, (x, dout, idx, gates), (out, dx, dgate) = _run("qwen3-30b-a3b", 512, 2)
    bad = idx.clone()
    bad[0, :64, :] = int(np.argmax(routing.mats[0, 0]))   # 64 tokens moved onto the hottest expert
    bad[0, :64, 1:] = (bad[0, :64, :1] + torch.arange(1, shape.top_k, device=bad.device)) % shape.num_experts
    dp.step(x, bad, gates, dout, out, dx, dgate)
    with pytest.raises(RuntimeError, match="step plan"):
        dp.check(sync=True)
    dp.check(sync=True)   # the flag is cleared once reported
    dp.close()


def test_step_input_validation():
    shape, routing, plan, dp, _, (x, dout, idx, gates), (out, dx, dgate) = _run("tiny", 256, 2)
    with pytest.raises(ValueError, match="idx must be torch.int32"):
        dp.step(x, idx.long(), gates, dout, out, dx, dgate)
    with pytest.raises(ValueError, match="gates must be torch.float32"):
        dp.step(x, idx, gates.bfloat16(), dout, out, dx, dgate)
    with pytest.raises(ValueError, match="shape"):
        dp.step(x[:, :128], idx[:, :128], gates[:, :128], dout[:, :128], out[:, :128], dx[:, :128], dgate[:, :128])
    with pytest.raises(ValueError, match="contiguous"):
        dp.step(x, idx.transpose(1, 2).contiguous().transpose(1, 2), gates, dout, out, dx, dgate)
    with pytest.raises(ValueError, match="cpu"):
        dp.step(x.cpu(), idx, gates, dout, out, dx, dgate)
    dp.close()


def test_per_plane_launch_settings():
    """Two data planes with different shapes / SM splits in one process keep their own settings:
    every GEMM and row-mover launch carries its plane's values (nothing process-global)."""
    from paper_2605_08639_b200 import kernels as Kmod
    seen = []
    orig = Kmod.grouped_gemm

    def spy(*a, sms=0, **kw):
        if not (kw.get("cta1") and kw.get("stream") is not None):   # opt-in side-stream tail launches
            seen.append(("gemm", sms))
        return orig(*a, sms=sms, **kw)

    a = _run("tiny", 256, 2, comm_sms=20)
    b = _run("qwen3-30b-a3b", 512, 2, comm_sms=28, row_movers="tma")
    dpa, dpb = a[3], b[3]
    assert (dpa.gemm_sms, dpa.comm_blocks) != (dpb.gemm_sms, dpb.comm_blocks)
    Kmod.grouped_gemm = spy
    try:
        calls = {}
        for dp, res in ((dpa, a), (dpb, b), (dpa, a)):
            seen.clear()
            orig_k = dp._k
            movers = []
            dp._k = lambda name, *args, _o=orig_k, _m=movers: (_m.append(args[-2]) if name in (
                "mb_scatter_rows", "mb_combine_rows") else None, _o(name, *args))
            (x, dout, idx, gates), (out, dx, dgate) = res[5], res[6]
            dp.step(x, idx, gates, dout, torch.empty_like(out), torch.empty_like(dx), torch.empty_like(dgate))
            del dp._k
            calls.setdefault(id(dp), []).append((set(s for _, s in seen), set(movers)))
        torch.cuda.synchronize()
        for dp in (dpa, dpb):
            for gemm_sms, mover_blocks in calls[id(dp)]:
                assert gemm_sms == {dp.gemm_sms}, (gemm_sms, dp.gemm_sms)
                assert mover_blocks == {dp.comm_blocks}, (mover_blocks, dp.comm_blocks)
    finally:
        Kmod.grouped_gemm = orig
    dpa.close()
    dpb.close()


def test_layout_without_pregated_activation():
    """MB_PREGATE=0 (the gate applied in the combine, gate*act written over Act by the dAct
    epilogue for dW2) still matches the oracle: the layer tests in a fresh process."""
    env = dict(os.environ, MB_PREGATE="0")
    ids = [f"{__file__}::test_layer_step_matches_oracle[{c}]" for c in ("tiny-256-2-step", "qwen3-30b-a3b-512-2-step",
                                                                       "tiny-256-4-micro_batch")]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *ids], env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "3 passed" in r.stdout
