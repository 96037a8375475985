"""TEST INFRASTRUCTURE: one rank of a multi-rank data-plane check (launched by
tests/test_multirank_gpu.py through torch.distributed.run; one process per rank, either one
GPU per rank over NCCL or every rank on cuda:0 with MB_OVERSUBSCRIBE=1 / gloo).

Every rank plans the step from the all-gathered K1 histograms, runs one training step of the
layer with replicas (ReLibra policy, GPU groups of --group), and checks against the CPU
restatement in oracle/moe_ref.py:
  * histogram, executed flow and the canonical permutation bit-exact (experts with >= 2
    copies included: round_split counts across copies, replicate.py:501-525);
  * out / dx / dgate of its tokens within the documented bf16 bounds (max-rel, L2, per row);
  * the fp32 gradients of its home experts after the replica-gradient push-back (every rank's
    tokens of every micro-batch) within the bounds, per expert;
  * with --migrate: a second batch whose hot set moved is planned, MoEDataPlane.migrate moves
    weights / fp32 gradients / expert state to the new owners (bit-exact), and a step of the
    new batch matches the oracle again.
Prints one JSON line per rank and exits 1 on any mismatch."""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import moe_ref  # noqa: E402
from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs  # noqa: E402
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile  # noqa: E402
from paper_2605_08639_b200.comm import init_distributed, local_device  # noqa: E402
from paper_2605_08639_b200.kernels import expert_histogram  # noqa: E402
from paper_2605_08639_b200.moe_layer import (MoEDataPlane, build_step_plan, deinterleave_w1,  # noqa: E402
                                             gather_routing, interleave_w1, plan_digest)
from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights  # noqa: E402


def step_and_check(dp, plan, comm, shape, routs, acts, wts, report, tag, steps=1):
    rank, world = comm.rank, comm.world
    MB = len(plan.mbs)
    me = routs[rank]
    x, dout = acts[rank][0].cuda(), acts[rank][1].cuda()
    idx, gates = torch.from_numpy(me.idx).cuda(), torch.from_numpy(me.gates).cuda()
    out, dx = torch.empty_like(x), torch.empty_like(x)
    dgate = torch.empty(MB, x.shape[1], shape.top_k, dtype=torch.float32, device="cuda")
    dp.zero_grads()
    for _ in range(steps):
        dp.step(x, idx, gates, dout, out, dx, dgate)
    dp.check(sync=True)
    comm.host_barrier()
    ok = True
    wg, wu, wd = (w.cuda() for w in wts)
    for m in range(MB):
        mbp = plan.mbs[m]
        if not np.array_equal(dp.counts[m].cpu().numpy(), moe_ref.histogram(me.idx[m], shape.num_experts)):
            ok = False
            report[f"{tag}counts_mb{m}"] = "MISMATCH"
        _, row_base = moe_ref.receive_layout(me.mats[m], plan.home, mbp.placement.replicas, mbp.counts, pad=128)
        ref_perm = moe_ref.canonical_permutation_fast(me.idx[m], rank, me.mats[m], plan.home, mbp.placement.replicas,
                                                      mbp.counts, row_base)
        if not np.array_equal(dp.perm[m].cpu().numpy(), ref_perm):
            ok = False
            report[f"{tag}perm_mb{m}"] = "MISMATCH"
        if not np.array_equal(moe_ref.executed_flow(me.mats[m], plan.home, mbp.placement.replicas, mbp.counts),
                              mbp.flow):
            ok = False
            report[f"{tag}flow_mb{m}"] = "MISMATCH"
        ref = moe_ref.moe_layer_fp32(x[m], idx[m], gates[m], wg, wu, wd, dout[m])
        for key, got in (("out", out[m]), ("dx", dx[m]), ("dgate", dgate[m])):
            c = moe_ref.close(got, ref[key])
            report[f"{tag}{key}_mb{m}"] = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in c.items()}
            ok &= c["ok"]
    # home-expert gradients after the push-back: every rank's tokens of every micro-batch
    gsum = None
    for r in range(world):
        for m in range(MB):
            rr = moe_ref.moe_layer_fp32(acts[r][0][m].cuda(), torch.from_numpy(routs[r].idx[m]).cuda(),
                                        torch.from_numpy(routs[r].gates[m]).cuda(), wg, wu, wd, acts[r][1][m].cuda())
            g = (rr["dWg"], rr["dWu"], rr["dWd"])
            gsum = g if gsum is None else tuple(a + b for a, b in zip(gsum, g))
    home = np.flatnonzero(plan.home == rank)
    hs = torch.from_numpy(home).cuda()
    gW1, gW2 = dp.grads()
    g_gate, g_up = deinterleave_w1(gW1)
    for key, got, ref in (("dWg", g_gate, gsum[0][hs] * steps), ("dWu", g_up, gsum[1][hs] * steps),
                          ("dWd", gW2, gsum[2][hs] * steps)):
        c = moe_ref.expert_grads_close(got, ref)
        report[f"{tag}{key}"] = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in c.items()}
        ok &= c["ok"]
    report[f"{tag}replica_contrib_experts"] = len(dp.replica_contrib)
    return ok, (x, dout)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--policy", default="relibra")
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--micro-batches", type=int, default=2)
    ap.add_argument("--zipf", type=float, default=1.5)
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--wgrad-mode", default="step")
    ap.add_argument("--replica-sets", type=int, default=2)
    ap.add_argument("--migrate", action="store_true")
    ap.add_argument("--min-copies", type=int, default=0, help="fail unless some expert has this many copies")
    ap.add_argument("--shared-layers", action="store_true",
                    help="a second MoE layer (own routing and weights) shares the first one's replica buffer")
    args = ap.parse_args()
    comm = init_distributed()
    rank, world = comm.rank, comm.world
    torch.cuda.set_device(local_device())
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    T, MB = args.tokens, args.micro_batches
    group = min(world, args.group or cfg["group"])
    topo = b200_box_topology(world, group, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=(0, 1, 2, 3)), replica=ReplicaConfig(cfg["slots"]))
    routs = [make_routing(shape, T, MB, world, r, zipf_s=args.zipf, shift=cfg["shift"]) for r in range(world)]
    # the routing every planner sees is the K1 histogram of each rank's tokens, all-gathered
    counts, _ = expert_histogram(torch.from_numpy(routs[rank].idx).cuda(), shape.num_experts)
    mats = gather_routing(comm, counts.cpu().numpy().astype(np.int64))
    report = {"rank": rank, "world": world, "policy": args.policy, "wgrad_mode": args.wgrad_mode,
              "replica_sets": args.replica_sets, "backend": comm.dist.get_backend() if comm.dist else None}
    ok = bool(np.array_equal(mats, routs[rank].mats))
    report["gathered_histograms"] = "ok" if ok else "MISMATCH"
    plan = build_step_plan(args.policy, mats, topo, model, topo.profile, cfgs, shape)
    digests = comm.all_gather_object(plan_digest(plan))
    ok &= len(set(digests)) == 1
    report["maxc"] = plan.maxc
    report["replicas_per_mb"] = [len(m.placement.replicas) for m in plan.mbs]
    if args.min_copies and plan.maxc < args.min_copies:
        ok = False
        report["min_copies"] = f"MISSING: maxc {plan.maxc} < {args.min_copies}"
    wts = make_weights(shape)
    plan_b = None
    if args.migrate:
        # batch B: the same popularity with the expert ids rotated (new hot set, new reorder plan)
        E = shape.num_experts
        rot = max(1, E // world // 2 + 1)
        routs_b = []
        for r in range(world):
            rb = make_routing(shape, T, MB, world, r, zipf_s=args.zipf, shift=cfg["shift"], seed=777)
            rb.idx = ((rb.idx + rot) % E).astype(np.int32)
            rb.mats = np.roll(rb.mats, rot, axis=2)
            routs_b.append(rb)
        plan_b = build_step_plan(args.policy, routs_b[0].mats, topo, model, topo.profile, cfgs, shape)
    rows_cap = max(plan.rows_cap, plan_b.rows_cap if plan_b is not None else 0)
    dp = MoEDataPlane(comm, shape, T, MB, plan, rows_cap=rows_cap, wgrad_mode=args.wgrad_mode,
                      replica_sets=args.replica_sets, expert_state={"tag": ((4,), torch.float32)})
    home_a = np.flatnonzero(plan.home == rank)
    wg, wu, wd = wts
    dp.set_weights(wg[home_a].cuda(), wu[home_a].cuda(), wd[home_a].cuda())
    dp.state["tag"].copy_(torch.tensor(home_a, dtype=torch.float32)[:, None].expand(-1, 4).cuda())
    acts = [make_activations(shape, T, MB, r) for r in range(world)]
    ok_a, _ = step_and_check(dp, plan, comm, shape, routs, acts, wts, report, "", steps=args.steps)
    ok &= ok_a
    report["memory"] = dp.memory_report()
    if args.shared_layers:
        # layer 2: its own routing and weights, the SAME layer-shared replica buffer; then layer 1
        # again (its replicas are pulled again after layer 2 used the slots)
        routs2 = [make_routing(shape, T, MB, world, r, zipf_s=args.zipf, shift=cfg["shift"], seed=4242)
                  for r in range(world)]
        plan2 = build_step_plan(args.policy, routs2[0].mats, topo, model, topo.profile, cfgs, shape)
        wts2 = make_weights(shape, seed=4321)
        dp2 = MoEDataPlane(comm, shape, T, MB, plan2, wgrad_mode=args.wgrad_mode, replica_buffer=dp.rb)
        home2 = np.flatnonzero(plan2.home == rank)
        dp2.set_weights(wts2[0][home2].cuda(), wts2[1][home2].cuda(), wts2[2][home2].cuda())
        acts2 = [make_activations(shape, T, MB, r, seed=123) for r in range(world)]
        ok2, _ = step_and_check(dp2, plan2, comm, shape, routs2, acts2, wts2, report, "L2_")
        ok3, _ = step_and_check(dp, plan, comm, shape, routs, acts, wts, report, "L1again_")
        report["shared_buffer_users"] = dp.rb.users
        report["layer2_replica_bytes_added"] = 0 if dp2.rb is dp.rb else -1
        ok &= ok2 and ok3 and dp2.rb is dp.rb
        dp2.close()
    if plan_b is not None:
        gW1, gW2 = dp.grads()
        mine = {int(e): (gW1[s].cpu(), gW2[s].cpu()) for s, e in enumerate(home_a)}
        grads = {}
        for d in comm.all_gather_object(mine):
            grads.update(d)
        comm.host_barrier()
        info = dp.migrate(plan_b)
        torch.cuda.synchronize()
        home_b = np.flatnonzero(plan_b.home == rank)
        checks = {
            "W1": torch.equal(dp.W1, interleave_w1(wg[home_b].cuda(), wu[home_b].cuda())),
            "W2": torch.equal(dp.W2, wd[home_b].cuda()),
            "state": torch.equal(dp.state["tag"][:, 0].cpu(), torch.tensor(home_b, dtype=torch.float32)),
            "gW1": all(torch.equal(dp.gW1[s].cpu(), grads[int(e)][0]) for s, e in enumerate(home_b)),
            "gW2": all(torch.equal(dp.gW2[s].cpu(), grads[int(e)][1]) for s, e in enumerate(home_b)),
        }
        report["migration"] = {k: ("ok" if v else "MISMATCH") for k, v in checks.items()}
        report["migration"].update(moved=info["experts_moved"], bytes_in=info["bytes_in"],
                                   home_changed=int((plan.home != plan_b.home).sum()))
        ok &= all(checks.values())
        ok_b, _ = step_and_check(dp, plan_b, comm, shape, routs_b, acts, wts, report, "B_")
        ok &= ok_b
    report["ok"] = bool(ok)
    print("MGPU " + json.dumps(report), flush=True)
    dp.close()
    comm.host_barrier()
    if comm.dist:
        comm.dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
