"""Multi-GPU parity check of the EP data plane (run with torchrun, one process per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_check.py [--config tiny] [--policy relibra]

Every rank runs one training step of the layer with the given policy (replicas included), then
checks against the CPU/fp32 oracle: permutation bit-exact (canonical permutation of the plan),
out / dx / dgate of its tokens and the fp32 gradients of its home experts (after the replica
gradient reduce) within rel 2e-2.  Prints one JSON line per rank; exits nonzero on mismatch.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import moe_ref  # noqa: E402
from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs  # noqa: E402
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile  # noqa: E402
from paper_2605_08639_b200.comm import init_distributed, local_device  # noqa: E402
from paper_2605_08639_b200.moe_layer import MoEDataPlane, build_step_plan, deinterleave_w1  # noqa: E402
from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--policy", default="relibra")
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--micro-batches", type=int, default=2)
    ap.add_argument("--zipf", type=float, default=1.5)
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--steps", type=int, default=1)
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
    me = routs[rank]
    plan = build_step_plan(args.policy, me.mats, topo, model, topo.profile, cfgs, shape)
    dp = MoEDataPlane(comm, shape, T, MB, plan)
    wg, wu, wd = make_weights(shape)
    home = np.flatnonzero(plan.home == rank)
    dp.set_weights(wg[home].cuda(), wu[home].cuda(), wd[home].cuda())
    dp.zero_grads()
    acts = [make_activations(shape, T, MB, r) for r in range(world)]
    x, dout = acts[rank][0].cuda(), acts[rank][1].cuda()
    idx = torch.from_numpy(me.idx).cuda()
    gates = torch.from_numpy(me.gates).cuda()
    out, dx = torch.empty_like(x), torch.empty_like(x)
    dgate = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    for _ in range(args.steps):
        dp.step(x, idx, gates, dout, out, dx, dgate)
    torch.cuda.synchronize()
    comm.host_barrier()
    report = {"rank": rank, "world": world, "policy": args.policy, "replicas": sum(len(m.placement.replicas)
                                                                                  for m in plan.mbs)}
    errs = {}
    ok = True
    wgc, wuc, wdc = wg.cuda(), wu.cuda(), wd.cuda()
    gsum = None
    for m in range(MB):
        mbp = plan.mbs[m]
        _, row_base = moe_ref.receive_layout(me.mats[m], plan.home, mbp.placement.replicas, mbp.counts, pad=128)
        ref_perm = moe_ref.canonical_permutation_fast(me.idx[m], rank, me.mats[m], plan.home, mbp.placement.replicas,
                                                      mbp.counts, row_base)
        if not np.array_equal(dp.perm[m].cpu().numpy(), ref_perm):
            ok = False
            errs[f"perm_mb{m}"] = "MISMATCH"
        flow = moe_ref.executed_flow(me.mats[m], plan.home, mbp.placement.replicas, mbp.counts)
        if not np.array_equal(flow, mbp.flow):
            ok = False
            errs[f"flow_mb{m}"] = "MISMATCH"
        ref = moe_ref.moe_layer_fp32(x[m], idx[m], gates[m], wgc, wuc, wdc, dout[m])
        for key, got in (("out", out[m]), ("dx", dx[m]), ("dgate", dgate[m])):
            e = moe_ref.rel_err(got, ref[key])
            errs[f"{key}_mb{m}"] = round(e, 5)
            ok &= e < 2e-2
        # weight grads need every rank's tokens
        for r in range(world):
            xr, dr = acts[r][0][m].cuda(), acts[r][1][m].cuda()
            rr = moe_ref.moe_layer_fp32(xr, torch.from_numpy(routs[r].idx[m]).cuda(),
                                        torch.from_numpy(routs[r].gates[m]).cuda(), wgc, wuc, wdc, dr)
            g = (rr["dWg"], rr["dWu"], rr["dWd"])
            gsum = g if gsum is None else tuple(a + b for a, b in zip(gsum, g))
    g_gate, g_up = deinterleave_w1(dp.gW1[:dp.M])
    hs = torch.from_numpy(home).cuda()
    for key, got, ref in (("dWg", g_gate, gsum[0][hs] * args.steps), ("dWu", g_up, gsum[1][hs] * args.steps),
                          ("dWd", dp.gW2[:dp.M], gsum[2][hs] * args.steps)):
        e = moe_ref.rel_err(got, ref)
        errs[key] = round(e, 5)
        ok &= e < 2e-2
    report["ok"] = bool(ok)
    report["errors"] = errs
    print(json.dumps(report), flush=True)
    dp.close()
    comm.host_barrier()
    if comm.dist:
        comm.dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
