"""Timeline of one bench step (torchrun, one process per GPU): start / end of every K4 launch
and comm phase relative to the step start, and the compute-stream gaps (where the GEMMs wait
for the comm stream).  Rank 0 prints one JSON line.

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/step_timeline.py [--config qwen3-30b-a3b]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs  # noqa: E402
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile  # noqa: E402
from paper_2605_08639_b200.comm import init_distributed, local_device  # noqa: E402
from paper_2605_08639_b200.kernels import expert_histogram  # noqa: E402
from paper_2605_08639_b200.moe_layer import MoEDataPlane, build_step_plan, gather_routing  # noqa: E402
from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3-30b-a3b")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--micro-batches", type=int, default=8)
    ap.add_argument("--policy", default="relibra")
    ap.add_argument("--back-to-back", type=int, default=1,
                    help="steps issued without a host sync; the last is reported (1 = synced single step)")
    args = ap.parse_args()
    comm = init_distributed()
    torch.cuda.set_device(local_device())
    rank, world = comm.rank, comm.world
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    T, MB = args.tokens, args.micro_batches
    topo = b200_box_topology(world, min(world, cfg["group"]), b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=tuple(range(4))), replica=ReplicaConfig(cfg["slots"]))
    r = make_routing(shape, T, MB, world, rank, zipf_s=1.0, shift=cfg["shift"], all_ranks=False)
    counts, _ = expert_histogram(torch.from_numpy(r.idx).cuda(), shape.num_experts)
    mats = gather_routing(comm, counts.cpu().numpy().astype(np.int64))
    plan = build_step_plan(args.policy, mats, topo, model, topo.profile, cfgs, shape)
    dp = MoEDataPlane(comm, shape, T, MB, plan)
    wg, wu, wd = make_weights_for(shape, np.flatnonzero(plan.home == rank))
    dp.set_weights(wg, wu, wd)
    x, dout = make_activations(shape, T, MB, rank)
    dev = {"x": x.cuda(), "dout": dout.cuda(), "idx": torch.from_numpy(r.idx).cuda(),
           "gates": torch.from_numpy(r.gates).cuda()}
    out, dx = torch.empty_like(dev["x"]), torch.empty_like(dev["x"])
    dgate = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    # warm-up, then (--back-to-back) steps issued without a host sync between them, as in the bench:
    # the last one is reported, so the host's lead over the GPU hides its launch work
    for it in range(3):
        dp.zero_grads()
        dp.step(dev["x"], dev["idx"], dev["gates"], dev["dout"], out, dx, dgate)
    torch.cuda.synchronize()
    comm.host_barrier()
    n = max(1, args.back_to_back)
    for it in range(n):
        dp.zero_grads()
        dp.timing = it == n - 1
        dp.gemm_events = []
        s0 = torch.cuda.Event(enable_timing=True)
        e0 = torch.cuda.Event(enable_timing=True)
        s0.record()
        dp.step(dev["x"], dev["idx"], dev["gates"], dev["dout"], out, dx, dgate)
        e0.record()
    torch.cuda.synchronize()
    ev = [(s0.elapsed_time(a), s0.elapsed_time(b), kd) for a, b, _, kd in dp.gemm_events]
    gemm = sorted([e for e in ev if not e[2].startswith("comm_")])
    gaps, prev = [], 0.0
    for a, b, kd in gemm:
        if a - prev > 0.02:
            gaps.append((round(prev, 3), round(a - prev, 3), kd))
        prev = max(prev, b)
    line = {"rank": rank, "world": world, "step_ms": round(s0.elapsed_time(e0), 3),
            "gemm_busy_ms": round(sum(b - a for a, b, _ in gemm), 3),
            "gemm_gaps (at, ms, next)": gaps, "tail_after_last_gemm_ms": round(s0.elapsed_time(e0) - prev, 3),
            "comm": [(round(a, 3), round(b - a, 3), kd[5:]) for a, b, kd in sorted(e for e in ev if e[2].startswith("comm_"))]}
    lines = comm.all_gather_object(line)
    if rank == 0:
        for ln in lines:
            print(json.dumps(ln), flush=True)
    dp.close()
    if comm.dist:
        comm.dist.barrier()
        comm.dist.destroy_process_group()


if __name__ == "__main__":
    main()
