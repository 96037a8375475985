"""Multi-GPU check of expert migration between batches (run with torchrun, one process per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_migrate.py [--config tiny]

Batch A is planned and stepped; batch B's routing has its hot experts moved, so the reorder
planner assigns experts differently and MoEDataPlane.migrate() moves weights, fp32 gradients and
per-expert state to their new owners.  Checks (per rank): migrated weights / state / gradients
bit-exact against the pre-migration values of the same experts, then a step of batch B against
the fp32 oracle (out / dx / dgate within rel 2e-2).  Prints one JSON line per rank.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import moe_ref  # noqa: E402
from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs  # noqa: E402
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile  # noqa: E402
from paper_2605_08639_b200.comm import init_distributed, local_device  # noqa: E402
from paper_2605_08639_b200.moe_layer import MoEDataPlane, build_step_plan, interleave_w1  # noqa: E402
from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--micro-batches", type=int, default=2)
    ap.add_argument("--zipf", type=float, default=1.5)
    args = ap.parse_args()
    comm = init_distributed()
    rank, world = comm.rank, comm.world
    torch.cuda.set_device(local_device())
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    E, T, MB = shape.num_experts, args.tokens, args.micro_batches
    topo = b200_box_topology(world, min(world, cfg["group"]), b200_profile(shape.hidden))
    model = ModelProfile(1, E, shape.top_k, shape.hidden, shape.ffn)
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=(0, 1, 2, 3)), replica=ReplicaConfig(cfg["slots"]))
    ra = make_routing(shape, T, MB, world, rank, zipf_s=args.zipf, shift=cfg["shift"])
    # batch B: the same popularity with the expert ids rotated (new hot set)
    rot = max(1, E // world // 2 + 1)
    rb = make_routing(shape, T, MB, world, rank, zipf_s=args.zipf, shift=cfg["shift"], seed=777)
    rb.idx = ((rb.idx + rot) % E).astype(np.int32)
    rb.mats = np.roll(rb.mats, rot, axis=2)
    pa = build_step_plan("relibra", ra.mats, topo, model, topo.profile, cfgs, shape)
    pb = build_step_plan("relibra", rb.mats, topo, model, topo.profile, cfgs, shape)
    dp = MoEDataPlane(comm, shape, T, MB, pa, rows_cap=max(pa.rows_cap, pb.rows_cap),
                      expert_state={"tag": ((4,), torch.float32)})
    wg, wu, wd = make_weights(shape)
    home_a = np.flatnonzero(pa.home == rank)
    dp.set_weights(wg[home_a].cuda(), wu[home_a].cuda(), wd[home_a].cuda())
    dp.state["tag"].copy_(torch.tensor(home_a, dtype=torch.float32)[:, None].expand(-1, 4).cuda())
    dp.zero_grads()
    acts = make_activations(shape, T, MB, rank)
    x, dout = acts[0].cuda(), acts[1].cuda()
    out, dx = torch.empty_like(x), torch.empty_like(x)
    dgate = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    dp.step(x, torch.from_numpy(ra.idx).cuda(), torch.from_numpy(ra.gates).cuda(), dout, out, dx, dgate)
    torch.cuda.synchronize()
    # every expert's accumulated gradient before the move, keyed by expert id
    mine = {int(e): (dp.gW1[s].cpu(), dp.gW2[s].cpu()) for s, e in enumerate(home_a)}
    grads = {}
    for d in comm.all_gather_object(mine):
        grads.update(d)
    comm.host_barrier()
    t0 = time.perf_counter()
    info = dp.migrate(pb)
    torch.cuda.synchronize()
    mig_ms = (time.perf_counter() - t0) * 1e3
    home_b = np.flatnonzero(pb.home == rank)
    ok = True
    errs = {"moved": info["experts_moved"], "bytes_in": info["bytes_in"], "migrate_ms": round(mig_ms, 3),
            "home_changed": int((pa.home != pb.home).sum())}
    w1_ref = interleave_w1(wg[home_b].cuda(), wu[home_b].cuda())
    checks = {
        "W1": torch.equal(dp.W1, w1_ref),
        "W2": torch.equal(dp.W2, wd[home_b].cuda()),
        "state": torch.equal(dp.state["tag"][:, 0].cpu(), torch.tensor(home_b, dtype=torch.float32)),
        "gW1": all(torch.equal(dp.gW1[s].cpu(), grads[int(e)][0]) for s, e in enumerate(home_b)),
        "gW2": all(torch.equal(dp.gW2[s].cpu(), grads[int(e)][1]) for s, e in enumerate(home_b)),
    }
    for k, v in checks.items():
        errs[k] = "ok" if v else "MISMATCH"
        ok &= v
    idx_b, gates_b = torch.from_numpy(rb.idx).cuda(), torch.from_numpy(rb.gates).cuda()
    dp.step(x, idx_b, gates_b, dout, out, dx, dgate)
    torch.cuda.synchronize()
    wgc, wuc, wdc = wg.cuda(), wu.cuda(), wd.cuda()
    for m in range(MB):
        ref = moe_ref.moe_layer_fp32(x[m], idx_b[m], gates_b[m], wgc, wuc, wdc, dout[m])
        for key, got in (("out", out[m]), ("dx", dx[m]), ("dgate", dgate[m])):
            e = moe_ref.rel_err(got, ref[key])
            errs[f"{key}_mb{m}"] = round(e, 5)
            ok &= e < 2e-2
    print(json.dumps({"rank": rank, "world": world, "ok": bool(ok), "checks": errs}), flush=True)
    dp.close()
    comm.host_barrier()
    if comm.dist:
        comm.dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
