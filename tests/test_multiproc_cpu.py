"""World-size-2 host logic over torch.distributed (gloo, CPU): every rank histograms its own
replayed routing, the counts are all-gathered into the (MB, G, E) trace, every rank runs the
planners, and the resulting step plans must be identical bit for bit on every rank (the data
plane relies on that: no size exchange happens during the step)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, policy, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_08639_b200 as mb
        from oracle import moe_ref
        from paper_2605_08639_b200.comm import Comm
        from paper_2605_08639_b200.moe_layer import build_step_plan, gather_routing, plan_digest
        from paper_2605_08639_b200.workload import SHAPES, make_routing
        comm = Comm()
        assert (comm.rank, comm.world) == (rank, world)
        cfg = SHAPES["qwen3-30b-a3b"]
        shape = cfg["shape"]
        own = make_routing(shape, 512, 3, world, rank, zipf_s=1.5, shift=cfg["shift"])
        local = np.stack([moe_ref.histogram(own.idx[m], shape.num_experts) for m in range(3)])
        mats = gather_routing(comm, local)
        assert np.array_equal(mats, own.mats)
        topo = mb.b200_box_topology(world, min(world, 4), mb.b200_profile(shape.hidden))
        model = mb.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
        cfgs = mb.SimConfigs(anneal=mb.AnnealConfig(seeds=(0, 1, 2)), replica=mb.ReplicaConfig(2))
        plan = build_step_plan(policy, mats, topo, model, topo.profile, cfgs, shape)
        digests = comm.all_gather_object(plan_digest(plan))
        out[rank] = (digests, plan.skew())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["relibra", "eplb_like"])
def test_world2_plans_identical(policy):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), policy, out), nprocs=world, join=True)
    d0, d1 = out[0][0], out[1][0]
    assert d0 == d1 and len(set(d0)) == 1


def _comm_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), MB_OVERSUBSCRIBE="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2605_08639_b200.comm import Comm, local_device
        comm = Comm()
        # max over ranks of the device-timed ms (the bench's max-over-ranks rule), gloo host path
        m = comm.max_over_ranks(1.5 + rank)
        g = comm.all_gather_tensor(torch.tensor([rank, 10 * rank], dtype=torch.int64))
        out[rank] = (m, g.tolist(), local_device())
    finally:
        dist.destroy_process_group()


def test_world4_oversubscribed_host_collectives():
    """MB_OVERSUBSCRIBE host side: gloo max-over-ranks and tensor all-gather; LOCAL_RANK folds
    onto the visible GPUs (none here: every rank maps to device 0)."""
    world = 4
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        m, g, dev = out[r]
        assert m == 1.5 + world - 1
        assert g == [[p, 10 * p] for p in range(world)]
        assert dev == 0
