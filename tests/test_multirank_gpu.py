"""Multi-rank data plane under the GPU suite: the replica path (layer-shared replica slots pulled
from the owners, replica-gradient push-back per micro-batch), the multi-copy canonical
permutation, peer scatter / combine over CUDA-IPC memory, the device barrier and expert
migration, each checked against the CPU oracle by tests/mgpu_worker.py on every rank.

Oversubscribed cases run 2 or 4 ranks on cuda:0 (MB_OVERSUBSCRIBE=1: gloo host group, CUDA IPC
between the ranks' processes, the ranks time-slice the GPU), so they run on a 1-GPU box; the
real multi-GPU case runs one rank per GPU over NCCL when the box has >= 2 GPUs."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(world, args, oversubscribe=True, timeout=900):
    env = dict(os.environ)
    env.pop("MB_COMM_SMS", None)
    if oversubscribe:
        env.update(MB_OVERSUBSCRIBE="1", CUDA_VISIBLE_DEVICES=env.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    cmd += [str(a) for a in args]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    reports = [json.loads(line[5:]) for line in proc.stdout.splitlines() if line.startswith("MGPU ")]
    return proc, reports


def _check(proc, reports, world):
    msg = proc.stdout[-4000:] + proc.stderr[-4000:]
    assert proc.returncode == 0, msg
    assert len(reports) == world, msg
    bad = [r for r in reports if not r["ok"]]
    assert not bad, json.dumps(bad)[:4000]
    return reports


@pytest.mark.parametrize("world,config,tokens,zipf,mode,sets,min_copies,migrate", [
    # 2 ranks, one group of 2, replicas (2 copies), both replica-weight set counts
    (2, "tiny", 256, 1.5, "step", 1, 2, False),
    # 4 ranks = one group of 4 at the Qwen3-30B-A3B shape: hot experts with 3+ copies
    (4, "qwen3-30b-a3b", 1024, 1.5, "step", 2, 3, False),
    (4, "qwen3-30b-a3b", 1024, 2.0, "micro_batch", 1, 3, False),
    # 4 ranks in one group, 4 copies of the hottest experts, then a new batch migrates experts
    (4, "tiny", 256, 2.0, "step", 2, 4, True),
])
def test_oversubscribed_replica_step(world, config, tokens, zipf, mode, sets, min_copies, migrate):
    args = ["--config", config, "--tokens", tokens, "--micro-batches", 3 if mode == "micro_batch" else 2,
            "--zipf", zipf, "--wgrad-mode", mode, "--replica-sets", sets, "--min-copies", min_copies,
            "--group", world]
    if migrate:
        args.append("--migrate")
    reports = _check(*_launch(world, args), world)
    assert max(r["maxc"] for r in reports) >= min_copies
    assert sum(r["replica_contrib_experts"] for r in reports) > 0, "no replica gradient was pushed back"
    if migrate:
        assert sum(r["migration"]["moved"] for r in reports) > 0


def test_oversubscribed_four_micro_batches_two_steps():
    """Step mode with 4 micro-batches, two steps: the last combine runs ahead of the third-to-last
    un-permute (schedule early_last), so B(3)'s replica gradients wait on a later un-permute's
    barrier before overwriting the ring set X(1) reads (replica_ring_guards)."""
    args = ["--config", "qwen3-30b-a3b", "--tokens", 1024, "--micro-batches", 4, "--zipf", 1.5, "--group", 4,
            "--replica-sets", 1, "--min-copies", 2, "--steps", 2]
    reports = _check(*_launch(4, args), 4)
    assert sum(r["replica_contrib_experts"] for r in reports) > 0


def test_oversubscribed_layers_share_the_replica_buffer():
    """Two MoE layers (own routing, own weights) share one layer-shared replica buffer: each layer's
    replicas are pulled into the same r slots right before use, gradients pushed back per
    micro-batch; both layers and a repeat of the first match the oracle."""
    args = ["--config", "qwen3-30b-a3b", "--tokens", 1024, "--micro-batches", 2, "--zipf", 1.5, "--group", 4,
            "--replica-sets", 1, "--min-copies", 2, "--shared-layers"]
    reports = _check(*_launch(4, args), 4)
    assert all(r["shared_buffer_users"] == 2 for r in reports)


def test_oversubscribed_two_groups():
    """EP=4 as two groups of 2: reordering across groups, replication inside a group."""
    args = ["--config", "qwen3-30b-a3b", "--tokens", 1024, "--micro-batches", 2, "--zipf", 1.5, "--group", 2,
            "--min-copies", 2]
    _check(*_launch(4, args), 4)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one rank per GPU over NCCL)")
def test_real_multi_gpu_replica_step():
    world = min(4, torch.cuda.device_count())
    args = ["--config", "qwen3-30b-a3b", "--tokens", 1024, "--micro-batches", 2, "--zipf", 1.5,
            "--min-copies", 2, "--migrate"]
    reports = _check(*_launch(world, args, oversubscribe=False), world)
    assert all(r["backend"] == "nccl" for r in reports)
