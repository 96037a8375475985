"""TEST INFRASTRUCTURE ONLY: the CPU reference arm of bench.py (--impl reference, cpu_baseline).

Times the reference's own CPU implementation of the path -- moebalance 0.1.0, built into
oracle/_ref by oracle/build_ref.sh (pure Python + numpy) -- on the bench's workload:
  * planners: sim.build_policy_bundle(trace, "relibra", ...) (reorder.anneal_reorder per layer,
    replicate.greedy_replicate + round_split per (micro-batch, layer); sim.py:214-280) over the
    step's (MB, 1, G, E) routing, at threads=1 and threads=nproc (sim.py:205-211);
  * the layer math the reference only models (costmodel.comp_time, costmodel.py:161-163): the
    fp32 port oracle/moe_ref.moe_layer_fp32 (torch CPU, every host thread) on a fixed token
    sample, so the number does not depend on a time budget.
Nothing here is on the product path."""

from __future__ import annotations

import os
import statistics
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def load_reference():
    """moebalance from oracle/_ref (built by oracle/build_ref.sh); None when absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "moebalance")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import moebalance
    return moebalance


def reference_planner_seconds(mb, mats: np.ndarray, shape, num_gpus: int, group: int, sa_chains: int, slots: int,
                              threads: int, reps: int = 3) -> float:
    """Median seconds of the reference's build_policy_bundle("relibra") for one step's routing
    (mats: (MB, G, E) counts), with the B200 rates the native planners use (cluster.b200_profile)."""
    from moebalance import sim
    flops, bw = 1376.6e12 / 3.0, 770e9 / 2.0
    hw = mb.HardwareProfile(flops_per_gpu=flops, bw_nvlink=bw, bw_rdma=bw, bytes_per_token=2.0 * shape.hidden)
    group = max(1, min(group, num_gpus))
    topo = mb.build_topology(num_gpus // group, group, hw)
    model = mb.ModelProfile(num_layers=1, num_experts=shape.num_experts, top_k=shape.top_k,
                            hidden_size=shape.hidden, intermediate_size=shape.ffn)
    trace = mb.RoutingTrace(model=model, topo=topo, matrices=np.ascontiguousarray(mats[:, None], dtype=np.uint32),
                            tokens_per_gpu=0, generator={})
    trace.validate()
    cfgs = sim.SimConfigs(anneal=mb.AnnealConfig(seeds=tuple(range(sa_chains))), replica=mb.ReplicaConfig(slots),
                          threads=threads)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        sim.build_policy_bundle(trace, "relibra", topo, model, hw, cfgs)
        times.append(time.perf_counter() - t0)
    return statistics.median(times)


def port_layer_tokens_per_s(cfg_name: str, zipf: float, threads: int, sample_tokens: int = 2048,
                            reps: int = 3) -> float:
    """Median tokens/s of the fp32 torch-CPU layer fwd+bwd (+ np.bincount histogram) over a
    fixed sample of `sample_tokens` tokens of one GPU's share."""
    import torch
    from oracle import moe_ref
    from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights
    torch.set_num_threads(threads)
    cfg = SHAPES[cfg_name]
    shape = cfg["shape"]
    wg, wu, wd = make_weights(shape)
    r = make_routing(shape, sample_tokens, 1, 1, 0, zipf_s=zipf, shift=cfg["shift"])
    x, dout = make_activations(shape, sample_tokens, 1, 0)
    idx, gates = torch.from_numpy(r.idx[0]), torch.from_numpy(r.gates[0])
    rates = []
    for _ in range(reps):
        t0 = time.perf_counter()
        moe_ref.histogram(r.idx[0], shape.num_experts)
        moe_ref.moe_layer_fp32(x[0], idx, gates, wg, wu, wd, dout[0])
        rates.append(sample_tokens / (time.perf_counter() - t0))
    return statistics.median(rates)
