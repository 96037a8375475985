"""Planner cost side by side: the REFERENCE's own planners (imported from /root/reference, this
container only) vs this package's native planners, on the bench's routing (Qwen3-30B-A3B shape,
8 micro-batches x 8192 tokens per GPU, Zipf 1.0), policy "relibra" = aggregate -> anneal_reorder
(default AnnealConfig: 16 chains) -> greedy_replicate + round_split per micro-batch.
Also checks that both produce the same bundle (assignment, replicas, fractions).

    PYTHONDONTWRITEBYTECODE=1 python tools/planner_timing.py > profiles/r01_planner_timing.json
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = "/root/reference/pkg/src"


def main():
    import paper_2605_08639_b200 as mb
    from paper_2605_08639_b200.workload import SHAPES, make_routing
    sys.path.insert(0, REF)
    import moebalance as ref
    from moebalance import sim as ref_sim
    ref.build_policy_bundle = ref_sim.build_policy_bundle
    ref.SimConfigs = ref_sim.SimConfigs

    cfg = SHAPES["qwen3-30b-a3b"]
    shape = cfg["shape"]
    out = {"host_cores": os.cpu_count(), "config": "qwen3-30b-a3b, MB=8, T=8192, zipf 1.0, relibra, 16 SA chains",
           "runs": []}
    for G, group in ((2, 2), (4, 4), (8, 4)):
        r = make_routing(shape, 8192, 8, G, 0, zipf_s=1.0, shift=cfg["shift"])
        mats = r.mats[:, None].astype(np.uint32)
        hw_kw = dict(flops_per_gpu=1376.6e12 / 3, bw_nvlink=770e9 / 2, bw_rdma=770e9 / 2,
                     bytes_per_token=2.0 * shape.hidden)
        res = {"gpus": G, "group": group}
        bundles = {}
        for name, lib, threads in (("reference", ref, 1), ("native_1thread", mb, 1), ("native", mb, 8)):
            hw = lib.HardwareProfile(**hw_kw)
            topo = lib.build_topology(G // group, group, hw)
            model = lib.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
            trace = lib.RoutingTrace(model=model, topo=topo, matrices=mats, tokens_per_gpu=8192)
            cfgs = lib.SimConfigs(replica=lib.ReplicaConfig(2), threads=threads)
            t0 = time.perf_counter()
            bundle, _ = lib.build_policy_bundle(trace, "relibra", topo, model, hw, cfgs)
            res[name + "_s"] = round(time.perf_counter() - t0, 4)
            bundles[name] = bundle
        a, b = bundles["reference"], bundles["native"]
        same = bool(np.array_equal(a.reorder[0].assignment, b.reorder[0].assignment))
        for key in a.replication.entries:
            ea, eb = a.replication.entries[key], b.replication.entries[key]
            same &= ea.placement.replicas == eb.placement.replicas
            same &= all(np.array_equal(ea.split.fractions[e], eb.split.fractions[e]) for e in ea.split.fractions)
        res["identical_bundles"] = same
        res["speedup_native_vs_reference"] = round(res["reference_s"] / res["native_s"], 1)
        out["runs"].append(res)
        print(json.dumps(res), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
