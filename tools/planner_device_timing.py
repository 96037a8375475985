"""Reorder planner on the host (C++ chains, OpenMP) vs on the GPU (mb_anneal_chains), same inputs:
the bench's Qwen3-30B-A3B routing aggregated over the step, default AnnealConfig (16 chains).
Prints one JSON line per G: wall times and whether the two plans are identical."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08639_b200 as mb  # noqa: E402
from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile  # noqa: E402
from paper_2605_08639_b200.workload import SHAPES, make_routing  # noqa: E402


def main():
    shape = SHAPES["qwen3-30b-a3b"]["shape"]
    model = mb.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    for G, grp in ((4, 4), (8, 4), (8, 8)):
        topo = b200_box_topology(G, grp, b200_profile(shape.hidden))
        r = make_routing(shape, 8192, 8, G, 0, zipf_s=1.0, shift=7)
        x = r.mats.sum(axis=0).astype(np.float64)   # (G, E) aggregate over micro-batches
        cfg = mb.AnnealConfig()
        extra = [mb.static_plan(shape.num_experts, topo)]
        mb.anneal_reorder_device(x, topo, model, topo.profile, mb.AnnealConfig(seeds=(0,), cooling_rate=0.9),
                                 extra_initial_plans=extra)  # warm-up (context, module load)
        t0 = time.perf_counter()
        host = mb.anneal_reorder(x, topo, model, topo.profile, cfg, extra_initial_plans=extra)
        t1 = time.perf_counter()
        dev, iters = mb.anneal_reorder_device(x, topo, model, topo.profile, cfg, extra_initial_plans=extra,
                                              return_iterations=True)
        t2 = time.perf_counter()
        t3 = time.perf_counter()
        host1 = mb.anneal_reorder(x, topo, model, topo.profile, cfg, extra_initial_plans=extra, threads=1)
        t4 = time.perf_counter()
        print(json.dumps({"G": G, "group": grp, "chains": len(cfg.seeds), "iterations": iters,
                          "host_ms": round((t1 - t0) * 1e3, 2), "host_threads": os.cpu_count(),
                          "host_1thread_ms": round((t4 - t3) * 1e3, 2), "device_ms": round((t2 - t1) * 1e3, 2),
                          "identical": host.assignment.tolist() == dev.assignment.tolist() == host1.assignment.tolist()}),
              flush=True)


def layers(L=48):
    """A whole model's reorder planning: L layers x 16 seeds (host: OpenMP over each layer's
    chains, layer after layer; device: every chain in one launch)."""
    shape = SHAPES["qwen3-30b-a3b"]["shape"]
    model = mb.ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    topo = b200_box_topology(8, 4, b200_profile(shape.hidden))
    xs = [make_routing(shape, 2048, 2, 8, 0, zipf_s=0.7 + 0.02 * li, shift=li).mats.sum(axis=0).astype(np.float64)
          for li in range(L)]
    cfg = mb.AnnealConfig()
    tm = {}
    t0 = time.perf_counter()
    dev, iters = mb.anneal_reorder_layers_device(xs, topo, model, topo.profile, cfg, timings=tm)
    t1 = time.perf_counter()
    host = [mb.anneal_reorder(x, topo, model, topo.profile, cfg) for x in xs]
    t2 = time.perf_counter()
    t1, t2 = t0 + (t2 - t1), t0 + (t2 - t1) + (t1 - t0)   # host_ms = t1 - t0, device_ms = t2 - t1
    print(json.dumps({"layers": L, "G": 8, "group": 4, "chains": L * len(cfg.seeds), "iterations": iters,
                      "host_ms": round((t1 - t0) * 1e3, 1), "host_threads": os.cpu_count(),
                      "device_ms": round((t2 - t1) * 1e3, 1), "device_breakdown_ms": {k: round(v, 1) for k, v in tm.items()},
                      "identical": all(a.assignment.tolist() == b.assignment.tolist() for a, b in zip(host, dev))}),
          flush=True)


if __name__ == "__main__":
    layers(1)   # warm-up: CUDA context + module load
    for L in (1, 8, 48):
        layers(L)
    main()
