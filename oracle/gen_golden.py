"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/ from the reference itself.

Imports moebalance from /root/reference/pkg/src (read-only; this container only) and records
inputs + outputs of the hot-path planner functions on the reference's own known-answer tests
and on seeded random instances at the BASELINE.json shapes.  Floats are stored with
float.hex() so the fixtures are exact.  The fixtures travel with the repo; the reference does not.

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def hw_tuple(hw):
    return [hw.flops_per_gpu.hex(), hw.bw_nvlink.hex(), hw.bw_rdma.hex(), float(hw.bytes_per_token).hex()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import moebalance as mb
    from moebalance import sim
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20261018)
    fx = {"generator": "oracle/gen_golden.py", "reference": "moebalance 0.1.0 (/root/reference/pkg)",
          "numpy": np.__version__, "cases": {}}
    C = fx["cases"]

    # ---------------------------------------------------------------- KATs of the reference tests
    unit = mb.HardwareProfile(6.0, 1e18, 1e18, 1.0)
    t2 = mb.build_topology(1, 2, unit)
    x = np.array([[12.0, 0.0], [0.0, 4.0]])
    model = mb.ModelProfile(num_layers=1, num_experts=2, top_k=1, hidden_size=1, intermediate_size=1)
    p, s = mb.greedy_replicate(x, mb.ReorderPlan(np.array([0, 1])), t2, model, unit, mb.ReplicaConfig(1))
    C["kat_twelve_vs_four"] = {"x": x.tolist(), "replicas": {str(k): v for k, v in p.replicas.items()},
                               "frac0": hexs(s.fractions[0]),
                               "comp": hexs(mb.compute_loads(x, np.array([0, 1]), t2, s.to_split_map(p)).comp)}
    pl = mb.ReplicaPlacement(home=np.array([0, 1]), replicas={0: [1]})
    xr = np.array([[10.0, 0.0], [0.0, 4.0]])
    C["kat_round_split"] = [
        {"frac": f, "counts": mb.round_split(mb.SplitPlan({0: np.array(f)}), pl, xr)[0].tolist()}
        for f in ([[1.0, 0.0], [1.0, 0.0]], [[0.5, 0.5], [0.5, 0.5]], [[2 / 3, 1 / 3], [1.0, 0.0]])]
    t22 = mb.build_topology(2, 2, mb.HardwareProfile(1.0, 1.0, 1.0, 1.0))
    C["kat_relay"] = {"cls": t22.class_matrix.tolist(), "relay": t22.relay_matrix.tolist()}
    xl = np.array([[5.0, 1.0, 0.0, 2.0], [0.0, 3.0, 4.0, 1.0]])
    C["kat_lpt"] = {"x": xl.tolist(), "assignment": mb.lpt_initial(xl, mb.build_topology(1, 2, unit)).assignment.tolist()}
    C["kat_skew"] = {"loads": [12, 4], "skew": mb.skewness([12, 4])}

    # ---------------------------------------------------------------- compute_loads with fractional splits
    cases = []
    for i in range(40):
        nodes, gpn = [(1, 2), (2, 2), (2, 4), (1, 8), (4, 2)][i % 5]
        g = nodes * gpn
        e = g * int(rng.integers(1, 4))
        hw = mb.HardwareProfile(6.0, float(rng.uniform(20, 200)), float(rng.uniform(5, 50)), 1.0)
        topo = mb.build_topology(nodes, gpn, hw)
        xx = rng.integers(0, 60, size=(g, e)).astype(float)
        home = rng.permutation(np.repeat(np.arange(g), e // g))
        splits = {}
        for ex in rng.choice(e, size=min(3, e), replace=False):
            cands = [q for q in range(g) if q // gpn == home[ex] // gpn and q != home[ex]]
            if not cands:
                continue
            k = 1 + int(rng.integers(1, len(cands) + 1))
            gp = [int(home[ex])] + [int(v) for v in rng.choice(cands, size=k - 1, replace=False)]
            splits[int(ex)] = (np.array(gp), rng.dirichlet(np.ones(k), size=g))
        lv = mb.compute_loads(xx, home, topo, splits)
        cases.append({"nodes": nodes, "gpn": gpn, "x": xx.tolist(), "home": home.tolist(),
                      "splits": [[ex, gp.tolist(), hexs(fr)] for ex, (gp, fr) in splits.items()],
                      "loads": {f: hexs(getattr(lv, f)) for f in ("comp", "nvlink_tx", "nvlink_rx", "rdma_tx", "rdma_rx")}})
    C["compute_loads"] = cases

    # ---------------------------------------------------------------- LPT / static / uniform / EPLB
    cases = []
    for i in range(60):
        g = [2, 4, 8][i % 3]
        e = g * int(rng.integers(1, 17))
        xx = rng.integers(0, 1000, size=(g, e))
        topo = mb.build_topology(max(1, g // 4), min(g, 4), unit)
        plan = mb.lpt_initial(xx, topo)
        loads = xx.astype(np.float64).sum(axis=0)
        ep = sim._eplb_replication(loads, plan.assignment, topo, 2)
        cases.append({"nodes": topo.num_nodes, "gpn": topo.gpus_per_node, "x": xx.tolist(),
                      "lpt": plan.assignment.tolist(), "static": mb.static_plan(e, topo).assignment.tolist(),
                      "eplb": [[k, v] for k, v in ep.replicas.items()]})
    C["lpt_static_eplb"] = cases
    mats = rng.integers(0, 50, size=(3, 1, 4, 16)).astype(np.uint32)
    tr = mb.RoutingTrace(model=mb.ModelProfile(1, 16, 2), topo=mb.build_topology(1, 4, unit), matrices=mats,
                         tokens_per_gpu=0)
    C["uniform"] = {"mats": mats.tolist(), "out": sim._uniform_matrices(tr).tolist()}

    # ---------------------------------------------------------------- simulated annealing
    cases = []
    n_sa = 8 if args.quick else 16
    for i in range(n_sa):
        nodes, gpn = [(2, 2), (2, 4), (1, 4), (4, 2)][i % 4]
        g = nodes * gpn
        e = g * int(rng.integers(2, 6))
        hw = mb.HardwareProfile(24.0, float(rng.uniform(20, 200)), float(rng.uniform(5, 50)), 1.0)
        topo = mb.build_topology(nodes, gpn, hw)
        model = mb.ModelProfile(1, e, 1, hidden_size=1, intermediate_size=1)
        xx = rng.integers(0, 50, size=(g, e)).astype(float)
        cfg = mb.AnnealConfig(seeds=(0, 1, 2, 3), cooling_rate=0.995)
        plan = mb.anneal_reorder(xx, topo, model, hw, cfg, extra_initial_plans=[mb.static_plan(e, topo)])
        cases.append({"nodes": nodes, "gpn": gpn, "hw": hw_tuple(hw), "x": xx.tolist(), "seeds": [0, 1, 2, 3],
                      "cooling": 0.995, "assignment": plan.assignment.tolist()})
    # Qwen3-30B-A3B shape (E=128, 2 groups x 4), default AnnealConfig: the production planner path
    big = []
    n_big = 1 if args.quick else 3
    for i in range(n_big):
        g, e = 8, 128
        hw = mb.HardwareProfile(1376.6e12 / 3, 770e9 / 2, 770e9 / 2, 4096.0)
        topo = mb.build_topology(2, 4, hw)
        model = mb.ModelProfile(1, e, 8, hidden_size=2048, intermediate_size=768)
        pop = (np.arange(e) + 1.0) ** -1.2
        pop = pop[np.random.default_rng(i).permutation(e)]
        pop /= pop.sum()
        xx = np.stack([np.random.default_rng(100 + i * 8 + j).multinomial(8 * 4096, pop) for j in range(g)]).astype(float)
        t0 = time.time()
        plan = mb.anneal_reorder(xx, topo, model, hw, mb.AnnealConfig(), extra_initial_plans=[mb.static_plan(e, topo)])
        big.append({"nodes": 2, "gpn": 4, "hw": hw_tuple(hw), "x": xx.tolist(), "h": 2048, "hp": 768,
                    "assignment": plan.assignment.tolist(), "ref_seconds": round(time.time() - t0, 2)})
    C["anneal_small"] = cases
    C["anneal_qwen3"] = big

    # ---------------------------------------------------------------- greedy replication + LP + round_split
    cases = []
    for i in range(120):
        nodes, gpn = [(1, 2), (1, 3), (2, 2), (1, 4), (2, 4)][i % 5]
        g = nodes * gpn
        e = g * int(rng.integers(1, 4))
        hw = mb.HardwareProfile(6.0, float(rng.uniform(20, 200)), float(rng.uniform(5, 50)), 1.0)
        topo = mb.build_topology(nodes, gpn, hw)
        model = mb.ModelProfile(1, e, 1, hidden_size=1, intermediate_size=1)
        xx = rng.integers(0, 30, size=(g, e)).astype(float)
        plan = mb.lpt_initial(xx, topo)
        r = int(rng.integers(0, 3))
        p, s = mb.greedy_replicate(xx, plan, topo, model, hw, mb.ReplicaConfig(r))
        counts = mb.round_split(s, p, xx)
        cases.append({"nodes": nodes, "gpn": gpn, "hw": hw_tuple(hw), "x": xx.tolist(), "home": plan.assignment.tolist(),
                      "slots": r, "replicas": [[k, v] for k, v in p.replicas.items()],
                      "fractions": [[k, list(v.shape), hexs(v)] for k, v in s.fractions.items()],
                      "counts": [[k, v.tolist()] for k, v in counts.items()]})
    C["greedy_small"] = cases
    big = []
    for i in range(4 if args.quick else 12):
        g, e = 8, 128
        hw = mb.HardwareProfile(1376.6e12 / 3, 770e9 / 2, 770e9 / 2, 4096.0)
        topo = mb.build_topology(2, 4, hw)
        model = mb.ModelProfile(1, e, 8, hidden_size=2048, intermediate_size=768)
        pop = (np.arange(e) + 1.0) ** -float(rng.uniform(0.5, 2.0))
        pop = pop[rng.permutation(e)]
        pop /= pop.sum()
        xx = np.stack([rng.multinomial(8 * 8192, pop) for _ in range(g)]).astype(float)
        plan = mb.lpt_initial(xx, topo)
        p, s = mb.greedy_replicate(xx, plan, topo, model, hw, mb.ReplicaConfig(2))
        counts = mb.round_split(s, p, xx)
        big.append({"nodes": 2, "gpn": 4, "hw": hw_tuple(hw), "x": xx.tolist(), "h": 2048, "hp": 768,
                    "home": plan.assignment.tolist(), "slots": 2,
                    "replicas": [[k, v] for k, v in p.replicas.items()],
                    "fractions": [[k, list(v.shape), hexs(v)] for k, v in s.fractions.items()],
                    "counts": [[k, v.tolist()] for k, v in counts.items()]})
    C["greedy_qwen3"] = big

    path = os.path.join(OUT, "planners.json")
    with open(path, "w") as f:
        json.dump(fx, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
