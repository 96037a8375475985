"""Plan files and the `solve` pipeline, wire-compatible with moebalance.

reorder.json      per-layer expert -> GPU arrays, optional sample -> GPU array, and the exact /
                  smoothed objective per layer (planio.py:25-52)
replication.json  per (micro_batch, layer): replica list, split rows (source_gpu, expert,
                  serving_gpu, fraction) and the objective (replicate.py:539-578)

`solve` is the reference CLI's `solve` command (cli.py:124-185) on this package's native
planners, including the data-locality sample placement (--sample-locality, reorder.py:365-568):
the files it writes are byte-identical to the reference's for the same trace and options
(tests/test_io_golden.py).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from . import loads as cm
from . import policies as sim
from . import reordering as ro
from . import replication as rep
from . import traces as rt


class PlanFormatError(ValueError):
    """Malformed or mismatched plan files (planio.py:21-22)."""


def chain_seeds(master_seed: int, count: int) -> tuple:
    """Annealing chain seeds derived from the master seed by fixed offsets (cli.py:39-41)."""
    return tuple(master_seed * 1000 + i for i in range(count))


def save_reorder_plan(path, trace_id: str, plans: list, objectives: list, sample_placement, config: dict) -> None:
    payload = {
        "version": 1,
        "trace_id": trace_id,
        "num_layers": len(plans),
        "plans": [np.asarray(p.assignment).tolist() for p in plans],
        "objectives": objectives,
        "sample_placement": np.asarray(sample_placement.source_gpu).tolist() if sample_placement else None,
        "config": config,
    }
    Path(path).write_text(json.dumps(payload, indent=2) + "\n")


def load_reorder_plan(path) -> dict:
    p = Path(path)
    if not p.is_file():
        raise FileNotFoundError(f"missing reorder plan file: {p}")
    data = json.loads(p.read_text())
    if data.get("version") != 1:
        raise PlanFormatError(f"unsupported reorder plan version in {p}")
    data["plans"] = [ro.ReorderPlan(np.asarray(a, dtype=np.int64)) for a in data["plans"]]
    if data.get("sample_placement") is not None:
        data["sample_placement"] = ro.SamplePlacement(np.asarray(data["sample_placement"], dtype=np.int64))
    return data


def replication_plan_to_dict(plan: rep.ReplicationPlan) -> dict:
    entries = []
    for (mb, layer) in sorted(plan.entries):
        entry = plan.entries[(mb, layer)]
        rows = []
        for e, frac in sorted(entry.split.fractions.items()):
            copies = entry.placement.copies(e)
            for j in range(frac.shape[0]):
                for col, gpu in enumerate(copies):
                    if frac[j, col] > 0:
                        rows.append([int(j), int(e), int(gpu), float(frac[j, col])])
        entries.append({
            "micro_batch": mb,
            "layer": layer,
            "replicas": [[int(e), int(g)] for e in sorted(entry.placement.replicas)
                         for g in entry.placement.replicas[e]],
            "splits": rows,
            "objective": entry.objective,
        })
    return {"version": 1, "entries": entries}


def replication_plan_from_dict(data: dict, home_per_layer: dict, num_gpus: int) -> rep.ReplicationPlan:
    plan = rep.ReplicationPlan()
    for entry in data["entries"]:
        mb, layer = entry["micro_batch"], entry["layer"]
        placement = rep.ReplicaPlacement(home=home_per_layer[layer])
        for e, g in entry["replicas"]:
            placement.replicas.setdefault(int(e), []).append(int(g))
        split = rep.SplitPlan()
        for j, e, gpu, value in entry["splits"]:
            e = int(e)
            if e not in split.fractions:
                split.fractions[e] = np.zeros((num_gpus, len(placement.copies(e))))
            split.fractions[e][int(j), placement.copies(e).index(int(gpu))] = value
        plan.entries[(mb, layer)] = rep.ReplicationEntry(placement=placement, split=split,
                                                         objective=entry["objective"])
    return plan


def save_replication_plan(path, trace_id: str, plan: rep.ReplicationPlan) -> None:
    payload = replication_plan_to_dict(plan)
    payload["trace_id"] = trace_id
    Path(path).write_text(json.dumps(payload, indent=2) + "\n")


def load_replication_plan(path, home_per_layer: dict, num_gpus: int) -> tuple:
    p = Path(path)
    if not p.is_file():
        raise FileNotFoundError(f"missing replication plan file: {p}")
    data = json.loads(p.read_text())
    if data.get("version") != 1:
        raise PlanFormatError(f"unsupported replication plan version in {p}")
    return replication_plan_from_dict(data, home_per_layer, num_gpus), data.get("trace_id", "")


def load_plan_bundle(plans_dir, trace: rt.RoutingTrace) -> sim.PlanBundle:
    """PlanBundle from a solve output directory, checked against the trace (planio.py:67-96)."""
    root = Path(plans_dir)
    reorder_path, replication_path = root / "reorder.json", root / "replication.json"
    if not reorder_path.is_file():
        raise FileNotFoundError(f"missing plan file for relibra: {reorder_path}")
    data = load_reorder_plan(reorder_path)
    if data["trace_id"] and data["trace_id"] != trace.trace_id():
        raise PlanFormatError(f"reorder plan {reorder_path} was solved for trace {data['trace_id']}, "
                              f"not {trace.trace_id()}")
    plans = data["plans"]
    if len(plans) != trace.model.num_layers:
        raise PlanFormatError("reorder plan layer count disagrees with the trace")
    homes = {layer: plans[layer].assignment for layer in range(len(plans))}
    if not replication_path.is_file():
        raise FileNotFoundError(f"missing plan file for relibra: {replication_path}")
    replication, rep_id = load_replication_plan(replication_path, homes, trace.topo.num_gpus)
    if rep_id and rep_id != trace.trace_id():
        raise PlanFormatError(f"replication plan {replication_path} belongs to a different trace")
    return sim.PlanBundle(reorder=plans, sample_placement=data.get("sample_placement"), replication=replication)


def solve(trace: rt.RoutingTrace, out_dir, seeds: int = 16, cooling: float = 0.9995, eps_frac: float = 1e-3,
          eps: float | None = None, beta: float = 20.0, replica_slots: int = 2, seed: int = 0,
          threads: int = 0, sample_locality: bool = False) -> sim.PlanBundle:
    """Inter-batch reorder per layer, optional data-locality sample placement, then intra-batch
    replication per (micro-batch, layer) on the (rewritten) matrices; writes reorder.json /
    replication.json (cli.py:124-185)."""
    topo, model, hw = trace.topo, trace.model, trace.topo.profile
    cfg = ro.AnnealConfig(seeds=chain_seeds(seed, seeds), cooling_rate=cooling, termination_eps=eps,
                          eps_frac=eps_frac, beta=beta)
    smoothing = cm.SmoothingConfig(beta=beta)
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    nthreads = threads if threads > 0 else None
    plans, objectives = [], []
    for layer in range(model.num_layers):
        agg = rt.aggregate_batch(trace, layer)
        plan = ro.anneal_reorder(agg, topo, model, hw, cfg,
                                 extra_initial_plans=[ro.static_plan(model.num_experts, topo)], threads=nthreads)
        est = cm.moe_time(cm.compute_loads(agg, plan.assignment, topo), model, hw, smoothing=smoothing)
        plans.append(plan)
        objectives.append({"exact": est.t_moe, "smoothed": est.t_moe_smoothed})
    placement = None
    if sample_locality:
        if trace.samples is None:
            raise ValueError("--sample-locality needs a trace with a sample table")
        placement = ro.anneal_sample_placement(trace, plans, topo, model, hw, cfg, threads=nthreads)
    matrices = (ro.rewrite_trace_matrices(trace, placement) if placement is not None
                else trace.matrices.astype(np.float64))
    replica_cfg = rep.ReplicaConfig(slots_per_gpu=replica_slots)
    replication = rep.ReplicationPlan()
    tasks = []
    for mb in range(trace.num_micro_batches):
        for layer in range(model.num_layers):
            tasks.append(((mb, layer), (lambda m=mb, l=layer: rep.greedy_replicate(
                matrices[m, l], plans[l], topo, model, hw, replica_cfg))))
    results = sim.solve_tasks(tasks, threads if threads > 0 else 1)
    for (mb, layer), (pl, split) in results.items():
        x = matrices[mb, layer]
        achieved = cm.moe_time(cm.compute_loads(x, plans[layer].assignment, topo,
                                                splits=split.to_split_map(pl)), model, hw).t_moe
        replication.entries[(mb, layer)] = rep.ReplicationEntry(pl, split, achieved)
    config_echo = {"seeds": seeds, "cooling": cooling, "eps_frac": eps_frac, "eps": eps, "beta": beta,
                   "replica_slots": replica_slots, "seed": seed, "sample_locality": bool(sample_locality)}
    tid = trace.trace_id()
    save_reorder_plan(out / "reorder.json", tid, plans, objectives, placement, config_echo)
    save_replication_plan(out / "replication.json", tid, replication)
    return sim.PlanBundle(reorder=plans, sample_placement=placement, replication=replication)
