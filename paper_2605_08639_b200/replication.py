"""Intra-batch expert replication: placement/split types, the token-split LP, the greedy
replicator and integer splitting.

Mirror of the hot-path part of ``moebalance.replicate`` (replicate.py:29-437, 497-534):
same dataclasses (``ReplicaPlacement.replicas`` keeps dict insertion order = copy order),
validation messages and errors.  The LP, the greedy loop and ``round_split`` run in
libmb_planner.so; ``round_split`` counts feed the dispatch tables of the data plane.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cluster import ClusterTopology, HardwareProfile
from .reordering import ReorderPlan

IMPROVE_RTOL = 1e-9
ENUM_GUARD = 2**20


class InstanceTooLargeError(ValueError):
    """Raised by exact enumeration beyond its guard (replicate.py:33-34)."""


@dataclass(frozen=True)
class ReplicaConfig:
    slots_per_gpu: int = 2

    def __post_init__(self) -> None:
        if self.slots_per_gpu < 0:
            raise ValueError("slots_per_gpu must be >= 0")


@dataclass
class ReplicaPlacement:
    home: np.ndarray
    replicas: dict = field(default_factory=dict)

    def copies(self, e: int) -> list:
        return [int(self.home[e])] + list(self.replicas.get(e, []))

    def slot_usage(self, num_gpus: int) -> np.ndarray:
        used = np.zeros(num_gpus, dtype=int)
        for gpus in self.replicas.values():
            for g in gpus:
                used[g] += 1
        return used

    def serving(self, gpu: int) -> list:
        own = {int(e) for e in np.flatnonzero(self.home == gpu)}
        own.update(e for e, gpus in self.replicas.items() if gpu in gpus)
        return sorted(own)


@dataclass
class SplitPlan:
    """fractions[e]: (G, len(copies(e))) per-source token fractions over the copies."""

    fractions: dict = field(default_factory=dict)

    def to_split_map(self, placement: ReplicaPlacement) -> dict:
        return {e: (np.array(placement.copies(e)), frac) for e, frac in self.fractions.items()}


@dataclass
class ReplicationEntry:
    placement: ReplicaPlacement
    split: SplitPlan
    objective: float


@dataclass
class ReplicationPlan:
    entries: dict = field(default_factory=dict)


def candidate_gpus(e: int, home: np.ndarray, topo: ClusterTopology) -> list:
    """Replica candidates: the home group minus the home GPU (replicate.py:104-107)."""
    h = int(home[e])
    return [g for g in topo.node_gpus(topo.node_of(h)) if g != h]


def validate_placement(placement: ReplicaPlacement, topo: ClusterTopology, cfg: ReplicaConfig | None = None) -> None:
    for e, gpus in placement.replicas.items():
        allowed = set(candidate_gpus(e, placement.home, topo))
        for g in gpus:
            if g not in allowed:
                raise ValueError(f"replica of expert {e} on GPU {g} leaves its home node or duplicates home")
        if len(set(gpus)) != len(gpus):
            raise ValueError(f"duplicate replica GPUs for expert {e}")
    if cfg is not None:
        used = placement.slot_usage(topo.num_gpus)
        if (used > cfg.slots_per_gpu).any():
            raise ValueError(f"replica slots exceeded: usage {used.tolist()}, limit {cfg.slots_per_gpu}")


def validate_split(split: SplitPlan, placement: ReplicaPlacement, x, tol: float = 1e-6) -> None:
    x = np.asarray(x, dtype=np.float64)
    for e, frac in split.fractions.items():
        k = len(placement.copies(e))
        if frac.shape != (x.shape[0], k):
            raise ValueError(f"split for expert {e} has shape {frac.shape}, expected {(x.shape[0], k)}")
        if frac.min() < -tol or frac.max() > 1 + tol:
            raise ValueError(f"split fractions for expert {e} escape [0, 1]")
        routed = x[:, e] > 0
        if routed.any():
            err = np.abs(frac[routed].sum(axis=1) - 1.0).max()
            if err > tol:
                raise ValueError(f"split for expert {e} violates conservation by {err:.3e}")


def _placement_csr(placement: ReplicaPlacement, order=None):
    keys = list(placement.replicas.keys()) if order is None else order
    experts, ptrs, gpus = [], [0], []
    for e in keys:
        experts.append(int(e))
        gpus.extend(int(g) for g in placement.replicas[e])
        ptrs.append(len(gpus))
    return nat.i32(experts), nat.i32(ptrs), nat.i32(gpus)


def _model_hw_args(model, hw: HardwareProfile):
    return (model.hidden_size, model.intermediate_size, hw.flops_per_gpu, hw.bw_nvlink, hw.bw_rdma,
            hw.bytes_per_token)


def solve_token_split_lp(x, placement: ReplicaPlacement, topo: ClusterTopology, model, hw: HardwareProfile) -> SplitPlan:
    """Optimal per-source fractions for a fixed placement (replicate.py:305-321)."""
    validate_placement(placement, topo)
    xs = nat.f64(x)
    g, num_experts = xs.shape
    home = nat.i64(placement.home)
    ex, pt, gp = _placement_csr(placement)
    out_e = np.zeros(max(len(ex), 1), dtype=np.int32)
    frac = np.zeros(max(num_experts * g * g, 1))
    lib = nat.planner()
    nat.check(lib.mbp_solve_token_split(nat.ptr(xs), topo.num_nodes, topo.gpus_per_node, num_experts, nat.ptr(home),
                                        *_model_hw_args(model, hw), len(ex), nat.ptr(ex), nat.ptr(pt), nat.ptr(gp),
                                        nat.ptr(out_e), nat.ptr(frac)), lib, "solve_token_split_lp")
    split = SplitPlan()
    off = 0
    for i in range(len(ex)):
        e = int(out_e[i])
        k = 1 + len(placement.replicas[e])
        split.fractions[e] = frac[off:off + g * k].reshape(g, k).copy()
        off += g * k
    validate_split(split, placement, xs)
    return split


def greedy_replicate(x, plan: ReorderPlan, topo: ClusterTopology, model, hw: HardwareProfile,
                     cfg: ReplicaConfig) -> tuple:
    """Algorithm 2 (replicate.py:365-437): replicate the bottleneck GPU's
    hottest expert onto the cheapest same-group GPU, re-solve the warm-started split LP, keep
    the step only if exact T_MoE improves by more than 1e-9 relative."""
    xs = nat.f64(x)
    g, num_experts = xs.shape
    home = nat.i64(plan.assignment)
    n_rep = np.zeros(1, dtype=np.int32)
    rep_e = np.zeros(num_experts, dtype=np.int32)
    rep_p = np.zeros(num_experts + 1, dtype=np.int32)
    rep_g = np.zeros(num_experts * g, dtype=np.int32)
    frac = np.zeros(num_experts * g * g)
    obj = np.zeros(1)
    lib = nat.planner()
    nat.check(lib.mbp_greedy_replicate(nat.ptr(xs), topo.num_nodes, topo.gpus_per_node, num_experts, nat.ptr(home),
                                       *_model_hw_args(model, hw), cfg.slots_per_gpu, nat.ptr(n_rep), nat.ptr(rep_e),
                                       nat.ptr(rep_p), nat.ptr(rep_g), nat.ptr(frac), nat.ptr(obj)),
              lib, "greedy_replicate")
    placement = ReplicaPlacement(home=np.asarray(plan.assignment))
    split = SplitPlan()
    off = 0
    for i in range(int(n_rep[0])):
        e = int(rep_e[i])
        gpus = [int(v) for v in rep_g[rep_p[i]:rep_p[i + 1]]]
        placement.replicas[e] = gpus
        k = 1 + len(gpus)
        split.fractions[e] = frac[off:off + g * k].reshape(g, k).copy()
        off += g * k
    validate_placement(placement, topo, cfg)
    validate_split(split, placement, xs)
    return placement, split


def round_split(split: SplitPlan, placement: ReplicaPlacement, x) -> dict:
    """Largest-remainder integer counts per (source, copy) (replicate.py:501-525)."""
    xs = nat.f64(x)
    g, num_experts = xs.shape
    order = list(split.fractions.keys())
    if not order:
        return {}
    ex = nat.i32(order)
    gpus, ptrs, fr = [], [0], []
    for e in order:
        frac = np.asarray(split.fractions[e], dtype=np.float64)
        k = frac.shape[1]
        cps = placement.copies(e)
        if len(cps) != k:  # fractions of a plan whose placement lost copies: pad with home
            cps = (cps + [cps[0]] * k)[:k]
        gpus.extend(cps[1:])
        ptrs.append(len(gpus))
        fr.append(np.ascontiguousarray(frac).ravel())
    gp, pt, ff = nat.i32(gpus), nat.i32(ptrs), nat.f64(np.concatenate(fr))
    counts = np.zeros(ff.size, dtype=np.int64)
    home = nat.i64(placement.home)
    lib = nat.planner()
    nat.check(lib.mbp_round_split(nat.ptr(xs), g, num_experts, nat.ptr(home), len(order), nat.ptr(ex), nat.ptr(pt),
                                  nat.ptr(gp), nat.ptr(ff), nat.ptr(counts)), lib, "round_split")
    out, off = {}, 0
    for e in order:
        k = split.fractions[e].shape[1]
        out[e] = counts[off:off + g * k].reshape(g, k).copy()
        off += g * k
    return out


def replica_memory(model, cfg: ReplicaConfig, scheme: str) -> int:
    """Replica-slot parameter bytes per GPU (replicate.py:528-534)."""
    if scheme == "per-layer":
        return model.num_layers * cfg.slots_per_gpu * model.param_bytes
    if scheme == "layer-shared":
        return cfg.slots_per_gpu * model.param_bytes
    raise ValueError(f"unknown buffer scheme {scheme!r}; expected 'per-layer' or 'layer-shared'")
