"""Inter-batch expert reordering (static blocks, LPT, simulated annealing).

Mirror of the hot-path part of ``moebalance.reorder`` (reorder.py:30-362).  The planners run
in libmb_planner.so: LPT and static are exact; the annealer reproduces the reference's numpy
PCG64 stream (SeedSequence(seed) per chain), swap proposals, Metropolis test and numpy's
summation order, and runs the chains of one layer in parallel threads (results gathered in
seed order, so the plan does not depend on the thread count).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as nat
from .cluster import ClusterTopology, HardwareProfile


@dataclass
class ReorderPlan:
    """Capacity-preserving expert -> GPU assignment of one layer."""

    assignment: np.ndarray

    def experts_on(self, gpu: int) -> np.ndarray:
        return np.flatnonzero(self.assignment == gpu)

    def copy(self) -> "ReorderPlan":
        return ReorderPlan(self.assignment.copy())

    def validate(self, topo: ClusterTopology) -> None:
        g = topo.num_gpus
        if len(self.assignment) % g:
            raise ValueError("expert count not divisible by GPU count")
        counts = np.bincount(self.assignment, minlength=g)
        per = len(self.assignment) // g
        if (counts != per).any():
            raise ValueError(f"plan is not capacity-preserving: counts {counts.tolist()}, expected {per} per GPU")


@dataclass(frozen=True)
class AnnealConfig:
    """Chain seeds, geometric cooling and LSE sharpness (reorder.py:53-78)."""

    seeds: tuple = tuple(range(16))
    cooling_rate: float = 0.9995
    termination_eps: float | None = None
    eps_frac: float = 1e-3
    beta: float = 20.0

    def __post_init__(self) -> None:
        if len(self.seeds) < 1:
            raise ValueError("need at least one annealing seed")
        if not 0 < self.cooling_rate < 1:
            raise ValueError(f"cooling_rate must be in (0, 1), got {self.cooling_rate}")
        if self.termination_eps is not None and not self.termination_eps > 0:
            raise ValueError("termination_eps must be > 0")
        if not self.eps_frac > 0:
            raise ValueError("eps_frac must be > 0")
        if not self.beta > 0:
            raise ValueError("beta must be > 0")

    def eps_for(self, theta0: float) -> float:
        return self.termination_eps if self.termination_eps is not None else self.eps_frac * theta0


@dataclass
class SamplePlacement:
    source_gpu: np.ndarray


def static_plan(num_experts: int, topo: ClusterTopology) -> ReorderPlan:
    """No-balancing baseline: experts [g*M, (g+1)*M) on GPU g (reorder.py:291-296)."""
    g = topo.num_gpus
    if num_experts % g:
        raise ValueError(f"{num_experts} experts not divisible by {g} GPUs")
    out = np.zeros(num_experts, dtype=np.int64)
    lib = nat.planner()
    nat.check(lib.mbp_static_plan(num_experts, g, nat.ptr(out)), lib, "static_plan")
    return ReorderPlan(out)


def lpt_initial(x_batch, topo: ClusterTopology) -> ReorderPlan:
    """Heaviest expert to the least-loaded open GPU, ties to the lower index (reorder.py:265-288)."""
    x = nat.f64(x_batch)
    g = topo.num_gpus
    if x.shape[1] % g:
        raise ValueError(f"{x.shape[1]} experts not divisible by {g} GPUs")
    out = np.zeros(x.shape[1], dtype=np.int64)
    lib = nat.planner()
    nat.check(lib.mbp_lpt_initial(nat.ptr(x), g, x.shape[1], nat.ptr(out)), lib, "lpt_initial")
    return ReorderPlan(out)


def anneal_reorder(x_batch, topo: ClusterTopology, model, hw: HardwareProfile, cfg: AnnealConfig,
                   extra_initial_plans: Sequence[ReorderPlan] = (), threads: int | None = None) -> ReorderPlan:
    """Swap SA from LPT; best exact T_MoE over [LPT, extra plans, chains in seed order]
    (reorder.py:329-362).  `threads` (extension): chain parallelism, default all cores."""
    x = nat.f64(x_batch)
    num_experts = x.shape[1]
    if num_experts % topo.num_gpus:
        raise ValueError(f"{num_experts} experts not divisible by {topo.num_gpus} GPUs")
    for plan in extra_initial_plans:
        plan.validate(topo)
    extra = nat.i64(np.stack([np.asarray(p.assignment) for p in extra_initial_plans])
                    if extra_initial_plans else np.zeros((0, num_experts)))
    seeds = np.ascontiguousarray([int(s) for s in cfg.seeds], dtype=np.uint64)
    out = np.zeros(num_experts, dtype=np.int64)
    iters = np.zeros(1, dtype=np.int64)
    nthreads = threads if threads is not None else (os.cpu_count() or 1)
    lib = nat.planner()
    nat.check(lib.mbp_anneal_reorder(
        nat.ptr(x), topo.num_nodes, topo.gpus_per_node, num_experts, model.hidden_size, model.intermediate_size,
        hw.flops_per_gpu, hw.bw_nvlink, hw.bw_rdma, hw.bytes_per_token, nat.ptr(seeds), len(seeds),
        cfg.cooling_rate, cfg.eps_frac, cfg.termination_eps if cfg.termination_eps is not None else -1.0,
        cfg.beta, nat.ptr(extra), len(extra_initial_plans), nthreads, nat.ptr(out), nat.ptr(iters)),
        lib, "anneal_reorder")
    return ReorderPlan(out)


def anneal_reorder_device(x_batch, topo: ClusterTopology, model, hw: HardwareProfile, cfg: AnnealConfig,
                          extra_initial_plans: Sequence[ReorderPlan] = (), device=None,
                          return_iterations: bool = False):
    """anneal_reorder with its chains on the GPU (GPU-side planning): the host
    prepares the LPT start, the shared contribution tensor and each seed's PCG64 state exactly as
    anneal_reorder does, the chains run as one GPU thread per seed (mb_anneal_chains), and the
    host picks the first minimum of the exact T_MoE over [LPT, extra plans, chains in seed order]
    (reorder.py:329-362).  Same arguments and result as anneal_reorder."""
    plans, iters = anneal_reorder_layers_device([x_batch], topo, model, hw, cfg, [extra_initial_plans], device)
    return (plans[0], iters) if return_iterations else plans[0]


def anneal_reorder_layers_device(x_layers, topo: ClusterTopology, model, hw: HardwareProfile, cfg: AnnealConfig,
                                 extra_initial_plans=None, device=None, timings: dict | None = None):
    """Every layer's reorder plan with all (layer, seed) chains in ONE device launch -- the
    paper's "one thread per (layer, seed)" solver at GPU width.  x_layers:
    per-layer (G, E) batch matrices; extra_initial_plans: per-layer sequences (or None).
    Returns ([ReorderPlan per layer], total chain iterations); `timings` (optional dict) receives
    host prepare / device chains / host select wall milliseconds."""
    import time

    import torch
    t0 = time.perf_counter()
    xs = [nat.f64(x) for x in x_layers]
    L = len(xs)
    if L == 0:
        return [], 0
    num_experts = xs[0].shape[1]
    G = topo.num_gpus
    if num_experts % G:
        raise ValueError(f"{num_experts} experts not divisible by {G} GPUs")
    extras = list(extra_initial_plans) if extra_initial_plans is not None else [()] * L
    if len(extras) != L:
        raise ValueError("need one extra-plan sequence per layer")
    for ex in extras:
        for plan in ex:
            plan.validate(topo)
    seeds = np.ascontiguousarray([int(s) for s in cfg.seeds], dtype=np.uint64)
    n = len(seeds)
    if n < 1:
        raise ValueError("need at least one annealing seed")
    base = np.zeros((L, num_experts), dtype=np.int64)
    contrib = np.zeros((L, num_experts, G, 5, G), dtype=np.float64)
    consts = np.zeros(5, dtype=np.float64)
    rng = np.zeros((L, n, 4), dtype=np.uint64)
    lib = nat.planner()
    args = (topo.num_nodes, topo.gpus_per_node, num_experts, model.hidden_size, model.intermediate_size,
            hw.flops_per_gpu, hw.bw_nvlink, hw.bw_rdma, hw.bytes_per_token, cfg.beta)
    for li, x in enumerate(xs):
        if x.shape != (G, num_experts):
            raise ValueError(f"layer {li}: expected a ({G}, {num_experts}) batch matrix, got {x.shape}")
        nat.check(lib.mbp_anneal_prepare(nat.ptr(x), *args, nat.ptr(seeds), n, nat.ptr(base[li]),
                                         nat.ptr(contrib[li]), nat.ptr(consts), nat.ptr(rng[li])), lib,
                  "anneal_prepare")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t1 = time.perf_counter()
    d_contrib = torch.from_numpy(contrib).to(dev)
    d_base = torch.from_numpy(base).to(dev)
    d_rng = torch.from_numpy(rng.view(np.int64)).to(dev)
    d_best = torch.empty((L * n, num_experts), dtype=torch.int64, device=dev)
    d_iters = torch.empty(L * n, dtype=torch.int64, device=dev)
    klib = nat.kernels()
    with torch.cuda.device(dev):
        nat.check(klib.mb_anneal_chains(d_contrib.data_ptr(), num_experts, G, d_base.data_ptr(), nat.ptr(consts),
                                        cfg.beta, d_rng.data_ptr(), L * n, n, cfg.cooling_rate, cfg.eps_frac,
                                        cfg.termination_eps if cfg.termination_eps is not None else -1.0,
                                        d_best.data_ptr(), d_iters.data_ptr(), nat.stream_ptr()),
                  klib, "mb_anneal_chains")
        best = d_best.cpu().numpy().reshape(L, n, num_experts)
        iters = int(d_iters.sum().item())
    t2 = time.perf_counter()
    plans = []
    for li, x in enumerate(xs):
        extra = [np.asarray(p.assignment, dtype=np.int64) for p in extras[li]]
        cands = np.ascontiguousarray(np.stack([base[li]] + extra + list(best[li])), dtype=np.int64)
        out = np.zeros(num_experts, dtype=np.int64)
        nat.check(lib.mbp_anneal_select(nat.ptr(x), *args, nat.ptr(cands), len(cands), nat.ptr(out)), lib,
                  "anneal_select")
        plans.append(ReorderPlan(out))
    if timings is not None:
        timings.update(prepare_ms=(t1 - t0) * 1e3, device_ms=(t2 - t1) * 1e3,
                       select_ms=(time.perf_counter() - t2) * 1e3)
    return plans, iters


def _sample_call(trace, plans, topo, model, hw, cfg, band, greedy_only, beta, threads):
    if trace.samples is None:
        raise ValueError("trace has no sample table")
    s = trace.samples
    L, E = trace.model.num_layers, trace.model.num_experts
    if len(plans) != L:
        raise ValueError(f"need one expert plan per layer ({L}), got {len(plans)}")
    counts = nat.f64(np.asarray(s.counts, dtype=np.float64).reshape(s.num_samples, L, E))
    mb = nat.i32(s.micro_batch)
    src = nat.i64(s.source_gpu)
    tok = nat.f64(np.asarray(s.tokens, dtype=np.float64))
    pl = nat.i64(np.stack([np.asarray(p.assignment) for p in plans]))
    seeds = np.ascontiguousarray([int(x) for x in (cfg.seeds if cfg else (0,))], dtype=np.uint64)
    out = np.zeros(s.num_samples, dtype=np.int64)
    lib = nat.planner()
    nat.check(lib.mbp_sample_placement(
        topo.num_nodes, topo.gpus_per_node, E, L, trace.num_micro_batches, s.num_samples, nat.ptr(counts),
        nat.ptr(mb), nat.ptr(src), nat.ptr(tok), nat.ptr(pl), model.hidden_size, model.intermediate_size,
        hw.flops_per_gpu, hw.bw_nvlink, hw.bw_rdma, hw.bytes_per_token, nat.ptr(seeds), len(seeds),
        cfg.cooling_rate if cfg else 0.5, cfg.eps_frac if cfg else 1e-3,
        (cfg.termination_eps if cfg and cfg.termination_eps is not None else -1.0), beta, band,
        1 if greedy_only else 0, threads if threads is not None else (os.cpu_count() or 1), nat.ptr(out)),
        lib, "sample_placement")
    return SamplePlacement(source_gpu=out)


def greedy_sample_initial(trace, plans: Sequence[ReorderPlan], topo: ClusterTopology, model, hw: HardwareProfile,
                          beta: float = 20.0, band: float = 0.10) -> SamplePlacement:
    """Longest-first greedy sample placement within the token band (reorder.py:457-487)."""
    return _sample_call(trace, plans, topo, model, hw, None, band, True, beta, 1)


def anneal_sample_placement(trace, plans: Sequence[ReorderPlan], topo: ClusterTopology, model, hw: HardwareProfile,
                            cfg: AnnealConfig, band: float = 0.10, threads: int | None = None) -> SamplePlacement:
    """Second annealing round: swap sample source GPUs under fixed expert plans; never worse
    than the greedy start in summed exact time (reorder.py:537-568).  `threads` (extension):
    chain parallelism, default all cores."""
    return _sample_call(trace, plans, topo, model, hw, cfg, band, False, cfg.beta, threads)


def apply_plan(x, plan: ReorderPlan, placement: SamplePlacement | None = None, trace=None,
               micro_batch: int | None = None, layer: int | None = None) -> np.ndarray:
    """One routing matrix under an expert plan and sample placement (reorder.py:575-607): expert
    relocation never changes matrix values; relocated samples move their counts between sources."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[1] != len(plan.assignment):
        raise ValueError(f"matrix has {x.shape[1]} experts, plan covers {len(plan.assignment)}")
    out = x.copy()
    if placement is None:
        return out
    if trace is None or trace.samples is None or micro_batch is None or layer is None:
        raise ValueError("sample relocation requires the trace with samples plus micro_batch and layer")
    s = trace.samples
    for i in np.flatnonzero(s.micro_batch == micro_batch):
        src, dst = int(s.source_gpu[i]), int(placement.source_gpu[i])
        if src == dst:
            continue
        counts = s.counts[i, layer].astype(np.float64)
        out[src] -= counts
        out[dst] += counts
    if out.min() < 0:
        raise ValueError("sample relocation produced negative counts; matrix does not match the trace")
    return out


def rewrite_trace_matrices(trace, placement: SamplePlacement) -> np.ndarray:
    """All (MB, L, G, E) matrices with sample rows moved to their new sources (reorder.py:610-627)."""
    s = trace.samples
    if s is None:
        raise ValueError("trace has no sample table")
    out = trace.matrices.astype(np.float64).copy()
    for i in range(s.num_samples):
        src, dst = int(s.source_gpu[i]), int(placement.source_gpu[i])
        if src == dst:
            continue
        counts = s.counts[i].astype(np.float64)  # (L, E)
        out[int(s.micro_batch[i]), :, src, :] -= counts
        out[int(s.micro_batch[i]), :, dst, :] += counts
    if out.min() < 0:
        raise ValueError("sample relocation produced negative counts")
    return out
