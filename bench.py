#!/usr/bin/env python
"""MoE-layer fwd+bwd tokens/s of the B200 ReLibra hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config qwen3-30b-a3b] [--zipf 1.0]
  torchrun --nproc-per-node N bench.py --gpus N ...           (one process per GPU, NCCL)
  python bench.py --impl reference ...                          (CPU reference arm, rank 0)

A step = one training step of one MoE layer over MB micro-batches of T tokens per GPU
(forward + backward incl. fp32 weight gradients) with replayed routing.  EP = N (all N GPUs
of one box; the reference's "node" = a GPU group of min(N, 4)).  Policies measured on the same
routing: ReLibra (headline `value`), no-balancing static EP, oracle-EPLB, and the balanced
ideal (uniform routing).  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd+bwd tokens/s"
PEAKS_FALLBACK = {"bf16_tflops_sustained": 1376.6, "bf16_tflops": 1667.1, "hbm_gbs": 6534.5}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


K4_TRAFFIC = os.path.join(ROOT, "profiles", "r02_launches_step_summary.json")


def k4_traffic_per_step(config: str, world: int, tokens: int, mbs: int):
    """DRAM bytes (read + write) of every K4 launch of ONE step, from the committed ncu launch list
    of that step of this bench command (the NVTX range "mb_step", dram__bytes_read.sum +
    dram__bytes_write.sum per launch, tools/ncu_step.sh); None for other configurations."""
    if (config, world, tokens, mbs) != ("qwen3-30b-a3b", 1, 8192, 8):
        return None
    try:
        return float(json.load(open(K4_TRAFFIC))["totals"]["k4_dram_bytes"])
    except (OSError, ValueError, KeyError):
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        pl = [float(s[7]) for s in self.samples if len(s) > 7 and s[7].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(pl) if pl else None}


# ----------------------------------------------------------------------------- CPU reference arm

REF_SAMPLE_TOKENS = 8192   # fixed layer-port sample per CPU-arm step (2048 spread 21% over 10 steps)


def cpu_reference_step(args, world, threads: int, reps: int = 1) -> dict:
    """One step of the CPU reference path on the host cores (oracle/ref_arm.py): the reference's
    own planners (moebalance from oracle/_ref: build_policy_bundle("relibra") over the step's
    routing, threads=1 and threads=nproc) plus the fp32 port of the layer fwd+bwd on a fixed
    token sample, combined as tokens/s of the whole step (every GPU's tokens on this host)."""
    from oracle import ref_arm
    from paper_2605_08639_b200.workload import SHAPES, make_routing
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    slots = cfg["slots"] if args.slots is None else args.slots
    group = min(world, args.group or cfg["group"])
    tokens_step = world * args.tokens * args.micro_batches
    layer_tps = ref_arm.port_layer_tokens_per_s(args.config, args.zipf, threads, sample_tokens=REF_SAMPLE_TOKENS,
                                                reps=reps)
    out = {"layer_port_tokens_per_s": layer_tps, "layer_sample_tokens": REF_SAMPLE_TOKENS}
    mb = ref_arm.load_reference()
    if mb is not None:
        r = make_routing(shape, args.tokens, args.micro_batches, world, 0, zipf_s=args.zipf, shift=hot_shift(args, cfg))
        out["planner_s_threads1"] = ref_arm.reference_planner_seconds(mb, r.mats, shape, world, group, args.sa_chains,
                                                                      slots, 1, reps=reps)
        out["planner_s_threadsN"] = ref_arm.reference_planner_seconds(mb, r.mats, shape, world, group,
                                                                      args.sa_chains, slots, threads, reps=reps)
        out["planner"] = "moebalance 0.1.0 (oracle/_ref) sim.build_policy_bundle('relibra')"
        planner_s = min(out["planner_s_threads1"], out["planner_s_threadsN"])
    else:
        out["planner"] = "unavailable (oracle/_ref not built: run oracle/build_ref.sh)"
        planner_s = 0.0
    out["step_s"] = planner_s + tokens_step / layer_tps
    out["value"] = tokens_step / out["step_s"]
    out["kind"] = "reference" if mb is not None else "port"
    out["sample"] = (f"per step: the reference's planners on the step's routing ({args.micro_batches} micro-batches x "
                     f"{world} GPUs, {args.sa_chains} SA chains) + the fp32 layer port at the rate of a fixed "
                     f"{REF_SAMPLE_TOKENS}-token sample, scaled to the step's {tokens_step} tokens")
    return out


def hot_shift(args, cfg):
    """Experts the hot set rotates by per micro-batch (config default unless --hot-shift)."""
    return cfg["shift"] if args.hot_shift is None else args.hot_shift


def synthetic_config(args, world):
    """The `config` object of a synthetic-routing run (both arms print the same one)."""
    from paper_2605_08639_b200.workload import SHAPES
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    return {"workload": f"{args.config} MoE layer fwd+bwd, EP={world}, replayed Zipf routing",
            "experts": shape.num_experts, "top_k": shape.top_k, "hidden": shape.hidden, "ffn": shape.ffn,
            "tokens_per_gpu": args.tokens, "micro_batches": args.micro_batches,
            "global_tokens_per_step": world * args.tokens * args.micro_batches, "policy": args.headline,
            "zipf_s": args.zipf, "hot_shift": hot_shift(args, cfg), "ep": world,
            "gpu_group": min(world, args.group or cfg["group"]),
            "replica_slots": cfg["slots"] if args.slots is None else args.slots, "sa_chains": args.sa_chains,
            "reorder_planner": "device" if args.device_planner else "host",
            **data_plane_config(world, shape, args),
            "l2": "inputs larger than L2 (per-step working set >> 126 MB)"}


def data_plane_config(world, shape, args=None):
    """Row-mover engine, SMs left to the comm stream, weight-gradient mode and replica weight
    sets (MoEDataPlane defaults / env overrides)."""
    from paper_2605_08639_b200 import moe_layer as ml
    movers = os.environ.get("MB_ROW_MOVERS") or ml.ROW_MOVERS.get(world, ml.ROW_MOVERS_MULTI)
    out = {"row_movers": movers, "comm_sms": ml.default_comm_sms(world, shape),
           "dispatch_tables": "device" if os.environ.get("MB_DEVICE_TABLES", "1") == "1" else "host",
           "activation": "pre-gated" if ml.PREGATE else "gate in combine"}
    if args is not None:
        out["wgrad_mode"] = args.wgrad_mode
        out["replica_sets"] = args.replica_sets or ml.default_replica_sets(shape)
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path (oracle/_ref
    planners + the fp32 layer port) on this host's cores, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    steps = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_step(args, world, threads)
        if i >= args.warmup:
            steps.append(r)
    value = statistics.median(r["value"] for r in steps)
    last = steps[-1]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(r["step_s"] for r in steps) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": synthetic_config(args, world),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": last["kind"],
                             "sample": last["sample"], "planner": last["planner"],
                             "planner_s_threads1": statistics.median(r.get("planner_s_threads1", 0.0) for r in steps),
                             "planner_s_threadsN": statistics.median(r.get("planner_s_threadsN", 0.0) for r in steps),
                             "layer_port_tokens_per_s": statistics.median(r["layer_port_tokens_per_s"] for r in steps),
                             "spread": (max(r["value"] for r in steps) - min(r["value"] for r in steps)) / value},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm

def _device_inputs(shape, T, MB, rank, routing):
    import torch
    from paper_2605_08639_b200.workload import make_activations
    xh, douth = make_activations(shape, T, MB, rank)
    dev = {"x": xh.cuda(), "dout": douth.cuda(), "idx": torch.from_numpy(routing.idx).cuda(),
           "gates": torch.from_numpy(routing.gates).cuda()}
    dev["out"] = torch.empty_like(dev["x"])
    dev["dx"] = torch.empty_like(dev["x"])
    dev["dgate"] = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")
    return dev


def _make_plane(comm, shape, T, MB, plan, **kw):
    from paper_2605_08639_b200.moe_layer import MoEDataPlane
    from paper_2605_08639_b200.workload import make_weights_for
    dp = MoEDataPlane(comm, shape, T, MB, plan, **kw)
    experts = np.flatnonzero(plan.home == comm.rank)
    wg, wu, wd = make_weights_for(shape, experts)
    dp.set_weights(wg, wu, wd)
    del wg, wu, wd
    dp.zero_grads()
    return dp


def _step(dp, dev):
    # one training step of the layer: optimizer.zero_grad() semantics (lazy: the first gradient
    # contribution stores instead of accumulating), then fwd + bwd over every micro-batch
    dp.zero_grads()
    dp.step(dev["x"], dev["idx"], dev["gates"], dev["dout"], dev["out"], dev["dx"], dev["dgate"])


def _timed_steps(comm, fn, steps):
    """Device time of `steps` calls of fn (CUDA events on the current stream, barrier + sync on
    both sides), max over ranks, per step."""
    import torch
    torch.cuda.synchronize()
    comm.host_barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    comm.host_barrier()
    return comm.max_over_ranks(s.elapsed_time(e) / steps)


def _plan(args, comm, policy, shape, routing, topo, model, cfgs, bundle=None):
    from paper_2605_08639_b200.moe_layer import build_step_plan, plan_digest, step_plan_from_bundle
    t0 = time.perf_counter()
    if bundle is not None:  # plan files (planio.solve / the reference's `solve`)
        plan = step_plan_from_bundle(policy, bundle, routing.mats, shape, layer=args.trace_layer)
    else:
        plan = build_step_plan(policy, routing.mats, topo, model, topo.profile, cfgs, shape)
    plan_ms = (time.perf_counter() - t0) * 1e3
    digests = comm.all_gather_object(plan_digest(plan))
    if len(set(digests)) != 1:
        raise RuntimeError(f"ranks disagree on the step plan: {digests}")
    return plan, plan_ms


def measure_detail(args, comm, dp, dev, plan, topo, model):
    """The headline policy's detailed run: K timed steps with per-launch CUDA events (GEMM kinds,
    comm phases), clocks sampled during the timed region, launch count, then e2e through the
    host-buffer API."""
    import torch
    from paper_2605_08639_b200.comm import local_device
    T, MB = args.tokens, args.micro_batches
    for _ in range(args.warmup):
        _step(dp, dev)
    torch.cuda.synchronize()
    comm.host_barrier()
    sampler = ClockSampler(local_device())
    sampler.start()
    time.sleep(0.15)
    dp.timing = True
    dp.gemm_events = []
    launches0 = dp.launches
    ms = _timed_steps(comm, lambda: _step(dp, dev), args.steps)
    clocks = sampler.stop()
    launches = (dp.launches - launches0) // args.steps
    dp.timing = False
    res = {"ms": ms, "launches": launches, "clocks": clocks, "rows": [dp.real_rows(m) for m in range(MB)],
           "rows_cap": plan.rows_cap}
    gev = [ev for ev in dp.gemm_events if not ev[3].startswith("comm_")]
    res["gemm_ms"] = sum(a.elapsed_time(b) for a, b, _, _ in gev) / args.steps
    res["gemm_flop"] = sum(f for _, _, f, _ in gev) / args.steps
    kinds = {}
    for a, b, f, kd in dp.gemm_events:
        ms_f = kinds.setdefault(kd, [0.0, 0.0])
        ms_f[0] += a.elapsed_time(b) / args.steps
        ms_f[1] += f / args.steps
    res["gemm_kinds"] = {kd: {"ms": round(v[0], 4), "tflops": round(v[1] / v[0] / 1e9, 1)}
                         for kd, v in kinds.items() if not kd.startswith("comm_") and v[0] > 0}
    # comm phases on the comm / copy streams (barriers included): NVLink bytes this rank moves / time
    res["comm_kinds"] = {kd[5:]: {"ms": round(v[0], 4), "nvlink_gb": round(v[1] / 1e9, 4),
                                  "gb_per_s": round(v[1] / v[0] / 1e6, 1) if v[0] > 0 else 0.0}
                         for kd, v in kinds.items() if kd.startswith("comm_")}
    res["gemm_launches"] = len(gev) // args.steps
    if os.environ.get("MB_NVTX_STEP") == "1":
        # one more step inside an NVTX range: ncu --nvtx --nvtx-include "mb_step/" profiles exactly it
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("mb_step")
        _step(dp, dev)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    # e2e through the host-buffer API (pinned host tensors, copies inside the timed region)
    host = {k: v.cpu().pin_memory() for k, v in dev.items()}
    for _ in range(2):
        dp.zero_grads()
        dp.step_host(host, dev)
    comm.host_barrier()
    t0 = time.perf_counter()
    n_e2e = max(2, min(args.steps, 5))
    for _ in range(n_e2e):
        dp.zero_grads()
        dp.step_host(host, dev)
    comm.host_barrier()
    res["e2e_ms"] = comm.max_over_ranks((time.perf_counter() - t0) * 1e3 / n_e2e)
    res["h2d"] = sum(host[k].numel() * host[k].element_size() for k in ("x", "idx", "gates", "dout"))
    res["d2h"] = sum(host[k].numel() * host[k].element_size() for k in ("out", "dx", "dgate"))
    del host
    return res


def check_step(args, comm, dp, dev, plan, shape):
    """--check (test infrastructure, off by default, after every timed region): the last step's
    outputs against the fp32 CPU restatement (oracle/moe_ref.py): out / dx / dgate of the first
    and last micro-batch on every rank; at EP=1 also the gradients of the 8 hottest and 8 coldest
    experts (the oracle needs every rank's tokens for the rest).  Returns {name: metrics}."""
    import torch
    from oracle import moe_ref
    from paper_2605_08639_b200.moe_layer import deinterleave_w1
    from paper_2605_08639_b200.workload import make_weights_for
    E, MB = shape.num_experts, args.micro_batches
    _step(dp, dev)
    dp.check(sync=True)
    wg, wu, wd = make_weights_for(shape, np.arange(E))
    out = {}
    for m in sorted({0, MB - 1}):
        ref = moe_ref.moe_layer_fp32(dev["x"][m], dev["idx"][m], dev["gates"][m], wg, wu, wd, dev["dout"][m])
        for key in ("out", "dx", "dgate"):
            out[f"{key}_mb{m}"] = moe_ref.close(dev[key][m], ref[key])
        del ref
    if comm.world == 1:
        load = plan.mats.sum(axis=(0, 1))
        order = np.argsort(-load, kind="stable")
        sel = torch.from_numpy(np.concatenate([order[:8], order[-8:]])).cuda()
        gsum = None
        for m in range(MB):
            keep = torch.isin(dev["idx"][m], sel)
            idx_m = torch.where(keep, dev["idx"][m], torch.full_like(dev["idx"][m], -1))
            r = moe_ref.moe_layer_fp32(dev["x"][m], idx_m, dev["gates"][m], wg, wu, wd, dev["dout"][m])
            g = (r["dWg"][sel], r["dWu"][sel], r["dWd"][sel])
            gsum = g if gsum is None else tuple(a + b for a, b in zip(gsum, g))
        gW1, gW2 = dp.grads()
        g_gate, g_up = deinterleave_w1(gW1[sel])
        for key, got, ref in (("dWg", g_gate, gsum[0]), ("dWu", g_up, gsum[1]), ("dWd", gW2[sel], gsum[2])):
            out[key + "_16_experts"] = moe_ref.expert_grads_close(got, ref)
    res = {k: {kk: (round(vv, 6) if isinstance(vv, float) else vv) for kk, vv in v.items()} for k, v in out.items()}
    oks = comm.all_gather_object(all(v["ok"] for v in out.values()))
    res["ok"] = bool(all(oks))
    return res


def measure_sequence(args, comm, shape, cfg, topo, model, cfgs):
    """Replay a sequence of batches whose hot set keeps shifting (each batch continues the
    micro-batch rotation of the last one); a batch is --batch-steps training steps under one
    plan.  Every batch is planned from its own routing, and expert migration -- bf16 weights,
    fp32 master weights and both Adam moments, the state an optimizer step leaves, moved by
    MoEDataPlane.migrate -- happens at every batch boundary inside the timed region
    (PAPER.md:390-392, 1081-1084).  Arms: "relibra_fresh" re-anneals every batch from scratch
    (the reference's planner: every batch's plan is independent, so most experts move);
    "relibra" prices migration into the choice (moe_layer.migration_aware_step_plan: the new
    annealed plan relabeled for overlap, or the current placement, whichever models faster
    over the batch including its migration); "static" never moves."""
    import torch
    from paper_2605_08639_b200.kernels import expert_histogram
    from paper_2605_08639_b200.moe_layer import gather_routing, migration_aware_step_plan
    from paper_2605_08639_b200.workload import make_routing
    rank, world = comm.rank, comm.world
    T, MB, NB, S = args.tokens, args.micro_batches, args.batches, args.batch_steps
    pdim = 3 * shape.hidden * shape.ffn
    state = {"master": ((pdim,), torch.float32), "adam_m": ((pdim,), torch.float32),
             "adam_v": ((pdim,), torch.float32)}
    bytes_per_expert = pdim * (2 + 3 * 4)
    routings = []
    for b in range(NB):
        r = make_routing(shape, T, MB, world, rank, zipf_s=args.zipf, shift=hot_shift(args, cfg), all_ranks=False,
                         mb_offset=b * MB)
        counts, _ = expert_histogram(torch.from_numpy(r.idx).cuda(), shape.num_experts)
        r.mats = gather_routing(comm, counts.cpu().numpy().astype(np.int64))
        routings.append(r)
    out = {}
    for arm in ("relibra", "relibra_fresh", "static"):
        plans, plan_ms, choices = [], [], []
        for b, r in enumerate(routings):
            if arm == "relibra" and b > 0:
                t0 = time.perf_counter()
                p, info = migration_aware_step_plan(plans[-1], r.mats, topo, model, topo.profile, cfgs, shape,
                                                    bytes_per_expert, steps_per_batch=S)
                ms = (time.perf_counter() - t0) * 1e3
                choices.append(info["choice"])
            else:
                p, ms = _plan(args, comm, "static" if arm == "static" else "relibra", shape, r, topo, model, cfgs)
            plans.append(p)
            plan_ms.append(ms)
        digests = comm.all_gather_object([plan_digest_of(p) for p in plans])
        if any(d != digests[0] for d in digests):
            raise RuntimeError("ranks disagree on the batch plans")
        dp = _make_plane(comm, shape, T, MB, plans[0], rows_cap=max(p.rows_cap for p in plans), expert_state=state,
                         wgrad_mode=args.wgrad_mode, replica_sets=args.replica_sets)
        tables = [dp.build_tables(p) for p in plans]
        devs = [_device_inputs(shape, T, MB, rank, r) for r in routings]
        moved = [0, 0]
        counting = [False]

        def switch(b):
            info = dp.migrate(tables[b], grads=False)   # after the optimizer step: gradients are zero
            if counting[0]:
                moved[0] += info["bytes_in"]
                moved[1] += info["experts_moved"]

        def run_sequence():
            for b in range(NB):
                if b:
                    switch(b)
                for _ in range(S):
                    _step(dp, devs[b])

        for _ in range(args.warmup):   # warm-up pass (also back to batch 0's placement below)
            _step(dp, devs[0])
        run_sequence()
        switch(0)
        total = []
        for rep_i in range(args.repeats):
            counting[0] = rep_i == 0          # moves of one pass over the sequence
            total.append(_timed_steps(comm, run_sequence, 1))
            counting[0] = False
            switch(0)   # not timed: back to batch 0's placement for the next repetition
        # the migrations alone (same moves, no steps): their share of the sequence
        mig_ms = _timed_steps(comm, lambda: [switch(b) for b in list(range(1, NB)) + [0]], 1) * (NB - 1) / NB
        tokens = world * T * MB * NB * S
        med = statistics.median(total)
        out[arm] = {"tokens_per_s": tokens / (med / 1e3), "ms_per_step": med / (NB * S),
                    "ms_per_step_min": min(total) / (NB * S), "ms_per_step_max": max(total) / (NB * S),
                    "migration_ms_per_batch": round(mig_ms / max(1, NB - 1), 4),
                    "migration_share": round(mig_ms / med, 4),
                    "experts_moved_in_per_batch_rank0": round(moved[1] / max(1, NB - 1), 2),
                    "migration_gb_in_per_batch_rank0": round(moved[0] / max(1, NB - 1) / 1e9, 4),
                    "planner_ms_per_batch": round(statistics.mean(plan_ms), 2),
                    "skew": round(float(np.mean([p.skew() for p in plans])), 4)}
        if choices:
            out[arm]["plan_choices"] = choices
        dp.close()
        del dp, devs, tables
        gc.collect()
        torch.cuda.empty_cache()
    for arm in ("relibra", "relibra_fresh"):
        out[arm]["speedup_vs_static"] = round(out["static"]["ms_per_step"] / out[arm]["ms_per_step"], 4)
    out["batches"], out["steps_per_batch"] = NB, S
    out["state_per_expert_bytes"] = bytes_per_expert
    out["state_per_expert"] = "bf16 weights + fp32 master weights + Adam m, v (what an optimizer step leaves)"
    return out


def plan_digest_of(plan):
    from paper_2605_08639_b200.moe_layer import plan_digest
    return plan_digest(plan)


def run_ours(args, comm):
    import torch
    from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs
    from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile
    from paper_2605_08639_b200.kernels import expert_histogram
    from paper_2605_08639_b200.moe_layer import gather_routing
    from paper_2605_08639_b200.replication import replica_memory
    from paper_2605_08639_b200.workload import SHAPES, make_routing
    rank, world = comm.rank, comm.world
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    group = min(world, args.group or cfg["group"])
    topo = b200_box_topology(world, group, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    slots = cfg["slots"] if args.slots is None else args.slots
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=tuple(range(args.sa_chains))), replica=ReplicaConfig(slots),
                      threads=1, device_anneal=args.device_planner)   # tasks in parallel threads measured slower (numpy BLAS lock)
    trace, bundle = None, None
    if args.trace:
        # replay a recorded count trace (routing.bin + manifest.json, either implementation):
        # tokens are realised per (micro-batch, source GPU) row with exactly the recorded counts
        from paper_2605_08639_b200 import planio
        from paper_2605_08639_b200.moe_layer import LayerShape
        from paper_2605_08639_b200.traces import load_trace
        trace = load_trace(args.trace)
        if trace.topo.num_gpus != world:
            raise SystemExit(f"trace has {trace.topo.num_gpus} GPUs, run with --gpus {trace.topo.num_gpus}")
        if trace.tokens_per_gpu <= 0:
            raise SystemExit("variable-token traces cannot be replayed on fixed token buffers")
        tm = trace.model
        shape = LayerShape(tm.num_experts, tm.top_k, tm.hidden_size, tm.intermediate_size)
        topo, group = trace.topo, trace.topo.gpus_per_node
        model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
        cfg = {"shape": shape, "shift": 0, "slots": slots, "group": group}
        args.micro_batches = trace.num_micro_batches
        trace_mats = trace.matrices.astype(np.int64)
        if args.plans:
            bundle = planio.load_plan_bundle(args.plans, trace)
            if bundle.sample_placement is not None:
                # data-locality placement: samples (and their tokens) start on their new GPUs
                from paper_2605_08639_b200.reordering import rewrite_trace_matrices
                trace_mats = rewrite_trace_matrices(trace, bundle.sample_placement).astype(np.int64)
        # token buffers hold the largest (micro-batch, GPU) row; shorter rows are padded with
        # dropped tokens (idx -1: no histogram count, no dispatch, zero output)
        args.tokens = int(trace_mats[:, args.trace_layer].sum(axis=-1).max()) // shape.top_k
    T, MB = args.tokens, args.micro_batches

    def routing_for(balanced):
        # each rank draws its own replayed routing, histograms it on the GPU (K1) and all-gathers
        # the counts into the (MB, G, E) trace every planner sees
        if trace is not None and not balanced:
            from paper_2605_08639_b200.traces import realize_tokens
            from paper_2605_08639_b200.workload import Routing
            idx = np.full((MB, T, shape.top_k), -1, dtype=np.int32)
            gts = np.zeros((MB, T, shape.top_k), dtype=np.float32)
            for m in range(MB):
                i_m, g_m = realize_tokens(trace_mats[m, args.trace_layer, rank], shape.top_k, seed=m * world + rank)
                idx[m, :len(i_m)], gts[m, :len(g_m)] = i_m, g_m
            r = Routing(idx=idx, gates=gts, mats=None)
        else:
            r = make_routing(shape, T, MB, world, rank, zipf_s=args.zipf, shift=hot_shift(args, cfg), balanced=balanced,
                             all_ranks=False)
        counts, _ = expert_histogram(torch.from_numpy(r.idx).cuda(), shape.num_experts)
        r.mats = gather_routing(comm, counts.cpu().numpy().astype(np.int64))
        if trace is not None and not balanced and not np.array_equal(r.mats, trace_mats[:, args.trace_layer]):
            raise RuntimeError("device histogram of the realised tokens differs from the trace counts")
        return r

    skewed = routing_for(False)
    balanced = routing_for(True)
    policies = [p for p in args.policies.split(",") if p]
    policies = [args.headline] + [p for p in policies if p != args.headline]
    if "relibra_box" in policies and group == world:
        policies.remove("relibra_box")   # one group already spans the box
    dp_kw = {"wgrad_mode": args.wgrad_mode, "replica_sets": args.replica_sets}

    def plan_of(pol):
        routing = balanced if pol == "balanced_oracle" else skewed
        if pol == "relibra_box":  # ReLibra with the whole NVSwitch box as one replication group
            box = b200_box_topology(world, world, b200_profile(shape.hidden))
            return routing, _plan(args, comm, "relibra", shape, routing, box, model, cfgs)
        return routing, _plan(args, comm, pol, shape, routing, topo, model, cfgs,
                              bundle=bundle if pol == "relibra" else None)

    # ---- headline: detailed run (per-launch events, clocks, e2e)
    routing, (plan, plan_ms) = plan_of(args.headline)
    dp = _make_plane(comm, shape, T, MB, plan, **dp_kw)
    dev = _device_inputs(shape, T, MB, rank, routing)
    head = measure_detail(args, comm, dp, dev, plan, topo, model)
    head["memory"] = dp.memory_report()
    check = check_step(args, comm, dp, dev, plan, shape) if args.check else None
    dp.close()
    del dp, dev
    gc.collect()
    torch.cuda.empty_cache()
    # ---- every policy on the same routing, interleaved: repeat r runs the policies in rotated
    # order (ABCD, BCDA, ...), each a fresh data plane with W warm-up and K timed steps
    results, failed, plans = {}, {}, {}
    for pol in policies:
        try:
            plans[pol] = plan_of(pol)
        except Exception as err:  # a comparison policy must not cost the headline line
            if pol == args.headline:
                raise
            failed[pol] = f"{type(err).__name__}: {err}"[:300]
    live = [p for p in policies if p in plans]
    times = {p: [] for p in live}
    for rep in range(args.repeats):
        for i in range(len(live)):
            pol = live[(i + rep) % len(live)]
            routing, (plan_p, pms) = plans[pol]
            try:
                dpp = _make_plane(comm, shape, T, MB, plan_p, **dp_kw)
                devp = _device_inputs(shape, T, MB, rank, routing)
                for _ in range(args.warmup):
                    _step(dpp, devp)
                times[pol].append(_timed_steps(comm, lambda: _step(dpp, devp), args.steps))
                dpp.close()
                del dpp, devp
            except Exception as err:
                if pol == args.headline:
                    raise
                failed[pol] = f"{type(err).__name__}: {err}"[:300]
            gc.collect()
            torch.cuda.empty_cache()
    for pol in live:
        if not times[pol]:
            continue
        plan_p, pms = plans[pol][1]
        med = statistics.median(times[pol])
        results[pol] = {"ms": med, "ms_min": min(times[pol]), "ms_max": max(times[pol]), "runs": len(times[pol]),
                        "plan_ms": pms, "skew": plan_p.skew(), "predicted_ms": plan_p.predicted_ms(topo, model,
                                                                                                     topo.profile)}
    tokens_step = world * T * MB
    ms_head = results[args.headline]["ms"]
    value = tokens_step / (ms_head / 1e3)
    peaks, peak_src = load_peaks()
    peak_tf = float(peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"]))
    gemm_tflops = head["gemm_flop"] / (head["gemm_ms"] / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_head, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": synthetic_config(args, world) if trace is None else {
            "workload": (f"trace {trace.trace_id()} layer {args.trace_layer} MoE layer fwd+bwd, EP={world}"
                         + (", plans from files" if bundle is not None else "")),
            "experts": shape.num_experts, "top_k": shape.top_k, "hidden": shape.hidden, "ffn": shape.ffn,
            "tokens_per_gpu": T, "micro_batches": MB, "global_tokens_per_step": tokens_step,
            "policy": args.headline, "ep": world, "gpu_group": group, "replica_slots": slots,
            "sa_chains": args.sa_chains, **data_plane_config(world, shape, args),
            "l2": "inputs larger than L2 (per-step working set >> 126 MB)"},
        "timing": (f"value / ms_per_step = median of {args.repeats} interleaved runs of {args.steps} timed steps "
                   f"(each after {args.warmup} warm-up steps; CUDA events, max over ranks); the headline's first "
                   f"extra run ({head['ms']:.3f} ms/step) carries the per-launch events, clocks and e2e"),
        "roofline": {"kernel": "K4 tcgen05 grouped GEMM (all fwd/dgrad/wgrad launches of the step)",
                     "bound": "tensor", "achieved": round(gemm_tflops, 1), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(gemm_tflops / peak_tf, 4),
                     "traffic": (None if trace is not None else
                                 k4_traffic_per_step(args.config, world, args.tokens, args.micro_batches)),
                     "traffic_unit": f"DRAM bytes per step over all K4 launches (ncu, {os.path.relpath(K4_TRAFFIC, ROOT)})",
                     "peak_source": f"bf16_tflops_sustained, {peak_src}",
                     "flops_per_step": head["gemm_flop"], "gemm_ms_per_step": round(head["gemm_ms"], 4),
                     "gemm_share_of_step": round(head["gemm_ms"] / head["ms"], 4),
                     "per_kind": head["gemm_kinds"]},
        "comm": head["comm_kinds"],
        "e2e": {"value": tokens_step / (head["e2e_ms"] / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": head["h2d"],
                "d2h_bytes_per_step": head["d2h"], "ms_per_step": head["e2e_ms"],
                "note": ("host<->device copies of every micro-batch inside the timed region (pinned memory); "
                         "at N>1 all ranks share the host's memory bandwidth")},
        "gpu_launches": head["launches"],
        "clocks": head["clocks"],
        "memory": dict(head["memory"], replica_memory_layer_shared=replica_memory(model, ReplicaConfig(slots),
                                                                                  "layer-shared")),
        "balance": {p: {"tokens_per_s": tokens_step / (r["ms"] / 1e3), "ms_per_step": r["ms"],
                        "ms_min": r["ms_min"], "ms_max": r["ms_max"], "runs": r["runs"], "skew": r["skew"],
                        "planner_ms": r["plan_ms"], "model_predicted_ms": round(r["predicted_ms"], 4)}
                    for p, r in results.items()},
    }
    if failed:
        line["balance"]["failed"] = failed
    if "static" in results:
        line["balance"]["speedup_vs_static"] = results["static"]["ms"] / ms_head
        line["balance"]["model_predicted_speedup_vs_static"] = (results["static"]["predicted_ms"]
                                                                / results[args.headline]["predicted_ms"])
    if "balanced_oracle" in results:
        line["balance"]["frac_of_balanced"] = results["balanced_oracle"]["ms"] / ms_head
        line["balance"]["model_predicted_frac_of_balanced"] = (results["balanced_oracle"]["predicted_ms"]
                                                               / results[args.headline]["predicted_ms"])
    if args.batches > 1 and trace is None:
        seq = measure_sequence(args, comm, shape, cfg, topo, model, cfgs)
        line["balance"]["shifting_batches"] = seq
        line["balance"]["relibra_with_migration"] = seq["relibra"]["tokens_per_s"]
        line["balance"]["relibra_fresh_with_migration"] = seq["relibra_fresh"]["tokens_per_s"]
    if check is not None:
        line["check"] = check
    if rank == 0 and world == 1 and not args.no_cpu_baseline and trace is None:
        r = cpu_reference_step(args, world, os.cpu_count() or 1, reps=2)
        line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": os.cpu_count(), "kind": r["kind"],
                                "sample": r["sample"], "planner": r["planner"],
                                **{k: r[k] for k in ("planner_s_threads1", "planner_s_threadsN",
                                                     "layer_port_tokens_per_s") if k in r}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if check is not None and not check["ok"]:
        raise SystemExit("--check: the timed configuration differs from the fp32 oracle")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen3-30b-a3b")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--micro-batches", type=int, default=8)
    ap.add_argument("--zipf", type=float, default=1.0)
    ap.add_argument("--hot-shift", type=int, default=None,
                    help="experts the hot set rotates by per micro-batch (default: the config's)")
    ap.add_argument("--slots", type=int, default=None)
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--sa-chains", type=int, default=8)
    ap.add_argument("--policies", default="relibra,static,eplb_like,balanced_oracle,relibra_box",
                    help="relibra_box = relibra with one replication group spanning all EP GPUs (run when EP > group)")
    ap.add_argument("--headline", default="relibra")
    ap.add_argument("--repeats", type=int, default=5,
                    help="interleaved repetitions of every policy (rotated order); value = the headline's median")
    ap.add_argument("--batches", type=int, default=4,
                    help="batches of the shifting-routing sequence (new plan + expert migration per batch); 1 = off")
    ap.add_argument("--batch-steps", type=int, default=4, help="training steps per batch of the sequence")
    ap.add_argument("--wgrad-mode", default="step", choices=["step", "micro_batch"])
    ap.add_argument("--replica-sets", type=int, default=None)
    ap.add_argument("--check", action="store_true",
                    help="after the timed runs, compare the last step with the fp32 oracle (test infrastructure)")
    ap.add_argument("--device-planner", action="store_true",
                    help="run the reorder planner's annealing chains on the GPU (identical plans)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", default=None, help="replay a recorded routing trace directory (manifest.json + "
                    "routing.bin) instead of synthetic Zipf routing")
    ap.add_argument("--trace-layer", type=int, default=0)
    ap.add_argument("--plans", default=None, help="with --trace: relibra uses the reorder.json / replication.json "
                    "of this solve output directory instead of planning")
    args = ap.parse_args()
    if args.headline not in args.policies.split(","):
        args.policies = args.headline + "," + args.policies
    if args.warmup < 3 and args.impl == "ours":
        print("bench: --warmup < 3 is below the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "reference":
        env_world = str(args.gpus)    # the CPU arm runs on rank 0 only: nothing to launch
    if env_world is None and args.gpus > 1:
        # `python bench.py --gpus N`: launch N ranks (one process per GPU, NCCL) ourselves
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(env_world or "1")
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; launch one process per GPU")
    rank = int(os.environ.get("RANK", "0"))
    if os.environ.get("NCCL_DEBUG") and not os.environ.get("NCCL_DEBUG_FILE"):
        # NCCL's log goes to stderr: stdout carries exactly one JSON line
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    from paper_2605_08639_b200.comm import init_distributed
    if world == 1:
        torch.cuda.set_device(0)
    comm = init_distributed()
    try:
        run_ours(args, comm)
    finally:
        if comm.dist:
            comm.dist.barrier()
            comm.dist.destroy_process_group()


if __name__ == "__main__":
    main()
