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


K4_TRAFFIC = os.path.join(ROOT, "profiles", "r01_launches_step2_summary.json")


def k4_traffic_per_step(config: str, world: int, tokens: int, mbs: int):
    """DRAM bytes (read + write) of every K4 launch of one step, from the committed ncu launch
    list of this same bench command (dram__bytes_read.sum + dram__bytes_write.sum per launch);
    None for other configurations (no capture)."""
    if (config, world, tokens, mbs) != ("qwen3-30b-a3b", 1, 8192, 8):
        return None
    try:
        rows = json.load(open(K4_TRAFFIC))
    except (OSError, ValueError):
        return None
    total = 0.0
    for key, r in rows.items():
        if not key.startswith("K4"):
            continue
        per_step = 2 if key.endswith("<1, 1, 1, 3>") else mbs   # wgrad: 2 launches per step
        total += (r["dram_read_per_launch"] + r["dram_write_per_launch"]) * per_step
    return total


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

def cpu_reference_sample(cfg_name: str, tokens: int, world: int, zipf: float, budget_s: float, threads: int):
    """The CPU path on a bounded sample (oracle port): np.bincount histogram + the fp32 layer
    fwd+bwd (SwiGLU experts, gate-weighted combine) on a token sample, all host threads.  The
    reference's planners are not in this arm (they cannot travel to the GPU box); their cost is
    measured beside the native planners in profiles/r01_planner_timing.json.
    Returns (tokens/s, sample description)."""
    import torch
    from oracle import moe_ref
    from paper_2605_08639_b200.workload import SHAPES, make_activations, make_routing, make_weights
    torch.set_num_threads(threads)
    cfg = SHAPES[cfg_name]
    shape = cfg["shape"]
    n = 256
    wg, wu, wd = make_weights(shape)
    done_tokens, elapsed = 0, 0.0
    while elapsed < budget_s:
        r = make_routing(shape, n, 1, 1, 0, zipf_s=zipf, shift=cfg["shift"])
        x, dout = make_activations(shape, n, 1, 0)
        t0 = time.perf_counter()
        moe_ref.histogram(r.idx[0], shape.num_experts)
        moe_ref.moe_layer_fp32(x[0], torch.from_numpy(r.idx[0]), torch.from_numpy(r.gates[0]), wg, wu, wd, dout[0])
        dt = time.perf_counter() - t0
        elapsed += dt
        done_tokens += n
        if dt < budget_s / 8:
            n *= 2
    tps = done_tokens / elapsed
    return tps, f"{done_tokens} tokens of {cfg_name} (1 GPU's share), fp32 torch CPU fwd+bwd + bincount, {elapsed:.1f}s"


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
            **data_plane_config(world, shape),
            "l2": "inputs larger than L2 (per-step working set >> 126 MB)"}


def data_plane_config(world, shape):
    """Row-mover engine and SMs left to the comm stream (MoEDataPlane defaults / env overrides)."""
    from paper_2605_08639_b200 import moe_layer as ml
    movers = os.environ.get("MB_ROW_MOVERS") or ml.ROW_MOVERS.get(world, ml.ROW_MOVERS_MULTI)
    return {"row_movers": movers, "comm_sms": ml.default_comm_sms(world, shape)}


def run_reference(args, rank, world):
    import torch
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        tps, sample = cpu_reference_sample(args.config, args.tokens, world, args.zipf,
                                           budget_s=2.0 if i < args.warmup else 4.0, threads=threads)
        if i >= args.warmup:
            vals.append(tps)
    # whole-job throughput: every GPU's share is independent CPU work on the same host
    value = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": synthetic_config(args, world),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm

def measure_policy(args, comm, policy, shape, cfg, routing, topo, model, cfgs, want_detail, bundle=None):
    import torch
    from paper_2605_08639_b200.comm import local_device
    from paper_2605_08639_b200.moe_layer import MoEDataPlane, build_step_plan, plan_digest
    from paper_2605_08639_b200.workload import make_activations, make_weights_for
    rank, world = comm.rank, comm.world
    T, MB = args.tokens, args.micro_batches
    t0 = time.perf_counter()
    if bundle is not None:  # plan files (planio.solve / the reference's `solve`)
        from paper_2605_08639_b200.moe_layer import step_plan_from_bundle
        plan = step_plan_from_bundle(policy, bundle, routing.mats, shape, layer=args.trace_layer)
    else:
        plan = build_step_plan(policy, routing.mats, topo, model, topo.profile, cfgs, shape)
    plan_ms = (time.perf_counter() - t0) * 1e3
    digests = comm.all_gather_object(plan_digest(plan))
    if len(set(digests)) != 1:
        raise RuntimeError(f"ranks disagree on the step plan: {digests}")
    dp = MoEDataPlane(comm, shape, T, MB, plan)
    experts = np.flatnonzero(plan.home == rank)
    wg, wu, wd = make_weights_for(shape, experts)
    dp.set_weights(wg, wu, wd)
    del wg, wu, wd
    dp.zero_grads()
    xh, douth = make_activations(shape, T, MB, rank)
    dev = {"x": xh.cuda(), "dout": douth.cuda(), "idx": torch.from_numpy(routing.idx).cuda(),
           "gates": torch.from_numpy(routing.gates).cuda()}
    dev["out"] = torch.empty_like(dev["x"])
    dev["dx"] = torch.empty_like(dev["x"])
    dev["dgate"] = torch.empty(MB, T, shape.top_k, dtype=torch.float32, device="cuda")

    def step():
        # one training step of the layer: optimizer.zero_grad() semantics (lazy: the weight-gradient
        # GEMMs store instead of accumulating), then fwd + bwd over every micro-batch
        dp.zero_grads()
        dp.step(dev["x"], dev["idx"], dev["gates"], dev["dout"], dev["out"], dev["dx"], dev["dgate"])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    comm.host_barrier()
    sampler = ClockSampler(local_device()) if want_detail else None
    if sampler:
        sampler.start()
        time.sleep(0.15)
    dp.timing = want_detail
    dp.gemm_events = []
    launches0 = dp.launches
    torch.cuda.synchronize()
    comm.host_barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    comm.host_barrier()
    clocks = sampler.stop() if sampler else None
    ms = s.elapsed_time(e) / args.steps
    launches = (dp.launches - launches0) // args.steps
    dp.timing = False
    ms_max = comm.max_over_ranks(ms)
    res = {"ms": ms_max, "plan_ms": plan_ms, "skew": plan.skew(), "launches": launches,
           "predicted_ms": plan.predicted_ms(topo, model, topo.profile),
           "rows": [dp.real_rows(m) for m in range(MB)], "rows_cap": plan.rows_cap}
    if want_detail:
        gev = [ev for ev in dp.gemm_events if not ev[3].startswith("comm_")]
        cev = [ev for ev in dp.gemm_events if ev[3].startswith("comm_")]
        gemm_ms = sum(a.elapsed_time(b) for a, b, _, _ in gev) / args.steps
        gemm_flop = sum(f for _, _, f, _ in gev) / args.steps
        kinds = {}
        for a, b, f, kd in dp.gemm_events:
            ms_f = kinds.setdefault(kd, [0.0, 0.0])
            ms_f[0] += a.elapsed_time(b) / args.steps
            ms_f[1] += f / args.steps
        res["gemm_kinds"] = {kd: {"ms": round(v[0], 4), "tflops": round(v[1] / v[0] / 1e9, 1)}
                             for kd, v in kinds.items() if not kd.startswith("comm_")}
        # comm phases on the comm stream (barriers included): NVLink bytes this rank moves / time
        res["comm_kinds"] = {kd[5:]: {"ms": round(v[0], 4), "nvlink_gb": round(v[1] / 1e9, 4),
                                      "gb_per_s": round(v[1] / v[0] / 1e6, 1) if v[0] > 0 else 0.0}
                             for kd, v in kinds.items() if kd.startswith("comm_")}
        res.update(gemm_ms=gemm_ms, gemm_flop=gemm_flop, gemm_launches=len(gev) // args.steps,
                   clocks=clocks)
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
        e2e_ms = (time.perf_counter() - t0) * 1e3 / n_e2e
        e2e_ms = comm.max_over_ranks(e2e_ms)
        res["e2e_ms"] = e2e_ms
        res["h2d"] = sum(host[k].numel() * host[k].element_size() for k in ("x", "idx", "gates", "dout"))
        res["d2h"] = sum(host[k].numel() * host[k].element_size() for k in ("out", "dx", "dgate"))
        del host
    dp.close()
    del dp, dev
    gc.collect()
    torch.cuda.empty_cache()
    return res


def run_ours(args, comm):
    import torch
    from paper_2605_08639_b200 import AnnealConfig, ModelProfile, ReplicaConfig, SimConfigs
    from paper_2605_08639_b200.cluster import b200_box_topology, b200_profile
    from paper_2605_08639_b200.kernels import expert_histogram
    from paper_2605_08639_b200.moe_layer import gather_routing
    from paper_2605_08639_b200.workload import SHAPES, make_routing
    rank, world = comm.rank, comm.world
    cfg = SHAPES[args.config]
    shape = cfg["shape"]
    group = min(world, args.group or cfg["group"])
    topo = b200_box_topology(world, group, b200_profile(shape.hidden))
    model = ModelProfile(1, shape.num_experts, shape.top_k, shape.hidden, shape.ffn)
    slots = cfg["slots"] if args.slots is None else args.slots
    cfgs = SimConfigs(anneal=AnnealConfig(seeds=tuple(range(args.sa_chains))), replica=ReplicaConfig(slots),
                      threads=min(8, os.cpu_count() or 1), device_anneal=args.device_planner)
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
    results = {}
    failed = {}
    policies = [args.headline] + [p for p in policies if p != args.headline]   # headline first
    for pol in policies:
        routing = balanced if pol == "balanced_oracle" else skewed
        try:
            if pol == "relibra_box":
                # ReLibra with the whole NVSwitch box as one replication group (group = EP)
                if group == world:
                    continue
                box = b200_box_topology(world, world, b200_profile(shape.hidden))
                results[pol] = measure_policy(args, comm, "relibra", shape, cfg, routing, box, model, cfgs,
                                              want_detail=False)
                continue
            results[pol] = measure_policy(args, comm, pol, shape, cfg, routing, topo, model, cfgs,
                                          want_detail=(pol == args.headline),
                                          bundle=bundle if pol == "relibra" else None)
        except Exception as err:  # a comparison policy must not cost the headline line
            if pol == args.headline:
                raise
            failed[pol] = f"{type(err).__name__}: {err}"[:300]
            torch.cuda.synchronize()
    head = results[args.headline]
    tokens_step = world * T * MB
    value = tokens_step / (head["ms"] / 1e3)
    peaks, peak_src = load_peaks()
    peak_tf = float(peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"]))
    gemm_tflops = head["gemm_flop"] / (head["gemm_ms"] / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": synthetic_config(args, world) if trace is None else {
            "workload": (f"trace {trace.trace_id()} layer {args.trace_layer} MoE layer fwd+bwd, EP={world}"
                         + (", plans from files" if bundle is not None else "")),
            "experts": shape.num_experts, "top_k": shape.top_k, "hidden": shape.hidden, "ffn": shape.ffn,
            "tokens_per_gpu": T, "micro_batches": MB, "global_tokens_per_step": tokens_step,
            "policy": args.headline, "ep": world, "gpu_group": group, "replica_slots": slots,
            "sa_chains": args.sa_chains, **data_plane_config(world, shape),
            "l2": "inputs larger than L2 (per-step working set >> 126 MB)"},
        "roofline": {"kernel": "K4 tcgen05 grouped GEMM (all fwd/dgrad/wgrad launches of the step)",
                     "bound": "tensor", "achieved": round(gemm_tflops, 1), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(gemm_tflops / peak_tf, 4),
                     "traffic": (None if trace is not None else
                                 k4_traffic_per_step(args.config, world, args.tokens, args.micro_batches)),
                     "traffic_unit": "DRAM bytes per step over all K4 launches (ncu, profiles/"
                                     "r01_launches_step2_summary.json)",
                     "peak_source": f"bf16_tflops_sustained, {peak_src}",
                     "flops_per_step": head["gemm_flop"], "gemm_ms_per_step": round(head["gemm_ms"], 4),
                     "gemm_share_of_step": round(head["gemm_ms"] / head["ms"], 4),
                     "per_kind": head["gemm_kinds"]},
        "comm": head["comm_kinds"],
        "e2e": {"value": tokens_step / (head["e2e_ms"] / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": head["h2d"],
                "d2h_bytes_per_step": head["d2h"], "ms_per_step": head["e2e_ms"]},
        "gpu_launches": head["launches"],
        "clocks": head["clocks"],
        "balance": {p: {"tokens_per_s": tokens_step / (r["ms"] / 1e3), "ms_per_step": r["ms"], "skew": r["skew"],
                        "planner_ms": r["plan_ms"], "model_predicted_ms": round(r["predicted_ms"], 4)}
                    for p, r in results.items()},
    }
    if failed:
        line["balance"]["failed"] = failed
    if "static" in results:
        line["balance"]["speedup_vs_static"] = results["static"]["ms"] / head["ms"]
    if "balanced_oracle" in results:
        line["balance"]["frac_of_balanced"] = results["balanced_oracle"]["ms"] / head["ms"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline and trace is None:
        tps, sample = cpu_reference_sample(args.config, T, world, args.zipf, budget_s=args.cpu_budget,
                                           threads=os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": tps, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)


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
    ap.add_argument("--device-planner", action="store_true",
                    help="run the reorder planner's annealing chains on the GPU (identical plans)")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", default=None, help="replay a recorded routing trace directory (manifest.json + "
                    "routing.bin) instead of synthetic Zipf routing")
    ap.add_argument("--trace-layer", type=int, default=0)
    ap.add_argument("--plans", default=None, help="with --trace: relibra uses the reorder.json / replication.json "
                    "of this solve output directory instead of planning")
    args = ap.parse_args()
    if args.headline not in args.policies.split(","):
        args.policies = args.headline + "," + args.policies
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    os.environ["NCCL_DEBUG"] = "WARN"  # keep NCCL's version banner off stdout: one JSON line only
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
