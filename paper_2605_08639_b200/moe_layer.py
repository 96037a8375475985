"""The MoE-layer training step under replayed routing, on B200.

This is the data plane the reference only models (sim.evaluate_bundle, sim.py:89-110:
flow_matrix -> comp = flow.sum(0) -> dispatch/combine link loads -> T = max comp + max comm).
One process per GPU; every rank runs, per step of MB micro-batches:

  K1  expert histogram of the local top-k indices (+ chunk scan)           histogram.cu
  K5  replica weight push into the replica slots of this step (owners)      copy engine, peer
  K2  stable-rank permutation -> (dst GPU, dst row) per (token, choice)    dispatch.cu
  K3  row scatter straight into peer receive buffers (dispatch A2A)         dispatch.cu
  K4  tcgen05 grouped GEMM: H = X W1^T (+SwiGLU), Y = Act W2^T              grouped_gemm*.cu
  K6  combine: out[t] = sum_i gate[t,i] * Y[perm(t,i)] over peer loads      dispatch.cu
  bwd K3 (raw dout scatter) -> K4 dAct with the combine backward fused in its epilogue
      (gate scaling, dgate partials, gate*act) -> K4 dX -> K6 un-permute sum + dgate gather
  once per step: K4 wgrad of every local slot, K contracted over all micro-batches (the fp32
      gradient-accumulation window), then K5^T: owners pull replica gradients from peers.

Two streams: the compute stream runs the GEMMs, the comm stream runs dispatch / combine and
every device barrier (totally ordered per rank), linked by per-micro-batch events, so the
NVLink all-to-all of one micro-batch overlaps the tensor-core work of another (two micro-batches
in flight, see schedule()).  Routing is replayed, so every count, row offset and replica is known
before the step: the host planners run once per step (StepPlan) and the kernels never exchange
sizes.  The same phases run one micro-batch at a time through begin_step / forward_mb /
backward_mb / end_step and the MoELayerFunction autograd entry.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import kernels as K
from . import policies as pol
from . import replication as rep
from . import traces as rt
from .cluster import ClusterTopology, HardwareProfile
from .comm import Comm, SymmetricArena

PAD = 128       # receive-slot row padding = GEMM M tile
# profiling only: skip the row movers (the GEMMs then run on stale / zero rows, which also draws
# less power -- do not read the result as the movers' cost)
_SKIP_ROWS = os.environ.get("MB_PROFILE_SKIP_ROWS", "0") == "1"
# SMs left to the comm stream while the persistent GEMM runs (measured on B200, qwen3 shape:
# N=4 step 24.1 ms with all 148 SMs in the GEMM, 19.7 ms with 28 left free)
# N=1: every SM to the GEMM (the 226 KB operand ring leaves no room for co-resident movers; the
# HBM-local movers fill the SMs between GEMM launches): 19.71 ms/step vs 20.13 with 20 SMs reserved
COMM_SMS = {1: 0, 2: 28, 4: 28}   # N=4 A/B: 28 SMs 18.41-18.60 ms vs 32 SMs 18.75-18.85
COMM_SMS_MULTI = 32                # N >= 8 (most NVLink rows per GPU) keeps the wider split
# Experts with a wide FFN do much more GEMM work per moved row (bytes / FLOP of a step = 4 / (9 h')):
# at h' >= 4096 the TMA movers keep up on 8 SMs (Mixtral-8x7B at N=4: 79.3-79.8 -> 71.8-74.0 ms per
# step with 140 GEMM SMs); Qwen3-235B (h' = 1536) is comm-bound on 16 (68.7-70.0 -> 73.0-73.2 ms).
COMM_SMS_WIDE_FFN = 8
WIDE_FFN = 4096
WIDE_HIDDEN = 4096   # 4096-wide token rows (Qwen3-235B): its N=4 numbers were measured with 32 comm SMs
# sets of the layer-shared replica weight slots (MoEDataPlane replica_sets; MB_REPLICA_SETS overrides):
# one set = exactly the paper's layer-shared buffer (replica_memory "layer-shared"); the backward
# pulls its replicas again.  N=4 Qwen3-30B-A3B (9 MiB experts): 19.40 ms/step with 1 set vs 19.30
# with 2.  Experts above REPLICA_SETS_BIG bytes (Mixtral-8x7B: 336 MiB) get a second set so the
# backward reuses the forward's pull instead of moving the expert over NVLink again.
REPLICA_SETS = 1
REPLICA_SETS_BIG = 64 << 20


def default_replica_sets(shape: "LayerShape") -> int:
    if os.environ.get("MB_REPLICA_SETS"):
        return int(os.environ["MB_REPLICA_SETS"])
    return REPLICA_SETS if 6 * shape.hidden * shape.ffn <= REPLICA_SETS_BIG else 2
# Row-mover engine per world size: "regs" = register-copy kernels (co-resident with the GEMM's
# CTAs on every SM), "tma" = cp.async.bulk kernels, one block on each of the COMM_SMS SMs the
# GEMM leaves free (bulk-copy scatter, register combine with a shared-memory reservation).
# Measured (profiles/r01_comm_engine.txt): at N=4 confined/32 SMs 18.85-19.04 ms
# vs regs 19.2-19.26 per step; at N=1 (HBM-local moves) regs is faster (18.8-19.3 vs >= 20.1).
ROW_MOVERS = {1: "regs"}
ROW_MOVERS_MULTI = "tma"
# with replicas (N>1) the last weight-gradient launch runs on every SM: by then the comm stream
# is idle (N=4: 18.9-19.0 -> 18.7-18.9 ms; at N=1 widening the single launch measured 3% slower).
# MB_WGRAD_ALL_SMS=0: A/B.
WGRAD_ALL_SMS = os.environ.get("MB_WGRAD_ALL_SMS", "1") == "1"
# per-micro-batch replica weight gradients on every SM instead of the GEMM's share (A/B: their
# ~2.4 waves of long tiles on the 60 GEMM clusters leave the last wave 40% full)
REPLICA_WGRAD_ALL_SMS = os.environ.get("MB_REPLICA_WGRAD_ALL_SMS", "0") == "1"
# 128-row tail blocks of odd groups in the single-CTA kernel beside the pair kernel (opt-in,
# MB_TAIL_TILES=1): measured no faster at N=1 (18.55-18.88 vs 18.57-18.78 ms/step; the tail kernel's
# 48 KB stages carry twice the B bytes per SM), so the pair kernel's half tiles stay the default
TAIL_TILES = os.environ.get("MB_TAIL_TILES", "0") == "1"
# non-gated F-mode GEMMs in the single-CTA (cta_group::1) kernel; MB_CTA1_F=0: the pair kernel (A/B)
CTA1_F = os.environ.get("MB_CTA1_F", "1") == "1"
CTA1_DACT = os.environ.get("MB_CTA1_DACT", "0") == "1"   # the gated dAct too (A/B)
# Pre-gated activation: the gate/up GEMM's epilogue writes gate*act, so the down GEMM yields gate*Y,
# the combine is a plain sum and the dAct epilogue no longer rewrites Act for dW2 (MB_PREGATE=0: the
# round-1 layout, gate applied in the combine and gate*act written by dAct)
PREGATE = os.environ.get("MB_PREGATE", "1") != "0"
# both weight gradients in one two-problem launch (mb_grouped_wgrad2); MB_WGRAD_MERGED=0: A/B
WGRAD_MERGED = os.environ.get("MB_WGRAD_MERGED", "1") == "1"
# overlap=False runs every phase in issue order on one stream with all SMs in the GEMM: at world 1
# (local row movers) it measured the same step time as the overlapped schedule (19.6 vs 19.4 ms).
CHUNK = 32      # tokens per permutation chunk
GATE_BLOCK = 128  # gate|up interleave block of W1 rows (= half the 256-wide SwiGLU tile)


@dataclass(frozen=True)
class LayerShape:
    num_experts: int
    top_k: int
    hidden: int
    ffn: int

    def check(self) -> None:
        if self.hidden % 256 or self.ffn % 256:
            raise ValueError("kernels need hidden % 256 == 0 and ffn % 256 == 0")


@dataclass
class MicroBatchPlan:
    placement: rep.ReplicaPlacement
    counts: dict                    # expert -> (G, copies) int64 (round_split)
    route_tab: np.ndarray           # [G][E][maxc][4]
    ncopies: np.ndarray             # [E]
    slot_tab: np.ndarray            # [G][max_slots][4] {row_begin, rows_real, rows_pad, expert}
    slot_w: np.ndarray              # [G][max_slots][2] {weight slot, replica}
    nslots: np.ndarray              # [G]
    total_rows: np.ndarray          # [G]
    flow: np.ndarray                # [G][G] rows src -> dst


@dataclass
class StepPlan:
    """Everything the step needs, identical on every rank (built from the gathered routing)."""

    policy: str
    shape: LayerShape
    world: int
    home: np.ndarray                # (E,) ReorderPlan.assignment
    mbs: list = field(default_factory=list)
    maxc: int = 1
    max_slots: int = 1
    rows_cap: int = PAD
    rep_experts: list = field(default_factory=list)   # per GPU: sorted experts replicated onto it this step
    slots: int = 0
    mats: np.ndarray | None = None  # (MB, G, E) routing counts the plan was built for
    tables: str = "host"            # where the split / dispatch tables were computed ("host" | "device")

    def predicted_ms(self, topo: ClusterTopology, model: rt.ModelProfile, hw: HardwareProfile) -> float:
        """The reference cost model's time for this step (sum over micro-batches of
        costmodel.moe_time, costmodel.py:205-213) with the executed integer splits, for
        predicted-vs-measured reporting (sim.evaluate_bundle, sim.py:64-110)."""
        from . import loads as cm
        total = 0.0
        for m, mbp in enumerate(self.mbs):
            x = self.mats[m].astype(np.float64)
            splits = {}
            for e, cnt in mbp.counts.items():
                col = x[:, e][:, None]
                frac = np.divide(cnt, col, out=np.zeros_like(cnt, dtype=np.float64), where=col > 0)
                frac[x[:, e] == 0, 0] = 1.0
                splits[e] = (np.array(mbp.placement.copies(e)), frac)
            total += cm.moe_time(cm.compute_loads(x, mbp.placement.home, topo, splits=splits), model, hw).t_moe
        return total * 1e3

    def executed_loads(self) -> np.ndarray:
        """(MB, G) GEMM rows per GPU actually executed (= costmodel comp with integer splits)."""
        return np.stack([mb.flow.sum(axis=0) for mb in self.mbs])

    def skew(self) -> float:
        """Mean over micro-batches of max/mean executed GPU load (routing.skewness, routing.py:483-493)."""
        return float(np.mean([rt.skewness(l) for l in self.executed_loads()]))

    def nvlink_rows(self) -> np.ndarray:
        """(MB, G) rows each GPU sends to other GPUs per A2A phase (off-diagonal flow)."""
        return np.stack([mb.flow.sum(axis=1) - np.diag(mb.flow) for mb in self.mbs])


def _device_tables_default() -> bool:
    """Integer split + dispatch tables on the GPU whenever one is present (MB_DEVICE_TABLES=0: host)."""
    return os.environ.get("MB_DEVICE_TABLES", "1") == "1" and torch.cuda.is_available()


def build_step_plan(policy: str, mats: np.ndarray, topo: ClusterTopology, model: rt.ModelProfile,
                    hw: HardwareProfile, cfgs: pol.SimConfigs, shape: LayerShape,
                    device_tables: bool | None = None) -> StepPlan:
    """Plan one step (one batch of MB micro-batches, one layer) from the gathered (MB, G, E)
    routing matrices, with the reference policies (sim.build_policy_bundle, sim.py:214-280).
    'balanced_oracle' is planned like 'static': its token routing must already be uniform.
    device_tables: the integer split and dispatch tables are computed on the GPU
    (mb_dispatch_tables) instead of the host planner library (identical tables); default: on
    when a GPU is present."""
    if device_tables is None:
        device_tables = _device_tables_default()
    trace = rt.build_trace(model, topo, mats[:, None], tokens_per_gpu=0)
    pol_name = "static" if policy == "balanced_oracle" else policy
    bundle, _ = pol.build_policy_bundle(trace, pol_name, topo, model, hw, cfgs)
    return step_plan_from_bundle(policy, bundle, mats, shape, layer=0, slots=cfgs.replica.slots_per_gpu,
                                 device_tables=device_tables)


def _device_dispatch_tables(x: np.ndarray, home: np.ndarray, placement, split, maxc: int, max_slots: int):
    """mb_dispatch_tables for one micro-batch: (counts dict, host tables..., device tables)."""
    g, e = x.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    order = list(placement.replicas.keys())
    ptrs, gpus, fr = [0], [], []
    for ex in order:
        cps = placement.copies(ex)
        frac = np.asarray(split.fractions[ex], dtype=np.float64)
        if frac.shape != (g, len(cps)):
            raise ValueError(f"fractions of expert {ex} have shape {frac.shape}, placement has {len(cps)} copies")
        gpus.extend(cps[1:])
        ptrs.append(len(gpus))
        fr.append(frac.ravel())
    i32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32).reshape(-1), device=dev)
    xd, hd = i32(x), i32(home)
    rep_e, rep_p, rep_g = i32(order if order else [0]), i32(ptrs), i32(gpus if gpus else [0])
    frac_d = torch.as_tensor(np.concatenate(fr) if fr else np.zeros(1), dtype=torch.float64, device=dev)
    ncnt = sum(g * (1 + len(placement.replicas[ex])) for ex in order)
    out = {"counts": torch.zeros(max(1, ncnt), dtype=torch.int64, device=dev),
           "route_tab": torch.empty((g, e, maxc, 4), dtype=torch.int32, device=dev),
           "ncopies": torch.empty(e, dtype=torch.int32, device=dev),
           "slot_tab": torch.empty((g, max_slots, 4), dtype=torch.int32, device=dev),
           "slot_w": torch.empty((g, max_slots, 2), dtype=torch.int32, device=dev),
           "nslots": torch.empty(g, dtype=torch.int32, device=dev),
           "total_rows": torch.empty(g, dtype=torch.int64, device=dev),
           "flow": torch.empty((g, g), dtype=torch.int64, device=dev),
           "error": torch.zeros(1, dtype=torch.int32, device=dev)}
    lib = nat.kernels()
    nat.check(lib.mb_dispatch_tables(g, e, xd.data_ptr(), hd.data_ptr(), len(order), rep_e.data_ptr(),
                                     rep_p.data_ptr(), rep_g.data_ptr(), frac_d.data_ptr(), PAD, maxc, max_slots,
                                     out["counts"].data_ptr(), out["route_tab"].data_ptr(), out["ncopies"].data_ptr(),
                                     out["slot_tab"].data_ptr(), out["slot_w"].data_ptr(), out["nslots"].data_ptr(),
                                     out["total_rows"].data_ptr(), out["flow"].data_ptr(), out["error"].data_ptr(),
                                     nat.stream_ptr()), lib, "mb_dispatch_tables")
    host = {k: v.cpu().numpy() for k, v in out.items()}
    if int(host["error"][0]):
        raise ValueError(f"mb_dispatch_tables: inconsistent plan (error bits {int(host['error'][0])})")
    counts, off = {}, 0
    for ex in order:
        k = 1 + len(placement.replicas[ex])
        counts[ex] = host["counts"][off:off + g * k].reshape(g, k).astype(np.int64)
        off += g * k
    return counts, host, out


def step_plan_from_bundle(policy: str, bundle: pol.PlanBundle, mats: np.ndarray, shape: LayerShape,
                          layer: int = 0, slots: int = 0, device_tables: bool | None = None) -> StepPlan:
    """Device tables of one layer's step from a PlanBundle (planned here, or loaded from the
    reorder.json / replication.json files of planio.solve or the reference's `solve`)."""
    if device_tables is None:
        device_tables = _device_tables_default()
    mbs_n, g, e = mats.shape
    home = np.asarray(bundle.reorder[layer].assignment, dtype=np.int64)
    if slots <= 0:  # loaded plans: the largest per-GPU replica count the files use
        slots = max([0] + [int(ent.placement.slot_usage(g).max())
                           for (mb, l), ent in bundle.replication.entries.items() if l == layer])
    plan = StepPlan(policy=policy, shape=shape, world=g, home=home, slots=slots, mats=np.asarray(mats))
    entries = []
    for mb in range(mbs_n):
        x = mats[mb].astype(np.float64)
        entry = bundle.replication.entries.get((mb, layer))
        if entry is None:
            placement, split = rep.ReplicaPlacement(home=home.copy()), rep.SplitPlan()
        else:
            placement, split = entry.placement, entry.split
        counts = None if device_tables else rep.round_split(split, placement, x)
        entries.append((placement, counts))
    plan.maxc = max([1] + [1 + len(p.replicas.get(ex, [])) for p, _ in entries for ex in p.replicas])
    per_gpu_rep = max([0] + [int(p.slot_usage(g).max()) for p, _ in entries])
    plan.max_slots = e // g + max(1, slots, per_gpu_rep)
    lib = nat.planner()
    if device_tables:
        for mb in range(mbs_n):
            entry = bundle.replication.entries.get((mb, layer))
            placement = entries[mb][0]
            split = entry.split if entry is not None else rep.SplitPlan()
            counts, h, d = _device_dispatch_tables(np.asarray(mats[mb]), home, placement, split, plan.maxc,
                                                   plan.max_slots)
            mbp = MicroBatchPlan(placement, counts, h["route_tab"], h["ncopies"], h["slot_tab"], h["slot_w"],
                                 h["nslots"], h["total_rows"], h["flow"])
            mbp.device = d          # the tables the kernels consume, computed on the GPU
            plan.mbs.append(mbp)
        plan.tables = "device"
    for mb, (placement, counts) in enumerate(entries if not device_tables else []):
        x = np.ascontiguousarray(mats[mb], dtype=np.int64)
        order = list(placement.replicas.keys())
        rep_e = nat.i32(order)
        ptrs, gpus, cnts = [0], [], []
        for ex in order:
            gpus.extend(placement.replicas[ex])
            ptrs.append(len(gpus))
            cnts.append(np.ascontiguousarray(counts[ex], dtype=np.int64).ravel())
        rep_p, rep_g = nat.i32(ptrs), nat.i32(gpus)
        cnt = nat.i64(np.concatenate(cnts) if cnts else np.zeros(0))
        route = np.zeros((g, e, plan.maxc, 4), dtype=np.int32)
        ncop = np.zeros(e, dtype=np.int32)
        slot_tab = np.zeros((g, plan.max_slots, 4), dtype=np.int32)
        slot_w = np.zeros((g, plan.max_slots, 2), dtype=np.int32)
        nslots = np.zeros(g, dtype=np.int32)
        total = np.zeros(g, dtype=np.int64)
        flow = np.zeros((g, g), dtype=np.int64)
        nat.check(lib.mbp_dispatch_plan(g, e, nat.ptr(x), nat.ptr(home), len(order), nat.ptr(rep_e), nat.ptr(rep_p),
                                        nat.ptr(rep_g), nat.ptr(cnt), PAD, plan.maxc, plan.max_slots, nat.ptr(route),
                                        nat.ptr(ncop), nat.ptr(slot_tab), nat.ptr(slot_w), nat.ptr(nslots),
                                        nat.ptr(total), nat.ptr(flow)), lib, "dispatch_plan")
        plan.mbs.append(MicroBatchPlan(placement, counts, route, ncop, slot_tab, slot_w, nslots, total, flow))
    plan.rows_cap = int(max(int(m.total_rows.max()) for m in plan.mbs))
    plan.rows_cap = max(PAD, (plan.rows_cap + PAD - 1) // PAD * PAD)
    plan.rep_experts = [sorted({int(ex) for m in plan.mbs for ex, gs in m.placement.replicas.items() if d in gs})
                        for d in range(g)]
    return plan


def migration_moves(old_home: np.ndarray, new_home: np.ndarray, world: int) -> list:
    """Per rank: [(new local slot, source rank, source local slot)] for every expert of its new
    home set.  Local slots order a rank's home experts ascending (as the receive layout does);
    an expert that stays on its rank may still change slot."""
    old_home, new_home = np.asarray(old_home), np.asarray(new_home)
    if old_home.shape != new_home.shape:
        raise ValueError("old and new assignments cover different expert counts")
    old_slot = {}
    for g in range(world):
        for s, e in enumerate(np.flatnonzero(old_home == g)):
            old_slot[int(e)] = s
    out = []
    for d in range(world):
        out.append([(s, int(old_home[e]), old_slot[int(e)]) for s, e in enumerate(np.flatnonzero(new_home == d))])
    return out


def gather_routing(comm: Comm, local_counts: np.ndarray) -> np.ndarray:
    """(MB, E) expert counts of this rank (the K1 histogram rows) -> (MB, G, E) of every rank,
    i.e. RoutingTrace.matrices[:, layer] (routing.py:151-168) assembled across processes."""
    rows = comm.all_gather_object(np.ascontiguousarray(local_counts, dtype=np.int64))
    return np.stack(rows, axis=1)


def plan_digest(plan: StepPlan) -> str:
    """sha256 of every table of a step plan: ranks must agree bit for bit before the step."""
    import hashlib
    h = hashlib.sha256(np.ascontiguousarray(plan.home).tobytes())
    for m in plan.mbs:
        for a in (m.route_tab, m.ncopies, m.slot_tab, m.slot_w, m.nslots, m.total_rows, m.flow):
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(repr(list(m.placement.replicas.items())).encode())
    return h.hexdigest()[:16]


# ----------------------------------------------------------------------------- weights


def interleave_w1(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[.., h', h] gate/up -> [.., 2h', h] with alternating 128-row gate/up blocks (the layout
    the SwiGLU epilogue consumes: one 256-wide N tile = 128 gate + 128 matching up columns)."""
    *lead, hp, h = w_gate.shape
    nb = hp // GATE_BLOCK
    g = w_gate.reshape(*lead, nb, GATE_BLOCK, h)
    u = w_up.reshape(*lead, nb, GATE_BLOCK, h)
    return torch.stack([g, u], dim=-3).reshape(*lead, 2 * hp, h)


def deinterleave_w1(w1: torch.Tensor) -> tuple:
    *lead, hp2, h = w1.shape
    nb = hp2 // (2 * GATE_BLOCK)
    v = w1.reshape(*lead, nb, 2, GATE_BLOCK, h)
    return v[..., 0, :, :].reshape(*lead, hp2 // 2, h), v[..., 1, :, :].reshape(*lead, hp2 // 2, h)


# ----------------------------------------------------------------------------- data plane


def default_comm_sms(world: int, shape: "LayerShape") -> int:
    """SMs left to the comm stream's row movers while the persistent GEMM runs (env
    MB_COMM_SMS overrides, for A/B runs)."""
    if os.environ.get("MB_COMM_SMS"):
        return int(os.environ["MB_COMM_SMS"])
    if world == 1:
        return COMM_SMS[1]
    if shape.ffn >= WIDE_FFN:
        return COMM_SMS_WIDE_FFN
    if shape.hidden >= WIDE_HIDDEN:
        return COMM_SMS_MULTI    # comm-bound 4096-wide rows (Qwen3-235B): the 32-SM split was measured
    return COMM_SMS.get(world, COMM_SMS_MULTI)


# the last micro-batch's combine ahead of the third-to-last un-permute on the comm stream (step
# mode): B(MB-1) is otherwise the one backward with no comm cover -- it waits for C(MB-1), queued
# behind X(MB-3); MB_EARLY_LAST_COMBINE=0: the plain rotation
EARLY_LAST_COMBINE = os.environ.get("MB_EARLY_LAST_COMBINE", "1") == "1"


def schedule(mb: int, wgrad_mode: str = "step", early_last: bool | None = None):
    """Per-rank issue order of one step, two micro-batches in flight (the two-batch overlap of
    EP training systems): compute runs F0 F1 B0 F2 B1 ... F(n-1) B(n-2) B(n-1), the comm stream
    D0 D1 C0 [D(m) C(m-1) X(m-2)]... so every all-to-all overlaps a GEMM phase of the neighbouring
    micro-batch, while each combine is still a global sync point: a rank can run at most one
    phase ahead of the slowest rank, so load imbalance is paid per micro-batch (as the
    reference's cost model sums it, sim.py:89-110), not averaged over the step.
    F = fwd GEMMs, B = bwd GEMMs (+ replica weight gradients), W = home weight gradients of one
    micro-batch (wgrad_mode "micro_batch" only), D = dispatch, C = combine + dout dispatch,
    X = dX un-permute + replica-gradient push-back to the owners.  early_last (step mode, default
    EARLY_LAST_COMBINE): the tail runs C(n-1) before X(n-3), so the last backward is not queued
    behind an un-permute (see replica_ring_guards for the ring-set ordering this changes)."""
    comp = [("F", 0)]
    per_mb = wgrad_mode == "micro_batch"
    for m in range(1, mb):
        comp += [("F", m), ("B", m - 1)] + ([("W", m - 1)] if per_mb else [])
    comp.append(("B", mb - 1))
    if per_mb:
        comp.append(("W", mb - 1))
    comm = [("D", 0)]
    if mb > 1:
        comm += [("D", 1)]
    comm.append(("C", 0))
    for m in range(2, mb):
        comm += [("D", m), ("C", m - 1), ("X", m - 2)]
    if mb > 1:
        comm += [("C", mb - 1), ("X", mb - 2)]
    comm.append(("X", mb - 1))
    if (EARLY_LAST_COMBINE if early_last is None else early_last) and wgrad_mode == "step" and mb >= 3:
        comm.remove(("X", mb - 3))
        comm.insert(comm.index(("C", mb - 1)) + 1, ("X", mb - 3))
    return comm, comp


def replica_ring_guards(comm: list, mb: int) -> dict:
    """{m: x}: B(m)'s replica weight gradients overwrite ring set m % GRAD_RING, which the owners
    read in X(m - GRAD_RING).  When C(m) -- whose barrier every rank reaches only after its earlier
    comm phases -- does not follow X(m - GRAD_RING) on the comm stream, B(m) waits instead for the
    start barrier of the next un-permute X(x) after it (every rank passes that barrier only after
    its own X(m - GRAD_RING))."""
    pos = {o: i for i, o in enumerate(comm)}
    guards = {}
    for m in range(GRAD_RING, mb):
        src = ("X", m - GRAD_RING)
        if pos[src] < pos[("C", m)]:
            continue
        later = [op for op in comm[pos[src] + 1:] if op[0] == "X"]
        if not later:
            raise RuntimeError(f"no un-permute barrier after X({m - GRAD_RING}) to guard B({m})")
        guards[m] = later[0][1]
    return guards


# micro-batch activation / receive buffer sets in wgrad_mode "micro_batch": D(m + 3) is the first
# phase to reuse micro-batch m's set, and every rank's comm stream reaches it only after X(m)'s
# barrier (all ranks finished B(m) / W(m)), so three sets suffice for the schedule above
RING_SETS = 3
# replica-gradient ring: B(m) writes set m % 2, the owners read it in X(m); B(m + 2) runs after
# C(m + 2)'s barrier, which every rank reaches after its X(m) push-back -- or, where the schedule's
# tail puts C(m + 2) first, after a later un-permute's barrier (replica_ring_guards)
GRAD_RING = 2
ACC_TASK = np.dtype([("dst", "<u8"), ("src", "<u8", (8,)), ("n", "<i8"), ("nsrc", "<i4"), ("store", "<i4")])
ERR_BITS = {1: "routing has more tokens for an expert than the step plan's counts (perm dropped them)",
            2: "device histogram differs from the counts the step plan was built for"}


# weight-gradient groups longest-K first (dW2 and dW1 of an expert side by side in the two-problem
# table), so the dynamic tile scheduler ends a launch on the short tiles; MB_WGRAD_LPT=0: expert order
WGRAD_LPT = os.environ.get("MB_WGRAD_LPT", "1") == "1"


def _wgrad_tables(tab: np.ndarray, dev) -> tuple:
    """(single-problem table, two-problem table) of a wgrad group table: the second lists every
    group twice, the copy flagged FLAG_PROBLEM2 (dW1 beside dW2 in one launch).  With WGRAD_LPT the
    groups are ordered by K blocks, longest first (each output tile is still computed by exactly
    one tile in a fixed K order, so the results do not depend on the order)."""
    if WGRAD_LPT and len(tab) > 1:
        tab = tab[np.argsort(-tab[:, 7].astype(np.int64), kind="stable")]
    t2 = tab.copy()
    t2[:, 3] |= K.FLAG_PROBLEM2
    if len(tab) * 2 > K.MAX_GROUPS:
        merged = None
    elif WGRAD_LPT:
        merged = np.stack([tab, t2], axis=1).reshape(-1, tab.shape[1])
    else:
        merged = np.concatenate([tab, t2])
    return (torch.from_numpy(np.ascontiguousarray(tab)).to(dev),
            None if merged is None else torch.from_numpy(np.ascontiguousarray(merged)).to(dev))


def _wgrad_table(rows: list) -> np.ndarray:
    tab = np.zeros((max(1, len(rows)), K.GROUP_FIELDS), dtype=np.int32)
    for i, row in enumerate(rows):
        tab[i] = row
    return tab[:len(rows)] if rows else tab[:0]


class ReplicaBuffer:
    """The paper's layer-shared replica buffer (replica_memory "layer-shared",
    replicate.py:528-534): `sets` x r replica weight slots of one expert shape per GPU plus the fp32
    replica-gradient ring, in their own symmetric arena, shared by every MoE layer
    (MoEDataPlane(..., replica_buffer=buf)) of a model.  Layers take turns: each (layer,
    micro-batch) phase pulls the replicas it needs into the slots right before its GEMM (after the
    slot's last use by any layer) and pushes the replica gradients back within the same
    micro-batch's backward, so the buffer never grows with the number of layers."""

    def __init__(self, comm: Comm, shape: LayerShape, slots: int, sets: int = 1,
                 device: torch.device | None = None):
        if slots < 1 or sets < 1:
            raise ValueError("a replica buffer needs >= 1 slot and >= 1 set")
        self.shape, self.slots, self.sets = shape, slots, sets
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        h, hp = shape.hidden, shape.ffn
        self.w1_bytes, self.w2_bytes = 2 * hp * h * 2, h * hp * 2
        self.g1_bytes, self.g2_bytes = 2 * hp * h * 4, h * hp * 4
        self.sizes = {"w1r": sets * slots * self.w1_bytes, "w2r": sets * slots * self.w2_bytes,
                      "rg1": GRAD_RING * slots * self.g1_bytes, "rg2": GRAD_RING * slots * self.g2_bytes}
        total = sum((v + 1023) // 1024 * 1024 for v in self.sizes.values()) + 4096
        self.arena = SymmetricArena(comm, total, self.device)
        self.off = {k: self.arena.alloc(v) for k, v in self.sizes.items()}
        A = self.arena
        self.W1r = A.local(self.off["w1r"], (sets, slots, 2 * hp, h), torch.bfloat16)
        self.W2r = A.local(self.off["w2r"], (sets, slots, h, hp), torch.bfloat16)
        self.rgW1 = A.local(self.off["rg1"], (GRAD_RING, slots, 2 * hp, h), torch.float32)
        self.rgW2 = A.local(self.off["rg2"], (GRAD_RING, slots, h, hp), torch.float32)
        # slot bookkeeping shared by the layers: per kind and set, the (layer, micro-batch) held,
        # the event after its last use, the event after its pull, an LRU stamp
        self.state = {kd: {"held": [None] * sets, "used": [None] * sets, "pulled": [None] * sets,
                           "seq": [0] * sets} for kd in ("w1", "w2")}
        self.done = set()      # (layer, micro-batch) whose backward is issued (no further use)
        self.seq = 0
        self.users = 0

    def invalidate(self, layer_token) -> None:
        """A new step of `layer_token`: its weights may have changed since the last pull."""
        for st in self.state.values():
            for i, tag in enumerate(st["held"]):
                if tag is not None and tag[0] == layer_token:
                    st["held"][i] = None
        self.done = {t for t in self.done if t[0] != layer_token}

    def nbytes(self) -> dict:
        return {"replica_weight_slots": self.sizes["w1r"] + self.sizes["w2r"],
                "replica_grad_ring": self.sizes["rg1"] + self.sizes["rg2"]}

    def close(self) -> None:
        self.arena.close()


class PlanTables:
    """A step plan's device tables for one data plane (MoEDataPlane.build_tables): built ahead,
    installed by load_plan / migrate without host work on the step's critical path."""

    def __init__(self, owner, plan: StepPlan, attrs: dict):
        self.owner, self.plan, self.attrs = owner, plan, attrs


class MoEDataPlane:
    """Per-rank device state for one MoE layer: home experts (+ fp32 gradients, optional expert
    state, double-banked for migration), the layer-shared replica slots, the replica-gradient
    ring, receive/activation buffers and the step tables.

    wgrad_mode "step" (default): weight gradients contract over every micro-batch of the step in
    one GEMM per weight (receive / activation buffers for all MB micro-batches stay resident);
    "micro_batch": each micro-batch's weight gradients are accumulated right after its backward
    (K = that micro-batch's rows), so only RING_SETS micro-batches of activations exist.
    replica_sets: sets of r replica weight slots (r = plan.slots); 1 = the paper's layer-shared
    buffer of exactly replica_memory(model, cfg, "layer-shared") bytes (replica weights are pulled
    again for the backward), 2 = double-buffered pulls."""

    def __init__(self, comm: Comm, shape: LayerShape, tokens: int, micro_batches: int, plan: StepPlan,
                 device: torch.device | None = None, comm_sms: int | None = None,
                 expert_state: dict | None = None, rows_cap: int = 0, overlap: bool | None = None,
                 row_movers: str | None = None, wgrad_mode: str | None = None, replica_sets: int | None = None,
                 replica_buffer: "ReplicaBuffer | None" = None):
        """expert_state: optional per-expert tensors that follow their expert when the reorder
        plan migrates it (e.g. optimizer moments): {name: (per-expert shape, torch dtype)}.
        rows_cap: receive rows per micro-batch to allocate (>= every plan this layer will load).
        overlap: run dispatch / combine on their own stream beside the GEMMs (default).
        row_movers: "regs" | "tma" scatter / combine engine (default per world size, ROW_MOVERS).
        replica_buffer: a ReplicaBuffer shared with the model's other MoE layers (default: this
        layer allocates its own)."""
        shape.check()
        self.comm, self.shape, self.T, self.MB = comm, shape, tokens, micro_batches
        self.rank, self.world = comm.rank, comm.world
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        if overlap is None and os.environ.get("MB_OVERLAP") in ("0", "1"):
            overlap = os.environ["MB_OVERLAP"] == "1"
        self.overlap = True if overlap is None else overlap
        wgrad_mode = wgrad_mode or os.environ.get("MB_WGRAD_MODE", "step")
        if wgrad_mode not in ("step", "micro_batch"):
            raise ValueError(f"wgrad_mode must be 'step' or 'micro_batch', got {wgrad_mode!r}")
        self.wgrad_mode = wgrad_mode
        if replica_sets is None:
            replica_sets = default_replica_sets(shape)
        if replica_sets < 1:
            raise ValueError("replica_sets must be >= 1")
        self.replica_sets = replica_sets
        if comm_sms is None:
            comm_sms = default_comm_sms(self.world, shape) if self.overlap else 0
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        # per-plane launch settings, passed with every launch (never process-global)
        self.gemm_sms, self.all_sms = max(2, sms - comm_sms), sms
        if row_movers is None:
            row_movers = os.environ.get("MB_ROW_MOVERS") or ROW_MOVERS.get(self.world, ROW_MOVERS_MULTI)
        if row_movers not in ("regs", "tma"):
            raise ValueError(f"row_movers must be 'regs' or 'tma', got {row_movers!r}")
        self.row_movers = row_movers
        self.comm_sms = comm_sms
        self.comm_blocks = comm_sms if (row_movers == "tma" and comm_sms > 0) else 0
        E, h, hp = shape.num_experts, shape.hidden, shape.ffn
        if E % self.world:
            raise ValueError(f"{E} experts not divisible by {self.world} GPUs")
        self.M = E // self.world
        self.R = max(plan.rows_cap, (rows_cap + PAD - 1) // PAD * PAD)
        self.slots = max(plan.slots, 1)
        if replica_buffer is None:
            replica_buffer = ReplicaBuffer(comm, shape, self.slots, replica_sets, self.device)
            self._owns_rb = True
        else:
            if replica_buffer.shape != shape or replica_buffer.slots < self.slots:
                raise ValueError("the shared replica buffer holds a different expert shape or fewer slots")
            self.slots, self.replica_sets = replica_buffer.slots, replica_buffer.sets
            self._owns_rb = False
        self.rb = replica_buffer
        self.rb.users += 1
        self.token = object()   # identity of this layer in the shared buffer's slot tags
        self.NA = micro_batches if wgrad_mode == "step" else min(micro_batches, RING_SETS)
        bf, f4 = 2, 4
        self.npart = hp // 64    # dgate partials per row (one per 64 features of h')
        R, NA = self.R, self.NA
        self.w1_bytes, self.w2_bytes = 2 * hp * h * bf, h * hp * bf
        self.g1_bytes, self.g2_bytes = 2 * hp * h * f4, h * hp * f4
        # ---- symmetric arena (peer-visible buffers; identical layout on every rank)
        sizes = {
            "xr": NA * R * h * bf, "y": NA * R * h * bf, "dyr": NA * R * h * bf, "dxp": NA * R * h * bf,
            "gate_r": NA * R * f4, "dgate_r": NA * R * self.npart * f4,
            # home-expert weights, fp32 gradients and expert state live in two banks: a migration
            # (new reorder plan) pulls every new home expert into the idle bank, then swaps
            "w1": self.M * self.w1_bytes, "w2": self.M * self.w2_bytes,
            "gw1": self.M * self.g1_bytes, "gw2": self.M * self.g2_bytes,
            "w1b": self.M * self.w1_bytes, "w2b": self.M * self.w2_bytes,
            "gw1b": self.M * self.g1_bytes, "gw2b": self.M * self.g2_bytes,
        }
        self.state_spec = {}
        for name, (eshape, dtype) in (expert_state or {}).items():
            nbytes = int(np.prod(eshape)) * torch.empty((), dtype=dtype).element_size()
            self.state_spec[name] = (tuple(eshape), dtype, nbytes)
            sizes["st_" + name] = sizes["st_" + name + "b"] = self.M * nbytes
        self.sizes = sizes
        total = sum((v + 1023) // 1024 * 1024 for v in sizes.values()) + 1024 * len(sizes)
        self.arena = SymmetricArena(comm, total, self.device)
        self.off = {key: self.arena.alloc(v) for key, v in sizes.items()}
        A = self.arena
        self.Xr = A.local(self.off["xr"], (NA, R, h), torch.bfloat16)
        self.Y = A.local(self.off["y"], (NA, R, h), torch.bfloat16)
        self.dYr = A.local(self.off["dyr"], (NA, R, h), torch.bfloat16)
        self.dXp = A.local(self.off["dxp"], (NA, R, h), torch.bfloat16)
        self.gate_r = A.local(self.off["gate_r"], (NA, R), torch.float32)
        self.dgate_r = A.local(self.off["dgate_r"], (NA, R, self.npart), torch.float32)
        # the layer-shared replica slots and replica-gradient ring (own, or shared by the layers)
        self.W1r, self.W2r, self.rgW1, self.rgW2 = self.rb.W1r, self.rb.W2r, self.rb.rgW1, self.rb.rgW2
        self.bank = 0
        self._bind_bank()
        # ---- local activations
        self.H = torch.empty((NA, R, 2 * hp), dtype=torch.bfloat16, device=self.device)
        self.Act = torch.empty((NA, R, hp), dtype=torch.bfloat16, device=self.device)
        self.dH = torch.empty((NA, R, 2 * hp), dtype=torch.bfloat16, device=self.device)
        # ---- per-micro-batch token-side buffers
        T, k, MB = tokens, shape.top_k, micro_batches
        self.perm = torch.empty((MB, T, k, 2), dtype=torch.int32, device=self.device)
        chunks = (T + CHUNK - 1) // CHUNK
        self.counts = torch.empty((MB, E), dtype=torch.int32, device=self.device)
        self.chunk_counts = torch.empty((MB, chunks, E), dtype=torch.int32, device=self.device)
        self.chunk_base = torch.empty((MB, chunks, E), dtype=torch.int32, device=self.device)
        # peer pointer tables [MB][world]: micro-batch m uses buffer set m % NA
        self.ptr_xr = self._set_table("xr", R * h * bf)
        self.ptr_y = self._set_table("y", R * h * bf)
        self.ptr_dyr = self._set_table("dyr", R * h * bf)
        self.ptr_dxp = self._set_table("dxp", R * h * bf)
        self.ptr_gate = self._set_table("gate_r", R * f4)
        self.ptr_dgate = self._set_table("dgate_r", R * self.npart * f4)
        # host-visible error flag the permutation / count-check kernels OR bits into
        lib = nat.kernels()
        hp_, dp_ = ctypes.c_void_p(), ctypes.c_void_p()
        nat.check(lib.mb_host_alloc_mapped(16, ctypes.byref(hp_), ctypes.byref(dp_)), lib, "mb_host_alloc_mapped")
        self._err_host, self.err_dev = hp_.value, dp_.value
        self._err_view = (ctypes.c_int32 * 4).from_address(self._err_host)
        self.xs = torch.cuda.Stream(device=self.device)      # comm stream: dispatch / combine / barriers
        # compute stream of the fused step: the caller's stream, or (MB_COMPUTE_PRIORITY=high) an own
        # high-priority stream, so GEMM CTAs are scheduled ahead of pending row-mover blocks
        self._ks = (torch.cuda.Stream(device=self.device, priority=-1)
                    if os.environ.get("MB_COMPUTE_PRIORITY") == "high" else None)
        self.cps = torch.cuda.Stream(device=self.device)     # copy-engine stream: replica weight pulls
        self.launches = 0
        self.timing = False       # record CUDA events around every K4 launch (bench roofline)
        self.gemm_events = []     # (start, end, algorithmic FLOPs, kind)
        self.load_plan(plan)

    def _set_table(self, key: str, stride: int) -> torch.Tensor:
        tab = np.array([[self.arena.peer_ptr(p, self.off[key]) + (m % self.NA) * stride for p in range(self.world)]
                        for m in range(self.MB)], dtype=np.int64)
        return torch.from_numpy(tab).to(self.device)

    def set_index(self, m: int) -> int:
        """Receive / activation buffer set of micro-batch m."""
        return m % self.NA

    def memory_report(self) -> dict:
        """Device bytes per GPU of the data plane's buffers (both banks of home state counted)."""
        s = self.sizes
        act = sum(s[k] for k in ("xr", "y", "dyr", "dxp", "gate_r", "dgate_r"))
        act += sum(t.numel() * t.element_size() for t in (self.H, self.Act, self.dH))
        return {**self.rb.nbytes(), "replica_sets": self.replica_sets, "replica_slots": self.slots,
                "replica_buffer_shared_by_layers": self.rb.users,
                "activations": act, "activation_sets": self.NA, "wgrad_mode": self.wgrad_mode,
                "home_weights_and_grads": sum(s[k] for k in ("w1", "w2", "gw1", "gw2", "w1b", "w2b", "gw1b", "gw2b")),
                "arena_total": self.arena.nbytes}

    # ------------------------------------------------------------------ helpers
    def _timed(self, amount: float, kind: str = "gemm", stream=None):
        """Context manager recording CUDA events around a launch sequence on `stream` (default:
        the current stream).  amount = algorithmic FLOPs (K4) or NVLink bytes (comm phases)."""
        dp = self

        class _T:
            def __enter__(self):
                if dp.timing:
                    self.s = torch.cuda.Event(enable_timing=True)
                    self.e = torch.cuda.Event(enable_timing=True)
                    self.s.record(stream)

            def __exit__(self, *a):
                if dp.timing:
                    self.e.record(stream)
                    dp.gemm_events.append((self.s, self.e, amount, kind))
        return _T()

    def remote_rows(self, m: int) -> tuple[int, int]:
        """(rows this rank sends to peers, rows peers send to it) in one A2A phase of micro-batch m."""
        f = self.plan.mbs[m].flow
        me = self.rank
        return int(f[me].sum() - f[me, me]), int(f[:, me].sum() - f[me, me])

    def real_rows(self, m: int) -> int:
        """Token rows this rank's experts serve in micro-batch m (padding excluded)."""
        return int(self.plan.mbs[m].flow[:, self.rank].sum())

    def errors(self) -> int:
        """Error bits the kernels reported so far (MB_ERR_*; read without a device sync)."""
        return int(self._err_view[0])

    def check(self, sync: bool = True) -> None:
        """Raise if a kernel flagged routing that differs from the step plan (optionally after a
        device synchronisation, so the last step is included)."""
        if sync:
            torch.cuda.synchronize(self.device)
        bits = self.errors()
        if bits:
            self._err_view[0] = 0
            msgs = [msg for b, msg in ERR_BITS.items() if bits & b]
            raise RuntimeError("MoE data plane: " + "; ".join(msgs))

    def _check_inputs(self, per_mb: bool, **tensors) -> None:
        """Validate the step's tensors at the API boundary (dtype, shape, contiguity, device)."""
        T, k, h, MB = self.T, self.shape.top_k, self.shape.hidden, self.MB
        lead = () if per_mb else (MB,)
        spec = {"x": (torch.bfloat16, lead + (T, h)), "dout": (torch.bfloat16, lead + (T, h)),
                "out": (torch.bfloat16, lead + (T, h)), "dx": (torch.bfloat16, lead + (T, h)),
                "idx": (torch.int32, lead + (T, k)), "gates": (torch.float32, lead + (T, k)),
                "dgate": (torch.float32, lead + (T, k))}
        for name, t in tensors.items():
            dtype, shp = spec[name]
            if not isinstance(t, torch.Tensor):
                raise TypeError(f"{name} must be a torch.Tensor")
            if t.dtype != dtype:
                raise ValueError(f"{name} must be {dtype} (got {t.dtype})")
            if tuple(t.shape) != shp:
                raise ValueError(f"{name} must have shape {list(shp)} (got {list(t.shape)}); the plane was built "
                                 f"for T={T}, top_k={k}, hidden={h}, micro_batches={MB}")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            if t.device != self.device:
                raise ValueError(f"{name} is on {t.device}, the data plane on {self.device}")

    # ------------------------------------------------------------------ plan upload
    def load_plan(self, plan) -> None:
        """Install a step plan (a StepPlan, or the PlanTables build_tables made from one)."""
        tables = plan if isinstance(plan, PlanTables) else self.build_tables(plan)
        if tables.owner is not self:
            raise ValueError("these plan tables were built for another data plane")
        self.plan = tables.plan
        self.tables = tables
        for key, val in tables.attrs.items():
            setattr(self, key, val)

    def build_tables(self, plan: StepPlan) -> "PlanTables":
        """Every device table of a step plan for this rank (uploaded now, installed by load_plan /
        migrate): per-micro-batch route / slot / GEMM group tables, the replicas this rank pulls,
        the weight-gradient tables and the replica-gradient push-back tasks."""
        if plan.rows_cap > self.R:
            raise ValueError(f"plan needs {plan.rows_cap} receive rows per micro-batch, buffers hold {self.R}")
        if len(plan.mbs) != self.MB:
            raise ValueError(f"plan has {len(plan.mbs)} micro-batches, the data plane {self.MB}")
        d, dev = self.rank, self.device
        E, MB, R = self.shape.num_experts, self.MB, self.R
        h, hp = self.shape.hidden, self.shape.ffn
        home = np.asarray(plan.home)
        home_experts = np.flatnonzero(home == d)
        nh = len(home_experts)
        local_of = np.zeros(E, dtype=np.int64)
        for g in range(self.world):
            mine = np.flatnonzero(home == g)
            local_of[mine] = np.arange(len(mine))
        loc_of_home = {int(ex): i for i, ex in enumerate(home_experts)}
        route, ncop, groups, slots, nsl, tails = [], [], [], [], [], []
        max_slots = plan.max_slots
        mb_rep = []               # per micro-batch: [(slot q, expert, owner rank, owner local index)]
        rep_rows = []             # per micro-batch: {(holder rank, expert): (slot q, real rows)}
        home_slots = []           # per micro-batch: {home expert: (row_begin, real rows)} on this rank
        rep_slots = []            # per micro-batch: {replicated expert: (row_begin, real rows, q)} on this rank
        for m, mbp in enumerate(plan.mbs):
            route.append(mbp.route_tab[d])
            ncop.append(mbp.ncopies)
            n = int(mbp.nslots[d])
            st = mbp.slot_tab[d].copy()
            st[n:] = 0  # unused entries all-zero (the batched pad-row zeroing relies on it)
            sw = mbp.slot_w[d]
            if int(sw[:n, 0][sw[:n, 1] > 0].max(initial=-1)) >= self.slots:
                raise ValueError("plan uses more replica slots than allocated")
            g = np.zeros((max_slots, K.GROUP_FIELDS), dtype=np.int32)
            g[:n, 0] = st[:n, 2]
            g[:n, 1] = st[:n, 0]
            g[:n, 2] = sw[:n, 0]
            g[:n, 3] = np.where(sw[:n, 1] > 0, K.FLAG_REPLICA, 0)
            g[:n, 6] = st[:n, 1]
            groups.append(g)
            # tail blocks: the last 128 rows of a slot with an odd number of 128-row blocks run in
            # the single-CTA kernel beside the pair kernel (which then sees whole 256-row tiles)
            pair_rows = (g[:n, 0] // 256) * 256
            has_tail = (g[:n, 0] - pair_rows) > 0
            gp = g.copy()
            gp[:n, 0] = pair_rows
            gt = g[:n][has_tail].copy()
            gt[:, 1] += pair_rows[has_tail]
            gt[:, 0] = 128
            gt[:, 6] = np.maximum(0, g[:n, 6][has_tail] - pair_rows[has_tail])
            n_pair_blocks, n_tail = int(pair_rows.sum()) // 256, int(has_tail.sum())
            tail_share = n_tail / max(1, n_tail + 2 * n_pair_blocks)   # SM-time share of the tails
            tails.append((gp, gt, tail_share))
            slots.append(st)
            nsl.append(n)
            mb_rep.append([(int(sw[s, 0]), int(st[s, 3]), int(home[st[s, 3]]), int(local_of[st[s, 3]]))
                           for s in range(n) if sw[s, 1] > 0])
            home_slots.append({int(st[s, 3]): (int(st[s, 0]), int(st[s, 1])) for s in range(n)
                               if sw[s, 1] == 0 and st[s, 1] > 0})
            rep_slots.append({int(st[s, 3]): (int(st[s, 0]), int(st[s, 1]), int(sw[s, 0])) for s in range(n)
                              if sw[s, 1] > 0 and st[s, 1] > 0})
            rr = {}
            for p in range(self.world):
                stt, sww = mbp.slot_tab[p], mbp.slot_w[p]
                for s in range(int(mbp.nslots[p])):
                    if sww[s, 1] and stt[s, 1] > 0:
                        rr[(p, int(stt[s, 3]))] = (int(sww[s, 0]), int(stt[s, 1]))
            rep_rows.append(rr)
        devs = [getattr(mbp, "device", None) for mbp in plan.mbs]
        if all(t is not None for t in devs):   # tables computed on the GPU (mb_dispatch_tables): use them as is
            route_dev = torch.stack([t["route_tab"][d] for t in devs])
            ncop_dev = torch.stack([t["ncopies"] for t in devs])
            slot_dev = torch.stack([t["slot_tab"][d] for t in devs])
        else:
            route_dev = torch.from_numpy(np.stack(route)).to(dev)
            ncop_dev = torch.from_numpy(np.stack(ncop)).to(dev)
            slot_dev = torch.from_numpy(np.stack(slots)).to(dev)
        at = {"home_experts": home_experts, "mb_rep": mb_rep, "nslots": nsl,
              "route_tab": route_dev, "ncopies": ncop_dev,
              "groups": torch.from_numpy(np.stack(groups)).to(dev),
              # per micro-batch (pair-kernel groups, tail groups or None, tail SM share)
              "tail_groups": [(torch.from_numpy(gp).to(dev), torch.from_numpy(gt).to(dev) if len(gt) else None, sh)
                              for gp, gt, sh in tails],
              "slot_tab": slot_dev,
              "expected": (torch.from_numpy(np.ascontiguousarray(plan.mats[:, d], dtype=np.int32)).to(dev)
                           if plan.mats is not None else None)}

        # ---- weight-gradient tables.  Contribution order per home expert (fresh step: the first
        # contribution stores, the rest accumulate): step mode X(0) .. X(MB-1) then the home wgrad;
        # micro-batch mode W(0) X(0) W(1) X(1) ...  (X = replica-gradient push-back)
        def r16(rows):
            return (rows + 15) // 16 * 16

        def group_row(segs, seg_rows, out_slot, flags):
            s0 = len(segs)
            segs.extend(seg_rows)
            tot = sum(r for _, r in seg_rows)
            kb = sum((r + 63) // 64 for _, r in seg_rows)
            return (tot, 0, out_slot, flags, s0, len(seg_rows), 0, kb)

        def seg_tensor(segs):
            return torch.from_numpy(np.asarray(segs if segs else [(0, 0)], dtype=np.int32).reshape(-1, 2)).to(dev)

        written = [False] * nh           # fresh step: has the expert's gradient been written yet
        replica_contrib = set()          # home local indices with replica gradients this step
        srcs_of = []                     # per m: {loc: [(holder, q)]}
        for m in range(MB):
            sm = {}
            for (p, ex), (q, _) in rep_rows[m].items():
                if p != d and int(home[ex]) == d:
                    sm.setdefault(loc_of_home[ex], []).append((p, q))
            for loc in sm:
                sm[loc].sort()
                if len(sm[loc]) > 8:
                    raise ValueError("more than 8 replicas of one expert in a micro-batch")
                replica_contrib.add(loc)
            srcs_of.append(sm)
        w_mb, rw_mb, acc_mb = [None] * MB, [None] * MB, [None] * MB
        nfl = {"rg1": 2 * hp * h, "rg2": h * hp}
        for m in range(MB):
            # replica wgrad of micro-batch m on this rank: store into ring set m % GRAD_RING
            segs, rows, a_rows = [], [], 0
            for ex, (r0, real, q) in sorted(rep_slots[m].items()):
                rows.append(group_row(segs, [(r0, r16(real))], q, 0))
                a_rows += real
            if rows:
                rw_mb[m] = (_wgrad_tables(_wgrad_table(rows), dev), seg_tensor(segs), a_rows)
            if self.wgrad_mode == "micro_batch":
                segs, rows_f, real = [], [], 0
                for ex, (r0, rr_) in sorted(home_slots[m].items()):
                    loc = loc_of_home[ex]
                    rows_f.append(group_row(segs, [(r0, r16(rr_))], loc, K.FLAG_ACCUMULATE if written[loc] else 0))
                    written[loc] = True
                    real += rr_
                if rows_f:
                    tab_f = _wgrad_table(rows_f)
                    tab_a = tab_f.copy()
                    tab_a[:, 3] |= K.FLAG_ACCUMULATE   # an accumulating step adds every contribution
                    w_mb[m] = (_wgrad_tables(tab_f, dev), _wgrad_tables(tab_a, dev), seg_tensor(segs), real)
            # owner push-back tasks of micro-batch m (fresh variant: first contribution stores)
            if srcs_of[m]:
                tasks = np.zeros(2 * len(srcs_of[m]), dtype=ACC_TASK)
                dst_other = np.zeros(2 * len(srcs_of[m]), dtype=np.uint64)   # the same in the other bank
                i = 0
                for loc in sorted(srcs_of[m]):
                    for key, gkey, size in (("rg1", "gw1", self.g1_bytes), ("rg2", "gw2", self.g2_bytes)):
                        tasks[i]["dst"] = self.arena.peer_ptr(d, self.off[gkey]) + loc * size
                        dst_other[i] = self.arena.peer_ptr(d, self.off[gkey + "b"]) + loc * size
                        for j, (p, q) in enumerate(srcs_of[m][loc]):
                            tasks[i]["src"][j] = (self.rb.arena.peer_ptr(p, self.rb.off[key])
                                                  + ((m % GRAD_RING) * self.slots + q) * size)
                        tasks[i]["n"], tasks[i]["nsrc"] = nfl[key], len(srcs_of[m][loc])
                        tasks[i]["store"] = 0 if written[loc] else 1
                        i += 1
                    written[loc] = True
                variants = []
                for bank in (0, 1):           # per gradient bank: (fresh, accumulating) task tables
                    tb = tasks.copy()
                    if bank:
                        tb["dst"] = dst_other
                    ta = tb.copy()
                    ta["store"] = 0
                    variants.append((torch.from_numpy(tb.view(np.uint8).copy()).to(dev),
                                     torch.from_numpy(ta.view(np.uint8).copy()).to(dev)))
                acc_mb[m] = (variants, len(tasks), int(tasks["n"].max()))
        at.update(w_mb=w_mb, rw_mb=rw_mb, acc_mb=acc_mb, replica_contrib=replica_contrib)
        # ---- step mode home wgrad: K contracted over every micro-batch; part B = experts without
        # replica gradients (runs right after the last backward), part A = the rest (after the last
        # push-back, accumulating onto it)
        wparts, idle_home = [], []
        if self.wgrad_mode == "step":
            segs, rows_a, rows_b = [], [], []
            for loc, ex in enumerate(home_experts):
                ex = int(ex)
                sr = [(self.set_index(m) * R + home_slots[m][ex][0], r16(home_slots[m][ex][1]))
                      for m in range(MB) if ex in home_slots[m]]
                if not sr:
                    if loc not in replica_contrib:
                        idle_home.append(loc)
                    continue
                real = sum(home_slots[m][ex][1] for m in range(MB) if ex in home_slots[m])
                (rows_a if loc in replica_contrib else rows_b).append((group_row(segs, sr, loc, 0), real))
            segs_t = seg_tensor(segs)
            for part_rows, part in ((rows_b, "B"), (rows_a, "A")):
                if not part_rows:
                    wparts.append(None)
                    continue
                tab = _wgrad_table([r for r, _ in part_rows])
                tab_fresh, tab_acc = tab.copy(), tab.copy()
                tab_acc[:, 3] |= K.FLAG_ACCUMULATE
                if part == "A":      # replica gradients were pushed back first: always accumulate
                    tab_fresh[:, 3] |= K.FLAG_ACCUMULATE
                wparts.append((_wgrad_tables(tab_fresh, dev), _wgrad_tables(tab_acc, dev), segs_t,
                               float(sum(r for _, r in part_rows)), part))
        else:
            idle_home = [loc for loc in range(nh) if not written[loc]]
        at.update(wparts=wparts, idle_home=idle_home)
        return PlanTables(self, plan, at)


    # ------------------------------------------------------------------ weights
    def _bind_bank(self) -> None:
        """Views of the current bank: W1/W2, fp32 gradients gW1/gW2, expert state."""
        sfx = "b" if self.bank else ""
        h, hp, A = self.shape.hidden, self.shape.ffn, self.arena
        self.off_w = {k: self.off[k + sfx] for k in ("w1", "w2", "gw1", "gw2")}
        self.W1 = A.local(self.off_w["w1"], (self.M, 2 * hp, h), torch.bfloat16)
        self.W2 = A.local(self.off_w["w2"], (self.M, h, hp), torch.bfloat16)
        self.gW1 = A.local(self.off_w["gw1"], (self.M, 2 * hp, h), torch.float32)
        self.gW2 = A.local(self.off_w["gw2"], (self.M, h, hp), torch.float32)
        self.state = {}
        for name, (eshape, dtype, _) in self.state_spec.items():
            off = self.off["st_" + name + sfx]
            self.off_w["st_" + name] = off
            self.state[name] = A.local(off, (self.M, *eshape), dtype)

    def migrate(self, plan, grads: bool = True) -> dict:
        """Switch to a step plan with a different reorder assignment (expert migration at a batch
        boundary): every rank pulls its new home experts' weights, fp32
        gradients and expert state from their old owners (copy engine over NVLink, or a local
        copy) into its idle bank, then all ranks swap banks and upload the new plan.  Collective:
        every rank calls it with the same plan.  grads=False skips the fp32 gradients (migration
        right after an optimizer step, when they are zero: the new bank's are zeroed instead).
        `plan` is a StepPlan or its prebuilt PlanTables.  Returns {experts_moved, bytes_in}."""
        tables = plan if isinstance(plan, PlanTables) else self.build_tables(plan)
        old_home, new_home = np.asarray(self.plan.home), np.asarray(tables.plan.home)
        if np.array_equal(old_home, new_home):      # same assignment: nothing moves
            self.load_plan(tables)
            return {"experts_moved": 0, "bytes_in": 0}
        moves = migration_moves(old_home, new_home, self.world)[self.rank]
        cur = torch.cuda.current_stream()
        cps, A, lib = self.cps, self.arena, nat.kernels()
        sfx_new = "" if self.bank else "b"
        items = [("w1", self.w1_bytes), ("w2", self.w2_bytes)]
        grads = grads and not getattr(self, "grads_pending_zero", False)
        if grads:
            items += [("gw1", self.g1_bytes), ("gw2", self.g2_bytes)]
        items += [("st_" + n, spec[2]) for n, spec in self.state_spec.items()]
        cps.wait_stream(cur)
        A.barrier(cps)  # every rank finished its last step: the current banks are stable
        moved = nbytes = 0
        for slot, src_rank, src_slot in moves:
            if src_rank != self.rank:
                moved += 1
            for key, size in items:
                src = A.peer_ptr(src_rank, self.off_w[key]) + src_slot * size
                dst = A.peer_ptr(self.rank, self.off[key + sfx_new]) + slot * size
                nat.check(lib.mb_memcpy_async(dst, src, size, cps.cuda_stream), lib, "migrate")
                if src_rank != self.rank:
                    nbytes += size
        A.barrier(cps)  # every pull has landed; the old banks may be reused
        cur.wait_stream(cps)
        self.bank ^= 1
        self._bind_bank()
        if not grads:
            self.zero_grads(lazy=True)
        self.load_plan(tables)
        return {"experts_moved": moved, "bytes_in": nbytes}

    def set_weights(self, w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor) -> None:
        """Home expert weights of this rank (ascending expert id): gate/up [M,h',h], down [M,h,h']."""
        self.W1.copy_(interleave_w1(w_gate, w_up))
        self.W2.copy_(w_down)

    def zero_grads(self, lazy: bool = True) -> None:
        """Reset the fp32 expert gradients.  lazy (default): no memset; the next step's first
        gradient contribution to each expert stores instead of accumulating (0 + x == x exactly),
        as a trainer's zero_grad() before backward would have it.  Read gradients through grads()
        to see the zeros before that step."""
        if lazy:
            self.grads_pending_zero = True
        else:
            self.gW1.zero_()
            self.gW2.zero_()
            self.grads_pending_zero = False

    def grads(self):
        """(gW1, gW2) of the current bank, materialising a pending lazy zero."""
        if getattr(self, "grads_pending_zero", False):
            self.zero_grads(lazy=False)
        return self.gW1, self.gW2

    # ------------------------------------------------------------------ step
    def _k(self, name, *args):
        if _SKIP_ROWS and name in ("mb_scatter_rows", "mb_combine_rows"):
            return  # profiling only (MB_PROFILE_SKIP_ROWS): GEMM timing without the row movers
        lib = nat.kernels()
        nat.check(getattr(lib, name)(*args), lib, name)
        self.launches += 1

    def _gemm(self, *args, sms=None, **kw):
        K.grouped_gemm(*args, sms=self.gemm_sms if sms is None else sms, **kw)
        self.launches += 1

    def forward_backward(self, x: torch.Tensor, idx: torch.Tensor, gates: torch.Tensor, dout: torch.Tensor,
                         out: torch.Tensor, dx: torch.Tensor, dgate: torch.Tensor, hooks=None) -> None:
        """One training step of the layer over MB micro-batches (inputs [MB, T, ...] on device).
        Writes out / dx / dgate and accumulates fp32 expert gradients.  Asynchronous with respect
        to the host; the current stream is ordered after all of it on return.  `hooks` (optional)
        gets inputs_ready(m, stream) (x, idx, gates of micro-batch m), optional dout_ready(m, stream),
        after_forward(m, stream), after_backward(m, stream).
        Runs the two-micro-batch-overlap schedule (schedule()); the same phases are available one
        micro-batch at a time through begin_step / forward_mb / backward_mb / end_step."""
        self._check_inputs(False, x=x, idx=idx, gates=gates, dout=dout, out=out, dx=dx, dgate=dgate)
        self.check(sync=False)
        ops = _StepOps(self, hooks, own_compute_stream=True)
        comm_fn = {"D": lambda m: ops.dispatch(m, x[m], idx[m], gates[m], idx, gates),
                   "C": lambda m: (ops.combine(m, gates[m], out[m]), ops.dout_dispatch(m, dout[m])),
                   "X": lambda m: ops.unpermute(m, dx[m], dgate[m])}
        comp_fn = {"F": ops.fwd_gemms, "B": ops.bwd_gemms, "W": ops.wgrad_mb}
        per_mb = self.wgrad_mode == "micro_batch"
        # comm op waits for this compute op of the same micro-batch; compute op for this comm op
        comm_needs = {"C": ("F", 0), "X": ("W" if per_mb else "B", 0)}
        comp_needs = {"F": ("D", 0), "B": ("C", 0), "W": ("X", -1)}
        comm_ops, comp_ops = schedule(self.MB, self.wgrad_mode)
        ops.ring_guard = replica_ring_guards(comm_ops, self.MB)
        ev_comm, ev_comp = {}, {}
        cs, xs = ops.cs, ops.xs
        ci = pi = 0
        # host issue order only has to respect the cross-stream event dependencies; each stream
        # then runs its own sequence in order on the device
        while ci < len(comm_ops) or pi < len(comp_ops):
            if ci < len(comm_ops):
                cop, cm = comm_ops[ci]
                dep = (comm_needs[cop][0], cm + comm_needs[cop][1]) if cop in comm_needs else None
                if dep is None or dep in ev_comp:
                    if dep is not None:
                        xs.wait_event(ev_comp[dep])
                    comm_fn[cop](cm)
                    ev_comm[(cop, cm)] = torch.cuda.Event()
                    ev_comm[(cop, cm)].record(xs)
                    ci += 1
                    continue
            op, m = comp_ops[pi]
            dep = (comp_needs[op][0], m + comp_needs[op][1])
            if dep[1] >= 0:
                if dep not in ev_comm:
                    raise RuntimeError(f"step schedule deadlock at {op}{m}")
                cs.wait_event(ev_comm[dep])
            with torch.cuda.stream(cs):
                comp_fn[op](m)
            ev_comp[(op, m)] = torch.cuda.Event()
            ev_comp[(op, m)].record(cs)
            pi += 1
        ops.finish(ev_comm.get(("X", self.MB - 1)))

    # ------------------------------------------------------------------ per-micro-batch API
    def begin_step(self) -> None:
        """Open a step for the per-micro-batch API."""
        if getattr(self, "_ops", None) is not None:
            raise RuntimeError("begin_step called twice without end_step")
        if self.wgrad_mode != "step":
            raise RuntimeError("the per-micro-batch API needs wgrad_mode='step' (its backward order is free, so "
                               "every micro-batch's activations stay resident)")
        self.check(sync=False)
        self._ops = _StepOps(self, None)

    def forward_mb(self, m: int, x: torch.Tensor, idx: torch.Tensor, gates: torch.Tensor,
                   out: torch.Tensor) -> None:
        """Forward of micro-batch m: dispatch, expert FFN, gate-weighted combine into out [T, h].
        Ordered after the current stream's work; the current stream waits for out."""
        ops = self._require_step()
        self._check_inputs(True, x=x, idx=idx, gates=gates, out=out)
        ops.xs.wait_stream(ops.cs)
        ops.dispatch(m, x, idx, gates)
        ops.cs.wait_stream(ops.xs)
        ops.fwd_gemms(m)
        ops.xs.wait_stream(ops.cs)
        ops.combine(m, gates, out)
        ops.cs.wait_stream(ops.xs)

    def backward_mb(self, m: int, dout: torch.Tensor, dx: torch.Tensor, dgate: torch.Tensor) -> None:
        """Backward of micro-batch m (after its forward_mb): dout dispatch, dAct with the fused
        combine backward, dX, replica weight gradients (pushed back to their owners), un-permute
        into dx [T, h] and dgate [T, k].  Home weight gradients are contracted over every
        micro-batch in end_step."""
        ops = self._require_step()
        self._check_inputs(True, dout=dout, dx=dx, dgate=dgate)
        ops.xs.wait_stream(ops.cs)
        ops.dout_dispatch(m, dout)
        ops.cs.wait_stream(ops.xs)
        ops.bwd_gemms(m)
        ops.xs.wait_stream(ops.cs)
        ops.unpermute(m, dx, dgate)
        ops.cs.wait_stream(ops.xs)

    def end_step(self) -> None:
        """Home weight gradients over the step's micro-batches."""
        ops = self._require_step()
        ops.finish(None)
        self._ops = None

    def _require_step(self):
        ops = getattr(self, "_ops", None)
        if ops is None:
            raise RuntimeError("call begin_step() first")
        return ops

    def _wgrad_prepare(self) -> bool:
        """Lazy zero_grads: zero the home experts no gradient contribution will write, report
        whether this step's first contributions store (fresh) or accumulate."""
        fresh = getattr(self, "grads_pending_zero", False)
        if fresh:
            for loc in self.idle_home:
                self.gW1[loc].zero_()
                self.gW2[loc].zero_()
            self.grads_pending_zero = False
        return fresh

    step = forward_backward

    def step_host(self, host: dict, dev: dict) -> None:
        """The user-facing step with HOST (pinned) tensors: micro-batch inputs are copied
        host->device on a copy stream while earlier micro-batches run, and out/dx/dgate are copied
        device->host as soon as they exist.  `dev` holds device staging tensors of the same
        shapes.  Synchronous: returns with the results on the host (raises if a kernel flagged
        routing that differs from the plan)."""
        for key in ("x", "idx", "gates", "dout", "out", "dx", "dgate"):
            if host[key].device.type != "cpu" or not host[key].is_pinned():
                raise ValueError(f"host[{key!r}] must be a pinned CPU tensor")
            if host[key].shape != dev[key].shape or host[key].dtype != dev[key].dtype:
                raise ValueError(f"host[{key!r}] and dev[{key!r}] differ in shape or dtype")
        cur = torch.cuda.current_stream()
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(device=self.device)
            self._d2h = torch.cuda.Stream(device=self.device)
        h2d, d2h = self._h2d, self._d2h
        ready, dready = {}, {}
        h2d.wait_stream(cur)
        # copy order follows the schedule's needs: the forward inputs of micro-batch m + 1 go
        # before the dout of micro-batch m (D(m+1) is issued before C(m))
        order = [("r", None)]   # every micro-batch's routing (small) first: D(0) prepares them all
        for m in range(self.MB):
            order.append(("f", m))
            if m >= 1:
                order.append(("b", m - 1))
        order.append(("b", self.MB - 1))
        # micro-batch 0's rows arrive in head_parts pieces and the last micro-batch's dx leaves in
        # as many: the scatter of the first piece and the read-back of the first piece overlap the
        # rest of the copy (only the step's head and tail copies are exposed)
        head_parts = tail_parts = 2
        last = self.MB - 1
        with torch.cuda.stream(h2d):
            for kind, m in order:
                if kind == "r":
                    for key in ("idx", "gates"):
                        dev[key].copy_(host[key], non_blocking=True)
                    rready = torch.cuda.Event()
                    rready.record(h2d)
                    continue
                if kind == "f":
                    evs = []
                    for t0, t1 in _token_parts(self.T, head_parts if m == 0 else 1):
                        dev["x"][m][t0:t1].copy_(host["x"][m][t0:t1], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(h2d)
                        evs.append(ev)
                    ready[m] = evs
                    continue
                dev["dout"][m].copy_(host["dout"][m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                dready[m] = ev
        T = self.T

        class _Hooks:
            def routing_ready(self, stream):
                stream.wait_event(rready)

            def input_parts(self, m):
                return len(ready[m])

            def inputs_ready(self, m, stream, part=0):
                stream.wait_event(ready[m][part])

            def dout_ready(self, m, stream):
                stream.wait_event(dready[m])

            def after_forward(self, m, stream):
                d2h.wait_stream(stream)
                with torch.cuda.stream(d2h):
                    host["out"][m].copy_(dev["out"][m], non_blocking=True)

            def output_parts(self, m):
                return tail_parts if m == last else 1

            def after_backward(self, m, stream, part=0):
                t0, t1 = _token_parts(T, self.output_parts(m))[part]
                d2h.wait_stream(stream)
                with torch.cuda.stream(d2h):
                    host["dx"][m][t0:t1].copy_(dev["dx"][m][t0:t1], non_blocking=True)
                    host["dgate"][m][t0:t1].copy_(dev["dgate"][m][t0:t1], non_blocking=True)

        # the compute stream reads the dispatched rows only, so only the comm stream waits on inputs
        self.forward_backward(dev["x"], dev["idx"], dev["gates"], dev["dout"], dev["out"], dev["dx"], dev["dgate"],
                              hooks=_Hooks())
        cur.wait_stream(d2h)
        cur.synchronize()
        self.check(sync=False)

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        self.arena.close()
        self.rb.users -= 1
        if self._owns_rb and self.rb.users == 0:
            self.rb.close()
        if self._err_host:
            nat.kernels().mb_host_free(self._err_host)
            self._err_host = 0


def _token_parts(T: int, parts: int):
    """[t0, t1) ranges splitting T tokens into `parts` near-equal pieces."""
    b = [T * i // parts for i in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts) if b[i + 1] > b[i]]


class _StepOps:
    """The phases of one step of a MoEDataPlane on its streams (compute: K4 GEMMs; comm:
    histogram / permutation / scatter / combine / replica-gradient push-back and every device
    barrier; copy: replica weight pulls).  Every rank must call the phases in the same order:
    each comm phase contains collective device barriers."""

    def __init__(self, dp: "MoEDataPlane", hooks=None, own_compute_stream: bool = False):
        """own_compute_stream (the fused step): the GEMMs run on the plane's compute stream (high
        priority with MB_COMPUTE_PRIORITY=high) joined to the caller's stream at both ends."""
        self.dp, self.hooks = dp, hooks
        self.user = torch.cuda.current_stream()
        self.fresh = dp._wgrad_prepare()    # (lazy zero of idle experts on the caller's stream)
        self.cs = dp._ks if (own_compute_stream and dp._ks is not None) else self.user
        if self.cs is not self.user:
            self.cs.wait_stream(self.user)
        self.xs = dp.xs if dp.overlap else self.cs
        self.st_x = self.xs.cuda_stream
        self.xs.wait_stream(self.user)
        dp.cps.wait_stream(self.user)
        self.first = True
        self.start_ev = None
        self.prepared = set()
        self.ring_guard, self.x_barrier_ev = {}, {}   # see replica_ring_guards
        # layer-shared replica weight slots: the buffer's bookkeeping (shared by the layers), this
        # layer's earlier pulls invalidated (its weights may have changed since)
        dp.rb.invalidate(dp.token)
        if not hasattr(dp, "_tail_stream"):
            dp._tail_stream = torch.cuda.Stream(device=dp.device)
        self.tail_stream = dp._tail_stream

    # -------------------------------------------------------------- replica weights (K5)
    def _replica_set(self, kind: str, m: int) -> int:
        """Set of `kind` replica slots holding micro-batch m's replica weights: pulled by this rank
        from the owners over NVLink (copy engine) into the least useful set, after that set's last
        use; the compute stream waits for the pull."""
        dp = self.dp
        rb = dp.rb
        st = rb.state[kind]
        need = dp.mb_rep[m]
        if not need:
            return 0
        tag = (dp.token, m)
        if tag in st["held"]:
            i = st["held"].index(tag)
        else:
            cand = list(range(rb.sets))
            free = [i for i in cand if st["held"][i] is None or st["held"][i] in rb.done]
            pool = free if free else cand
            i = min(pool, key=lambda j: st["seq"][j])
            cps, A, lib = dp.cps, dp.arena, nat.kernels()
            if st["used"][i] is not None:
                cps.wait_event(st["used"][i])    # the slot's last reader (any layer)
            if self.start_ev is not None:
                cps.wait_event(self.start_ev)
            size = dp.w1_bytes if kind == "w1" else dp.w2_bytes
            base = rb.off["w1r" if kind == "w1" else "w2r"] + i * rb.slots * size
            with dp._timed(len(need) * size, "comm_replica_pull", cps):
                for q, _, owner, loc in need:
                    src = A.peer_ptr(owner, dp.off_w[kind]) + loc * size
                    nat.check(lib.mb_memcpy_async(rb.arena.peer_ptr(dp.rank, base) + q * size, src, size,
                                                  cps.cuda_stream), lib, "replica pull")
            ev = torch.cuda.Event()
            ev.record(cps)
            st["pulled"][i] = ev
            st["held"][i] = tag
        self.cs.wait_event(st["pulled"][i])
        return i

    def _replica_used(self, kind: str, i: int, m: int) -> None:
        if not self.dp.mb_rep[m]:
            return
        rb = self.dp.rb
        st = rb.state[kind]
        ev = torch.cuda.Event()
        ev.record(self.cs)
        st["used"][i] = ev
        rb.seq += 1
        st["seq"][i] = rb.seq

    # -------------------------------------------------------------- comm stream
    def _first_barrier(self):
        if self.first:
            self.dp.arena.barrier(self.xs)  # all ranks: previous step drained (buffers may be rewritten)
            self.start_ev = torch.cuda.Event()
            self.start_ev.record(self.xs)
            self.first = False

    def prepare(self, m0, m1, idx, gates, rows=True):
        """Routing side of micro-batches [m0, m1) in one launch per kernel: K1 histogram (+ the
        check against the plan's counts), chunk scan, and (rows) pad-row zeroing and K2 stable
        ranks (+ gates into the serving ranks' receive slots).  idx / gates are the [MB, T, k]
        step tensors (routing is replayed, so every micro-batch's permutation can be built before
        its rows move)."""
        dp, xs, st = self.dp, self.xs, self.st_x
        sh = dp.shape
        T, k, h, E = dp.T, sh.top_k, sh.hidden, sh.num_experts
        nb = m1 - m0
        if nb <= 0:
            return
        if self.hooks and hasattr(self.hooks, "routing_ready"):
            self.hooks.routing_ready(xs)
        dp._k("mb_expert_histogram", idx[m0].data_ptr(), nb, T, k, E, dp.counts[m0].data_ptr(),
              dp.chunk_counts[m0].data_ptr(), CHUNK, st)
        if dp.expected is not None:
            dp._k("mb_check_counts", dp.counts[m0].data_ptr(), dp.expected[m0].data_ptr(), nb * E, dp.err_dev,
                  2, st)
        dp._k("mb_chunk_scan", dp.chunk_counts[m0].data_ptr(), dp.chunk_base[m0].data_ptr(), nb,
              (T + CHUNK - 1) // CHUNK, E, st)
        if not rows:
            return
        dp._k("mb_zero_pad_rows_nb", dp.Xr[dp.set_index(m0)].data_ptr(), dp.R, dp.slot_tab[m0].data_ptr(),
              dp.plan.max_slots, nb, h, st)
        self._first_barrier()
        dp._k("mb_permute_rank_nb", idx[m0].data_ptr(), T, k, gates[m0].data_ptr(), E, dp.chunk_base[m0].data_ptr(),
              CHUNK, dp.route_tab[m0].data_ptr(), dp.ncopies[m0].data_ptr(), dp.plan.maxc,
              dp.ptr_gate[m0].data_ptr(), dp.world, dp.perm[m0].data_ptr(), nb, dp.err_dev, st)
        self.prepared.update(range(m0, m1))

    def dispatch(self, m, x, idx, gates, idx_all=None, gates_all=None):
        """D(m): routing side of m (unless prepared), K3 scatter into every rank's receive rows.
        With the step's [MB, ...] routing tensors (idx_all / gates_all), D(0) also prepares
        micro-batches 1..MB-1 once its rows have landed (wgrad_mode "step"; with the micro-batch
        buffer ring only their histograms: rows and gates of a set are written at its own D)."""
        dp, xs, st = self.dp, self.xs, self.st_x
        sh = dp.shape
        T, k, h = dp.T, sh.top_k, sh.hidden
        ring = dp.NA < dp.MB
        with dp._timed(dp.remote_rows(m)[0] * 2 * h, "comm_dispatch", xs):
            if m not in self.prepared:
                if ring and idx_all is not None and m == 0:
                    self.prepare(0, dp.MB, idx_all, gates_all, rows=False)
                self._prepare_one(m, idx, gates, histogram=not (ring and idx_all is not None))
            # the host-buffer step lands micro-batch 0's rows in parts: scatter each as it arrives
            parts = self.hooks.input_parts(m) if self.hooks and hasattr(self.hooks, "input_parts") else 1
            for p, (t0, t1) in enumerate(_token_parts(T, parts)):
                if self.hooks:
                    self.hooks.inputs_ready(m, xs, p)
                dp._k("mb_scatter_rows", x[t0:].data_ptr(), t1 - t0, k, h, dp.perm[m][t0:].data_ptr(),
                      dp.ptr_xr[m].data_ptr(), dp.comm_blocks, st)
            dp.arena.barrier(xs)  # rows of micro-batch m have landed everywhere
        if idx_all is not None and m == 0 and not ring:
            # after D(0)'s barrier, beside F(0): only pad rows (disjoint from the real rows peers
            # may already be storing) and this rank's own tables / receive gates are written
            self.prepare(1, dp.MB, idx_all, gates_all)

    def _prepare_one(self, m, idx, gates, histogram=True):
        """Routing side of micro-batch m from its own [T, k] tensors."""
        dp, xs, st = self.dp, self.xs, self.st_x
        sh = dp.shape
        T, k, h, E = dp.T, sh.top_k, sh.hidden, sh.num_experts
        if histogram:
            if self.hooks and hasattr(self.hooks, "routing_ready"):
                self.hooks.routing_ready(xs)
            dp._k("mb_expert_histogram", idx.data_ptr(), 1, T, k, E, dp.counts[m].data_ptr(),
                  dp.chunk_counts[m].data_ptr(), CHUNK, st)
            if dp.expected is not None:
                dp._k("mb_check_counts", dp.counts[m].data_ptr(), dp.expected[m].data_ptr(), E, dp.err_dev, 2, st)
            dp._k("mb_chunk_scan", dp.chunk_counts[m].data_ptr(), dp.chunk_base[m].data_ptr(), 1,
                  (T + CHUNK - 1) // CHUNK, E, st)
        self._first_barrier()
        dp._k("mb_zero_pad_rows", dp.Xr[dp.set_index(m)].data_ptr(), dp.slot_tab[m].data_ptr(), dp.nslots[m], h, st)
        dp._k("mb_permute_rank", idx.data_ptr(), T, k, gates.data_ptr(), E, dp.chunk_base[m].data_ptr(), CHUNK,
              dp.route_tab[m].data_ptr(), dp.ncopies[m].data_ptr(), dp.plan.maxc, dp.ptr_gate[m].data_ptr(),
              dp.perm[m].data_ptr(), dp.err_dev, st)
        self.prepared.add(m)

    def combine(self, m, gates, out):
        """K6: out[t] = sum_i gate * Y[perm(t, i)] over peer loads (PREGATE: the rows already
        hold gate * Y, so a plain sum)."""
        dp, xs = self.dp, self.xs
        h = dp.shape.hidden
        with dp._timed(dp.remote_rows(m)[0] * 2 * h, "comm_combine", xs):
            dp.arena.barrier(xs)  # Y of micro-batch m complete on every rank
            dp._k("mb_combine_rows", dp.ptr_y[m].data_ptr(), dp.perm[m].data_ptr(),
                  None if PREGATE else gates.data_ptr(), dp.T,
                  dp.shape.top_k, h, out.data_ptr(), None, None, 1, dp.comm_blocks, self.st_x)
            if self.hooks:
                self.hooks.after_forward(m, xs)

    def dout_dispatch(self, m, dout):
        """Backward K3: the raw dout rows follow the forward permutation."""
        dp, xs = self.dp, self.xs
        h = dp.shape.hidden
        with dp._timed(dp.remote_rows(m)[0] * 2 * h, "comm_dout_dispatch", xs):
            if self.hooks and hasattr(self.hooks, "dout_ready"):
                self.hooks.dout_ready(m, xs)
            dp._k("mb_scatter_rows", dout.data_ptr(), dp.T, dp.shape.top_k, h, dp.perm[m].data_ptr(),
                  dp.ptr_dyr[m].data_ptr(), dp.comm_blocks, self.st_x)
            dp.arena.barrier(xs)  # dout rows of micro-batch m have landed everywhere

    def unpermute(self, m, dx, dgate):
        """X(m): dX un-permute (sum over the k copies) + dgate gather, then (owners) the replica
        gradients of micro-batch m pushed back into the home experts' fp32 gradients."""
        dp, xs = self.dp, self.xs
        h = dp.shape.hidden
        with dp._timed(dp.remote_rows(m)[0] * 2 * h, "comm_unpermute", xs):
            dp.arena.barrier(xs)  # dX rows / dgate partials / replica gradients of m complete everywhere
            if m in self.ring_guard.values():
                self.x_barrier_ev[m] = torch.cuda.Event()
                self.x_barrier_ev[m].record(xs)
            # the host-buffer step reads the last micro-batch's dx back in parts, each as it is done
            parts = self.hooks.output_parts(m) if self.hooks and hasattr(self.hooks, "output_parts") else 1
            for p, (t0, t1) in enumerate(_token_parts(dp.T, parts)):
                dp._k("mb_combine_rows", dp.ptr_dxp[m].data_ptr(), dp.perm[m][t0:].data_ptr(), None, t1 - t0,
                      dp.shape.top_k, h, dx[t0:].data_ptr(), dp.ptr_dgate[m].data_ptr(), dgate[t0:].data_ptr(),
                      dp.npart, dp.comm_blocks, self.st_x)
                if self.hooks:
                    self.hooks.after_backward(m, xs, p)
        acc = dp.acc_mb[m]
        if acc is not None:
            variants, n, max_n = acc
            tasks_fresh, tasks_acc = variants[dp.bank]
            with dp._timed(n * (max_n * 4), "comm_replica_grad_pushback", xs):
                dp._k("mb_accumulate_f32_tasks", (tasks_fresh if self.fresh else tasks_acc).data_ptr(), n, max_n,
                      self.st_x)

    # -------------------------------------------------------------- compute stream
    def _fgemm(self, m, mode, A, B0, **kw):
        """One F-mode GEMM of micro-batch m.  The non-gated modes run in the single-CTA member of
        the pair family (128-row tiles, no half tiles: EP=1 ragged rows fwd1 1123 vs 1069, dX 1133 vs
        1036, fwd2 1026 vs 979 TFLOP/s; equal on even 4096-row groups); the gated dAct in the pair
        kernel.  With TAIL_TILES (opt-in) the pair kernel's odd tail blocks run in the single-CTA
        kernel on a side stream instead."""
        dp = self.dp
        ng = dp.nslots[m]
        if CTA1_F and (mode != K.GEMM_DGRAD_DSWIGLU_GATED or CTA1_DACT):
            dp._gemm(mode, A, B0, dp.groups[m][:ng], cta1=True, **kw)
            return
        gp, gt, share = dp.tail_groups[m]
        if not TAIL_TILES or gt is None:
            dp._gemm(mode, A, B0, dp.groups[m][:ng], **kw)
            return
        ts = self.tail_stream
        ts.wait_stream(self.cs)
        tail_sms = int(min(64, max(2, round(dp.gemm_sms * share))))
        K.grouped_gemm(mode, A, B0, gt, cta1=True, sms=tail_sms, stream=ts, **kw)
        dp.launches += 1
        dp._gemm(mode, A, B0, gp[:ng], **kw)
        self.cs.wait_stream(ts)

    def fwd_gemms(self, m):
        """F(m): gate/up GEMM + SwiGLU, down GEMM."""
        dp = self.dp
        h, hp = dp.shape.hidden, dp.shape.ffn
        ng = dp.nslots[m]
        if ng:
            a = dp.set_index(m)
            rows = dp.real_rows(m)
            i1 = self._replica_set("w1", m)
            with dp._timed(4.0 * rows * h * hp, "fwd_swiglu"):
                self._fgemm(m, K.GEMM_FWD_SWIGLU, dp.Xr[a], dp.W1, N=2 * hp, K=h, C=dp.H[a], C2=dp.Act[a],
                            B1=dp.W1r[i1], row_scale=dp.gate_r[a] if PREGATE else None)
            self._replica_used("w1", i1, m)
            i2 = self._replica_set("w2", m)
            with dp._timed(2.0 * rows * h * hp, "fwd_down"):
                self._fgemm(m, K.GEMM_FWD_STORE, dp.Act[a], dp.W2, N=h, K=hp, C=dp.Y[a], B1=dp.W2r[i2])
            self._replica_used("w2", i2, m)

    def bwd_gemms(self, m):
        """B(m): dAct with the combine backward + dSwiGLU fused in its epilogue, dX, then the
        weight gradients of the replicas this rank served (stored into the gradient ring)."""
        dp = self.dp
        h, hp = dp.shape.hidden, dp.shape.ffn
        ng = dp.nslots[m]
        if ng:
            a = dp.set_index(m)
            rows = dp.real_rows(m)
            i2 = self._replica_set("w2", m)
            # dAct = dout.W2 with the combine backward fused in the epilogue: gate applied per row,
            # dgate partials <dout.W2, act> = <dout, Y>; Act already holds gate*act for dW2
            # (PREGATE; otherwise the epilogue writes it over Act)
            with dp._timed(2.0 * rows * h * hp, "dgrad_act_gated"):
                self._fgemm(m, K.GEMM_DGRAD_DSWIGLU_GATED, dp.dYr[a], dp.W2, N=hp, K=h, C=dp.dH[a],
                            C2=None if PREGATE else dp.Act[a], aux=dp.H[a], B1=dp.W2r[i2], row_scale=dp.gate_r[a],
                            row_partial=dp.dgate_r[a])
            self._replica_used("w2", i2, m)
            i1 = self._replica_set("w1", m)
            with dp._timed(4.0 * rows * h * hp, "dgrad_x"):
                self._fgemm(m, K.GEMM_DGRAD_STORE, dp.dH[a], dp.W1, N=h, K=2 * hp, C=dp.dXp[a], B1=dp.W1r[i1])
            self._replica_used("w1", i1, m)
        dp.rb.done.add((dp.token, m))
        rw = dp.rw_mb[m]
        if rw is not None:
            tabs, segs, rrows = rw
            a, q = dp.set_index(m), m % GRAD_RING
            if m in self.ring_guard:   # ring set q: every owner has read it (X(m - GRAD_RING))
                ev = self.x_barrier_ev.get(self.ring_guard[m])
                if ev is None:
                    raise RuntimeError(f"replica-gradient ring guard of B({m}) issued before X({self.ring_guard[m]})")
                self.cs.wait_event(ev)
            with dp._timed(6.0 * rrows * h * hp, "wgrad_replica"):
                self._wgrad_launch(tabs, segs, dp.dYr[a], dp.Act[a], dp.rgW2[q], dp.dH[a], dp.Xr[a], dp.rgW1[q],
                                   sms=dp.all_sms if REPLICA_WGRAD_ALL_SMS else None)

    def _wgrad_launch(self, tabs, segs, dY, act, c2, dh, xr, c1, sms=None):
        """dW2 (C2 (+)= dY^T act) and dW1 (C1 (+)= dH^T X) of the groups in `tabs`: one two-problem
        launch (mb_grouped_wgrad2) unless MB_WGRAD_MERGED=0 or the doubled table is too long."""
        dp = self.dp
        h, hp = dp.shape.hidden, dp.shape.ffn
        single, merged = tabs
        R = dY.numel() // h
        if WGRAD_MERGED and merged is not None:
            K.grouped_wgrad2(dY.view(R, h), act.view(R, hp), c2, dh.view(R, 2 * hp), xr.view(R, h), c1, merged,
                             segs=segs, sms=dp.gemm_sms if sms is None else sms)
            dp.launches += 1
            return
        dp._gemm(K.GEMM_WGRAD, dY.view(R, h), act.view(R, hp), single, M=h, N=hp, C=c2, c_slot_stride=h * hp,
                 segs=segs, sms=sms)
        dp._gemm(K.GEMM_WGRAD, dh.view(R, 2 * hp), xr.view(R, h), single, M=2 * hp, N=h, C=c1,
                 c_slot_stride=2 * hp * h, segs=segs, sms=sms)

    def wgrad_mb(self, m):
        """W(m) (wgrad_mode "micro_batch"): home weight gradients of micro-batch m, K = its rows."""
        dp = self.dp
        w = dp.w_mb[m]
        if w is None:
            return
        tabs_fresh, tabs_acc, segs, rows = w
        h, hp = dp.shape.hidden, dp.shape.ffn
        a = dp.set_index(m)
        with dp._timed(6.0 * rows * h * hp, "wgrad"):
            self._wgrad_launch(tabs_fresh if self.fresh else tabs_acc, segs, dp.dYr[a], dp.Act[a], dp.gW2, dp.dH[a],
                               dp.Xr[a], dp.gW1)

    def _wgrad_step(self, part, sms):
        dp = self.dp
        tabs_fresh, tabs_acc, segs, rows, _ = part
        h, hp = dp.shape.hidden, dp.shape.ffn
        with dp._timed(6.0 * rows * h * hp, "wgrad"):
            self._wgrad_launch(tabs_fresh if self.fresh else tabs_acc, segs, dp.dYr, dp.Act, dp.gW2, dp.dH, dp.Xr,
                               dp.gW1, sms=sms)

    def finish(self, last_x_ev):
        """Step mode: home weight gradients over every micro-batch (part B: experts without
        replica gradients, right after the last backward; part A: the rest, after the last
        replica-gradient push-back, on every SM); then every stream joins the current one."""
        dp, cs, xs = self.dp, self.cs, self.xs
        with torch.cuda.stream(cs):
            if dp.wgrad_mode == "step":
                part_b, part_a = dp.wparts
                if part_b is not None:
                    self._wgrad_step(part_b, None)
                if part_a is not None:
                    if last_x_ev is not None:
                        cs.wait_event(last_x_ev)
                    else:
                        cs.wait_stream(xs)
                    # the comm stream is idle by now: the last weight-gradient launch takes every SM
                    self._wgrad_step(part_a, dp.all_sms if (WGRAD_ALL_SMS and dp.overlap) else None)
        cs.wait_stream(xs)
        cs.wait_stream(dp.cps)
        if cs is not self.user:
            self.user.wait_stream(cs)


class MoELayerFunction(torch.autograd.Function):
    """torch.autograd entry for one micro-batch of a MoEDataPlane step:

        dp.begin_step()
        outs = [MoELayerFunction.apply(x[m], gates[m], dp, idx[m], m) for m in range(MB)]
        ... loss.backward()        # runs backward_mb for every micro-batch
        dp.end_step()              # home weight gradients into dp.gW1 / gW2

    Differentiable in x ([T, h] bf16) and gates ([T, k] fp32); the expert weight gradients
    accumulate inside the data plane (fp32, all micro-batches of the step in one contraction;
    replica gradients pushed back per micro-batch).  Every rank must run the same micro-batches
    in the same order (collective barriers)."""

    @staticmethod
    def forward(ctx, x, gates, dp, idx, m):
        out = torch.empty_like(x)
        dp.forward_mb(m, x.contiguous(), idx.contiguous(), gates.contiguous(), out)
        ctx.dp, ctx.m = dp, m
        ctx.k = idx.shape[-1]
        return out

    @staticmethod
    def backward(ctx, dout):
        dp, m = ctx.dp, ctx.m
        dx = torch.empty_like(dout)
        dgate = torch.empty(dout.shape[0], ctx.k, dtype=torch.float32, device=dout.device)
        dp.backward_mb(m, dout.contiguous(), dx, dgate)
        return dx, dgate, None, None, None


# ----------------------------------------------------------------------------- batch boundaries


def relabel_for_overlap(new_home: np.ndarray, old_home: np.ndarray, topo: ClusterTopology) -> np.ndarray:
    """The GPU relabeling of `new_home` (a permutation of GPU ids that maps whole groups onto
    groups, so replicas stay inside a group) that keeps the most experts where `old_home` has
    them: max sum_e [pi(new_home[e]) == old_home[e]] as two nested assignment problems (GPUs
    inside each pair of groups, then groups).  The relabeled plan balances the same loads; its
    modelled time differs only through which token rows stay local."""
    g, gs = topo.num_gpus, topo.gpus_per_node
    ng = g // gs
    new_home, old_home = np.asarray(new_home, dtype=np.int64), np.asarray(old_home, dtype=np.int64)
    overlap = np.zeros((g, g), dtype=np.int64)   # [new gpu, old gpu]
    np.add.at(overlap, (new_home, old_home), 1)

    def best_assignment(mat):
        try:
            from scipy.optimize import linear_sum_assignment
            r, c = linear_sum_assignment(-mat)
            return list(c[np.argsort(r)]), int(mat[r, c].sum())
        except ImportError:   # small groups: exhaustive
            import itertools
            best, perm = -1, None
            for p in itertools.permutations(range(mat.shape[0])):
                v = int(sum(mat[i, p[i]] for i in range(len(p))))
                if v > best:
                    best, perm = v, list(p)
            return perm, best

    inner, gval = {}, np.zeros((ng, ng), dtype=np.int64)
    for a in range(ng):
        for b in range(ng):
            sub = overlap[a * gs:(a + 1) * gs, b * gs:(b + 1) * gs]
            inner[(a, b)], gval[a, b] = best_assignment(sub)
    outer, _ = best_assignment(gval)
    pi = np.zeros(g, dtype=np.int64)
    for a in range(ng):
        b = outer[a]
        for i, j in enumerate(inner[(a, b)]):
            pi[a * gs + i] = b * gs + j
    return pi[new_home]


def migration_aware_step_plan(prev: "StepPlan", mats: np.ndarray, topo: ClusterTopology, model: rt.ModelProfile,
                              hw: HardwareProfile, cfgs: pol.SimConfigs, shape: LayerShape,
                              bytes_per_expert: float, steps_per_batch: int = 1, link_bw: float = 700e9) -> tuple:
    """ReLibra's plan for the next batch with the expert migration it implies priced in (the
    reference plans every batch from scratch and does not model migration; PAPER.md:1081-1084
    reports it as overhead): the annealing reorder of the new batch (seeded with the current
    placement as an extra initial plan), relabeled for the largest overlap with the current
    placement, against keeping the current placement; each candidate is scored as
    steps_per_batch x its modelled step time (greedy replication per micro-batch) + the time to
    pull its incoming experts (bytes_per_expert per expert, max over ranks, over NVLink).
    Returns (StepPlan, info)."""
    from . import reordering as ro
    trace = rt.build_trace(model, topo, mats[:, None], tokens_per_gpu=0)
    agg = rt.aggregate_batch(trace, 0)
    new = ro.anneal_reorder(agg, topo, model, hw, cfgs.anneal,
                            extra_initial_plans=[ro.static_plan(model.num_experts, topo),
                                                 ro.ReorderPlan(np.asarray(prev.home, dtype=np.int64).copy())])
    relabeled = relabel_for_overlap(new.assignment, prev.home, topo)
    cands = {"keep": np.asarray(prev.home, dtype=np.int64), "reorder": relabeled}
    scored = {}
    for name, home in cands.items():
        bundle = pol.replication_bundle(trace, [ro.ReorderPlan(home.copy())], topo, model, hw, cfgs)
        plan = step_plan_from_bundle("relibra", bundle, mats, shape, layer=0, slots=cfgs.replica.slots_per_gpu)
        moved_in = np.array([int(((home == d) & (prev.home != d)).sum()) for d in range(topo.num_gpus)])
        mig_s = float(moved_in.max()) * bytes_per_expert / link_bw
        t = steps_per_batch * plan.predicted_ms(topo, model, hw) / 1e3 + mig_s
        scored[name] = (t, plan, int(moved_in.sum()), mig_s)
    choice = min(scored, key=lambda k: (scored[k][0], k != "keep"))
    t, plan, moved, mig_s = scored[choice]
    info = {"choice": choice, "experts_moved": moved, "predicted_migration_ms": mig_s * 1e3,
            "predicted_batch_ms": {k: v[0] * 1e3 for k, v in scored.items()},
            "moved_without_relabel": int((new.assignment != prev.home).sum())}
    return plan, info
