"""Per-GPU load accounting and the MoE time model.

Mirror of ``moebalance.costmodel`` (costmodel.py:19-213).  ``flow_matrix`` and
``compute_loads`` run in the C++ planner library (libmb_planner.so, mbp_compute_loads) with
numpy's exact reduction order, so loads are bit-identical to the reference's; the
elementwise time conversions stay in numpy exactly as the reference writes them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .cluster import ClusterTopology, HardwareProfile

SPLIT_TOL = 1e-6

SplitMap = dict  # expert -> (serving GPUs (k,), fractions (G, k))


@dataclass(frozen=True)
class SmoothingConfig:
    beta: float = 20.0

    def __post_init__(self) -> None:
        if not self.beta > 0:
            raise ValueError(f"beta must be > 0, got {self.beta!r}")


@dataclass
class LoadVector:
    comp: np.ndarray
    nvlink_tx: np.ndarray
    nvlink_rx: np.ndarray
    rdma_tx: np.ndarray
    rdma_rx: np.ndarray
    expert_load: np.ndarray

    def comm_rows(self) -> np.ndarray:
        return np.stack([self.nvlink_tx, self.nvlink_rx, self.rdma_tx, self.rdma_rx])


@dataclass
class CostEstimate:
    comp_times: np.ndarray
    comm_times: np.ndarray
    t_moe: float
    t_moe_smoothed: float | None = None


def _check_split_entry(x, placement, e, gpus, frac, num_experts) -> None:
    if not 0 <= e < num_experts:
        raise ValueError(f"split entry for unknown expert {e}")
    if placement[e] not in gpus:
        raise ValueError(f"split for expert {e} omits its home GPU {placement[e]}")
    if frac.shape != (x.shape[0], len(gpus)):
        raise ValueError(f"split fractions for expert {e} have shape {frac.shape}, expected {(x.shape[0], len(gpus))}")
    if frac.min() < -SPLIT_TOL or frac.max() > 1 + SPLIT_TOL:
        raise ValueError(f"split fractions for expert {e} outside [0, 1]")
    routed = x[:, e] > 0
    if routed.any():
        err = np.abs(frac[routed].sum(axis=1) - 1.0).max()
        if err > SPLIT_TOL:
            raise ValueError(f"split fractions for expert {e} violate conservation by {float(err):.3e}")


def _native_loads(x, placement, topo: ClusterTopology, splits: SplitMap | None, want_flow: bool):
    g = topo.num_gpus
    num_experts = x.shape[1]
    experts, ptrs, gpus_flat, fracs = [], [0], [], []
    for e, (gpus, frac) in (splits or {}).items():
        gpus = np.asarray(gpus)
        frac = np.asarray(frac, dtype=np.float64)
        _check_split_entry(x, placement, int(e), gpus, frac, num_experts)
        experts.append(int(e))
        gpus_flat.extend(int(v) for v in gpus)
        ptrs.append(len(gpus_flat))
        fracs.append(np.ascontiguousarray(frac).ravel())
    xs = nat.f64(x)
    pl = nat.i64(placement)
    se, sp, sg = nat.i32(experts), nat.i32(ptrs), nat.i32(gpus_flat)
    sf = nat.f64(np.concatenate(fracs) if fracs else np.zeros(0))
    out = np.zeros((5, g))
    flow = np.zeros((g, g)) if want_flow else None
    lib = nat.planner()
    nat.check(lib.mbp_compute_loads(nat.ptr(xs), topo.num_nodes, topo.gpus_per_node, num_experts, nat.ptr(pl),
                                    len(experts), nat.ptr(se), nat.ptr(sp), nat.ptr(sg), nat.ptr(sf),
                                    nat.ptr(out), nat.ptr(flow)), lib, "compute_loads")
    return out, flow


def flow_matrix(x, placement, topo: ClusterTopology, splits: SplitMap | None = None) -> np.ndarray:
    """(G, G) flow[src, serving GPU] (costmodel.py:91-108)."""
    x = np.asarray(x, dtype=np.float64)
    return _native_loads(x, np.asarray(placement), topo, splits, True)[1]


def compute_loads(x, placement, topo: ClusterTopology, splits: SplitMap | None = None) -> LoadVector:
    """Computation and the four link loads per GPU, dispatch + mirrored combine (costmodel.py:127-158)."""
    x = np.asarray(x, dtype=np.float64)
    g = topo.num_gpus
    placement = np.asarray(placement)
    if placement.shape != (x.shape[1],):
        raise ValueError(f"placement covers {placement.shape} experts, routing matrix has {x.shape[1]}")
    if placement.min() < 0 or placement.max() >= g:
        raise ValueError("placement references GPU ids outside the topology")
    if x.shape[0] != g:
        raise ValueError(f"routing matrix has {x.shape[0]} source rows, topology has {g} GPUs")
    out, _ = _native_loads(x, placement, topo, splits, False)
    return LoadVector(comp=out[0], nvlink_tx=out[1], nvlink_rx=out[2], rdma_tx=out[3], rdma_rx=out[4],
                      expert_load=x.sum(axis=0))


def comp_time(load, model, hw: HardwareProfile):
    """6 h h' L / F seconds (costmodel.py:161-163)."""
    return 6.0 * model.hidden_size * model.intermediate_size * np.asarray(load, dtype=np.float64) / hw.flops_per_gpu


def comm_row_times(loads: LoadVector, hw: HardwareProfile) -> np.ndarray:
    rows = loads.comm_rows() * hw.bytes_per_token
    rows[0:2] /= hw.bw_nvlink
    rows[2:4] /= hw.bw_rdma
    return rows


def comm_time(loads: LoadVector, hw: HardwareProfile) -> np.ndarray:
    return comm_row_times(loads, hw).max(axis=0)


def lse(values, beta: float) -> float:
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise ValueError("lse of an empty vector")
    if not beta > 0:
        raise ValueError(f"beta must be > 0, got {beta!r}")
    m = v.max()
    return float(m + np.log(np.exp(beta * (v - m)).sum()) / beta)


def smoothed_moe_time(loads: LoadVector, model, hw: HardwareProfile, cfg: SmoothingConfig) -> float:
    comp = comp_time(loads.comp, model, hw)
    rows = comm_row_times(loads, hw)
    inner = np.array([lse(rows[:, g], cfg.beta) for g in range(rows.shape[1])])
    return lse(comp, cfg.beta) + lse(inner, cfg.beta)


def moe_time(loads: LoadVector, model, hw: HardwareProfile, smoothing: SmoothingConfig | None = None) -> CostEstimate:
    """max comp time + max comm time (Eq. 6; costmodel.py:202-213)."""
    comp = comp_time(loads.comp, model, hw)
    comm = comm_time(loads, hw)
    est = CostEstimate(comp_times=comp, comm_times=comm, t_moe=float(comp.max() + comm.max()))
    if smoothing is not None:
        est.t_moe_smoothed = smoothed_moe_time(loads, model, hw, smoothing)
    return est
