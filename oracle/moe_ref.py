"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): CPU restatement of the data plane.

Everything here is written independently of the product code (no import of
paper_2605_08639_b200) so that it can check it.
"""

from __future__ import annotations

import numpy as np
import torch


# ----------------------------------------------------------------------------- integer path

def histogram(idx: np.ndarray, num_experts: int) -> np.ndarray:
    """x[e] = #{(t,i): idx[t,i] == e}: one row of RoutingTrace.matrices (routing.py:151-168).
    Entries outside [0, E) (dropped choices, idx = -1) are not counted."""
    v = np.asarray(idx, dtype=np.int64).ravel()
    v = v[(v >= 0) & (v < num_experts)]
    return np.bincount(v, minlength=num_experts).astype(np.int64)


def copies_of(e: int, home, replicas: dict) -> list:
    """ReplicaPlacement.copies (replicate.py:55-56): [home] + replicas in insertion order."""
    return [int(home[e])] + [int(g) for g in replicas.get(e, [])]


def split_counts(x: np.ndarray, home, replicas: dict, counts: dict, j: int, e: int) -> list:
    """Integer tokens of (source j, expert e) per copy: round_split counts, or all at home."""
    if e in counts and e in replicas:
        return [int(v) for v in counts[e][j]]
    return [int(x[j, e])]


def receive_layout(x: np.ndarray, home, replicas: dict, counts: dict, pad: int = 128):
    """Receive layout of every GPU (defined by this build): slots = home experts ascending,
    then replicated experts ascending; inside a slot, source GPU ascending; slots padded to
    `pad` rows.  Returns (slots[d] = [(expert, copy, row_begin, rows_real, rows_pad)],
    row_base[(j, e, c)] = first destination row of source j's share of copy c)."""
    g, num_experts = x.shape
    slots, row_base = [], {}
    for d in range(g):
        mine = []
        for e in range(num_experts):
            if int(home[e]) == d:
                mine.append((e, 0))
        for e in range(num_experts):
            cps = copies_of(e, home, replicas)
            for c in range(1, len(cps)):
                if cps[c] == d:
                    mine.append((e, c))
        row = 0
        out = []
        for e, c in mine:
            begin = row
            real = 0
            for j in range(g):
                row_base[(j, e, c)] = begin + real
                real += split_counts(x, home, replicas, counts, j, e)[c]
            padded = -(-real // pad) * pad
            out.append((e, c, begin, real, padded))
            row += padded
        slots.append(out)
    return slots, row_base


def executed_flow(x: np.ndarray, home, replicas: dict, counts: dict) -> np.ndarray:
    """flow[j, d] = token rows source j sends to GPU d (costmodel.flow_matrix, costmodel.py:91-108,
    with the fractions replaced by their round_split integers)."""
    g, num_experts = x.shape
    flow = np.zeros((g, g), dtype=np.int64)
    for j in range(g):
        for e in range(num_experts):
            for c, d in enumerate(copies_of(e, home, replicas)):
                flow[j, d] += split_counts(x, home, replicas, counts, j, e)[c]
    return flow


def canonical_permutation(idx: np.ndarray, j: int, x: np.ndarray, home, replicas: dict, counts: dict,
                          row_base: dict) -> np.ndarray:
    """perm[t, i] = (dst GPU, dst row) for source GPU j, (t, i) enumerated row-major; the
    stable rank r of (t, i) among j's entries of expert e picks copy c = min{c: r < cum[c]}.
    Dropped choices (idx outside [0, E)) map to (-1, -1)."""
    t_n, k = idx.shape
    num_experts = len(home)
    perm = np.full((t_n, k, 2), -1, dtype=np.int32)
    seen = {}
    for t in range(t_n):
        for i in range(k):
            e = int(idx[t, i])
            if not 0 <= e < num_experts:
                continue
            r = seen.get(e, 0)
            seen[e] = r + 1
            cnt = split_counts(x, home, replicas, counts, j, e)
            cps = copies_of(e, home, replicas)
            acc = 0
            for c, n in enumerate(cnt):
                if r < acc + n or c == len(cnt) - 1:
                    perm[t, i] = (cps[c], row_base[(j, e, c)] + r - acc)
                    break
                acc += n
    return perm


def canonical_permutation_fast(idx: np.ndarray, j: int, x, home, replicas, counts, row_base) -> np.ndarray:
    """Vectorised equivalent of canonical_permutation (stable argsort by expert)."""
    flat = np.asarray(idx, dtype=np.int64).ravel()
    order = np.argsort(flat, kind="stable")
    sorted_e = flat[order]
    starts = np.searchsorted(sorted_e, sorted_e, side="left")
    rank = np.empty_like(flat)
    rank[order] = np.arange(flat.size) - starts
    out = np.full((flat.size, 2), -1, dtype=np.int64)
    for e in np.unique(flat):
        if not 0 <= e < len(home):
            continue  # dropped choice
        sel = flat == e
        r = rank[sel]
        cnt = np.asarray(split_counts(x, home, replicas, counts, j, int(e)))
        cum = np.cumsum(cnt)
        c = np.minimum(np.searchsorted(cum, r, side="right"), len(cnt) - 1)
        before = np.concatenate([[0], cum[:-1]])[c]
        cps = np.asarray(copies_of(int(e), home, replicas))
        base = np.asarray([row_base[(j, int(e), int(cc))] for cc in range(len(cnt))])
        out[sel, 0] = cps[c]
        out[sel, 1] = base[c] + r - before
    return out.reshape(idx.shape + (2,)).astype(np.int32)


# ----------------------------------------------------------------------------- layer math

def moe_layer_fp32(x: torch.Tensor, idx: torch.Tensor, gates: torch.Tensor, w_gate: torch.Tensor,
                   w_up: torch.Tensor, w_down: torch.Tensor, dout: torch.Tensor) -> dict:
    """fp32 SwiGLU expert FFN (three GEMMs per expert) with top-k gate-weighted
    combine and its backward:
        h_g = x Wg^T, h_u = x Wu^T, a = silu(h_g) * h_u, y = a Wd^T, out[t] = sum_i gate[t,i] y_{e(t,i)}[t]
    Where a token's expert runs (home or any replica) does not change the math; replicas hold
    identical weights and their gradients are summed at the owner.
    Returns out, dx, dgate, dWg, dWu, dWd (fp32)."""
    x = x.float()
    dout = dout.float()
    gates = gates.float()
    t_n, k = idx.shape
    num_experts = w_gate.shape[0]
    out = torch.zeros_like(x)
    dx = torch.zeros_like(x)
    dgate = torch.zeros(t_n, k, dtype=torch.float32, device=x.device)
    dwg = torch.zeros_like(w_gate, dtype=torch.float32)
    dwu = torch.zeros_like(w_up, dtype=torch.float32)
    dwd = torch.zeros_like(w_down, dtype=torch.float32)
    flat_e = idx.reshape(-1).long()
    flat_t = torch.arange(t_n, device=x.device).repeat_interleave(k)
    flat_g = gates.reshape(-1)
    for e in range(num_experts):
        sel = torch.nonzero(flat_e == e).flatten()
        if sel.numel() == 0:
            continue
        tok = flat_t[sel]
        g = flat_g[sel][:, None]
        xe = x[tok]
        wg, wu, wd = w_gate[e].float(), w_up[e].float(), w_down[e].float()
        hg, hu = xe @ wg.T, xe @ wu.T
        s = torch.sigmoid(hg)
        a = hg * s * hu
        y = a @ wd.T
        out.index_add_(0, tok, g * y)
        do = dout[tok]
        dgate.view(-1)[sel] = (do * y).sum(dim=1)
        dy = g * do
        da = dy @ wd
        dwd[e] += dy.T @ a
        dhu = da * hg * s
        dhg = da * hu * s * (1 + hg * (1 - s))
        dwg[e] += dhg.T @ xe
        dwu[e] += dhu.T @ xe
        dx.index_add_(0, tok, dhg @ wg + dhu @ wu)
    return {"out": out, "dx": dx, "dgate": dgate, "dWg": dwg, "dWu": dwu, "dWd": dwd}


def rel_err(got: torch.Tensor, ref: torch.Tensor) -> float:
    """max |got - ref| / max |ref| (the documented bf16 tolerance metric, bound 2e-2)."""
    got, ref = got.float(), ref.float()
    den = ref.abs().max().clamp_min(1e-12)
    return float((got - ref.to(got.device)).abs().max() / den)


def rel_l2(got: torch.Tensor, ref: torch.Tensor) -> float:
    """||got - ref||_2 / ||ref||_2 over the whole tensor (normalised L2)."""
    got, ref = got.float(), ref.float().to(got.device)
    return float((got - ref).norm() / ref.norm().clamp_min(1e-30))


def row_rel(got: torch.Tensor, ref: torch.Tensor, floor: float = 0.25) -> float:
    """max over rows (last dim = a row) of ||got_row - ref_row|| / max(||ref_row||, floor x RMS row
    norm): every row is judged on its own scale (cold experts, small tokens), not on the tensor's
    maximum; the floor keeps rows that are small by cancellation (a dgate dot product near 0,
    whose rounding error scales with its operands, not its value) from dominating."""
    got, ref = got.float(), ref.float().to(got.device)
    g2, r2 = got.reshape(-1, got.shape[-1]), ref.reshape(-1, ref.shape[-1])
    rn = r2.norm(dim=1)
    rms = rn.pow(2).mean().sqrt()
    if float(rms) == 0.0:
        return float((g2 - r2).abs().max()) if g2.numel() else 0.0
    return float(((g2 - r2).norm(dim=1) / torch.maximum(rn, floor * rms)).max())


# documented bf16 tolerances of the data plane against this fp32 restatement (north_star: rel 2e-2)
TOL_MAX_REL = 2e-2     # max |d| / max |ref|
TOL_L2 = 1e-2          # normalised L2 of the whole tensor
TOL_ROW = 5e-2         # per row (token row of out / dx, k choices of dgate, per-expert gradient slice)


def close(got: torch.Tensor, ref: torch.Tensor) -> dict:
    """All three error measures and whether each is inside its documented bound."""
    m = {"max_rel": rel_err(got, ref), "l2": rel_l2(got, ref), "row": row_rel(got, ref)}
    m["ok"] = m["max_rel"] < TOL_MAX_REL and m["l2"] < TOL_L2 and m["row"] < TOL_ROW
    return m


def expert_grads_close(got: torch.Tensor, ref: torch.Tensor) -> dict:
    """Per-expert gradients [experts, rows, cols]: every expert judged on its own norm (cold
    experts included), plus the whole-tensor measures."""
    m = close(got, ref)
    per = [rel_l2(got[i], ref[i]) for i in range(got.shape[0]) if float(ref[i].float().abs().max()) > 0]
    m["expert_l2_max"] = max(per) if per else 0.0
    m["ok"] = m["ok"] and m["expert_l2_max"] < TOL_ROW
    return m
