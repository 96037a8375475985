"""Synthetic workload of the benchmark and tests: replayed token routing, layer weights and
upstream gradients, plus the named shapes of BASELINE.json.

Data is synthetic by construction (no network, no checkpoints): Zipf-skewed Gumbel-top-k
routing with a hot set rotating every micro-batch, weights
N(0, h^-1/2) bf16, activations and upstream gradients N(0, 1) bf16.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .moe_layer import LayerShape
from .traces import ZipfRouting

SHAPES = {
    # BASELINE.json configs
    "tiny": dict(shape=LayerShape(num_experts=8, top_k=2, hidden=512, ffn=512), shift=1, slots=2, group=2),
    "qwen3-30b-a3b": dict(shape=LayerShape(num_experts=128, top_k=8, hidden=2048, ffn=768), shift=7, slots=2, group=4),
    "mixtral-8x7b": dict(shape=LayerShape(num_experts=8, top_k=2, hidden=4096, ffn=14336), shift=1, slots=1, group=4),
    "qwen3-235b-a22b": dict(shape=LayerShape(num_experts=128, top_k=8, hidden=4096, ffn=1536), shift=7, slots=2,
                            group=4),
}


@dataclass
class Routing:
    idx: np.ndarray     # [MB, T, k] int32 (this rank)
    gates: np.ndarray   # [MB, T, k] float32
    mats: np.ndarray    # [MB, G, E] int64 counts of every rank (np.bincount, host side)


def make_routing(shape: LayerShape, tokens: int, micro_batches: int, world: int, rank: int, zipf_s: float = 1.0,
                 shift: int = 7, seed: int = 20261018, balanced: bool = False, all_ranks: bool = True,
                 mb_offset: int = 0) -> Routing:
    """This rank's token-level indices/gates and (all_ranks) every rank's counts via np.bincount.
    With all_ranks=False only this rank's row of `mats` is filled (the caller histograms on the
    device and all-gathers, see moe_layer.gather_routing).  mb_offset: index of the first
    micro-batch in the run (a sequence of batches continues the hot-set rotation)."""
    gen = ZipfRouting(shape.num_experts, shape.top_k, tokens, zipf_s=zipf_s, shift=shift, seed=seed,
                      balanced=balanced)
    mats = np.zeros((micro_batches, world, shape.num_experts), dtype=np.int64)
    idx = np.zeros((micro_batches, tokens, shape.top_k), dtype=np.int32)
    gates = np.zeros((micro_batches, tokens, shape.top_k), dtype=np.float32)
    for m in range(micro_batches):
        for j in range(world) if all_ranks else (rank,):
            i_j, g_j = gen.sample(m + mb_offset, 0, j)
            mats[m, j] = np.bincount(i_j.ravel(), minlength=shape.num_experts)
            if j == rank:
                idx[m], gates[m] = i_j, g_j
    return Routing(idx=idx, gates=gates, mats=mats)


def make_weights(shape: LayerShape, seed: int = 1234, device="cpu"):
    """Logical expert weights (bf16): gate/up [E, h', h], down [E, h, h']."""
    gen = torch.Generator(device="cpu").manual_seed(seed)
    e, h, hp = shape.num_experts, shape.hidden, shape.ffn
    wg = (torch.randn(e, hp, h, generator=gen) * h ** -0.5).bfloat16()
    wu = (torch.randn(e, hp, h, generator=gen) * h ** -0.5).bfloat16()
    wd = (torch.randn(e, h, hp, generator=gen) * hp ** -0.5).bfloat16()
    return wg.to(device), wu.to(device), wd.to(device)


def make_weights_for(shape: LayerShape, experts: np.ndarray, seed: int = 1234, device="cuda"):
    """Weights of a subset of experts generated directly on the device (deterministic per expert),
    for shapes too large to materialise every expert on the host."""
    h, hp = shape.hidden, shape.ffn
    out = [torch.empty((len(experts), hp, h), dtype=torch.bfloat16, device=device),
           torch.empty((len(experts), hp, h), dtype=torch.bfloat16, device=device),
           torch.empty((len(experts), h, hp), dtype=torch.bfloat16, device=device)]
    for i, e in enumerate(experts):
        gen = torch.Generator(device=device).manual_seed(seed * 100003 + int(e))
        out[0][i] = (torch.randn(hp, h, generator=gen, device=device) * h ** -0.5).bfloat16()
        out[1][i] = (torch.randn(hp, h, generator=gen, device=device) * h ** -0.5).bfloat16()
        out[2][i] = (torch.randn(h, hp, generator=gen, device=device) * hp ** -0.5).bfloat16()
    return out


def make_activations(shape: LayerShape, tokens: int, micro_batches: int, rank: int, seed: int = 99, device="cpu"):
    """Token activations x and upstream gradients dout [MB, T, h] bf16 of one rank."""
    gen = torch.Generator(device="cpu").manual_seed(seed + 7919 * rank)
    x = torch.randn(micro_batches, tokens, shape.hidden, generator=gen).bfloat16()
    dout = torch.randn(micro_batches, tokens, shape.hidden, generator=gen).bfloat16()
    return x.to(device), dout.to(device)
