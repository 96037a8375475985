"""Micro-benchmark of the K4 grouped GEMM modes at MoE-layer shapes (CUDA events).

usage: python tools/bench_gemm.py [--rows-per-group 512] [--groups 128] [--h 2048] [--hp 768]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08639_b200 import kernels as K  # noqa: E402


def timeit(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows-per-group", type=int, default=512)
    ap.add_argument("--groups", type=int, default=128)
    ap.add_argument("--h", type=int, default=2048)
    ap.add_argument("--hp", type=int, default=768)
    ap.add_argument("--only", default="")
    ap.add_argument("--cublas", action="store_true",
                    help="also time torch.bmm (cuBLAS) on the same balanced shapes, plain GEMMs without epilogues")
    ap.add_argument("--zipf-rows", action="store_true",
                    help="group rows = micro-batch 0 of the bench's skewed Qwen3 routing at EP=1 (128-padded)")
    ap.add_argument("--single", action="store_true",
                    help="F modes in the single-CTA (cta_group::1, 128-row tile) member of the pair family")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    G, r, h, hp = a.groups, a.rows_per_group, a.h, a.hp
    R = G * r
    dev = "cuda"
    rows = [r] * G
    if a.zipf_rows:
        from paper_2605_08639_b200.workload import SHAPES, make_routing
        rt = make_routing(SHAPES["qwen3-30b-a3b"]["shape"], 8192, 1, 1, 0)
        rows = [int((c + 127) // 128 * 128) for c in rt.mats[0, 0]]
        G = len(rows)
    a0 = [sum(rows[:i]) for i in range(G)]
    R = sum(rows)
    groups = K.make_groups(rows, a0, list(range(G)))
    wg = K.make_groups(rows, a0, list(range(G)), [K.FLAG_ACCUMULATE] * G)
    X = torch.randn(R, h, device=dev).bfloat16()
    W1 = (torch.randn(G, 2 * hp, h, device=dev) * 0.02).bfloat16()
    W2 = (torch.randn(G, h, hp, device=dev) * 0.02).bfloat16()
    H = torch.empty(R, 2 * hp, device=dev).bfloat16()
    Act = torch.empty(R, hp, device=dev).bfloat16()
    Y = torch.empty(R, h, device=dev).bfloat16()
    dY = torch.randn(R, h, device=dev).bfloat16()
    dH = torch.empty(R, 2 * hp, device=dev).bfloat16()
    dX = torch.empty(R, h, device=dev).bfloat16()
    gW1 = torch.zeros(G, 2 * hp, h, device=dev)
    gW2 = torch.zeros(G, h, hp, device=dev)
    flop = 2.0 * R * h * hp
    if a.single:   # every F-mode launch below runs the single-CTA kernel
        _gg = K.grouped_gemm

        def _single(mode, *args, **kw):
            return _gg(mode, *args, cta1=(mode != K.GEMM_WGRAD), **kw)
        K.grouped_gemm = _single
    global timeit
    _t = timeit
    timeit = lambda fn: _t(fn, iters=a.iters, warmup=a.warmup)
    only = set(a.only.split(",")) if a.only else None
    res = {}
    if not only or "fwd1_swiglu" in only: res["fwd1_swiglu"] = (timeit(lambda: K.grouped_gemm(K.GEMM_FWD_SWIGLU, X, W1, groups, N=2 * hp, K=h, C=H, C2=Act)), 2 * flop)
    if not only or "fwd2_store" in only: res["fwd2_store"] = (timeit(lambda: K.grouped_gemm(K.GEMM_FWD_STORE, Act, W2, groups, N=h, K=hp, C=Y)), flop)
    if not only or "dgrad_dswiglu" in only: res["dgrad_dswiglu"] = (timeit(lambda: K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU, dY, W2, groups, N=hp, K=h, C=dH, aux=H)), flop)
    gate = torch.rand(R, device=dev)
    part = torch.empty(R, hp // 64, device=dev)
    if only and "dgrad_gated_noact" in only:  # pre-gated layout: no gate*act rewrite
        res["dgrad_gated_noact"] = (timeit(lambda: K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dY, W2, groups, N=hp, K=h, C=dH, aux=H, row_scale=gate, row_partial=part)), flop)
    if only and "fwd1_pregated" in only:
        res["fwd1_pregated"] = (timeit(lambda: K.grouped_gemm(K.GEMM_FWD_SWIGLU, X, W1, groups, N=2 * hp, K=h, C=H, C2=Act, row_scale=gate)), 2 * flop)
    if only and "dgrad_gated" in only: res["dgrad_gated"] = (timeit(lambda: K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dY, W2, groups, N=hp, K=h, C=dH, C2=Act, aux=H, row_scale=gate, row_partial=part)), flop)
    if not only or "dgrad_dx" in only: res["dgrad_dx"] = (timeit(lambda: K.grouped_gemm(K.GEMM_DGRAD_STORE, dH, W1, groups, N=h, K=2 * hp, C=dX)), 2 * flop)
    if not only or "wgrad_w2" in only: res["wgrad_w2"] = (timeit(lambda: K.grouped_gemm(K.GEMM_WGRAD, dY, Act, wg, M=h, N=hp, C=gW2, c_slot_stride=h * hp)), flop)
    if not only or "wgrad_w1" in only: res["wgrad_w1"] = (timeit(lambda: K.grouped_gemm(K.GEMM_WGRAD, dH, X, wg, M=2 * hp, N=h, C=gW1, c_slot_stride=2 * hp * h)), 2 * flop)
    if only and "wgrad2" in only:
        # the step's weight-gradient launch: both weights of every group in one two-problem launch,
        # K = the group's rows over 8 micro-batches (wgrad_mode "step")
        R8 = 8 * R
        dY8 = torch.randn(R8, h, device=dev).bfloat16()
        act8 = torch.randn(R8, hp, device=dev).bfloat16()
        dH8 = torch.randn(R8, 2 * hp, device=dev).bfloat16()
        X8 = torch.randn(R8, h, device=dev).bfloat16()
        tab = K.make_groups([8 * r for r in rows], [8 * a for a in a0], list(range(G)))
        tab2 = tab.clone()
        tab2[:, 3] |= K.FLAG_PROBLEM2
        merged = torch.cat([tab, tab2])
        res["wgrad2"] = (timeit(lambda: K.grouped_wgrad2(dY8, act8, gW2, dH8, X8, gW1, merged)), 3 * 8 * flop)
    out = {k: {"ms": round(v[0], 4), "tflops": round(v[1] / v[0] / 1e9, 1)} for k, v in res.items()}
    tot_ms = sum(v[0] for v in res.values())
    if not only:
        out["total"] = {"ms": round(tot_ms, 4), "tflops": round(9 * flop / tot_ms / 1e9, 1)}
    if a.cublas:
        # library baseline: batched cuBLAS GEMMs of the same (balanced) shapes, bf16 in / bf16 out
        Xb = X.view(G, r, h)
        W1t = W1.transpose(1, 2).contiguous()   # [G, h, 2h']
        W2t = W2.transpose(1, 2).contiguous()   # [G, h', h]
        Hb = torch.empty(G, r, 2 * hp, device=dev).bfloat16()
        Ab = Act.view(G, r, hp)
        dYb = dY.view(G, r, h)
        dHb = torch.randn(G, r, 2 * hp, device=dev).bfloat16()
        cub = {
            "fwd1": (lambda: torch.bmm(Xb, W1t), 2 * flop),
            "fwd2": (lambda: torch.bmm(Ab, W2t), flop),
            "dgrad_act": (lambda: torch.bmm(dYb, W2), flop),
            "dgrad_x": (lambda: torch.bmm(dHb, W1), 2 * flop),
            "wgrad_w2": (lambda: torch.bmm(dYb.transpose(1, 2), Ab), flop),
            "wgrad_w1": (lambda: torch.bmm(dHb.transpose(1, 2), Xb), 2 * flop),
        }
        out["cublas"] = {}
        for k, (fn, fl) in cub.items():
            ms = timeit(fn)
            out["cublas"][k] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}
        del Hb
    print(json.dumps({"shape": {"groups": G, "rows": r, "h": h, "hp": hp}, "gemm": out}))


if __name__ == "__main__":
    main()
