"""K4 tcgen05 grouped GEMM vs a plain PyTorch fp32 reference of the same contraction.

Tolerance: bf16 operands, fp32 accumulation; bf16 outputs are compared at rel 2e-2
(north_star's documented bf16 tolerance), fp32 wgrad outputs at rel 1e-3 of the max.
"""

import pytest
import torch

from paper_2605_08639_b200 import kernels as K

pytestmark = pytest.mark.gpu

DEV = "cuda"


def rel_err(got, ref):
    return ((got.float() - ref.float()).abs().max() / ref.float().abs().max().clamp_min(1e-6)).item()


def _row_groups(rows):
    a0 = [0]
    for r in rows[:-1]:
        a0.append(a0[-1] + r)
    return a0, sum(rows)


@pytest.mark.parametrize("rows", [[128], [256, 0, 384, 128], [128] * 9])
def test_fwd_store(rows):
    torch.manual_seed(0)
    N, Kd = 512, 256
    a0, R = _row_groups(rows)
    S = len(rows)
    slots = list(reversed(range(S)))
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    W = (torch.randn(S, N, Kd, device=DEV) * Kd ** -0.5).bfloat16()
    C = torch.full((R, N), float("nan"), device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_FWD_STORE, A, W, K.make_groups(rows, a0, slots), N=N, K=Kd, C=C)
    torch.cuda.synchronize()
    for g, r in enumerate(rows):
        if r == 0:
            continue
        ref = A[a0[g]:a0[g] + r].float() @ W[slots[g]].float().T
        assert rel_err(C[a0[g]:a0[g] + r], ref) < 2e-2


def test_fwd_replica_map():
    torch.manual_seed(1)
    N, Kd = 256, 128
    rows = [128, 256, 128]
    a0, R = _row_groups(rows)
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    Wh = torch.randn(2, N, Kd, device=DEV).bfloat16()
    Wr = torch.randn(3, N, Kd, device=DEV).bfloat16()
    C = torch.zeros(R, N, device=DEV).bfloat16()
    groups = K.make_groups(rows, a0, [1, 2, 0], [0, K.FLAG_REPLICA, 0])
    K.grouped_gemm(K.GEMM_FWD_STORE, A, Wh, groups, N=N, K=Kd, C=C, B1=Wr)
    torch.cuda.synchronize()
    refs = [A[0:128].float() @ Wh[1].float().T, A[128:384].float() @ Wr[2].float().T, A[384:].float() @ Wh[0].float().T]
    assert rel_err(C, torch.cat(refs)) < 2e-2


def test_fwd_swiglu():
    torch.manual_seed(2)
    hp, Kd = 256, 256        # h' = 256 -> 2h' = 512 = two 256-wide tiles (gate|up blocks of 128)
    rows = [128, 256]
    a0, R = _row_groups(rows)
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    W = (torch.randn(2, 2 * hp, Kd, device=DEV) * Kd ** -0.5).bfloat16()
    H = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
    Act = torch.zeros(R, hp, device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_FWD_SWIGLU, A, W, K.make_groups(rows, a0, [0, 1]), N=2 * hp, K=Kd, C=H, C2=Act)
    torch.cuda.synchronize()
    for g, r in enumerate(rows):
        h = A[a0[g]:a0[g] + r].float() @ W[g].float().T
        assert rel_err(H[a0[g]:a0[g] + r], h) < 2e-2
        hb = h.view(r, -1, 2, 128)
        act = (torch.nn.functional.silu(hb[:, :, 0]) * hb[:, :, 1]).reshape(r, hp)
        assert rel_err(Act[a0[g]:a0[g] + r], act) < 2e-2


@pytest.mark.parametrize("cta1", [False, True])
def test_fwd_swiglu_pregated(cta1):
    """row_scale: the activation leaves scaled by the row's gate, pad rows (past rows_real) zero;
    H is unscaled.  Odd 128-row blocks exercise the pair kernel's half tiles."""
    torch.manual_seed(12)
    hp, Kd = 256, 256
    rows, real = [384, 128], [300, 128]
    a0, R = _row_groups(rows)
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    W = (torch.randn(2, 2 * hp, Kd, device=DEV) * Kd ** -0.5).bfloat16()
    gate = torch.rand(R, device=DEV)
    H = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
    Act = torch.full((R, hp), float("nan"), device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_FWD_SWIGLU, A, W, K.make_groups(rows, a0, [0, 1], rows_real=real), N=2 * hp, K=Kd,
                   C=H, C2=Act, row_scale=gate, cta1=cta1)
    torch.cuda.synchronize()
    for g, r in enumerate(rows):
        h = A[a0[g]:a0[g] + r].float() @ W[g].float().T
        assert rel_err(H[a0[g]:a0[g] + r], h) < 2e-2
        hb = H[a0[g]:a0[g] + r].float().view(r, -1, 2, 128)   # the act is computed from bf16 H
        act = (torch.nn.functional.silu(hb[:, :, 0]) * hb[:, :, 1]).reshape(r, hp)
        sl = slice(a0[g], a0[g] + real[g])
        assert rel_err(Act[sl], gate[sl, None] * act[:real[g]]) < 2e-2
        assert torch.all(Act[a0[g] + real[g]:a0[g] + r] == 0)


def test_dgrad_store():
    torch.manual_seed(3)
    N, Kd = 512, 384
    rows = [256, 128]
    a0, R = _row_groups(rows)
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    W = (torch.randn(2, Kd, N, device=DEV) * Kd ** -0.5).bfloat16()   # [slot][K][N], N contiguous
    C = torch.zeros(R, N, device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_DGRAD_STORE, A, W, K.make_groups(rows, a0, [1, 0]), N=N, K=Kd, C=C)
    torch.cuda.synchronize()
    ref = torch.cat([A[:256].float() @ W[1].float(), A[256:].float() @ W[0].float()])
    assert rel_err(C, ref) < 2e-2


def test_dgrad_dswiglu():
    torch.manual_seed(4)
    hp, hd = 256, 512         # dAct = dY[R,h] . W2[h,h'] ; H/dH [R, 2h'] gate|up blocks of 128
    rows = [128, 128]
    a0, R = _row_groups(rows)
    dY = torch.randn(R, hd, device=DEV).bfloat16()
    W2 = (torch.randn(2, hd, hp, device=DEV) * hd ** -0.5).bfloat16()
    H = torch.randn(R, 2 * hp, device=DEV).bfloat16()
    dH = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU, dY, W2, K.make_groups(rows, a0, [0, 1]), N=hp, K=hd, C=dH, aux=H)
    torch.cuda.synchronize()
    for g in range(2):
        sl = slice(a0[g], a0[g] + rows[g])
        da = dY[sl].float() @ W2[g].float()
        hb = H[sl].float().view(rows[g], -1, 2, 128)
        gt, up = hb[:, :, 0].reshape(rows[g], hp), hb[:, :, 1].reshape(rows[g], hp)
        s = torch.sigmoid(gt)
        dg = da * up * s * (1 + gt * (1 - s))
        du = da * gt * s
        ref = torch.stack([dg.view(rows[g], -1, 128), du.view(rows[g], -1, 128)], dim=2).reshape(rows[g], 2 * hp)
        assert rel_err(dH[sl], ref) < 2e-2


@pytest.mark.parametrize("rows,real", [([256, 128], [200, 128]), ([384, 128, 512], [300, 77, 512])])
def test_dgrad_dswiglu_gated(rows, real):
    """Fused combine-backward: raw dout rows in, gate per row, dgate partials, gate*act out.
    Odd multiples of 128 rows exercise the M=128 tail tiles of the CTA-pair kernel."""
    torch.manual_seed(7)
    hp, hd = 512, 256
    a0, R = _row_groups(rows)
    dout = torch.randn(R, hd, device=DEV).bfloat16()
    W2 = (torch.randn(2, hd, hp, device=DEV) * hd ** -0.5).bfloat16()
    H = torch.randn(R, 2 * hp, device=DEV).bfloat16()
    gate = torch.rand(R, device=DEV)
    dH = torch.full((R, 2 * hp), float("nan"), device=DEV).bfloat16()
    actg = torch.full((R, hp), float("nan"), device=DEV).bfloat16()
    part = torch.zeros(R, hp // 64, device=DEV)
    S = len(rows)
    W2 = (torch.randn(S, hd, hp, device=DEV) * hd ** -0.5).bfloat16()
    K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dout, W2, K.make_groups(rows, a0, list(range(S)), rows_real=real),
                   N=hp, K=hd, C=dH, C2=actg, aux=H, row_scale=gate, row_partial=part)
    torch.cuda.synchronize()
    for g in range(S):
        sl = slice(a0[g], a0[g] + real[g])
        raw = dout[sl].float() @ W2[g].float()
        hb = H[sl].float().view(real[g], -1, 2, 128)
        gt, up = hb[:, :, 0].reshape(real[g], hp), hb[:, :, 1].reshape(real[g], hp)
        s = torch.sigmoid(gt)
        act = gt * s * up
        da = gate[sl, None] * raw
        dg = da * up * s * (1 + gt * (1 - s))
        du = da * gt * s
        ref = torch.stack([dg.view(real[g], -1, 128), du.view(real[g], -1, 128)], dim=2).reshape(real[g], 2 * hp)
        assert rel_err(dH[sl], ref) < 2e-2
        assert rel_err(actg[sl], gate[sl, None] * act) < 2e-2
        assert rel_err(part[sl].sum(1), (raw * act).sum(1)) < 2e-2
        pad = slice(a0[g] + real[g], a0[g] + rows[g])
        assert torch.all(dH[pad] == 0) and torch.all(actg[pad] == 0)
    # without C2 (the data plane's pre-gated layout): same dH and partials, nothing else written
    dH2 = torch.full_like(dH, float("nan"))
    part2 = torch.zeros_like(part)
    K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dout, W2, K.make_groups(rows, a0, list(range(S)), rows_real=real),
                   N=hp, K=hd, C=dH2, aux=H, row_scale=gate, row_partial=part2)
    torch.cuda.synchronize()
    for g in range(S):
        sl = slice(a0[g], a0[g] + real[g])
        assert torch.equal(dH2[sl], dH[sl]) and torch.equal(part2[sl], part[sl])


def test_single_cta_path_matches_pair():
    torch.manual_seed(8)
    N, Kd = 512, 256
    rows = [384, 128]
    a0, R = _row_groups(rows)
    A = torch.randn(R, Kd, device=DEV).bfloat16()
    W = (torch.randn(2, N, Kd, device=DEV) * Kd ** -0.5).bfloat16()
    C1 = torch.zeros(R, N, device=DEV).bfloat16()
    C2 = torch.zeros(R, N, device=DEV).bfloat16()
    g = K.make_groups(rows, a0, [1, 0])
    K.grouped_gemm(K.GEMM_FWD_STORE, A, W, g, N=N, K=Kd, C=C1)
    K.grouped_gemm(K.GEMM_FWD_STORE, A, W, g, N=N, K=Kd, C=C2, single_cta=True)
    torch.cuda.synchronize()
    assert rel_err(C1, C2) < 1e-2


def test_wgrad_accumulate():
    torch.manual_seed(5)
    Md, Nd = 256, 512
    krows = [64, 0, 192, 128]
    a0, R = _row_groups(krows)
    slots = [2, 0, 1, 3]
    flags = [K.FLAG_ACCUMULATE, 0, 0, K.FLAG_ACCUMULATE]
    A = torch.randn(R, Md, device=DEV).bfloat16()
    B = torch.randn(R, Nd, device=DEV).bfloat16()
    C0 = torch.randn(4, Md, Nd, device=DEV)
    C = C0.clone()
    K.grouped_gemm(K.GEMM_WGRAD, A, B, K.make_groups(krows, a0, slots, flags), M=Md, N=Nd, C=C,
                   c_slot_stride=Md * Nd)
    torch.cuda.synchronize()
    for g, r in enumerate(krows):
        s = slots[g]
        if r == 0:
            assert torch.equal(C[s], C0[s])
            continue
        ref = A[a0[g]:a0[g] + r].float().T @ B[a0[g]:a0[g] + r].float()
        if flags[g] & K.FLAG_ACCUMULATE:
            ref = ref + C0[s]
        assert rel_err(C[s], ref) < 1e-3


def test_wgrad_segments_16_rows():
    """K split over segments whose row counts are multiples of 16 (partial last k-blocks)."""
    torch.manual_seed(9)
    Md, Nd = 256, 256
    R = 1024
    A = torch.randn(R, Md, device=DEV).bfloat16()
    B = torch.randn(R, Nd, device=DEV).bfloat16()
    segs_g = [[(0, 48), (128, 16), (512, 112)], [(256, 64), (640, 208)], [(900, 16)]]
    segs, seg_begin, seg_count, tot, kblocks = [], [], [], [], []
    for sg in segs_g:
        seg_begin.append(len(segs))
        seg_count.append(len(sg))
        segs.extend(sg)
        tot.append(sum(r for _, r in sg))
        kblocks.append(sum((r + 63) // 64 for _, r in sg))
    groups = K.make_groups(tot, [0] * 3, [2, 0, 1], [0, K.FLAG_ACCUMULATE, 0], seg_begin, seg_count,
                           kblocks=kblocks)
    C0 = torch.randn(3, Md, Nd, device=DEV)
    C = C0.clone()
    K.grouped_gemm(K.GEMM_WGRAD, A, B, groups, M=Md, N=Nd, C=C, c_slot_stride=Md * Nd,
                   segs=torch.tensor(segs, dtype=torch.int32, device=DEV))
    torch.cuda.synchronize()
    for g, (sg, slot) in enumerate(zip(segs_g, [2, 0, 1])):
        ref = sum(A[a:a + r].float().T @ B[a:a + r].float() for a, r in sg)
        if g == 1:
            ref = ref + C0[slot]
        assert rel_err(C[slot], ref) < 1e-3


def test_histogram_matches_bincount():
    torch.manual_seed(6)
    E, k = 128, 8
    idx = torch.stack([torch.randperm(E, device=DEV)[:k] for _ in range(1000)]).int()
    idx = idx.view(2, 500, k).contiguous()
    counts, chunks = K.expert_histogram(idx, E, chunk_tokens=32)
    torch.cuda.synchronize()
    for b in range(2):
        ref = torch.bincount(idx[b].flatten().long(), minlength=E)
        assert torch.equal(counts[b].long(), ref)
        assert torch.equal(chunks[b].sum(0).long(), ref)


def test_fused_combine_backward_matches_unfused_path():
    """The gated dSwiGLU epilogue (combine backward fused into the dAct GEMM) against the unfused
    path: mb_combine_bwd_expert (dY = gate*dout, dgate = <dout, Y>) then the plain dSwiGLU GEMM."""
    import numpy as np
    from paper_2605_08639_b200 import _native as nat
    torch.manual_seed(13)
    hp, hd = 512, 256
    rows, real = [384, 256], [300, 256]
    a0, R = _row_groups(rows)
    H = torch.randn(R, 2 * hp, device=DEV).bfloat16()
    hb = H.float().view(R, -1, 2, 128)   # gate|up interleaved in blocks of 128
    Act = (torch.nn.functional.silu(hb[:, :, 0]) * hb[:, :, 1]).reshape(R, hp).bfloat16()
    W2 = (torch.randn(2, hd, hp, device=DEV) * hd ** -0.5).bfloat16()
    g = K.make_groups(rows, a0, [0, 1], rows_real=real)
    Y = torch.zeros(R, hd, device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_FWD_STORE, Act, W2, g, N=hd, K=hp, C=Y)
    dout = torch.randn(R, hd, device=DEV).bfloat16()
    gate = torch.rand(R, device=DEV)
    # fused
    dH1 = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
    actg = torch.zeros(R, hp, device=DEV).bfloat16()
    part = torch.zeros(R, hp // 64, device=DEV)
    K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dout, W2, g, N=hp, K=hd, C=dH1, C2=actg, aux=H, row_scale=gate,
                   row_partial=part)
    # unfused
    slot_tab = torch.tensor([[a0[i], real[i], rows[i], i] for i in range(2)], dtype=torch.int32, device=DEV)
    dy = dout.clone()
    dgate = torch.zeros(R, device=DEV)
    lib = nat.kernels()
    nat.check(lib.mb_combine_bwd_expert(dy.data_ptr(), Y.data_ptr(), gate.data_ptr(), dgate.data_ptr(),
                                        slot_tab.data_ptr(), 2, R, hd, nat.stream_ptr()), lib, "combine_bwd")
    dH2 = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
    K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU, dy, W2, g, N=hp, K=hd, C=dH2, aux=H)
    torch.cuda.synchronize()
    for i in range(2):
        sl = slice(a0[i], a0[i] + real[i])
        assert rel_err(dH1[sl], dH2[sl]) < 2e-2
        assert rel_err(part[sl].sum(1), dgate[sl]) < 2e-2
        pad = slice(a0[i] + real[i], a0[i] + rows[i])
        assert torch.all(dH1[pad] == 0) and torch.all(dy[pad] == 0)


def test_wgrad_two_problems_one_launch():
    """mb_grouped_wgrad2: dW2 and dW1 of every group in one dynamically scheduled launch are
    bit-identical to the two single-problem launches (same tiles, same K order)."""
    torch.manual_seed(11)
    h, hp = 512, 256
    R = 1024
    dY = torch.randn(R, h, device=DEV).bfloat16()
    act = torch.randn(R, hp, device=DEV).bfloat16()
    dH = torch.randn(R, 2 * hp, device=DEV).bfloat16()
    X = torch.randn(R, h, device=DEV).bfloat16()
    segs_g = [[(0, 48), (512, 112)], [(256, 64), (640, 208)], [(900, 16)]]
    segs, seg_begin, seg_count, tot, kblocks = [], [], [], [], []
    for sg in segs_g:
        seg_begin.append(len(segs))
        seg_count.append(len(sg))
        segs.extend(sg)
        tot.append(sum(r for _, r in sg))
        kblocks.append(sum((r + 63) // 64 for _, r in sg))
    flags = [0, K.FLAG_ACCUMULATE, 0]
    single = K.make_groups(tot, [0] * 3, [2, 0, 1], flags, seg_begin, seg_count, kblocks=kblocks)
    merged = torch.cat([single, single.clone()])
    merged[3:, 3] |= K.FLAG_PROBLEM2
    segs_t = torch.tensor(segs, dtype=torch.int32, device=DEV)
    C2a, C1a = torch.randn(3, h, hp, device=DEV), torch.randn(3, 2 * hp, h, device=DEV)
    C2b, C1b = C2a.clone(), C1a.clone()
    K.grouped_gemm(K.GEMM_WGRAD, dY, act, single, M=h, N=hp, C=C2a, c_slot_stride=h * hp, segs=segs_t)
    K.grouped_gemm(K.GEMM_WGRAD, dH, X, single, M=2 * hp, N=h, C=C1a, c_slot_stride=2 * hp * h, segs=segs_t)
    K.grouped_wgrad2(dY, act, C2b, dH, X, C1b, merged, segs=segs_t)
    torch.cuda.synchronize()
    assert torch.equal(C2a, C2b) and torch.equal(C1a, C1b)
    ref = sum(dY[a:a + r].float().T @ act[a:a + r].float() for a, r in segs_g[2])
    assert rel_err(C2b[1], ref) < 1e-3


@pytest.mark.parametrize("rows", [[128, 128, 128], [384, 128, 256]])
@pytest.mark.parametrize("mode", ["fwd_swiglu", "fwd_store", "dgrad_store", "dgrad_gated"])
def test_single_cta_variant_matches_pair(mode, rows):
    """The single-CTA (cta_group::1, 128-row tiles) member of the pair family gives the pair
    kernel's results, on groups of one and of several 128-row blocks (odd and even)."""
    torch.manual_seed(13)
    h, hp, G = 512, 256, 3
    a0 = [sum(rows[:i]) for i in range(G)]
    R = sum(rows)
    real = [rows[0], rows[1] - 28, 1 + rows[2] // 2]
    groups = K.make_groups(rows, a0, [2, 0, 1], rows_real=real)
    X = torch.randn(R, h, device=DEV).bfloat16()
    W1 = (torch.randn(G, 2 * hp, h, device=DEV) * 0.05).bfloat16()
    W2 = (torch.randn(G, h, hp, device=DEV) * 0.05).bfloat16()
    outs = []
    for tail in (False, True):
        if mode == "fwd_swiglu":
            H = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
            Act = torch.zeros(R, hp, device=DEV).bfloat16()
            K.grouped_gemm(K.GEMM_FWD_SWIGLU, X, W1, groups, N=2 * hp, K=h, C=H, C2=Act, cta1=tail)
            outs.append((H, Act))
        elif mode == "fwd_store":
            A = torch.randn(R, hp, generator=torch.Generator(device="cuda").manual_seed(3), device=DEV).bfloat16()
            Y = torch.zeros(R, h, device=DEV).bfloat16()
            K.grouped_gemm(K.GEMM_FWD_STORE, A, W2, groups, N=h, K=hp, C=Y, cta1=tail)
            outs.append((Y,))
        elif mode == "dgrad_store":
            dH = torch.randn(R, 2 * hp, generator=torch.Generator(device="cuda").manual_seed(4), device=DEV).bfloat16()
            dX = torch.zeros(R, h, device=DEV).bfloat16()
            K.grouped_gemm(K.GEMM_DGRAD_STORE, dH, W1, groups, N=h, K=2 * hp, C=dX, cta1=tail)
            outs.append((dX,))
        else:
            dY = torch.randn(R, h, generator=torch.Generator(device="cuda").manual_seed(5), device=DEV).bfloat16()
            H = torch.randn(R, 2 * hp, generator=torch.Generator(device="cuda").manual_seed(6), device=DEV).bfloat16()
            gate = torch.rand(R, generator=torch.Generator(device="cuda").manual_seed(7), device=DEV)
            dH = torch.zeros(R, 2 * hp, device=DEV).bfloat16()
            act = torch.zeros(R, hp, device=DEV).bfloat16()
            part = torch.zeros(R, hp // 64, device=DEV)
            K.grouped_gemm(K.GEMM_DGRAD_DSWIGLU_GATED, dY, W2, groups, N=hp, K=h, C=dH, C2=act, aux=H,
                           row_scale=gate, row_partial=part, cta1=tail)
            outs.append((dH, act, part))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert rel_err(b, a) < 1e-3, mode
