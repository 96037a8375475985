"""Thin Python wrappers over the sm_100a data-plane C-ABI (``include/mb_kernels.h``).

Every wrapper takes CUDA tensors, launches on the current torch stream and returns
immediately.  Shapes/dtypes are checked here; the kernels themselves never allocate.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat

GEMM_FWD_STORE = 0
GEMM_FWD_SWIGLU = 1
GEMM_DGRAD_STORE = 2
GEMM_DGRAD_DSWIGLU = 3
GEMM_WGRAD = 4
GEMM_DGRAD_DSWIGLU_GATED = 5

GROUP_FIELDS = 8  # int32 rows, a0, slot, flags, seg_begin, seg_count, rows_real, kblocks
FLAG_ACCUMULATE = 1
FLAG_REPLICA = 2
FLAG_PROBLEM2 = 4   # grouped_wgrad2: the group belongs to the second problem (dW1)
MAX_GROUPS = 256    # groups per launch (kMaxGroups)


def _lib():
    return nat.kernels()


def _need_cuda(*tensors):
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("data-plane ops take CUDA tensors (there is no CPU path)")


def make_groups(rows, a0, slot, flags=None, seg_begin=None, seg_count=None, rows_real=None, kblocks=None,
                device="cuda") -> torch.Tensor:
    """Pack per-group (rows, a0, slot, flags, seg_begin, seg_count, rows_real, kblocks) into the
    int32 [G, 8] table.  kblocks (wgrad): sum over the group's K segments of ceil(rows / 64)."""
    n = len(rows)
    z = [0] * n
    flags = z if flags is None else flags
    seg_begin = z if seg_begin is None else seg_begin
    seg_count = z if seg_count is None else seg_count
    rows_real = rows if rows_real is None else rows_real
    kblocks = z if kblocks is None else kblocks
    tab = np.zeros((n, GROUP_FIELDS), dtype=np.int32)
    for c, v in enumerate((rows, a0, slot, flags, seg_begin, seg_count, rows_real, kblocks)):
        tab[:, c] = np.asarray(v, dtype=np.int64)
    return torch.from_numpy(tab).to(device)


def expert_histogram(idx: torch.Tensor, num_experts: int, chunk_tokens: int = 32,
                     counts: torch.Tensor | None = None, chunk_counts: torch.Tensor | None = None):
    """K1: idx [NB, T, k] int32 -> counts [NB, E] int32 (u32 values), chunk counts [NB, chunks, E]."""
    _need_cuda(idx)
    if idx.dim() == 2:
        idx = idx.unsqueeze(0)
    if idx.dtype != torch.int32 or not idx.is_contiguous():
        raise ValueError("idx must be a contiguous int32 [NB, T, k] tensor")
    nb, t, k = idx.shape
    chunks = (t + chunk_tokens - 1) // chunk_tokens
    if counts is None:
        counts = torch.empty((nb, num_experts), dtype=torch.int32, device=idx.device)
    if chunk_counts is None:
        chunk_counts = torch.empty((nb, max(chunks, 1), num_experts), dtype=torch.int32, device=idx.device)
    lib = _lib()
    nat.check(lib.mb_expert_histogram(idx.data_ptr(), nb, t, k, num_experts, counts.data_ptr(),
                                      chunk_counts.data_ptr(), chunk_tokens, nat.stream_ptr()),
              lib, "mb_expert_histogram")
    return counts, chunk_counts


def grouped_gemm(mode: int, A: torch.Tensor, B0: torch.Tensor, groups: torch.Tensor, *, M: int = 0, N: int,
                 K: int = 0, C: torch.Tensor, C2: torch.Tensor | None = None, aux: torch.Tensor | None = None,
                 B1: torch.Tensor | None = None, c_slot_stride: int = 0,
                 segs: torch.Tensor | None = None, row_scale: torch.Tensor | None = None,
                 row_partial: torch.Tensor | None = None, single_cta: bool = False, sms: int = 0,
                 stream=None, cta1: bool = False) -> None:
    """K4: tcgen05 grouped GEMM; see include/mb_kernels.h for the five modes.  sms > 0: SMs the
    persistent grid covers for this launch (0 = the process default); stream: default current.
    cta1: the single-CTA member of the pair kernel family (cta_group::1, 128 x 256 tiles, no half
    tiles: a group pays at most 127 padded rows) -- the default of the data plane's non-gated
    F-mode launches (measured faster than the pair on ragged expert groups, equal on even ones)."""
    _need_cuda(A, B0, groups, C, C2, aux, B1)
    for t in (A, B0, B1):
        if t is not None and (t.dtype != torch.bfloat16 or not t.is_contiguous()):
            raise ValueError("GEMM operands must be contiguous bf16")
    if groups.dtype != torch.int32 or groups.dim() != 2 or groups.shape[1] != GROUP_FIELDS:
        raise ValueError("groups must be an int32 [G, 4] table")
    a_cols = A.shape[-1]
    a_rows = A.numel() // a_cols
    b_cols = B0.shape[-1]
    b0_rows = B0.numel() // b_cols
    b1_rows = 0 if B1 is None else B1.numel() // b_cols
    ldc = C.shape[-1]
    ldc2 = 0 if C2 is None else C2.shape[-1]
    ld_aux = 0 if aux is None else aux.shape[-1]
    lib = _lib()
    nat.check(lib.mb_grouped_gemm(mode | (0x100 if single_cta else 0) | (0x200 if cta1 else 0), A.data_ptr(), a_rows,
                                  a_cols,
                                  B0.data_ptr(), b0_rows, nat.ptr(B1), b1_rows, b_cols, groups.data_ptr(),
                                  nat.ptr(segs), groups.shape[0], M, N, K,
                                  C.data_ptr(), ldc, c_slot_stride, nat.ptr(C2), ldc2, nat.ptr(aux), ld_aux,
                                  nat.ptr(row_scale), nat.ptr(row_partial), int(sms), nat.stream_ptr(stream)),
              lib, "mb_grouped_gemm")


def grouped_wgrad2(A0: torch.Tensor, B0: torch.Tensor, C0: torch.Tensor, A1: torch.Tensor, B1: torch.Tensor,
                   C1: torch.Tensor, groups: torch.Tensor, segs: torch.Tensor | None = None, sms: int = 0,
                   stream=None) -> None:
    """K4 wgrad of both FFN weights in one launch: groups without FLAG_PROBLEM2 give
    C0[slot] (+)= A0^T B0 (A0 [K, M0], B0 [K, N0]), groups with it C1[slot] (+)= A1^T B1."""
    _need_cuda(A0, B0, C0, A1, B1, C1, groups)
    for t in (A0, B0, A1, B1):
        if t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError("wgrad operands must be contiguous bf16")
    for t in (C0, C1):
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError("wgrad outputs must be contiguous fp32")
    if groups.dtype != torch.int32 or groups.dim() != 2 or groups.shape[1] != GROUP_FIELDS:
        raise ValueError("groups must be an int32 [G, 8] table")
    k_rows = A0.numel() // A0.shape[-1]
    if any(t.numel() // t.shape[-1] != k_rows for t in (B0, A1, B1)):
        raise ValueError("wgrad operands must have the same number of K rows")
    M0, N0, M1, N1 = A0.shape[-1], B0.shape[-1], A1.shape[-1], B1.shape[-1]
    lib = _lib()
    nat.check(lib.mb_grouped_wgrad2(A0.data_ptr(), B0.data_ptr(), M0, N0, C0.data_ptr(), A1.data_ptr(),
                                    B1.data_ptr(), M1, N1, C1.data_ptr(), k_rows, groups.data_ptr(), nat.ptr(segs),
                                    groups.shape[0], int(sms), nat.stream_ptr(stream)), lib, "mb_grouped_wgrad2")
