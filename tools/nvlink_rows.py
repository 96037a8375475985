"""Single-process NVLink row movers (for ncu): GPU 0 scatters token rows into a receive buffer on
GPU 1 (peer access over NVLink) and combines them back, with the same kernels and engines the data
plane uses (register movers on every SM, or the confined bulk-copy movers on `--blocks` SMs).
One process, so ncu can profile it (`tools/ncu_nvlink.sh`); prints GB/s per phase.

  python tools/nvlink_rows.py [--tokens 8192 --k 8 --h 2048 --blocks 28]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08639_b200 import _native as nat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--h", type=int, default=2048)
    ap.add_argument("--blocks", type=int, default=28, help="confined bulk-copy movers on this many SMs (0: registers)")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    if torch.cuda.device_count() < 2:
        raise SystemExit("needs 2 GPUs")
    torch.cuda.set_device(0)
    from cuda.bindings import runtime as cudart   # cuda-python: GPU 0 may load / store GPU 1 memory
    err = cudart.cudaDeviceEnablePeerAccess(1, 0)[0]
    if err not in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
        raise SystemExit(f"cudaDeviceEnablePeerAccess: {err}")
    lib = nat.kernels()
    T, k, h = a.tokens, a.k, a.h
    rows = T * k
    x = torch.randn(T, h, device="cuda:0").bfloat16()
    local = torch.empty(rows, h, dtype=torch.bfloat16, device="cuda:0")
    with torch.cuda.device(1):
        remote = torch.empty(rows, h, dtype=torch.bfloat16, device="cuda:1")
    torch.cuda.set_device(0)
    g = torch.Generator().manual_seed(1)
    # every choice goes to GPU 1 (all remote), distinct rows
    perm = torch.empty(T * k, 2, dtype=torch.int32)
    perm[:, 0] = 1
    perm[:, 1] = torch.randperm(rows, generator=g).to(torch.int32)
    perm = perm.cuda()
    ptrs = torch.tensor([local.data_ptr(), remote.data_ptr()], dtype=torch.int64, device="cuda:0")
    gates = torch.rand(T, k, generator=g).cuda()
    out = torch.empty(T, h, dtype=torch.bfloat16, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream

    def scatter():
        nat.check(lib.mb_scatter_rows(x.data_ptr(), T, k, h, perm.data_ptr(), ptrs.data_ptr(), a.blocks, st), lib, "s")

    def combine():
        nat.check(lib.mb_combine_rows(ptrs.data_ptr(), perm.data_ptr(), gates.data_ptr(), T, k, h, out.data_ptr(), None,
                                      None, 1, a.blocks, st), lib, "c")

    res = {}
    for name, fn in (("scatter", scatter), ("combine", combine)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / a.iters
        res[name] = {"ms": round(ms, 4), "nvlink_gb_s": round(rows * h * 2 / ms / 1e6, 1)}
    print(json.dumps({"tokens": T, "k": k, "h": h, "blocks": a.blocks or "registers", "bytes_per_phase": rows * h * 2,
                      **res}))


if __name__ == "__main__":
    main()
