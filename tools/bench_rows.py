"""Row-mover micro-benchmark: K3 scatter and K6 combine alone, register-copy vs TMA bulk kernels.

  python tools/bench_rows.py                                   (1 GPU: HBM copies)
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_rows.py   (NVLink)

Each rank owns T tokens x k choices; every choice goes to a uniformly random rank (the rows a
source sends to one rank land in that rank's region [src * T * k, ...) at random positions).
Checks that both engines write identical receive rows / identical combine outputs, then times
each engine at several SM counts.  GB/s counts bytes written by scatter (all k rows) and bytes
read by combine; `remote` is the NVLink share.  Prints one JSON line per configuration on rank 0.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_08639_b200 import _native as nat  # noqa: E402
from paper_2605_08639_b200.comm import SymmetricArena, init_distributed, local_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--blocks", default="0,8,12,16,20,28,40,74,148")
    args = ap.parse_args()
    comm = init_distributed()
    torch.cuda.set_device(local_device())
    rank, world = comm.rank, comm.world
    T, k, h = args.tokens, args.k, args.hidden
    lib = nat.kernels()
    rows_per_src = T * k
    npart = 12
    arena = SymmetricArena(comm, world * rows_per_src * (h * 2 + npart * 4) + (1 << 20),
                           torch.device("cuda", local_device()))
    off = arena.alloc(world * rows_per_src * h * 2)
    off_s = arena.alloc(world * rows_per_src * npart * 4)
    arena.local(off_s, (world * rows_per_src, npart), torch.float32).copy_(
        torch.rand(world * rows_per_src, npart, generator=torch.Generator().manual_seed(7 + rank)))
    sptrs = arena.peer_table(off_s)[0].contiguous()
    dgate = torch.empty(T, k, dtype=torch.float32, device="cuda")
    recv = arena.local(off, (world * rows_per_src, h), torch.bfloat16)
    ptrs = arena.peer_table(off)[0].contiguous()
    g = torch.Generator().manual_seed(1000 + rank)
    x = torch.randn(T, h, generator=g).to(torch.bfloat16).cuda()
    dst = torch.randint(0, world, (T * k,), generator=g)
    perm = torch.empty(T * k, 2, dtype=torch.int32)
    perm[:, 0] = dst.to(torch.int32)
    for d in range(world):
        sel = torch.nonzero(dst == d).flatten()
        perm[sel, 1] = (rank * rows_per_src + torch.randperm(rows_per_src, generator=g)[: len(sel)]).to(torch.int32)
    perm = perm.cuda()
    gates = torch.rand(T, k, generator=g).cuda()
    out = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
    remote_frac = float((perm[:, 0] != rank).float().mean())
    st = torch.cuda.current_stream().cuda_stream

    def scatter():
        nat.check(lib.mb_scatter_rows(x.data_ptr(), T, k, h, perm.data_ptr(), ptrs.data_ptr(), -1, st), lib, "scatter")

    def combine():
        nat.check(lib.mb_combine_rows(ptrs.data_ptr(), perm.data_ptr(), gates.data_ptr(), T, k, h, out.data_ptr(),
                                      None, None, 1, -1, st), lib, "combine")

    def unpermute():
        nat.check(lib.mb_combine_rows(ptrs.data_ptr(), perm.data_ptr(), None, T, k, h, out.data_ptr(),
                                      sptrs.data_ptr(), dgate.data_ptr(), npart, -1, st), lib, "unpermute")

    def sync():
        torch.cuda.synchronize()
        comm.host_barrier()

    # parity: both engines, same inputs
    res = {}
    for nb in (0, 20):
        nat.check(lib.mb_set_comm_blocks(nb), lib, "set_comm_blocks")
        recv.zero_()
        sync()
        scatter()
        sync()
        r = recv.clone()
        combine()
        sync()
        o = out.clone()
        unpermute()
        sync()
        res[nb] = (r, o, out.clone(), dgate.clone())
    same_scatter = bool(torch.equal(res[0][0], res[20][0]))
    same_combine = bool(torch.equal(res[0][1], res[20][1]))
    same_unpermute = bool(torch.equal(res[0][2], res[20][2]) and torch.equal(res[0][3], res[20][3]))
    del res
    nbytes = T * k * h * 2
    for nb in [int(b) for b in args.blocks.split(",")]:
        for name, fn in (("scatter", scatter), ("combine", combine), ("unpermute", unpermute)):
            nat.check(lib.mb_set_comm_blocks(nb), lib, "set_comm_blocks")
            if nb == 0 and name == "scatter":
                os.environ.pop("MB_COMM_GRID", None)
            for _ in range(3):
                fn()
            sync()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.iters):
                fn()
            e.record()
            sync()
            ms = comm.max_over_ranks(s.elapsed_time(e) / args.iters)
            if rank == 0:
                print(json.dumps({"op": name, "engine": "tma" if nb else "regs", "blocks": nb or "148x8",
                                  "world": world, "ms": round(ms, 4), "gb_s": round(nbytes / ms / 1e6, 1),
                                  "remote_gb_s": round(nbytes * remote_frac / ms / 1e6, 1),
                                  "parity": {"scatter": same_scatter, "combine": same_combine,
                                             "unpermute": same_unpermute}}), flush=True)
    nat.check(lib.mb_set_comm_blocks(0), lib, "set_comm_blocks")
    sync()
    arena.close()
    if comm.dist:
        comm.dist.destroy_process_group()


if __name__ == "__main__":
    main()
