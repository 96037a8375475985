"""Measured NVLink peak of this box (the denominator for the comm phases' GB/s): copy-engine
peer copies GPU0 -> GPU1 (one direction) and both directions at once, 1 GiB, best of 10, CUDA
events; and a 4-GPU all-to-all of copy-engine copies when 4 GPUs are visible.  One JSON line."""
import json

import torch


def timed(fn, streams, iters=10):
    best = float("inf")
    for _ in range(iters):
        for s in streams:
            s.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in streams]
        for (a, _), s in zip(ev, streams):
            a.record(s)
        fn()
        for (_, b), s in zip(ev, streams):
            b.record(s)
        for s in streams:
            s.synchronize()
        best = min(best, max(a.elapsed_time(b) for a, b in ev))
    return best


def main():
    n = torch.cuda.device_count()
    nbytes = 1 << 30
    bufs = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
    dst = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
    streams = [torch.cuda.Stream(device=f"cuda:{i}") for i in range(n)]
    out = {"gpus": n, "bytes": nbytes}

    def one_way():
        with torch.cuda.stream(streams[0]):
            dst[1].copy_(bufs[0], non_blocking=True)
    ms = timed(one_way, streams[:1])
    out["one_direction_gb_s"] = round(nbytes / ms / 1e6, 1)

    def both_ways():
        with torch.cuda.stream(streams[0]):
            dst[1].copy_(bufs[0], non_blocking=True)
        with torch.cuda.stream(streams[1]):
            dst[0].copy_(bufs[1], non_blocking=True)
    ms = timed(both_ways, streams[:2])
    out["bidirectional_per_direction_gb_s"] = round(nbytes / ms / 1e6, 1)
    if n >= 4:
        chunk = nbytes // 4

        def all_to_all():
            for i in range(4):
                with torch.cuda.stream(streams[i]):
                    for j in range(4):
                        if j != i:
                            dst[j][i * chunk:(i + 1) * chunk].copy_(bufs[i][j * chunk:(j + 1) * chunk],
                                                                    non_blocking=True)
        ms = timed(all_to_all, streams[:4])
        out["all_to_all_4gpu_send_gb_s_per_gpu"] = round(3 * chunk / ms / 1e6, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
