"""One-process-per-GPU plumbing for the 8xB200 box: a symmetric CUDA-IPC arena (every rank
allocates the same layout, exports one handle and opens every peer's), device-side
barriers over flags in that arena, and host-side object exchange through torch.distributed.

The reference has no communication code (bandwidths are modelled, topology.py:29-47); this
is the transport the data plane writes through: kernels receive peer base pointers and
load/store rows over NVLink5 directly.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _native as nat

BARRIER_TIMEOUT_NS = 20_000_000_000  # 20 s, then the kernel traps instead of hanging the GPU


class _CudaView:
    """__cuda_array_interface__ shim so torch can wrap raw device memory without copying."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.bfloat16: ("<i2", torch.int16), torch.float32: ("<f4", None), torch.int32: ("<i4", None),
            torch.int64: ("<i8", None), torch.uint8: ("|u1", None), torch.float16: ("<f2", None)}


def wrap(ptr: int, shape, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    typestr, carrier = _TYPESTR[dtype]
    t = torch.as_tensor(_CudaView(ptr, shape, typestr), device=device)
    return t.view(dtype) if carrier is not None else t


class Comm:
    """Rank/world bookkeeping; world == 1 needs no torch.distributed."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.rank = self.dist.get_rank() if self.dist else 0
        self.world = self.dist.get_world_size() if self.dist else 1

    def all_gather_object(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def all_gather_tensor(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t.unsqueeze(0)
        if self.dist.get_backend() == "gloo":  # oversubscribed test mode: host-side gather
            parts = [torch.empty_like(t, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, t.contiguous().cpu())
            return torch.stack(parts).to(t.device)
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.contiguous())
        return out

    def max_over_ranks(self, value: float) -> float:
        """Max of a per-rank scalar (device-timed milliseconds) over all ranks."""
        if self.world == 1:
            return float(value)
        dev = "cpu" if self.dist.get_backend() == "gloo" else "cuda"
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def host_barrier(self) -> None:
        if self.world > 1:
            self.dist.barrier()


class SymmetricArena:
    """Same-sized IPC allocation on every rank; `peer_ptr(p, off)` is rank p's byte `off`."""

    HEADER = 4096  # barrier flags (world u32) + epoch + error flag live at the start

    def __init__(self, comm: Comm, nbytes: int, device: torch.device):
        self.comm = comm
        self.device = device
        self.nbytes = int(nbytes) + self.HEADER
        lib = nat.kernels()
        self._lib = lib
        base = ctypes.c_void_p()
        hsize = lib.mb_ipc_handle_size()
        handle = ctypes.create_string_buffer(hsize)
        nat.check(lib.mb_ipc_malloc(self.nbytes, ctypes.byref(base), handle), lib, "mb_ipc_malloc")
        self.base = base.value
        handles = comm.all_gather_object(handle.raw)
        self.peer_base = []
        self._opened = []
        for p, h in enumerate(handles):
            if p == comm.rank:
                self.peer_base.append(self.base)
                continue
            pb = ctypes.c_void_p()
            hb = ctypes.create_string_buffer(h, len(h))
            nat.check(lib.mb_ipc_open(hb, ctypes.byref(pb)), lib, "mb_ipc_open")
            self.peer_base.append(pb.value)
            self._opened.append(pb.value)
        self._next = self.HEADER
        # barrier state: flags[world] at 0, epoch at 512, error flag at 520
        self.flag_ptrs = torch.tensor([b for b in self.peer_base], dtype=torch.int64, device=device)
        self.epoch_ptr = self.base + 512
        self.error_ptr = self.base + 520

    def alloc(self, nbytes: int, align: int = 1024) -> int:
        off = (self._next + align - 1) // align * align
        if off + nbytes > self.nbytes:
            raise MemoryError(f"arena exhausted: need {off + nbytes} of {self.nbytes} bytes")
        self._next = off + int(nbytes)
        return off

    def local(self, off: int, shape, dtype) -> torch.Tensor:
        return wrap(self.base + off, shape, dtype, self.device)

    def peer_ptr(self, rank: int, off: int) -> int:
        return self.peer_base[rank] + off

    def peer_table(self, off: int, stride_bytes: int = 0, count: int = 1) -> torch.Tensor:
        """int64 device table [count][world] of peer pointers base_p + off + i * stride."""
        tab = np.array([[self.peer_base[p] + off + i * stride_bytes for p in range(self.comm.world)]
                        for i in range(count)], dtype=np.int64)
        return torch.from_numpy(tab).to(self.device)

    def barrier(self, stream=None) -> None:
        """Device-side barrier on `stream` (no host sync); a no-op for world == 1."""
        if self.comm.world == 1:
            return
        nat.check(self._lib.mb_peer_barrier(self.flag_ptrs.data_ptr(), self.comm.rank, self.comm.world, self.epoch_ptr,
                                            BARRIER_TIMEOUT_NS, self.error_ptr, nat.stream_ptr(stream)),
                  self._lib, "mb_peer_barrier")

    def close(self) -> None:
        for p in self._opened:
            self._lib.mb_ipc_close(p)
        self._opened = []
        if self.base:
            self._lib.mb_device_free(self.base)
            self.base = 0


def local_device() -> int:
    """CUDA device of this rank: LOCAL_RANK, folded onto the visible GPUs when more ranks than
    GPUs run (MB_OVERSUBSCRIBE=1: a correctness test of an EP=8 job on a 2- or 4-GPU box; the
    ranks sharing a GPU time-slice, so timings from that mode mean nothing)."""
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MB_OVERSUBSCRIBE") == "1":
        return local % max(1, torch.cuda.device_count())
    return local


def init_distributed() -> Comm:
    """torchrun-style env (RANK/WORLD_SIZE/LOCAL_RANK/MASTER_*): NCCL process group, one GPU per
    rank (gloo under MB_OVERSUBSCRIBE=1: NCCL refuses two ranks on one GPU)."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and not dist.is_initialized():
        dev = local_device()
        torch.cuda.set_device(dev)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if os.environ.get("MB_OVERSUBSCRIBE") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return Comm()
