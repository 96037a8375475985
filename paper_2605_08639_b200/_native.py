"""ctypes bindings for the two native libraries (built in-tree by ``csrc/Makefile``).

``libmb_sm100.so``   sm_100a data-plane kernels, C-ABI in ``include/mb_kernels.h``
``libmb_planner.so`` C++ host planners,        C-ABI in ``include/mb_planner.h``

There is no fallback: if a library is missing the import of the op that needs it raises
``NativeLibraryError``.  Nonzero status codes raise ``ValueError`` (invalid argument) or
``RuntimeError`` (CUDA / solver failure) with the library's thread-local message.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_int = ctypes.c_int
c_char_p = ctypes.c_char_p


class NativeLibraryError(RuntimeError):
    """A required native library is missing or failed to load."""


class LPError(RuntimeError):
    """Numerical failure or malformed input in the simplex solver (mirrors moebalance.lp.LPError)."""


_KERNEL_SIGS = {
    "mb_last_error": (c_char_p, []),
    "mb_version": (c_int, []),
    "mb_expert_histogram": (c_int, [c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "mb_set_gemm_sms": (c_int, [c_int]),
    "mb_grouped_gemm": (
        c_int,
        [c_int, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_int, c_int, c_int, c_int,
         c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp],
    ),
}

_KERNEL_SIGS.update({
    "mb_grouped_wgrad2": (c_int, [c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_i64, c_vp, c_vp,
                                  c_int, c_i32, c_vp]),
    "mb_chunk_scan": (c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "mb_permute_rank": (c_int, [c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp,
                                c_vp]),
    "mb_permute_rank_nb": (c_int, [c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_i32,
                                   c_vp, c_i32, c_vp, c_vp]),
    "mb_check_counts": (c_int, [c_vp, c_vp, c_i64, c_vp, c_i32, c_vp]),
    "mb_dispatch_tables": (c_int, [c_i32, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp,
                                   c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mb_zero_pad_rows_nb": (c_int, [c_vp, c_i64, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "mb_scatter_rows": (c_int, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "mb_set_comm_blocks": (c_int, [c_i32]),
    "mb_anneal_chains": (c_int, [c_vp, c_i32, c_i32, c_vp, c_vp, c_dbl, c_vp, c_i32, c_i32, c_dbl, c_dbl, c_dbl, c_vp,
                                 c_vp, c_vp]),
    "mb_combine_rows": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp]),
    "mb_combine_bwd_expert": (c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i32, c_vp]),
    "mb_zero_pad_rows": (c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "mb_accumulate_f32": (c_int, [c_vp, c_vp, c_i32, c_i64, c_vp]),
    "mb_accumulate_f32_tasks": (c_int, [c_vp, c_i32, c_i64, c_vp]),
    "mb_ipc_malloc": (c_int, [c_i64, ctypes.POINTER(c_vp), c_vp]),
    "mb_ipc_handle_size": (c_int, []),
    "mb_ipc_open": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "mb_ipc_close": (c_int, [c_vp]),
    "mb_device_free": (c_int, [c_vp]),
    "mb_host_alloc_mapped": (c_int, [c_i64, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)]),
    "mb_host_free": (c_int, [c_vp]),
    "mb_memcpy_async": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "mb_peer_barrier": (c_int, [c_vp, c_i32, c_i32, c_vp, c_i64, c_vp, c_vp]),
})

_PLANNER_SIGS: dict = {
    "mbp_last_error": (c_char_p, []),
    "mbp_use_numpy_blas": (c_int, [c_char_p, c_char_p]),
    "mbp_numpy_blas_active": (c_int, []),
    "mbp_static_plan": (c_int, [c_i32, c_i32, c_vp]),
    "mbp_lpt_initial": (c_int, [c_vp, c_i32, c_i32, c_vp]),
    "mbp_anneal_prepare": (c_int, [c_vp, c_i32, c_i32, c_i32, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl,
                                   c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mbp_anneal_select": (c_int, [c_vp, c_i32, c_i32, c_i32, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl,
                                  c_vp, c_i32, c_vp]),
    "mbp_anneal_reorder": (c_int, [c_vp, c_i32, c_i32, c_i32, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_vp,
                                   c_i32, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "mbp_compute_loads": (c_int, [c_vp, c_i32, c_i32, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mbp_sample_placement": (c_int, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                     c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_vp, c_i32, c_dbl, c_dbl, c_dbl, c_dbl,
                                     c_dbl, c_i32, c_i32, c_vp]),
    "mbp_greedy_replicate": (c_int, [c_vp, c_i32, c_i32, c_i32, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl,
                                     c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mbp_solve_token_split": (c_int, [c_vp, c_i32, c_i32, c_i32, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl,
                                      c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mbp_round_split": (c_int, [c_vp, c_i32, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mbp_eplb_replication": (c_int, [c_vp, c_i32, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "mbp_uniform_matrices": (c_int, [c_vp, c_i64, c_i32, c_vp]),
    "mbp_dispatch_plan": (c_int, [c_i32, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32,
                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
}

_libs: dict[str, ctypes.CDLL] = {}


def _load(name: str, sigs: dict) -> ctypes.CDLL:
    if name in _libs:
        return _libs[name]
    path = LIB_DIR / name
    if not path.is_file():
        raise NativeLibraryError(
            f"{path} is missing: build it with `make -C {LIB_DIR.parent / 'csrc'}` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    try:
        lib = ctypes.CDLL(str(path), mode=os.RTLD_LOCAL)
    except OSError as err:
        raise NativeLibraryError(f"failed to load {path}: {err}") from err
    for fn, (res, args) in sigs.items():
        f = getattr(lib, fn)
        f.restype = res
        f.argtypes = args
    _libs[name] = lib
    return lib


def kernels() -> ctypes.CDLL:
    # MB_KERNELS_LIB selects an alternative build in lib/ (A/B experiments of kernel variants)
    return _load(os.environ.get("MB_KERNELS_LIB", "libmb_sm100.so"), _KERNEL_SIGS)


def planner() -> ctypes.CDLL:
    fresh = "libmb_planner.so" not in _libs
    lib = _load("libmb_planner.so", _PLANNER_SIGS)
    if fresh and os.environ.get("MB_PLANNER_NUMPY_BLAS", "1") != "0":
        path = numpy_blas_path()
        if path:
            lib.mbp_use_numpy_blas(path.encode(), b"scipy_")
    return lib


def numpy_blas_path() -> str | None:
    """numpy's bundled ILP64 OpenBLAS (the library numpy's matmul calls), if present."""
    try:
        import numpy as np
        for d in (Path(np.__file__).resolve().parent.parent / "numpy.libs",):
            for p in sorted(d.glob("libscipy_openblas64_*.so")):
                return str(p)
    except Exception:  # pragma: no cover
        return None
    return None


def register_planner_sigs(sigs: dict) -> None:
    _PLANNER_SIGS.update(sigs)


def check(status: int, lib: ctypes.CDLL, what: str) -> None:
    if status == 0:
        return
    if hasattr(lib, "mbp_last_error"):
        msg = lib.mbp_last_error()
    else:
        msg = lib.mb_last_error() if hasattr(lib, "mb_last_error") else None
    msg = msg.decode() if isinstance(msg, bytes) else str(msg)
    if status == 1:
        raise ValueError(f"{what}: {msg}")
    if status == 5:
        raise LPError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (status {status}): {msg}")


def f64(a):
    import numpy as np
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    import numpy as np
    return np.ascontiguousarray(a, dtype=np.int64)


def i32(a):
    import numpy as np
    return np.ascontiguousarray(a, dtype=np.int32)


def ptr(t) -> int | None:
    """Raw pointer of a torch tensor / numpy array (None for None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
