"""Routing traces: the (micro-batch, layer, source GPU, expert) count contract, its metrics,
and the token-level replayed routing that produces it.

Mirror of the hot-path part of ``moebalance.routing`` (routing.py:27-212, 476-518): same
``ModelProfile`` / ``RoutingTrace`` fields, validation messages, ``aggregate_batch``,
``skewness``, ``hot_expert_intersection``.  The reference draws COUNTS directly
(routing.py:414-418); the data plane needs TOKENS, so ``ZipfRouting`` generates per-token
top-k choices (Gumbel-top-k over a Zipf popularity whose hot set rotates every micro-batch,
SURVEY.md section 8d) and ``trace_from_routing`` histograms them on the GPU (kernel K1) into a
``RoutingTrace`` whose matrices equal np.bincount of the indices bit for bit.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .cluster import ClusterTopology, HardwareProfile, build_topology

U32_MAX = 2**32 - 1
DEFAULT_HIDDEN_SIZE = 1024
DEFAULT_INTERMEDIATE_SIZE = 512


class TraceFormatError(ValueError):
    """Malformed or internally inconsistent routing trace."""


@dataclass(frozen=True)
class ModelProfile:
    """MoE dimensions (routing.py:53-84): param_bytes = 3 * 2 * h * h' (bf16 SwiGLU expert)."""

    num_layers: int
    num_experts: int
    top_k: int
    hidden_size: int = DEFAULT_HIDDEN_SIZE
    intermediate_size: int = DEFAULT_INTERMEDIATE_SIZE
    expert_param_bytes: int | None = None

    def __post_init__(self) -> None:
        if self.num_layers < 1 or self.num_experts < 1:
            raise ValueError("model needs at least one layer and one expert")
        if not 1 <= self.top_k <= self.num_experts:
            raise ValueError(f"top_k {self.top_k} outside [1, {self.num_experts}]")
        if self.hidden_size < 1 or self.intermediate_size < 1:
            raise ValueError("hidden/intermediate sizes must be positive")

    @property
    def param_bytes(self) -> int:
        if self.expert_param_bytes is not None:
            return self.expert_param_bytes
        return 6 * self.hidden_size * self.intermediate_size

    def experts_per_gpu(self, topo: ClusterTopology) -> int:
        if self.num_experts % topo.num_gpus:
            raise ValueError(f"{self.num_experts} experts not divisible by {topo.num_gpus} GPUs")
        return self.num_experts // topo.num_gpus


MANIFEST_VERSION = 1
MANIFEST_REQUIRED = ("version", "num_layers", "num_experts", "top_k", "num_micro_batches", "num_nodes",
                     "gpus_per_node", "tokens_per_gpu", "flops_per_gpu", "bw_nvlink_Bps", "bw_rdma_Bps",
                     "bytes_per_token")


@dataclass
class SampleTable:
    """Per-sample counts [sample][layer][expert] u32 and each sample's micro-batch, source GPU and
    token length (routing.py:137-149; samples.bin / samples.json)."""

    counts: np.ndarray
    micro_batch: np.ndarray
    source_gpu: np.ndarray
    tokens: np.ndarray

    @property
    def num_samples(self) -> int:
        return int(self.counts.shape[0])


@dataclass
class RoutingTrace:
    """matrices[mb, layer, src_gpu, expert] (u32) token-to-expert assignment counts."""

    model: ModelProfile
    topo: ClusterTopology
    matrices: np.ndarray
    tokens_per_gpu: int
    samples: object | None = None
    generator: dict = field(default_factory=dict)

    @property
    def num_micro_batches(self) -> int:
        return self.matrices.shape[0]

    def matrix(self, micro_batch: int, layer: int) -> np.ndarray:
        return self.matrices[micro_batch, layer]

    def manifest(self) -> dict:
        hw = self.topo.profile
        m = {
            "version": 1, "num_layers": self.model.num_layers, "num_experts": self.model.num_experts,
            "top_k": self.model.top_k, "num_micro_batches": self.num_micro_batches,
            "num_nodes": self.topo.num_nodes, "gpus_per_node": self.topo.gpus_per_node,
            "tokens_per_gpu": self.tokens_per_gpu, "flops_per_gpu": hw.flops_per_gpu,
            "bw_nvlink_Bps": hw.bw_nvlink, "bw_rdma_Bps": hw.bw_rdma, "bytes_per_token": hw.bytes_per_token,
            "hidden_size": self.model.hidden_size, "intermediate_size": self.model.intermediate_size,
            "expert_param_bytes": self.model.param_bytes, "has_samples": self.samples is not None,
        }
        if self.generator:
            m["generator"] = self.generator
        return m

    def trace_id(self) -> str:
        """sha256 over the manifest and the little-endian u32 matrices (routing.py:170-174)."""
        h = hashlib.sha256(json.dumps(self.manifest(), sort_keys=True).encode())
        h.update(np.ascontiguousarray(self.matrices, dtype="<u4").tobytes())
        return h.hexdigest()[:16]

    def validate(self) -> None:
        """Shape and row-sum invariants of routing.py:176-195."""
        mb, layers, g, e = self.matrices.shape
        if layers != self.model.num_layers or e != self.model.num_experts:
            raise TraceFormatError("matrix dimensions disagree with the model profile")
        if g != self.topo.num_gpus:
            raise TraceFormatError("matrix dimensions disagree with the topology")
        self.model.experts_per_gpu(self.topo)
        sums = self.matrices.astype(np.int64).sum(axis=3)
        if (sums % self.model.top_k).any():
            raise TraceFormatError("row sums are not divisible by top_k")
        if (sums != sums[:, :1, :]).any():
            raise TraceFormatError("per-GPU token counts differ across layers of one micro-batch")
        if self.tokens_per_gpu > 0 and (sums != self.tokens_per_gpu * self.model.top_k).any():
            raise TraceFormatError(
                f"row sums do not match tokens_per_gpu * top_k = {self.tokens_per_gpu * self.model.top_k}")
        if self.samples is not None:
            self._validate_samples()

    def _validate_samples(self) -> None:
        """Sample table consistency (routing.py:197-212)."""
        s = self.samples
        mb, layers, g, e = self.matrices.shape
        if s.counts.shape[1:] != (layers, e):
            raise TraceFormatError("sample counts disagree with trace dimensions")
        if not (len(s.micro_batch) == len(s.source_gpu) == len(s.tokens) == s.counts.shape[0]):
            raise TraceFormatError("sample index and sample counts disagree in length")
        if s.micro_batch.min(initial=0) < 0 or s.micro_batch.max(initial=0) >= mb:
            raise TraceFormatError("sample micro_batch out of range")
        if s.source_gpu.min(initial=0) < 0 or s.source_gpu.max(initial=0) >= g:
            raise TraceFormatError("sample source_gpu out of range")
        rebuilt = np.zeros((mb, layers, g, e), dtype=np.int64)
        np.add.at(rebuilt, (s.micro_batch, slice(None), s.source_gpu), s.counts.astype(np.int64))
        if (rebuilt != self.matrices.astype(np.int64)).any():
            raise TraceFormatError("per-GPU sums over samples do not reproduce the routing matrices")


def save_trace(trace: RoutingTrace, path) -> None:
    """manifest.json + routing.bin (+ samples.bin / samples.json), byte-compatible with
    moebalance.routing.save_trace (routing.py:240-256)."""
    trace.validate()
    if trace.matrices.max(initial=0) > U32_MAX:
        raise TraceFormatError("token counts exceed the u32 trace format")
    out = Path(path)
    out.mkdir(parents=True, exist_ok=True)
    (out / "manifest.json").write_text(json.dumps(trace.manifest(), indent=2, sort_keys=True) + "\n")
    (out / "routing.bin").write_bytes(np.ascontiguousarray(trace.matrices, dtype="<u4").tobytes())
    if trace.samples is not None:
        s = trace.samples
        (out / "samples.bin").write_bytes(np.ascontiguousarray(s.counts, dtype="<u4").tobytes())
        index = [{"micro_batch": int(s.micro_batch[i]), "source_gpu": int(s.source_gpu[i]),
                  "tokens": int(s.tokens[i])} for i in range(s.num_samples)]
        (out / "samples.json").write_text(json.dumps({"samples": index}, indent=2) + "\n")


def load_trace(path) -> RoutingTrace:
    """Read a trace directory written by either implementation (routing.py:259-322), validating
    every invariant; errors are TraceFormatError (a ValueError) as in the reference."""
    root = Path(path)
    mpath = root / "manifest.json"
    if not mpath.is_file():
        raise TraceFormatError(f"missing manifest: {mpath}")
    try:
        man = json.loads(mpath.read_text())
    except json.JSONDecodeError as err:
        raise TraceFormatError(f"malformed manifest: {err}") from err
    missing = [k for k in MANIFEST_REQUIRED if k not in man]
    if missing:
        raise TraceFormatError(f"manifest missing keys: {', '.join(missing)}")
    if man["version"] != MANIFEST_VERSION:
        raise TraceFormatError(f"unsupported trace version {man['version']}")
    model = ModelProfile(num_layers=man["num_layers"], num_experts=man["num_experts"], top_k=man["top_k"],
                         hidden_size=man.get("hidden_size", DEFAULT_HIDDEN_SIZE),
                         intermediate_size=man.get("intermediate_size", DEFAULT_INTERMEDIATE_SIZE),
                         expert_param_bytes=man.get("expert_param_bytes"))
    topo = build_topology(man["num_nodes"], man["gpus_per_node"],
                          HardwareProfile(flops_per_gpu=man["flops_per_gpu"], bw_nvlink=man["bw_nvlink_Bps"],
                                          bw_rdma=man["bw_rdma_Bps"], bytes_per_token=man["bytes_per_token"]))
    shape = (man["num_micro_batches"], model.num_layers, topo.num_gpus, model.num_experts)
    bpath = root / "routing.bin"
    if not bpath.is_file():
        raise TraceFormatError(f"missing routing.bin in {root}")
    payload = bpath.read_bytes()
    expected = int(np.prod(shape)) * 4
    if len(payload) != expected:
        raise TraceFormatError(f"routing.bin holds {len(payload)} bytes, manifest implies {expected}")
    matrices = np.frombuffer(payload, dtype="<u4").reshape(shape).copy()
    samples = _load_samples(root, shape) if man.get("has_samples") else None
    trace = RoutingTrace(model=model, topo=topo, matrices=matrices, tokens_per_gpu=man["tokens_per_gpu"],
                         samples=samples, generator=man.get("generator", {}))
    trace.validate()
    return trace


def _load_samples(root: Path, shape: tuple) -> SampleTable:
    bpath, ipath = root / "samples.bin", root / "samples.json"
    if not bpath.is_file() or not ipath.is_file():
        raise TraceFormatError("manifest declares samples but sample files are missing")
    index = json.loads(ipath.read_text())["samples"]
    _, layers, _, experts = shape
    payload = bpath.read_bytes()
    expected = len(index) * layers * experts * 4
    if len(payload) != expected:
        raise TraceFormatError(f"samples.bin holds {len(payload)} bytes, index implies {expected}")
    counts = np.frombuffer(payload, dtype="<u4").reshape(len(index), layers, experts).copy()
    return SampleTable(counts=counts, micro_batch=np.array([s["micro_batch"] for s in index], dtype=np.int32),
                       source_gpu=np.array([s["source_gpu"] for s in index], dtype=np.int32),
                       tokens=np.array([s["tokens"] for s in index], dtype=np.int32))


def realize_tokens(counts: np.ndarray, top_k: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Token-level routing for one (micro-batch, layer, source GPU) count row of a recorded trace:
    idx [T, k] int32 whose np.bincount equals `counts` exactly, each token with k distinct experts,
    and softmax gates [T, k] float32.  Expert ids are laid out count-descending and dealt
    column-major over the T x k grid (a run of c <= T ids never lands twice in one row); the
    rows are then shuffled with `seed`.  Lets count traces (routing.bin) drive the data plane."""
    counts = np.asarray(counts, dtype=np.int64)
    total = int(counts.sum())
    if total % top_k:
        raise TraceFormatError("row sum is not divisible by top_k")
    T = total // top_k
    if counts.max(initial=0) > T:
        raise TraceFormatError("an expert count exceeds the token count: no distinct top-k realisation")
    order = np.argsort(-counts, kind="stable")
    ids = np.repeat(order, counts[order]).astype(np.int32)
    idx = ids.reshape(top_k, T).T.copy()
    rng = np.random.default_rng(seed)
    idx = idx[rng.permutation(T)]
    logits = rng.standard_normal((T, top_k)).astype(np.float32)
    gates = np.exp(logits - logits.max(axis=1, keepdims=True))
    gates = (gates / gates.sum(axis=1, keepdims=True)).astype(np.float32)
    return np.ascontiguousarray(idx), gates


def aggregate_batch(trace: RoutingTrace, layer: int) -> np.ndarray:
    """int64 sum of one layer's matrices over the micro-batches (routing.py:476-480)."""
    if not 0 <= layer < trace.model.num_layers:
        raise ValueError(f"layer {layer} out of range [0, {trace.model.num_layers})")
    return trace.matrices[:, layer].astype(np.int64).sum(axis=0)


def skewness(loads) -> float:
    """max / mean load; 1.0 = perfectly balanced (routing.py:483-493)."""
    v = np.asarray(loads, dtype=np.float64).ravel()
    if v.size == 0:
        raise ValueError("skewness of an empty load vector")
    if v.min() < 0:
        raise ValueError("loads must be non-negative")
    tot = v.sum()
    if tot == 0:
        raise ValueError("skewness undefined for an all-zero load vector")
    return float(v.max() * v.size / tot)


def top_k_experts(expert_loads: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest loads, ties toward the lower index."""
    loads = np.asarray(expert_loads, dtype=np.float64)
    return np.lexsort((np.arange(len(loads)), -loads))[:k]


def hot_expert_intersection(trace: RoutingTrace, layer: int, k: int) -> np.ndarray:
    """|top_k(mb) & top_k(mb+1)| / k for adjacent micro-batches (routing.py:502-518)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    if k > trace.model.num_experts:
        raise ValueError(f"k = {k} exceeds the expert count {trace.model.num_experts}")
    if trace.num_micro_batches < 2:
        raise ValueError("need at least two micro-batches")
    if not 0 <= layer < trace.model.num_layers:
        raise ValueError(f"layer {layer} out of range")
    hot = [set(top_k_experts(trace.matrices[m, layer].astype(np.int64).sum(axis=0), k).tolist())
           for m in range(trace.num_micro_batches)]
    return np.array([len(a & b) / k for a, b in zip(hot[:-1], hot[1:])])


# ----------------------------------------------------------------------------- token routing


@dataclass(frozen=True)
class ZipfRouting:
    """Replayed top-k routing with Zipf(s) expert popularity and a hot set that rotates by
    `shift` ranks every micro-batch.  `balanced=True` yields the
    balanced-ideal routing instead: token t takes experts (t*k + i) mod E, whose counts equal
    sim._uniform_matrices (sim.py:127-139) exactly."""

    num_experts: int
    top_k: int
    tokens: int
    zipf_s: float = 1.0
    shift: int = 7
    seed: int = 20261018
    balanced: bool = False

    def popularity(self, micro_batch: int) -> np.ndarray:
        e = self.num_experts
        perm = np.random.default_rng(self.seed).permutation(e)
        weights = (np.arange(e, dtype=np.float64) + 1.0) ** (-self.zipf_s)
        p = np.empty(e)
        p[perm[(np.arange(e) + micro_batch * self.shift) % e]] = weights
        return p / p.sum()

    def sample(self, micro_batch: int, layer: int, src_gpu: int) -> tuple[np.ndarray, np.ndarray]:
        """(idx [T,k] int32, gates [T,k] float32) for one (micro-batch, layer, source GPU)."""
        t, k, e = self.tokens, self.top_k, self.num_experts
        rng = np.random.default_rng([self.seed + 1000 * micro_batch + layer, src_gpu])
        if self.balanced:
            idx = ((np.arange(t, dtype=np.int64)[:, None] * k + np.arange(k)[None, :]) % e).astype(np.int32)
            logits = rng.standard_normal((t, k))
        else:
            scores = np.log(self.popularity(micro_batch))[None, :] + rng.gumbel(size=(t, e))
            part = np.argpartition(-scores, k - 1, axis=1)[:, :k]
            order = np.argsort(-np.take_along_axis(scores, part, axis=1), axis=1, kind="stable")
            idx = np.take_along_axis(part, order, axis=1).astype(np.int32)
            logits = np.take_along_axis(scores, idx.astype(np.int64), axis=1)
        z = logits - logits.max(axis=1, keepdims=True)
        gates = np.exp(z)
        gates = (gates / gates.sum(axis=1, keepdims=True)).astype(np.float32)
        return np.ascontiguousarray(idx), np.ascontiguousarray(gates)


def routing_matrix_from_indices(idx_per_gpu: list[np.ndarray], num_experts: int) -> np.ndarray:
    """(G, E) counts from per-GPU [T,k] index arrays on the host (np.bincount); the device
    path is kernels.expert_histogram."""
    return np.stack([np.bincount(np.asarray(i).ravel(), minlength=num_experts) for i in idx_per_gpu]).astype(np.uint32)


def build_trace(model: ModelProfile, topo: ClusterTopology, matrices: np.ndarray, tokens_per_gpu: int,
                generator: dict | None = None) -> RoutingTrace:
    """RoutingTrace over (MB, L, G, E) counts, validated."""
    trace = RoutingTrace(model=model, topo=topo, matrices=np.ascontiguousarray(matrices, dtype=np.uint32),
                         tokens_per_gpu=tokens_per_gpu, generator=dict(generator or {}))
    trace.validate()
    return trace
