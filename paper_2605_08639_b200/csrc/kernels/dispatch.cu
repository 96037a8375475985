// K2/K3/K6: token permutation, dispatch and combine over NVLink peer pointers.
//
// The reference only MODELS this traffic: costmodel.flow_matrix (costmodel.py:91-108) gives
// flow[src, serving GPU] from the routing matrix, the placement and the split fractions;
// replicate.round_split (replicate.py:501-525) turns fractions into whole tokens; combine is
// the mirror of dispatch (costmodel.py:149-150).  Here the same integers drive real row moves.
//
// Canonical permutation P (defined by this build, identical in oracle/moe_ref.py):
//   on source GPU j enumerate (t, i) row-major; e = idx[t,i]; r = stable rank of (t,i) among the
//   entries of GPU j routed to e; copy c = min{c : r < cum_end[e][c]} where cum_end are the
//   prefix sums of the integer split counts of (j, e) over copies [home] + replicas
//   (ReplicaPlacement.copies, replicate.py:55-56); destination (gpu, row) =
//   (copies[c], row_base[e][c] + r - cum_end[e][c-1]).
//   row_base is fixed by the receive layout of the destination GPU: slots (home experts
//   ascending, then replicated experts ascending) x source GPU ascending x rank, each slot padded
//   to a multiple of 128 rows (the GEMM M tile).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "capi_common.cuh"
#include "sm100_ptx.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

constexpr int32_t kErrRoutingMismatch = MB_ERR_ROUTING_MISMATCH;

// ------------------------------------------------------------------ chunk prefix scan
// chunk_base[b][c][e] = sum_{c' < c} chunk_counts[b][c'][e]   (one warp per expert column)
__global__ void __launch_bounds__(256) chunk_scan_kernel(const uint32_t* __restrict__ chunk_counts,
                                                         uint32_t* __restrict__ chunk_base, int chunks, int E) {
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const uint32_t* cc = chunk_counts + static_cast<int64_t>(b) * chunks * E;
  uint32_t* cb = chunk_base + static_cast<int64_t>(b) * chunks * E;
  const int per = (chunks + 31) / 32;
  for (int e = blockIdx.x * warps + warp; e < E; e += gridDim.x * warps) {
    const int c0 = lane * per;
    const int c1 = min(c0 + per, chunks);
    uint32_t s = 0;
    for (int c = c0; c < c1; ++c) s += cc[static_cast<int64_t>(c) * E + e];
    uint32_t incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    uint32_t run = incl - s;
    for (int c = c0; c < c1; ++c) {
      cb[static_cast<int64_t>(c) * E + e] = run;
      run += cc[static_cast<int64_t>(c) * E + e];
    }
  }
}

// ------------------------------------------------------------------ K2 stable-rank permutation
// One warp per chunk of `chunk_tokens` tokens; ranks are stable in row-major (t, i) order.
// route_tab: [E][maxc][4] int32 {cum_end, dst_gpu, dst_row_base, 0}; ncopies[E].
// Batched over micro-batches on blockIdx.y (per-micro-batch tables at fixed strides; dst_gate
// holds `world` pointers per micro-batch).
__global__ void __launch_bounds__(128) permute_rank_kernel(
    const int32_t* __restrict__ idx, int64_t T, int k, const float* __restrict__ gate, int E,
    const uint32_t* __restrict__ chunk_base, int chunk_tokens, const int4* __restrict__ route_tab,
    const int32_t* __restrict__ ncopies, int maxc, float* const* __restrict__ dst_gate, int2* __restrict__ perm,
    int world, int32_t* __restrict__ error_flag) {
  extern __shared__ uint32_t running_all[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunk = blockIdx.x * (blockDim.x >> 5) + warp;
  {
    const int64_t b = blockIdx.y;
    const int64_t chunks = (T + chunk_tokens - 1) / chunk_tokens;
    idx += b * T * k;
    if (gate) gate += b * T * k;
    chunk_base += b * chunks * E;
    route_tab += b * E * maxc;
    ncopies += b * E;
    if (dst_gate) dst_gate += b * world;
    perm += b * T * k;
  }
  uint32_t* running = running_all + warp * E;
  for (int e = lane; e < E; e += 32) running[e] = 0;
  __syncwarp();
  const int64_t t0 = static_cast<int64_t>(chunk) * chunk_tokens;
  if (t0 >= T) return;
  const int64_t t1 = min(t0 + chunk_tokens, T);
  const int64_t n0 = t0 * k, n1 = t1 * k;
  const uint32_t* base = chunk_base + static_cast<int64_t>(chunk) * E;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t s = n0; s < n1; s += 32) {
    const int64_t n = s + lane;
    const bool valid = n < n1;
    const int e = valid ? idx[n] : -1;
    const bool ok = valid && e >= 0 && e < E;
    const unsigned peers = __match_any_sync(0xffffffffu, ok ? e : -1);
    const int leader = __ffs(peers) - 1;
    uint32_t first = 0;
    if (ok && lane == leader) {
      first = base[e] + running[e];
      running[e] += __popc(peers);
    }
    first = __shfl_sync(0xffffffffu, first, leader);
    __syncwarp();
    if (!ok) {
      if (valid) perm[n] = make_int2(-1, -1);
      continue;
    }
    const uint32_t r = first + __popc(peers & lt_mask);
    const int nc = ncopies[e];
    const int4* tab = route_tab + static_cast<int64_t>(e) * maxc;
    int prev = 0, c = 0;
    int4 ent = tab[0];
    while (c + 1 < nc && static_cast<int>(r) >= ent.x) {
      prev = ent.x;
      ent = tab[++c];
    }
    if (static_cast<int>(r) >= ent.x) {
      // more tokens of expert e than the plan's split counts: the routing differs from the
      // (replayed) counts the tables were built for.  Drop the choice instead of writing past
      // the receive slot, and flag it (the host raises).
      perm[n] = make_int2(-1, -1);
      if (error_flag) atomicOr(error_flag, kErrRoutingMismatch);
      continue;
    }
    const int row = ent.z + static_cast<int>(r) - prev;
    perm[n] = make_int2(ent.y, row);
    if (gate && dst_gate) dst_gate[ent.y][row] = gate[n];
  }
}

// ------------------------------------------------------------------ routing / plan consistency
// counts[i] (K1 histogram) must equal expected[i] (the counts the step plan was built from);
// a mismatch sets `code` in the host-visible error flag.  The permutation kernel additionally
// drops (perm = -1) any choice whose rank falls past its expert's planned rows.
__global__ void __launch_bounds__(256) check_counts_kernel(const uint32_t* __restrict__ counts,
                                                           const int32_t* __restrict__ expected, int64_t n,
                                                           int32_t* __restrict__ error_flag, int32_t code) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (counts[i] != static_cast<uint32_t>(expected[i])) atomicOr(error_flag, code);
}

// ------------------------------------------------------------------ K3 scatter (dispatch A2A)
// Warp per token: the row is read once (128-bit loads) and stored to every (gpu, row) of its
// k choices, straight into the (possibly peer, NVLink-mapped) receive buffers.
template <int VPL>
__global__ void __launch_bounds__(256) scatter_rows_kernel(const uint4* __restrict__ x, int64_t T, int k, int h,
                                                           const int2* __restrict__ perm, void* const* __restrict__ dst_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int vrow = h >> 3;  // uint4 per row
  for (int64_t t = warp_global; t < T; t += nwarps) {
    const uint4* src = x + t * vrow;
    for (int col0 = 0; col0 < vrow; col0 += 32 * VPL) {
      uint4 v[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int col = col0 + j * 32 + lane;
        if (col < vrow) v[j] = __ldg(src + col);
      }
      for (int i = 0; i < k; ++i) {
        const int2 pr = perm[t * k + i];
        if (pr.x < 0) continue;
        uint4* dst = reinterpret_cast<uint4*>(dst_rows[pr.x]) + static_cast<int64_t>(pr.y) * vrow;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int col = col0 + j * 32 + lane;
          if (col < vrow) dst[col] = v[j];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K6 combine (un-permute)
// out[t] = sum_i w[t,i] * rows[perm(t,i)]  (fp32, fixed i order), w = gate or 1.
// Optionally gathers a per-row scalar (dgate) back into [T,k] order.
template <int VPL>
__global__ void __launch_bounds__(256) combine_rows_kernel(const void* const* __restrict__ src_rows, const int2* __restrict__ perm,
                                                           const float* __restrict__ gate, int64_t T, int k, int h,
                                                           uint4* __restrict__ out, const float* const* __restrict__ src_scalar,
                                                           float* __restrict__ scalar_out, int npart) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int vrow = h >> 3;
  for (int64_t t = warp_global; t < T; t += nwarps) {
    if (scalar_out && lane < k) {
      // per-row scalar = sum of its npart partials (fixed order: deterministic)
      const int2 pr = perm[t * k + lane];
      float s = 0.0f;
      if (pr.x >= 0) {
        const float* src = src_scalar[pr.x] + static_cast<int64_t>(pr.y) * npart;
        for (int q = 0; q < npart; ++q) s += src[q];
      }
      scalar_out[t * k + lane] = s;
    }
    for (int col0 = 0; col0 < vrow; col0 += 32 * VPL) {
      float acc[VPL][8];
#pragma unroll
      for (int j = 0; j < VPL; ++j)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j][q] = 0.0f;
      for (int i = 0; i < k; ++i) {
        const int2 pr = perm[t * k + i];
        if (pr.x < 0) continue;
        const float w = gate ? gate[t * k + i] : 1.0f;
        const uint4* src = reinterpret_cast<const uint4*>(src_rows[pr.x]) + static_cast<int64_t>(pr.y) * vrow;
        uint4 v[VPL];
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int col = col0 + j * 32 + lane;
          if (col < vrow) v[j] = src[col];
        }
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const uint32_t u[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[j][2 * q] += w * bf16lo(u[q]);
            acc[j][2 * q + 1] += w * bf16hi(u[q]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int col = col0 + j * 32 + lane;
        if (col < vrow)
          out[t * vrow + col] = make_uint4(pack_bf16x2(acc[j][0], acc[j][1]), pack_bf16x2(acc[j][2], acc[j][3]),
                                           pack_bf16x2(acc[j][4], acc[j][5]), pack_bf16x2(acc[j][6], acc[j][7]));
      }
    }
  }
}

// ------------------------------------------------------------------ TMA row movers
// The same two operations with the copy engine of each SM (cp.async.bulk) instead of register
// copies.  A block owns most of an SM's shared memory, so it never co-resides with a GEMM CTA
// (the row movers stay on the SMs the persistent GEMM leaves free), and each SM keeps ~190 KB of
// rows in flight -- what a remote (NVLink) copy needs to cover its latency.
constexpr int kTmaBarBytes = 1024;  // mbarriers at the start of dynamic shared memory

// K3: warp w streams tokens t = gw, gw + nwarps, ...: token j is bulk-loaded into buffer j % nbuf
// (one 128-bit-aligned row), then lanes 0..k-1 each bulk-store it to one (gpu, row) of the token's
// choices.  Loads run nbuf - 1 tokens ahead; a buffer is refilled once the stores that read it
// (the warp's previous bulk group) have drained it.
__global__ void __launch_bounds__(256, 1) scatter_rows_tma_kernel(const uint8_t* __restrict__ x, int64_t T, int k,
                                                                  int row_bytes, const int2* __restrict__ perm,
                                                                  void* const* __restrict__ dst_rows, int nbuf) {
  extern __shared__ __align__(1024) uint8_t smem_t[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_t) + warp * nbuf;
  uint8_t* buf = smem_t + kTmaBarBytes + static_cast<int64_t>(warp) * nbuf * row_bytes;
  if (lane == 0) {
    for (int b = 0; b < nbuf; ++b) mbar_init(&bar[b], 1);
    fence_proxy_async_smem();
  }
  __syncwarp();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * nw;
  if (gw >= T) return;
  const int64_t n = (T - gw + nwarps - 1) / nwarps;
  auto load = [&](int64_t j) {
    const int b = static_cast<int>(j % nbuf);
    mbar_arrive_expect_tx(&bar[b], row_bytes);
    bulk_load_1d(buf + static_cast<int64_t>(b) * row_bytes, x + (gw + j * nwarps) * row_bytes, row_bytes, &bar[b]);
  };
  if (lane == 0)
    for (int64_t j = 0; j < nbuf - 1 && j < n; ++j) load(j);
  int2 pr = make_int2(-1, -1);
  if (lane < k) pr = perm[gw * k + lane];
  for (int64_t j = 0; j < n; ++j) {
    const int b = static_cast<int>(j % nbuf);
    const int64_t t = gw + j * nwarps;
    // next token's choices while this one's row lands
    int2 pr_next = make_int2(-1, -1);
    if (lane < k && j + 1 < n) pr_next = perm[(t + nwarps) * k + lane];
    mbar_wait(&bar[b], static_cast<uint32_t>((j / nbuf) & 1));
    for (int i = lane; i < k; i += 32) {
      const int2 p = i < 32 ? pr : perm[t * k + i];
      if (p.x >= 0)
        bulk_store_1d(reinterpret_cast<uint8_t*>(dst_rows[p.x]) + static_cast<int64_t>(p.y) * row_bytes,
                      buf + static_cast<int64_t>(b) * row_bytes, row_bytes);
    }
    bulk_commit();
    pr = pr_next;
    const int64_t jn = j + nbuf - 1;
    if (jn < n) {
      bulk_wait_read<1>();  // token j-1's stores have read the buffer token jn lands in
      __syncwarp();
      if (lane == 0) load(jn);
    }
  }
  bulk_wait<0>();
}

// K6: block-cooperative.  A producer warp keeps a ring of nslot token slots in flight: for each
// token its lanes 0..k-1 bulk-load the k full rows (local or peer, one cp.async.bulk of 2h bytes
// each -- the TMA unit's cost is per operation, so whole rows move ~4x the bytes per op of 1 KB
// pieces) plus, for the dX un-permute, the rows' dgate partials; the (gpu, row, weight) triples
// go into the slot beside them.  kConsumers warps reduce a landed slot together (warp w owns
// columns w*32 + lane + 256*r) in fp32 with the fixed i order and arithmetic of
// combine_rows_kernel (bit-identical results) and release the slot on its empty barrier.
constexpr int kConsumers = 8;
// nsplit > 1: a slot holds one 1/nsplit column piece of the token's k rows (more, smaller slots in
// flight for the same shared memory); work item = (token, piece).
template <int KMAX>
__global__ void __launch_bounds__(32 * (kConsumers + 1), 1)
    combine_rows_tma_kernel(const void* const* __restrict__ src_rows, const int2* __restrict__ perm,
                            const float* __restrict__ gate, int64_t T, int k, int h, uint4* __restrict__ out,
                            const float* const* __restrict__ src_scalar, float* __restrict__ scalar_out, int npart,
                            int nslot, int nsplit) {
  extern __shared__ __align__(1024) uint8_t smem_t[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row_bytes = h * 2, vrow = h >> 3;
  const int piece_bytes = row_bytes / nsplit, pvrow = vrow / nsplit;
  const bool scal = scalar_out != nullptr;
  const int side_bytes = KMAX * 16 + (scal ? KMAX * npart * 4 : 0);  // npart % 4 == 0 (host check)
  const int64_t slot_bytes = static_cast<int64_t>(KMAX) * piece_bytes + side_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_t);
  uint64_t* empty = full + nslot;
  auto rows_of = [&](int s) { return smem_t + kTmaBarBytes + s * slot_bytes; };
  auto meta = [&](int s) { return reinterpret_cast<int4*>(rows_of(s) + static_cast<int64_t>(KMAX) * piece_bytes); };
  auto scl = [&](int s) {
    return reinterpret_cast<float*>(rows_of(s) + static_cast<int64_t>(KMAX) * piece_bytes + KMAX * 16);
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < nslot; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kConsumers);
    }
    fence_proxy_async_smem();
  }
  __syncthreads();
  const int64_t n = (T - blockIdx.x + gridDim.x - 1) / gridDim.x;  // tokens of this block
  if (static_cast<int64_t>(blockIdx.x) >= T) return;
  if (warp == kConsumers) {
    // ------------------------------------------------ producer
    // permutation entries are loaded a batch of kTB tokens at a time (lane = token-in-batch *
    // KMAX + choice), one batch ahead, so their global-load latency overlaps the slot waits
    constexpr int kTB = 32 / KMAX;
    const int ub = lane / KMAX, ci = lane % KMAX;
    auto fetch = [&](int64_t b, int2& p, float& w) {
      p = make_int2(-1, -1);
      w = 0.0f;
      const int64_t j = b * kTB + ub;
      if (ci < k && j < n) {
        const int64_t t = blockIdx.x + j * gridDim.x;
        p = perm[t * k + ci];
        w = gate ? gate[t * k + ci] : 1.0f;
      }
    };
    int2 pc, pn;
    float wc, wn;
    fetch(0, pc, wc);
    for (int64_t b = 0; b * kTB < n; ++b) {
      fetch(b + 1, pn, wn);
      for (int u = 0; u < kTB; ++u) {
        const int64_t jt = b * kTB + u;
        if (jt >= n) break;
        const bool mine = ub == u;
        const unsigned valid = __ballot_sync(0xffffffffu, mine && pc.x >= 0);
        for (int part = 0; part < nsplit; ++part) {
          const int64_t j = jt * nsplit + part;
          const int s = static_cast<int>(j % nslot);
          mbar_wait(&empty[s], static_cast<uint32_t>(((j / nslot) & 1) ^ 1));
          const bool with_scal = scal && part == 0;
          if (mine) meta(s)[ci] = make_int4(pc.x, pc.y, __float_as_int(wc), 0);
          if (lane == 0)
            mbar_arrive_expect_tx(&full[s], __popc(valid) * (piece_bytes + (with_scal ? npart * 4 : 0)));
          __syncwarp();
          if (mine && pc.x >= 0) {
            bulk_load_1d(rows_of(s) + static_cast<int64_t>(ci) * piece_bytes,
                         reinterpret_cast<const uint8_t*>(src_rows[pc.x]) + static_cast<int64_t>(pc.y) * row_bytes +
                             static_cast<int64_t>(part) * piece_bytes,
                         piece_bytes, &full[s]);
            if (with_scal)
              bulk_load_1d(scl(s) + ci * npart, src_scalar[pc.x] + static_cast<int64_t>(pc.y) * npart, npart * 4,
                           &full[s]);
          }
        }
      }
      pc = pn;
      wc = wn;
    }
    return;
  }
  // -------------------------------------------------- consumers
  for (int64_t j = 0; j < n * nsplit; ++j) {
    const int s = static_cast<int>(j % nslot);
    const int64_t t = blockIdx.x + (j / nsplit) * gridDim.x;
    const int part = static_cast<int>(j % nsplit);
    mbar_wait(&full[s], static_cast<uint32_t>((j / nslot) & 1));
    const int4* m = meta(s);
    if (scal && part == 0 && warp == 0 && lane < k) {
      float sc = 0.0f;
      if (m[lane].x >= 0) {
        const float* src = scl(s) + lane * npart;
        for (int qq = 0; qq < npart; ++qq) sc += src[qq];
      }
      scalar_out[t * k + lane] = sc;
    }
    const uint4* rows = reinterpret_cast<const uint4*>(rows_of(s));
    for (int col = warp * 32 + lane; col < pvrow; col += 32 * kConsumers) {
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
      uint4 u4[KMAX];
#pragma unroll
      for (int i = 0; i < KMAX; ++i)
        if (i < k && m[i].x >= 0) u4[i] = rows[static_cast<int64_t>(i) * pvrow + col];
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        if (i >= k) break;
        const int4 mi = m[i];
        if (mi.x < 0) continue;
        const float wi = __int_as_float(mi.z);
        const uint32_t u[4] = {u4[i].x, u4[i].y, u4[i].z, u4[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc[2 * e] += wi * bf16lo(u[e]);
          acc[2 * e + 1] += wi * bf16hi(u[e]);
        }
      }
      out[t * vrow + static_cast<int64_t>(part) * pvrow + col] =
          make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                     pack_bf16x2(acc[6], acc[7]));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// K6, confined register variant: warp per token, all k rows of a column chunk loaded before any
// is accumulated (k * VPL 128-bit loads in flight per lane; the fixed-i fp32 accumulation of
// combine_rows_kernel, so results are bit-identical).  Launched one 512-thread block per free SM
// with a shared-memory reservation that keeps it off the GEMM's SMs.
template <int KMAX, int VPL>
__global__ void __launch_bounds__(512, 1) combine_rows_mlp_kernel(const void* const* __restrict__ src_rows,
                                                                  const int2* __restrict__ perm,
                                                                  const float* __restrict__ gate, int64_t T, int k,
                                                                  int h, uint4* __restrict__ out,
                                                                  const float* const* __restrict__ src_scalar,
                                                                  float* __restrict__ scalar_out, int npart) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int vrow = h >> 3;
  for (int64_t t = warp_global; t < T; t += nwarps) {
    int2 p = make_int2(-1, -1);
    float w = 0.0f;
    if (lane < k) {
      p = perm[t * k + lane];
      w = gate ? gate[t * k + lane] : 1.0f;
    }
    float sc = 0.0f;
    if (scalar_out && lane < k && p.x >= 0) {
      const float* src = src_scalar[p.x] + static_cast<int64_t>(p.y) * npart;
      for (int q = 0; q < npart; ++q) sc += src[q];
    }
    const uint4* rowp[KMAX];
    float wi[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      const int px = __shfl_sync(0xffffffffu, p.x, i);
      const int py = __shfl_sync(0xffffffffu, p.y, i);
      wi[i] = __shfl_sync(0xffffffffu, w, i);
      rowp[i] = (i < k && px >= 0)
                    ? reinterpret_cast<const uint4*>(src_rows[px]) + static_cast<int64_t>(py) * vrow
                    : nullptr;
    }
    for (int col0 = 0; col0 < vrow; col0 += 32 * VPL) {
      uint4 u[KMAX][VPL];
#pragma unroll
      for (int i = 0; i < KMAX; ++i)
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int col = col0 + j * 32 + lane;
          if (rowp[i] && col < vrow) u[i][j] = rowp[i][col];
        }
      float acc[VPL][8];
#pragma unroll
      for (int j = 0; j < VPL; ++j)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[j][q] = 0.0f;
#pragma unroll
      for (int i = 0; i < KMAX; ++i) {
        if (!rowp[i]) continue;
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const uint32_t uu[4] = {u[i][j].x, u[i][j].y, u[i][j].z, u[i][j].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[j][2 * q] += wi[i] * bf16lo(uu[q]);
            acc[j][2 * q + 1] += wi[i] * bf16hi(uu[q]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int col = col0 + j * 32 + lane;
        if (col < vrow)
          out[t * vrow + col] = make_uint4(pack_bf16x2(acc[j][0], acc[j][1]), pack_bf16x2(acc[j][2], acc[j][3]),
                                           pack_bf16x2(acc[j][4], acc[j][5]), pack_bf16x2(acc[j][6], acc[j][7]));
      }
    }
    if (scalar_out && lane < k) scalar_out[t * k + lane] = sc;
  }
}

// ------------------------------------------------------------------ slot-table helpers
// slot_tab: [nslots][4] int32 {row_begin, rows_real, rows_pad, expert}; slots tile [0, total) in order.
__device__ __forceinline__ int find_slot(const int4* __restrict__ slots, int nslots, int64_t row) {
  int lo = 0, hi = nslots - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (slots[mid].x <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Expert-side combine backward (local to the serving GPU):
//   dY[row] = gate[row] * dout[row] (in place), dgate[row] = <dout[row], Y[row]>; pad rows -> 0.
template <int VPL>
__global__ void __launch_bounds__(256) combine_bwd_expert_kernel(uint4* __restrict__ dout_rows, const uint4* __restrict__ y_rows,
                                                                 const float* __restrict__ gate_rows, float* __restrict__ dgate_rows,
                                                                 const int4* __restrict__ slots, int nslots, int64_t total_rows, int h) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int vrow = h >> 3;
  for (int64_t row = warp_global; row < total_rows; row += nwarps) {
    const int4 sl = slots[find_slot(slots, nslots, row)];
    const bool real = row < static_cast<int64_t>(sl.x) + sl.y;
    uint4* d = dout_rows + row * vrow;
    if (!real) {
      for (int col = lane; col < vrow; col += 32) d[col] = make_uint4(0, 0, 0, 0);
      if (lane == 0 && dgate_rows) dgate_rows[row] = 0.0f;
      continue;
    }
    const float g = gate_rows[row];
    const uint4* y = y_rows + row * vrow;
    float dot = 0.0f;
    for (int col0 = 0; col0 < vrow; col0 += 32 * VPL) {
      uint4 dv[VPL], yv[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int col = col0 + j * 32 + lane;
        if (col < vrow) { dv[j] = d[col]; yv[j] = y[col]; }
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int col = col0 + j * 32 + lane;
        if (col >= vrow) continue;
        const uint32_t du[4] = {dv[j].x, dv[j].y, dv[j].z, dv[j].w};
        const uint32_t yu[4] = {yv[j].x, yv[j].y, yv[j].z, yv[j].w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float d0 = bf16lo(du[q]), d1 = bf16hi(du[q]);
          dot += d0 * bf16lo(yu[q]) + d1 * bf16hi(yu[q]);
          o[q] = pack_bf16x2(g * d0, g * d1);
        }
        d[col] = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
    if (lane == 0 && dgate_rows) dgate_rows[row] = dot;
  }
}

// Zero the pad rows [row_begin + rows_real, row_begin + rows_pad) of every slot.
// blockIdx.y = micro-batch (rows / slot tables at fixed strides; unused slot entries are all-zero)
__global__ void __launch_bounds__(256) zero_pad_rows_kernel(uint4* __restrict__ rows, const int4* __restrict__ slots, int h,
                                                            int64_t rows_stride, int slots_stride) {
  rows += blockIdx.y * rows_stride * (h >> 3);
  const int4 sl = slots[static_cast<int64_t>(blockIdx.y) * slots_stride + blockIdx.x];
  const int vrow = h >> 3;
  const int64_t r0 = static_cast<int64_t>(sl.x) + sl.y, r1 = static_cast<int64_t>(sl.x) + sl.z;
  const int64_t n = (r1 - r0) * vrow;
  uint4* base = rows + r0 * vrow;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) base[i] = make_uint4(0, 0, 0, 0);
}

// dst[i] += sum_s srcs[s][i]  (fp32, sources in list order: deterministic replica-grad reduce)
__global__ void __launch_bounds__(256) accumulate_f32_kernel(float4* __restrict__ dst, const float4* const* __restrict__ srcs,
                                                             int nsrc, int64_t n4) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = dst[i];
    for (int s = 0; s < nsrc; ++s) {
      const float4 b = srcs[s][i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    dst[i] = a;
  }
}

// Batched replica-gradient push-back: task b adds (or, first contribution, stores) the sum of its
// sources in list order into its destination -- one launch per micro-batch covers every home
// expert whose replicas served rows (replica gradients accumulate at the owner).
struct AccTask {
  float* dst;
  const float* src[MB_ACC_MAX_SRC];
  int64_t n;      // floats, multiple of 4
  int32_t nsrc;
  int32_t store;  // 1: dst = sum(src) (the expert's first gradient contribution of a fresh step)
};
static_assert(sizeof(AccTask) == 8 + 8 * MB_ACC_MAX_SRC + 16, "AccTask layout is part of the C-ABI");

__global__ void __launch_bounds__(256) accumulate_tasks_kernel(const AccTask* __restrict__ tasks) {
  const AccTask& t = tasks[blockIdx.y];
  float4* dst = reinterpret_cast<float4*>(t.dst);
  const int64_t n4 = t.n >> 2;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = t.store ? make_float4(0.f, 0.f, 0.f, 0.f) : dst[i];
    for (int s = 0; s < t.nsrc; ++s) {
      const float4 b = reinterpret_cast<const float4*>(t.src[s])[i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    dst[i] = a;
  }
}

// Row-moving kernels run concurrently with the persistent GEMM.  comm_smem() > 0 reserves that
// much dynamic shared memory per block so the blocks cannot co-reside with a GEMM CTA (they
// stay on the SMs the GEMM leaves free); comm_grid() caps the grid (experiment knobs:
// MB_COMM_SMEM, MB_COMM_GRID).
inline int comm_smem() {
  static int v = -1;
  if (v < 0) { const char* e = std::getenv("MB_COMM_SMEM"); v = e ? std::atoi(e) : 0; }
  return v;
}
inline int64_t comm_grid() {
  static int64_t v = -1;
  if (v < 0) { const char* e = std::getenv("MB_COMM_GRID"); v = e ? std::atoll(e) : 0; }
  return v;
}

// TMA row movers (scatter_rows_tma_kernel / combine_rows_tma_kernel): number of blocks, one per
// SM; 0 = the register-copy kernels (mb_set_comm_blocks, env MB_COMM_BLOCKS overrides).
// A call's own value (>= 0: a data plane passes its engine) wins over the process default.
static int g_comm_blocks = 0;
inline int comm_blocks(int per_call) {
  if (per_call >= 0) return per_call;
  if (const char* e = std::getenv("MB_COMM_BLOCKS")) return std::atoi(e);
  return g_comm_blocks;
}
constexpr int kTmaSmemBudget = 192 * 1024;

inline int grid_for(int64_t work_items, int per_block) {
  int64_t g = (work_items + per_block - 1) / per_block;
  const int64_t cap = comm_grid() > 0 ? comm_grid() : static_cast<int64_t>(device_sm_count()) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace mb

using namespace mb;

extern "C" int mb_chunk_scan(const uint32_t* chunk_counts, uint32_t* chunk_base, int64_t nb, int32_t chunks, int32_t E,
                             void* stream) {
  MB_CHECK_ARG(chunk_counts && chunk_base && nb >= 0 && chunks >= 0 && E >= 1, "bad chunk scan args");
  if (nb == 0 || chunks == 0) return MB_OK;
  dim3 grid((E + 7) / 8, static_cast<unsigned>(nb));
  chunk_scan_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(chunk_counts, chunk_base, chunks, E);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_permute_rank(const int32_t* idx, int64_t T, int32_t k, const float* gate, int32_t E,
                               const uint32_t* chunk_base, int32_t chunk_tokens, const int32_t* route_tab,
                               const int32_t* ncopies, int32_t maxc, float* const* dst_gate, int32_t* perm,
                               int32_t* error_flag, void* stream) {
  MB_CHECK_ARG(T >= 0 && k >= 1 && E >= 1 && E <= 2048 && chunk_tokens >= 1 && maxc >= 1, "bad permute args");
  MB_CHECK_ARG(idx && chunk_base && route_tab && ncopies && perm, "null permute operand");
  if (T == 0) return MB_OK;
  const int64_t chunks = (T + chunk_tokens - 1) / chunk_tokens;
  const int wpb = 4;
  const int64_t grid = (chunks + wpb - 1) / wpb;
  permute_rank_kernel<<<static_cast<unsigned>(grid), 32 * wpb, wpb * E * sizeof(uint32_t),
                        reinterpret_cast<cudaStream_t>(stream)>>>(
      idx, T, k, gate, E, chunk_base, chunk_tokens, reinterpret_cast<const int4*>(route_tab), ncopies, maxc, dst_gate,
      reinterpret_cast<int2*>(perm), 0, error_flag);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_permute_rank_nb(const int32_t* idx, int64_t T, int32_t k, const float* gate, int32_t E,
                                  const uint32_t* chunk_base, int32_t chunk_tokens, const int32_t* route_tab,
                                  const int32_t* ncopies, int32_t maxc, float* const* dst_gate, int32_t world,
                                  int32_t* perm, int32_t nb, int32_t* error_flag, void* stream) {
  MB_CHECK_ARG(T >= 0 && k >= 1 && E >= 1 && E <= 2048 && chunk_tokens >= 1 && maxc >= 1 && nb >= 0 && world >= 1,
               "bad permute args");
  MB_CHECK_ARG(idx && chunk_base && route_tab && ncopies && perm, "null permute operand");
  if (T == 0 || nb == 0) return MB_OK;
  const int64_t chunks = (T + chunk_tokens - 1) / chunk_tokens;
  const int wpb = 4;
  dim3 grid(static_cast<unsigned>((chunks + wpb - 1) / wpb), static_cast<unsigned>(nb));
  permute_rank_kernel<<<grid, 32 * wpb, wpb * E * sizeof(uint32_t), reinterpret_cast<cudaStream_t>(stream)>>>(
      idx, T, k, gate, E, chunk_base, chunk_tokens, reinterpret_cast<const int4*>(route_tab), ncopies, maxc, dst_gate,
      reinterpret_cast<int2*>(perm), world, error_flag);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}


extern "C" int mb_set_comm_blocks(int32_t blocks) {
  MB_CHECK_ARG(blocks >= 0, "blocks must be >= 0 (0 = register-copy row movers)");
  g_comm_blocks = blocks;
  return MB_OK;
}

extern "C" int mb_scatter_rows(const void* x, int64_t T, int32_t k, int32_t h, const int32_t* perm,
                               void* const* dst_rows, int32_t comm_blocks_call, void* stream) {
  MB_CHECK_ARG(x && perm && dst_rows && T >= 0 && k >= 1 && h >= 8 && h % 8 == 0, "bad scatter args");
  if (T == 0) return MB_OK;
  if (const int nb = comm_blocks(comm_blocks_call); nb > 0) {
    const int row_bytes = 2 * h;
    int warps = 8, nbuf = 0;
    while (warps > 1 && (nbuf = (kTmaSmemBudget - kTmaBarBytes) / (warps * row_bytes)) < 3) warps >>= 1;
    nbuf = (kTmaSmemBudget - kTmaBarBytes) / (warps * row_bytes);
    if (nbuf > 128 / warps) nbuf = 128 / warps;
    if (nbuf >= 2) {
      const int smem = kTmaBarBytes + warps * nbuf * row_bytes;
      MB_CUDA_TRY(cudaFuncSetAttribute(scatter_rows_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      scatter_rows_tma_kernel<<<nb, 32 * warps, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
          reinterpret_cast<const uint8_t*>(x), T, k, row_bytes, reinterpret_cast<const int2*>(perm), dst_rows, nbuf);
      MB_CUDA_TRY(cudaGetLastError());
      return MB_OK;
    }
  }
  const int grid = grid_for(T, 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int vrow = h / 8;
  if (vrow <= 64)
    scatter_rows_kernel<2><<<grid, 256, comm_smem(), s>>>(reinterpret_cast<const uint4*>(x), T, k, h, reinterpret_cast<const int2*>(perm), dst_rows);
  else if (vrow <= 128)
    scatter_rows_kernel<4><<<grid, 256, comm_smem(), s>>>(reinterpret_cast<const uint4*>(x), T, k, h, reinterpret_cast<const int2*>(perm), dst_rows);
  else
    scatter_rows_kernel<8><<<grid, 256, comm_smem(), s>>>(reinterpret_cast<const uint4*>(x), T, k, h, reinterpret_cast<const int2*>(perm), dst_rows);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_combine_rows(const void* const* src_rows, const int32_t* perm, const float* gate, int64_t T, int32_t k,
                               int32_t h, void* out, const float* const* src_scalar, float* scalar_out,
                               int32_t npart, int32_t comm_blocks_call, void* stream) {
  MB_CHECK_ARG(src_rows && perm && out && T >= 0 && k >= 1 && k <= 32 && h >= 8 && h % 8 == 0, "bad combine args");
  MB_CHECK_ARG((scalar_out == nullptr) == (src_scalar == nullptr), "src_scalar and scalar_out go together");
  MB_CHECK_ARG(npart >= 1, "npart must be >= 1");
  if (T == 0) return MB_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int vrow = h / 8;
  const int2* pr = reinterpret_cast<const int2*>(perm);
  uint4* o = reinterpret_cast<uint4*>(out);
  const char* ce = std::getenv("MB_COMBINE_ENGINE");
  if (const int nb = comm_blocks(comm_blocks_call); nb > 0 && k <= 8 && !(ce && std::string(ce) == "tma")) {
    // confined register engine: the smem reservation keeps the blocks off the GEMM's SMs
    constexpr int kReserve = 100 * 1024;
    const int kmax = k <= 2 ? 2 : k <= 4 ? 4 : 8;
    auto launch = [&](auto kern) -> int {
      MB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kReserve));
      kern<<<nb, 512, kReserve, s>>>(src_rows, pr, gate, T, k, h, o, src_scalar, scalar_out, npart);
      MB_CUDA_TRY(cudaGetLastError());
      return MB_OK;
    };
    if (kmax == 2) return launch(combine_rows_mlp_kernel<2, 4>);
    if (kmax == 4) return launch(combine_rows_mlp_kernel<4, 2>);
    return launch(combine_rows_mlp_kernel<8, 2>);
  }
  if (const int nb = comm_blocks(comm_blocks_call); nb > 0 && k <= 16 && (!scalar_out || (npart % 4 == 0 && npart <= 64))) {
    const int kmax = k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : 16;
    // whole rows per slot (MB_COMBINE_SPLIT=n: 1/n pieces -- measured n times slower: the cost is
    // per bulk operation, not per byte)
    int nsplit = 1;
    if (const char* e = std::getenv("MB_COMBINE_SPLIT")) nsplit = std::max(1, std::atoi(e));
    auto slot_of = [&](int ns) {
      return static_cast<int64_t>(kmax) * (2 * h / ns) + kmax * 16 + (scalar_out ? kmax * npart * 4 : 0);
    };
    const int64_t slot_bytes = slot_of(nsplit);
    int nslot = static_cast<int>((kTmaSmemBudget - kTmaBarBytes) / slot_bytes);
    if (nslot > 64) nslot = 64;
    if (nslot >= 2 && (2 * h) % (16 * nsplit) == 0) {
      const int smem = kTmaBarBytes + static_cast<int>(nslot * slot_bytes);
      auto launch = [&](auto kern) -> int {
        MB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        kern<<<nb, 32 * (kConsumers + 1), smem, s>>>(src_rows, pr, gate, T, k, h, o, src_scalar, scalar_out, npart,
                                                     nslot, nsplit);
        MB_CUDA_TRY(cudaGetLastError());
        return MB_OK;
      };
      if (kmax == 2) return launch(combine_rows_tma_kernel<2>);
      if (kmax == 4) return launch(combine_rows_tma_kernel<4>);
      if (kmax == 8) return launch(combine_rows_tma_kernel<8>);
      return launch(combine_rows_tma_kernel<16>);
    }
  }
  const int grid = grid_for(T, 8);
  if (vrow <= 64)
    combine_rows_kernel<2><<<grid, 256, comm_smem(), s>>>(src_rows, pr, gate, T, k, h, o, src_scalar, scalar_out, npart);
  else if (vrow <= 128)
    combine_rows_kernel<4><<<grid, 256, comm_smem(), s>>>(src_rows, pr, gate, T, k, h, o, src_scalar, scalar_out, npart);
  else
    combine_rows_kernel<8><<<grid, 256, comm_smem(), s>>>(src_rows, pr, gate, T, k, h, o, src_scalar, scalar_out, npart);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_combine_bwd_expert(void* dout_rows, const void* y_rows, const float* gate_rows, float* dgate_rows,
                                     const int32_t* slot_tab, int32_t nslots, int64_t total_rows, int32_t h,
                                     void* stream) {
  MB_CHECK_ARG(dout_rows && y_rows && gate_rows && slot_tab && nslots >= 0 && h % 8 == 0, "bad combine_bwd args");
  if (total_rows == 0 || nslots == 0) return MB_OK;
  const int grid = grid_for(total_rows, 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int vrow = h / 8;
  const int4* sl = reinterpret_cast<const int4*>(slot_tab);
  if (vrow <= 64)
    combine_bwd_expert_kernel<2><<<grid, 256, 0, s>>>(reinterpret_cast<uint4*>(dout_rows), reinterpret_cast<const uint4*>(y_rows), gate_rows, dgate_rows, sl, nslots, total_rows, h);
  else if (vrow <= 128)
    combine_bwd_expert_kernel<4><<<grid, 256, 0, s>>>(reinterpret_cast<uint4*>(dout_rows), reinterpret_cast<const uint4*>(y_rows), gate_rows, dgate_rows, sl, nslots, total_rows, h);
  else
    combine_bwd_expert_kernel<8><<<grid, 256, 0, s>>>(reinterpret_cast<uint4*>(dout_rows), reinterpret_cast<const uint4*>(y_rows), gate_rows, dgate_rows, sl, nslots, total_rows, h);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_zero_pad_rows(void* rows, const int32_t* slot_tab, int32_t nslots, int32_t h, void* stream) {
  MB_CHECK_ARG(rows && slot_tab && nslots >= 0 && h % 8 == 0, "bad zero_pad args");
  if (nslots == 0) return MB_OK;
  zero_pad_rows_kernel<<<nslots, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint4*>(rows), reinterpret_cast<const int4*>(slot_tab), h, 0, 0);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_zero_pad_rows_nb(void* rows, int64_t rows_stride, const int32_t* slot_tab, int32_t max_slots,
                                   int32_t nb, int32_t h, void* stream) {
  MB_CHECK_ARG(rows && slot_tab && max_slots >= 0 && nb >= 0 && rows_stride >= 0 && h % 8 == 0, "bad zero_pad args");
  if (max_slots == 0 || nb == 0) return MB_OK;
  dim3 grid(static_cast<unsigned>(max_slots), static_cast<unsigned>(nb));
  zero_pad_rows_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint4*>(rows), reinterpret_cast<const int4*>(slot_tab), h, rows_stride, max_slots);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_accumulate_f32(float* dst, const float* const* srcs, int32_t nsrc, int64_t n, void* stream) {
  MB_CHECK_ARG(dst && (nsrc == 0 || srcs) && n % 4 == 0, "bad accumulate args (n must be a multiple of 4)");
  if (n == 0 || nsrc == 0) return MB_OK;
  accumulate_f32_kernel<<<grid_for(n / 4, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(dst), reinterpret_cast<const float4* const*>(srcs), nsrc, n / 4);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_check_counts(const uint32_t* counts, const int32_t* expected, int64_t n, int32_t* error_flag,
                               int32_t code, void* stream) {
  MB_CHECK_ARG(counts && expected && error_flag && n >= 0 && code != 0, "bad check_counts args");
  if (n == 0) return MB_OK;
  check_counts_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024)), 256, 0,
                        reinterpret_cast<cudaStream_t>(stream)>>>(counts, expected, n, error_flag, code);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" int mb_accumulate_f32_tasks(const void* tasks, int32_t ntasks, int64_t max_n, void* stream) {
  MB_CHECK_ARG(ntasks >= 0 && ntasks <= 65535 && max_n >= 0 && max_n % 4 == 0 && (ntasks == 0 || tasks),
               "bad accumulate task args");
  if (ntasks == 0 || max_n == 0) return MB_OK;
  const int per_task = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((max_n / 4 + 255) / 256,
                                                                                  std::max(1, 2 * device_sm_count() / ntasks))));
  dim3 grid(static_cast<unsigned>(per_task), static_cast<unsigned>(ntasks));
  accumulate_tasks_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const AccTask*>(tasks));
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}
