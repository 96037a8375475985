// K1: warp-aggregated expert-load histogram over replayed top-k routing.
//
// counts[b][e] = #{(t,i) : idx[b][t][i] == e} for every (micro-batch, layer) batch b in ONE
// launch: this is exactly one source row of RoutingTrace.matrices (routing.py:151-168), the
// u32 [mb][layer][src][expert] layout of routing.bin (routing.py:3-13).  The per-chunk
// counts are kept so the permutation kernel (K2) can derive stable per-expert ranks
// without a second pass over the indices.
//
// HBM-bound: T*k*4 B read + E*4 B written per batch.  Grid = (chunks, batches); each CTA
// owns one chunk of `chunk_tokens` tokens, privatises E bins in shared memory and
// aggregates equal experts inside a warp with __match_any_sync before the smem atomic.
#include "capi_common.cuh"
#include "sm100_ptx.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

__global__ void __launch_bounds__(256) expert_histogram_kernel(const int32_t* __restrict__ idx, int64_t tokens,
                                                               int topk, int num_experts, uint32_t* __restrict__ counts,
                                                               uint32_t* __restrict__ chunk_counts, int chunk_tokens) {
  extern __shared__ uint32_t bins[];
  const int chunk = blockIdx.x;
  const int64_t b = blockIdx.y;
  const int num_chunks = gridDim.x;
  for (int e = threadIdx.x; e < num_experts; e += blockDim.x) bins[e] = 0;
  __syncthreads();

  const int64_t t0 = static_cast<int64_t>(chunk) * chunk_tokens;
  const int64_t t1 = (t0 + chunk_tokens < tokens) ? (t0 + chunk_tokens) : tokens;
  const int64_t n = (t1 - t0) * topk;
  const int32_t* src = idx + (b * tokens + t0) * topk;
  const int lane = lane_id();
  // vectorised 16-byte loads when the chunk start is aligned (always true for k*chunk%4==0)
  for (int64_t base = static_cast<int64_t>(threadIdx.x) * 4; base < n; base += static_cast<int64_t>(blockDim.x) * 4) {
    int v[4];
    if (base + 3 < n && ((reinterpret_cast<uintptr_t>(src + base) & 15) == 0)) {
      const int4 q = *reinterpret_cast<const int4*>(src + base);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = (base + j < n) ? src[base + j] : -1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = (v[j] >= 0 && v[j] < num_experts) ? v[j] : -1;
      const unsigned active = __activemask();
      const unsigned peers = __match_any_sync(active, e);
      const int leader = __ffs(peers) - 1;
      if (lane == leader && e >= 0) atomicAdd(&bins[e], static_cast<uint32_t>(__popc(peers)));
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < num_experts; e += blockDim.x) {
    const uint32_t c = bins[e];
    if (chunk_counts) chunk_counts[(b * num_chunks + chunk) * num_experts + e] = c;
    if (c) atomicAdd(&counts[b * num_experts + e], c);
  }
}

}  // namespace mb

using namespace mb;

extern "C" int mb_expert_histogram(const int32_t* idx, int64_t nb, int64_t tokens, int32_t topk, int32_t num_experts,
                                   uint32_t* counts, uint32_t* chunk_counts, int32_t chunk_tokens, void* stream) {
  MB_CHECK_ARG(nb >= 0 && tokens >= 0 && topk >= 1 && num_experts >= 1 && num_experts <= 4096,
               "bad histogram shape nb=%lld T=%lld k=%d E=%d", (long long)nb, (long long)tokens, topk, num_experts);
  MB_CHECK_ARG(chunk_tokens >= 1, "chunk_tokens must be >= 1");
  MB_CHECK_ARG(counts != nullptr, "counts is null");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (nb == 0) return MB_OK;
  MB_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * nb * num_experts, s));
  if (tokens == 0) {
    return MB_OK;
  }
  MB_CHECK_ARG(idx != nullptr, "idx is null");
  const int64_t chunks = (tokens + chunk_tokens - 1) / chunk_tokens;
  MB_CHECK_ARG(chunks <= 0x7fffffff && nb <= 65535, "too many chunks/batches");
  dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(nb));
  expert_histogram_kernel<<<grid, 256, num_experts * sizeof(uint32_t), s>>>(idx, tokens, topk, num_experts, counts,
                                                                          chunk_counts, chunk_tokens);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

extern "C" const char* mb_last_error(void) { return g_last_error.c_str(); }
extern "C" int mb_version(void) { return 1; }
