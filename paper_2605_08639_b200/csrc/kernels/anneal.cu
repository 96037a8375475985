// GPU-side planning: the simulated-annealing chains of the inter-batch expert
// reordering planner, one warp per (layer, seed) chain.
//
// Device restatement of reorder._run_chain (reorder.py:299-326) as the host planner runs it
// (csrc/planner/reorder.cpp run_chain): swap proposals from numpy's PCG64 stream
// (Generator.integers(0, E) = 32-bit Lemire on the buffered next_uint32; Generator.random() =
// (next_uint64 >> 11) * 2^-53), O(G) swap delta on the shared contribution tensor, LSE_beta
// surrogate with numpy's pairwise summation order, Metropolis test drawing random() only when
// diff >= 0 (reorder.py:319), contribution refresh every 4096 accepted swaps (reorder.py:27),
// best plan on strict improvement.  The warp's lanes split the O(G) element work (delta, times,
// exponentials); every sum keeps the host's exact order (numpy's pairwise order for the LSE
// sums, sequential over experts for the refresh); lane 0 owns the random stream and the
// Metropolis draw.  Built with -fmad=false so every product / sum rounds as on the host.  exp / log are CUDA's double-precision functions (<= 1 ulp), so a plan can differ
// from the host's only where a decision hinges on the last bit of a surrogate value; the GPU
// tests compare against the reference's plans.
#include <cstdint>

#include "capi_common.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

constexpr int kSaMaxG = 32;
constexpr int kSaMaxE = 1024;
constexpr int kRefreshEvery = 4096;

typedef unsigned __int128 u128;

struct DevPCG64 {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;
  __device__ void step() {
    const u128 mult = (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
  }
  __device__ uint64_t next64() {
    step();
    const uint64_t hi = static_cast<uint64_t>(state >> 64), lo = static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    const uint64_t v = hi ^ lo;
    return (v >> rot) | (v << ((-rot) & 63));
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t n = next64();
    has32 = true;
    buf32 = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n & 0xFFFFFFFFu);
  }
  __device__ double random() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
  __device__ uint32_t bounded(uint32_t n) {
    const uint32_t rng = n - 1u;
    if (rng == 0) return 0;
    uint64_t m = static_cast<uint64_t>(next32()) * n;
    uint32_t left = static_cast<uint32_t>(m & 0xFFFFFFFFu);
    if (left < n) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % n;
      while (left < threshold) {
        m = static_cast<uint64_t>(next32()) * n;
        left = static_cast<uint32_t>(m & 0xFFFFFFFFu);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }
};

struct SaConsts {
  double comp_unit, row_units[4], beta;
};

constexpr int kSaWarps = 4;                    // chains per block (one warp each)
constexpr int kSaQ = (5 * kSaMaxG + 31) / 32;  // loads5 elements per lane

struct SaWarpSmem {
  int32_t assign[kSaMaxE];
  double tv[5 * kSaMaxG];  // per-element times of the candidate loads
  double ex[5 * kSaMaxG];  // exp(beta * (t - max)) of one LSE
};

// numpy pairwise_sum of a[0..n) (n <= 128) by the whole warp, in numpy's exact order: lanes
// 0..7 run the eight strided accumulators, the tree and the tail are evaluated identically by
// every lane.
__device__ double np_sum_warp(const double* a, int n, int lane) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  const int body = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    r = a[lane];
    for (int i = 8; i < body; i += 8) r += a[i + lane];
  }
  double rr[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) rr[j] = __shfl_sync(0xffffffffu, r, j);
  double res = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
  for (int i = body; i < n; ++i) res += a[i];
  return res;
}

// reorder._lse: m + log(sum(exp(beta * (v - m)))) / beta (max is exact in any order)
__device__ double lse_warp(const double* v, int n, double beta, double* ex, int lane) {
  double m = -INFINITY;
  for (int i = lane; i < n; i += 32) m = fmax(m, v[i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  for (int i = lane; i < n; i += 32) ex[i] = exp(beta * (v[i] - m));
  __syncwarp();
  const double s = np_sum_warp(ex, n, lane);
  __syncwarp();
  return m + log(s) / beta;
}

// One warp per chain: lanes own loads5 elements i = lane + 32q; lane 0 owns the random stream.
__global__ void __launch_bounds__(32 * kSaWarps) anneal_chains_kernel(
    const double* __restrict__ contrib, int E, int G, const int64_t* __restrict__ base, SaConsts c,
    const uint64_t* __restrict__ rng4, int nchains, int chains_per_layer, double cooling, double eps_frac,
    double term_eps, int64_t* __restrict__ best_out, int64_t* __restrict__ iters_out) {
  __shared__ SaWarpSmem smem_all[kSaWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chain = blockIdx.x * kSaWarps + warp;
  if (chain >= nchains) return;
  SaWarpSmem& sm = smem_all[warp];
  {  // layer-batched: chain c anneals layer c / chains_per_layer (its own contrib and start)
    const int64_t layer = chain / chains_per_layer;
    contrib += layer * E * G * 5 * G;
    base += layer * E;
  }
  const int n5 = 5 * G;
  auto cc = [&](int e, int host) { return contrib + (static_cast<int64_t>(e) * G + host) * n5; };
  auto unit = [&](int i) { return i < G ? c.comp_unit : c.row_units[(i - G) / G]; };
  for (int e = lane; e < E; e += 32) sm.assign[e] = static_cast<int32_t>(base[e]);
  __syncwarp();
  double l5[kSaQ], d5[kSaQ];
  auto refresh = [&]() {  // contrib[arange(E), assignment].sum(axis=0): sequential over experts
#pragma unroll
    for (int q = 0; q < kSaQ; ++q) {
      const int i = lane + 32 * q;
      double acc = 0.0;
      if (i < n5)
        for (int e = 0; e < E; ++e) acc += cc(e, sm.assign[e])[i];
      l5[q] = acc;
    }
  };
  auto smoothed = [&](const double* add) {  // add == nullptr: loads5 itself, else loads5 + add
#pragma unroll
    for (int q = 0; q < kSaQ; ++q) {
      const int i = lane + 32 * q;
      if (i < n5) sm.tv[i] = (add ? l5[q] + add[q] : l5[q]) * unit(i);
    }
    __syncwarp();
    const double a = lse_warp(sm.tv, G, c.beta, sm.ex, lane);
    const double b = lse_warp(sm.tv + G, 4 * G, c.beta, sm.ex, lane);
    return a + b;
  };
  refresh();
  DevPCG64 rng;
  const uint64_t* r4 = rng4 + 4 * static_cast<int64_t>(chain);
  rng.state = (static_cast<u128>(r4[0]) << 64) | r4[1];
  rng.inc = (static_cast<u128>(r4[2]) << 64) | r4[3];
  int64_t* best = best_out + static_cast<int64_t>(chain) * E;
  for (int e = lane; e < E; e += 32) best[e] = sm.assign[e];
  double t_cur = smoothed(nullptr);
  double theta = t_cur > 0 ? t_cur : 1.0;
  const double eps = term_eps > 0 ? term_eps : eps_frac * theta;
  double best_t = t_cur;
  int64_t iters = 0;
  int since_refresh = 0;
  if (G >= 2 && E >= 2) {
    while (theta > eps) {
      int ea = 0, eb = 0;
      if (lane == 0) {
        while (true) {
          ea = static_cast<int>(rng.bounded(static_cast<uint32_t>(E)));
          eb = static_cast<int>(rng.bounded(static_cast<uint32_t>(E)));
          if (ea != eb && sm.assign[ea] != sm.assign[eb]) break;
        }
      }
      ea = __shfl_sync(0xffffffffu, ea, 0);
      eb = __shfl_sync(0xffffffffu, eb, 0);
      const int ga = sm.assign[ea], gb = sm.assign[eb];
      const double *aga = cc(ea, ga), *agb = cc(ea, gb), *bga = cc(eb, ga), *bgb = cc(eb, gb);
#pragma unroll
      for (int q = 0; q < kSaQ; ++q) {
        const int i = lane + 32 * q;
        d5[q] = i < n5 ? agb[i] - aga[i] + bga[i] - bgb[i] : 0.0;
      }
      const double t_new = smoothed(d5);
      const double diff = t_new - t_cur;
      int accept = diff < 0;
      if (lane == 0 && !accept) accept = rng.random() < exp(-fmin(diff / theta, 745.0));
      accept = __shfl_sync(0xffffffffu, accept, 0);
      if (accept) {
#pragma unroll
        for (int q = 0; q < kSaQ; ++q) l5[q] += d5[q];
        __syncwarp();
        if (lane == 0) {
          sm.assign[ea] = gb;
          sm.assign[eb] = ga;
        }
        __syncwarp();
        if (++since_refresh >= kRefreshEvery) {
          refresh();
          since_refresh = 0;
        }
        t_cur = t_new;
        if (t_cur < best_t) {
          best_t = t_cur;
          for (int e = lane; e < E; e += 32) best[e] = sm.assign[e];
        }
      }
      theta *= cooling;
      ++iters;
    }
  }
  if (lane == 0) iters_out[chain] = iters;
}

}  // namespace mb

using namespace mb;

extern "C" int mb_anneal_chains(const double* contrib, int32_t E, int32_t G, const int64_t* base,
                                const double* consts, double beta, const uint64_t* rng, int32_t nchains,
                                int32_t chains_per_layer, double cooling, double eps_frac, double term_eps,
                                int64_t* best, int64_t* iters, void* stream) {
  MB_CHECK_ARG(contrib && base && consts && rng && best && iters, "null anneal operand");
  MB_CHECK_ARG(chains_per_layer >= 1 && nchains % chains_per_layer == 0, "nchains must be layers x chains_per_layer");
  MB_CHECK_ARG(G >= 1 && G <= kSaMaxG && E >= 1 && E <= kSaMaxE && E % G == 0 && nchains >= 0,
               "anneal dims: 1 <= G <= %d, 1 <= E <= %d, G | E", kSaMaxG, kSaMaxE);
  MB_CHECK_ARG(cooling > 0.0 && cooling < 1.0, "cooling must be in (0, 1)");
  if (nchains == 0) return MB_OK;
  SaConsts c;
  c.comp_unit = consts[0];
  for (int r = 0; r < 4; ++r) c.row_units[r] = consts[1 + r];
  c.beta = beta;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // one warp per chain, kSaWarps chains per block
  anneal_chains_kernel<<<(nchains + kSaWarps - 1) / kSaWarps, 32 * kSaWarps, 0, s>>>(
      contrib, E, G, base, c, rng, nchains, chains_per_layer, cooling, eps_frac, term_eps, best, iters);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}
