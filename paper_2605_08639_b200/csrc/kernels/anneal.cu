// GPU-side planning: the simulated-annealing chains of the inter-batch expert
// reordering planner, one GPU thread per seed.
//
// Device restatement of reorder._run_chain (reorder.py:299-326) as the host planner runs it
// (csrc/planner/reorder.cpp run_chain): swap proposals from numpy's PCG64 stream
// (Generator.integers(0, E) = 32-bit Lemire on the buffered next_uint32; Generator.random() =
// (next_uint64 >> 11) * 2^-53), O(G) swap delta on the shared contribution tensor, LSE_beta
// surrogate with numpy's pairwise summation order, Metropolis test drawing random() only when
// diff >= 0 (reorder.py:319), contribution refresh every 4096 accepted swaps (reorder.py:27),
// best plan on strict improvement.  Built with -fmad=false so every product / sum rounds as on
// the host.  exp / log are CUDA's double-precision functions (<= 1 ulp), so a plan can differ
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

// numpy pairwise_sum (n <= 4 * kSaMaxG = 128 here: no recursion)
__device__ double np_sum_dev(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

__device__ double vmax_dev(const double* a, int n) {
  double m = a[0];
  for (int i = 1; i < n; ++i)
    if (a[i] > m || isnan(a[i])) m = a[i];
  return m;
}

__device__ double lse_dev(const double* v, int n, double beta, double* scratch) {
  const double m = vmax_dev(v, n);
  for (int i = 0; i < n; ++i) scratch[i] = exp(beta * (v[i] - m));
  return m + log(np_sum_dev(scratch, n)) / beta;
}

struct SaConsts {
  double comp_unit, row_units[4], beta;
};

struct SaChain {
  const double* contrib;  // [E][G][5][G]
  int E, G;
  SaConsts c;
  int32_t assign[kSaMaxE];
  double loads5[5 * kSaMaxG], comp_t[kSaMaxG], rows_t[4 * kSaMaxG], scratch[4 * kSaMaxG];
  int since_refresh = 0;

  __device__ const double* cc(int e, int host) const { return contrib + (static_cast<int64_t>(e) * G + host) * 5 * G; }
  __device__ void refresh() {
    for (int i = 0; i < 5 * G; ++i) loads5[i] = 0.0;
    for (int e = 0; e < E; ++e) {
      const double* p = cc(e, assign[e]);
      for (int i = 0; i < 5 * G; ++i) loads5[i] += p[i];
    }
    since_refresh = 0;
  }
  __device__ double smoothed(const double* l5) {
    for (int g = 0; g < G; ++g) comp_t[g] = l5[g] * c.comp_unit;
    for (int r = 0; r < 4; ++r)
      for (int g = 0; g < G; ++g) rows_t[r * G + g] = l5[(r + 1) * G + g] * c.row_units[r];
    return lse_dev(comp_t, G, c.beta, scratch) + lse_dev(rows_t, 4 * G, c.beta, scratch);
  }
};

__global__ void __launch_bounds__(32) anneal_chains_kernel(const double* __restrict__ contrib, int E, int G,
                                                           const int64_t* __restrict__ base, SaConsts consts,
                                                           const uint64_t* __restrict__ rng4, int nchains,
                                                           double cooling, double eps_frac, double term_eps,
                                                           int64_t* __restrict__ best_out,
                                                           int64_t* __restrict__ iters_out) {
  const int chain = blockIdx.x * blockDim.x + threadIdx.x;
  if (chain >= nchains) return;
  SaChain st;
  st.contrib = contrib;
  st.E = E;
  st.G = G;
  st.c = consts;
  for (int e = 0; e < E; ++e) st.assign[e] = static_cast<int32_t>(base[e]);
  st.refresh();
  DevPCG64 rng;
  const uint64_t* r4 = rng4 + 4 * static_cast<int64_t>(chain);
  rng.state = (static_cast<u128>(r4[0]) << 64) | r4[1];
  rng.inc = (static_cast<u128>(r4[2]) << 64) | r4[3];
  int64_t* best = best_out + static_cast<int64_t>(chain) * E;
  for (int e = 0; e < E; ++e) best[e] = st.assign[e];
  double t_cur = st.smoothed(st.loads5);
  double theta = t_cur > 0 ? t_cur : 1.0;
  const double eps = term_eps > 0 ? term_eps : eps_frac * theta;
  double best_t = t_cur;
  int64_t iters = 0;
  if (G >= 2 && E >= 2) {
    double delta[5 * kSaMaxG], cand[5 * kSaMaxG];
    while (theta > eps) {
      int ea, eb;
      while (true) {
        ea = static_cast<int>(rng.bounded(static_cast<uint32_t>(E)));
        eb = static_cast<int>(rng.bounded(static_cast<uint32_t>(E)));
        if (ea != eb && st.assign[ea] != st.assign[eb]) break;
      }
      const int ga = st.assign[ea], gb = st.assign[eb];
      const double *aga = st.cc(ea, ga), *agb = st.cc(ea, gb), *bga = st.cc(eb, ga), *bgb = st.cc(eb, gb);
      for (int i = 0; i < 5 * G; ++i) {
        delta[i] = agb[i] - aga[i] + bga[i] - bgb[i];
        cand[i] = st.loads5[i] + delta[i];
      }
      const double t_new = st.smoothed(cand);
      const double diff = t_new - t_cur;
      bool accept = diff < 0;
      if (!accept) accept = rng.random() < exp(-fmin(diff / theta, 745.0));
      if (accept) {
        for (int i = 0; i < 5 * G; ++i) st.loads5[i] += delta[i];
        st.assign[ea] = gb;
        st.assign[eb] = ga;
        if (++st.since_refresh >= kRefreshEvery) st.refresh();
        t_cur = t_new;
        if (t_cur < best_t) {
          best_t = t_cur;
          for (int e = 0; e < E; ++e) best[e] = st.assign[e];
        }
      }
      theta *= cooling;
      ++iters;
    }
  }
  iters_out[chain] = iters;
}

}  // namespace mb

using namespace mb;

extern "C" int mb_anneal_chains(const double* contrib, int32_t E, int32_t G, const int64_t* base,
                                const double* consts, double beta, const uint64_t* rng, int32_t nchains,
                                double cooling, double eps_frac, double term_eps, int64_t* best, int64_t* iters,
                                void* stream) {
  MB_CHECK_ARG(contrib && base && consts && rng && best && iters, "null anneal operand");
  MB_CHECK_ARG(G >= 1 && G <= kSaMaxG && E >= 1 && E <= kSaMaxE && E % G == 0 && nchains >= 0,
               "anneal dims: 1 <= G <= %d, 1 <= E <= %d, G | E", kSaMaxG, kSaMaxE);
  MB_CHECK_ARG(cooling > 0.0 && cooling < 1.0, "cooling must be in (0, 1)");
  if (nchains == 0) return MB_OK;
  SaConsts c;
  c.comp_unit = consts[0];
  for (int r = 0; r < 4; ++r) c.row_units[r] = consts[1 + r];
  c.beta = beta;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // one thread per chain; per-chain state lives in local memory (L1-resident)
  anneal_chains_kernel<<<(nchains + 31) / 32, 32, 0, s>>>(contrib, E, G, base, c, rng, nchains, cooling, eps_frac,
                                                          term_eps, best, iters);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}
