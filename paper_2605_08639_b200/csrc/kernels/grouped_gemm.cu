// Host launcher + C-ABI for the K4 tcgen05 grouped GEMM (grouped_gemm.cuh: 1-CTA 128xBN
// tiles; grouped_gemm_pair.cuh: CTA-pair 256x256 tiles, the default when the shape allows).
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "grouped_gemm_pair.cuh"
#include "capi_common.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

static int gemm_sms(int per_call);

template <bool kW, bool kAmn, bool kBmn, int BN, int kEpi>
static int launch_gemm(const GemmParams& p, cudaStream_t stream) {
  auto kern = grouped_gemm_kernel<kW, kAmn, kBmn, BN, kEpi>;
  static bool attr_set = false;
  if (!attr_set) {
    MB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<BN>::kSmemBytes));
    attr_set = true;
  }
  kern<<<device_sm_count(), 192, GemmCfg<BN>::kSmemBytes, stream>>>(p);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}

template <bool kW, bool kAmn, bool kBmn, int kEpi, bool kPair = true>
static int launch_pair(const GemmParams& p, cudaStream_t stream, int sms) {
  auto kern = kPair ? grouped_gemm_pair_kernel<kW, kAmn, kBmn, kEpi> : grouped_gemm_single_kernel<kW, kAmn, kBmn, kEpi>;
  using Cfg = PairCfg<kEpi, kPair>;
  static bool attr_set = false;
  if (!attr_set) {
    MB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    attr_set = true;
  }
  const int grid = kPair ? (gemm_sms(sms) & ~1) : gemm_sms(sms);
  static unsigned long long* prof = nullptr;
#ifdef MB_GEMM_PROFILE
  const bool profile = std::getenv("MB_GEMM_PROF") != nullptr;
#else
  const bool profile = false;
#endif
  GemmParams q = p;
  // dynamic tile scheduling: a zeroed counter per launch from a small ring (concurrent launches on
  // different streams never share one); MB_GEMM_STATIC=1 keeps the static stride (A/B)
  static int* counters = nullptr;
  static std::atomic<unsigned> next_counter{0};
  constexpr unsigned kCounters = 256;
  static const bool static_sched = [] {
    const char* e = std::getenv("MB_GEMM_STATIC");
    return e && e[0] == '1';
  }();
  if (!static_sched) {
    if (!counters) {
      int* c = nullptr;
      MB_CUDA_TRY(cudaMalloc(&c, kCounters * 32 * sizeof(int)));
      MB_CUDA_TRY(cudaMemset(c, 0, kCounters * 32 * sizeof(int)));
      counters = c;
    }
    q.tile_counter = counters + (next_counter.fetch_add(1) % kCounters) * 32;   // own 128-byte line
    MB_CUDA_TRY(cudaMemsetAsync(q.tile_counter, 0, sizeof(int), stream));
  }
  if (profile) {
    if (!prof) MB_CUDA_TRY(cudaMalloc(&prof, 8 * sizeof(unsigned long long)));
    MB_CUDA_TRY(cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), stream));
    q.prof = prof;
  }
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, stream>>>(q);
  MB_CUDA_TRY(cudaGetLastError());
  if (profile) {  // profiling only: synchronous readback, per-cluster averages in cycles
    unsigned long long h[8];
    MB_CUDA_TRY(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, stream));
    MB_CUDA_TRY(cudaStreamSynchronize(stream));
    const double n = grid / 2;
    std::fprintf(stderr, "[gemm-prof] epi=%d W=%d kernel=%.0f producer_wait_empty=%.0f mma_wait_full=%.0f "
                 "mma_wait_tempty=%.0f epi_wait_tfull=%.0f cycles/cluster\n", kEpi, (int)kW, h[4] / n, h[0] / n,
                 h[1] / n, h[2] / n, h[3] / n);
  }
  return MB_OK;
}

// SMs the persistent GEMM occupies: the per-call value (a data plane passes its own split), else
// the process default (mb_set_gemm_sms / MB_GEMM_SMS, default all).  The SMs left free run the
// dispatch / combine kernels the comm stream runs concurrently.
static int g_gemm_sms = 0;
static int gemm_sms(int per_call) {
  const int n = device_sm_count();
  int v = g_gemm_sms;
  if (const char* e = std::getenv("MB_GEMM_SMS")) v = std::atoi(e);
  if (per_call > 0) v = per_call;
  return (v >= 2 && v <= n) ? v : n;
}

static bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("MB_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace mb

using namespace mb;

extern "C" int mb_grouped_wgrad2(const void* A0, const void* B0, int32_t M0, int32_t N0, void* C0, const void* A1,
                                 const void* B1, int32_t M1, int32_t N1, void* C1, int64_t k_rows,
                                 const void* groups, const void* segs, int num_groups, int32_t gemm_sms,
                                 void* stream) {
  MB_CHECK_ARG(num_groups >= 0 && num_groups <= kMaxGroups, "num_groups %d outside [0, %d]", num_groups, kMaxGroups);
  MB_CHECK_ARG(A0 && B0 && C0 && A1 && B1 && C1 && groups && k_rows > 0, "null wgrad operand");
  MB_CHECK_ARG(M0 % 256 == 0 && N0 % 256 == 0 && M1 % 256 == 0 && N1 % 256 == 0,
               "two-problem wgrad needs M and N multiples of 256 (M0=%d N0=%d M1=%d N1=%d)", M0, N0, M1, N1);
  if (num_groups == 0) return MB_OK;
  GemmParams p{};
  p.groups = reinterpret_cast<const GemmGroup*>(groups);
  p.segs = reinterpret_cast<const GemmSeg*>(segs);
  p.num_groups = num_groups;
  p.M = M0; p.N = N0; p.M2 = M1; p.N2 = N1; p.K = 0;
  p.C = C0; p.ldc = N0; p.c_slot_stride = static_cast<int64_t>(M0) * N0;
  if (const char* dbg = std::getenv("MB_GEMM_DEBUG")) p.debug = std::atoi(dbg);
  int rc;
  // problem 0 (groups without flag 4): A0 [k_rows, M0], B0 [k_rows, N0] -> C0 [slots][M0][N0]
  if ((rc = make_tmap_bf16_2d(&p.tmA, A0, M0, k_rows, int64_t(M0) * 2, 64, 64))) return rc;
  if ((rc = make_tmap_bf16_2d(&p.tmB0, B0, N0, k_rows, int64_t(N0) * 2, 64, 64))) return rc;
  if ((rc = make_tmap_2d(&p.tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, C0, N0, static_cast<uint64_t>(M0) * kMaxGroups,
                         int64_t(N0) * 4, 32, 32)))
    return rc;
  // problem 1 (flag 4): A1 [k_rows, M1], B1 [k_rows, N1] -> C1 [slots][M1][N1]
  if ((rc = make_tmap_bf16_2d(&p.tmAh, A1, M1, k_rows, int64_t(M1) * 2, 64, 64))) return rc;
  if ((rc = make_tmap_bf16_2d(&p.tmB0h, B1, N1, k_rows, int64_t(N1) * 2, 64, 64))) return rc;
  if ((rc = make_tmap_2d(&p.tmC2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, C1, N1, static_cast<uint64_t>(M1) * kMaxGroups,
                         int64_t(N1) * 4, 32, 32)))
    return rc;
  p.tmB1 = p.tmB0;
  p.tmB1h = p.tmB0h;
  // MB_WGRAD_CTA1=1: the single-CTA (cta_group::1, 128-row tile) member of the family (A/B)
  static const bool cta1 = [] {
    const char* e = std::getenv("MB_WGRAD_CTA1");
    return e && e[0] == '1';
  }();
  if (cta1) return launch_pair<true, true, true, EPI_ACC_F32, false>(p, reinterpret_cast<cudaStream_t>(stream), gemm_sms);
  return launch_pair<true, true, true, EPI_ACC_F32>(p, reinterpret_cast<cudaStream_t>(stream), gemm_sms);
}

extern "C" int mb_set_gemm_sms(int sms) {
  MB_CHECK_ARG(sms >= 0, "sms must be >= 0 (0 = all)");
  g_gemm_sms = sms;
  return MB_OK;
}

extern "C" int mb_grouped_gemm(int mode, const void* A, int64_t a_rows, int64_t a_cols, const void* B0,
                               int64_t b0_rows, const void* B1, int64_t b1_rows, int64_t b_cols,
                               const void* groups, const void* segs, int num_groups, int M, int N, int K, void* C,
                               int64_t ldc, int64_t c_slot_stride, void* C2, int64_t ldc2, const void* aux,
                               int64_t ld_aux, const float* row_scale, float* row_partial, int32_t gemm_sms,
                               void* stream) {
  const bool force_single = (mode & 0x100) != 0 || !pair_enabled();
  // 0x200: the single-CTA member of the pair family (cta_group::1, 128 x 256 tiles) -- the tail
  // blocks of groups with an odd number of 128-row blocks run at full tensor efficiency there
  const bool tail = (mode & 0x200) != 0;
  mode &= 0xff;
  MB_CHECK_ARG(!tail || (mode != MB_GEMM_WGRAD && N % 256 == 0), "single-CTA tail launches are F-mode, N %% 256 == 0");
  MB_CHECK_ARG(num_groups >= 0 && num_groups <= kMaxGroups, "num_groups %d outside [0, %d]", num_groups, kMaxGroups);
  MB_CHECK_ARG(A && B0 && C && groups, "null operand pointer");
  MB_CHECK_ARG(a_cols % 64 == 0 && b_cols % 64 == 0, "operand widths must be multiples of 64");
  if (num_groups == 0) return MB_OK;
  if (!B1) { B1 = B0; b1_rows = b0_rows; }
  GemmParams p{};
  p.groups = reinterpret_cast<const GemmGroup*>(groups);
  p.segs = reinterpret_cast<const GemmSeg*>(segs);
  p.num_groups = num_groups;
  p.M = M; p.N = N; p.K = K;
  p.C = C; p.ldc = ldc; p.c_slot_stride = c_slot_stride;
  p.C2 = C2; p.ldc2 = ldc2; p.aux = aux; p.ld_aux = ld_aux;
  p.rscale = row_scale; p.rpart = row_partial;
  if (const char* dbg = std::getenv("MB_GEMM_DEBUG")) p.debug = std::atoi(dbg);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool pair = !force_single && N % 256 == 0 && (mode != MB_GEMM_WGRAD || M % 256 == 0);
  int rc;
  if (pair || tail || mode == MB_GEMM_DGRAD_DSWIGLU_GATED) {
    // epilogue TMA store maps: 32-row x 128-byte boxes (64 bf16 / 32 fp32 columns)
    if (mode == MB_GEMM_WGRAD) {
      MB_CHECK_ARG(c_slot_stride == static_cast<int64_t>(M) * ldc, "wgrad output must be [slots][M][ldc]");
      if ((rc = make_tmap_2d(&p.tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, C, ldc, static_cast<uint64_t>(M) * kMaxGroups,
                             ldc * 4, 32, 32)))
        return rc;
    } else {
      MB_CHECK_ARG(ldc % 64 == 0 && (!C2 || ldc2 % 64 == 0), "output widths must be multiples of 64");
      // dSwiGLU epilogues move 32-feature chunks (32 rows x 64 B boxes, 64B swizzle); the others
      // 32 rows x 128 B boxes (128B swizzle)
      const bool heavy = mode == MB_GEMM_DGRAD_DSWIGLU || mode == MB_GEMM_DGRAD_DSWIGLU_GATED;
      const uint32_t bw = heavy ? 32 : 64;
      const CUtensorMapSwizzle sz = heavy ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
      if ((rc = make_tmap_bf16_2d(&p.tmC, C, ldc, a_rows, ldc * 2, bw, 32, sz))) return rc;
      if (C2 && (rc = make_tmap_bf16_2d(&p.tmC2, C2, ldc2, a_rows, ldc2 * 2, bw, 32, sz))) return rc;
      if (aux && (rc = make_tmap_bf16_2d(&p.tmAux, aux, ld_aux, a_rows, ld_aux * 2, bw, 32, sz))) return rc;
    }
  }
  switch (mode) {
    case MB_GEMM_FWD_STORE:
    case MB_GEMM_FWD_SWIGLU: {
      MB_CHECK_ARG(N % 256 == 0 && K % 64 == 0 && a_cols == K && b_cols == K, "fwd GEMM shape N=%d K=%d", N, K);
      const uint32_t bbox = (pair || tail) ? 128 : 256;
      if ((rc = make_tmap_bf16_2d(&p.tmA, A, a_cols, a_rows, a_cols * 2, 64, 128))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB0, B0, b_cols, b0_rows, b_cols * 2, 64, bbox))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB1, B1, b_cols, b1_rows, b_cols * 2, 64, bbox))) return rc;
      if (pair) {  // tail tiles
        if ((rc = make_tmap_bf16_2d(&p.tmAh, A, a_cols, a_rows, a_cols * 2, 64, 64))) return rc;
        if ((rc = make_tmap_bf16_2d(&p.tmB0h, B0, b_cols, b0_rows, b_cols * 2, 64, 64))) return rc;
        if ((rc = make_tmap_bf16_2d(&p.tmB1h, B1, b_cols, b1_rows, b_cols * 2, 64, 64))) return rc;
      }
      if (mode == MB_GEMM_FWD_STORE)
        return tail ? launch_pair<false, false, false, EPI_STORE_BF16, false>(p, s, gemm_sms)
               : pair ? launch_pair<false, false, false, EPI_STORE_BF16>(p, s, gemm_sms)
                      : launch_gemm<false, false, false, 256, EPI_STORE_BF16>(p, s);
      MB_CHECK_ARG(C2 != nullptr, "SwiGLU epilogue needs the activation output");
      MB_CHECK_ARG(!row_scale || pair || tail, "gate-scaled SwiGLU needs the CTA-pair kernel family");
      return tail ? launch_pair<false, false, false, EPI_SWIGLU, false>(p, s, gemm_sms)
             : pair ? launch_pair<false, false, false, EPI_SWIGLU>(p, s, gemm_sms)
                    : launch_gemm<false, false, false, 256, EPI_SWIGLU>(p, s);
    }
    case MB_GEMM_DGRAD_DSWIGLU_GATED: {
      MB_CHECK_ARG((!force_single || tail) && N % 256 == 0 && K % 64 == 0 && a_cols == K && b_cols == N,
                   "gated dSwiGLU GEMM needs the CTA-pair kernel family and N %% 256 == 0 (N=%d K=%d)", N, K);
      MB_CHECK_ARG(aux && row_scale && row_partial, "gated dSwiGLU needs H, gate and partials");
      if ((rc = make_tmap_bf16_2d(&p.tmA, A, a_cols, a_rows, a_cols * 2, 64, 128))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmAh, A, a_cols, a_rows, a_cols * 2, 64, 64))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB0, B0, b_cols, b0_rows, b_cols * 2, 64, 64))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB1, B1, b_cols, b1_rows, b_cols * 2, 64, 64))) return rc;
      return tail ? launch_pair<false, false, true, EPI_DSWIGLU_GATED, false>(p, s, gemm_sms)
                  : launch_pair<false, false, true, EPI_DSWIGLU_GATED>(p, s, gemm_sms);
    }
    case MB_GEMM_DGRAD_STORE:
    case MB_GEMM_DGRAD_DSWIGLU: {
      MB_CHECK_ARG(K % 64 == 0 && a_cols == K && b_cols == N, "dgrad GEMM shape N=%d K=%d", N, K);
      if ((rc = make_tmap_bf16_2d(&p.tmA, A, a_cols, a_rows, a_cols * 2, 64, 128))) return rc;
      if (pair && (rc = make_tmap_bf16_2d(&p.tmAh, A, a_cols, a_rows, a_cols * 2, 64, 64))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB0, B0, b_cols, b0_rows, b_cols * 2, 64, 64))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB1, B1, b_cols, b1_rows, b_cols * 2, 64, 64))) return rc;
      if (mode == MB_GEMM_DGRAD_STORE) {
        MB_CHECK_ARG(N % 256 == 0, "dgrad N=%d must be a multiple of 256", N);
        return tail ? launch_pair<false, false, true, EPI_STORE_BF16, false>(p, s, gemm_sms)
               : pair ? launch_pair<false, false, true, EPI_STORE_BF16>(p, s, gemm_sms)
                      : launch_gemm<false, false, true, 256, EPI_STORE_BF16>(p, s);
      }
      MB_CHECK_ARG(N % 128 == 0 && aux != nullptr, "dSwiGLU epilogue needs N%%128==0 and H");
      return tail ? launch_pair<false, false, true, EPI_DSWIGLU, false>(p, s, gemm_sms)
             : pair ? launch_pair<false, false, true, EPI_DSWIGLU>(p, s, gemm_sms)
                    : launch_gemm<false, false, true, 128, EPI_DSWIGLU>(p, s);
    }
    case MB_GEMM_WGRAD: {
      MB_CHECK_ARG(M % 128 == 0 && N % 256 == 0 && a_cols == M && b_cols == N, "wgrad GEMM shape M=%d N=%d", M, N);
      if ((rc = make_tmap_bf16_2d(&p.tmA, A, a_cols, a_rows, a_cols * 2, 64, 64))) return rc;
      if ((rc = make_tmap_bf16_2d(&p.tmB0, B0, b_cols, b0_rows, b_cols * 2, 64, 64))) return rc;
      p.tmB1 = p.tmB0;
      return pair ? launch_pair<true, true, true, EPI_ACC_F32>(p, s, gemm_sms)
                  : launch_gemm<true, true, true, 256, EPI_ACC_F32>(p, s);
    }
    default:
      return set_error(MB_EINVAL, "unknown grouped GEMM mode %d", mode);
  }
}
