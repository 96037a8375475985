// K4: tcgen05 grouped GEMM for the expert FFN (forward, dgrad and wgrad).
//
// One persistent, warp-specialized kernel template serves every contraction of the
// SwiGLU expert FFN ("three GEMMs per expert"; 6hh' FLOP per row
// forward, costmodel.comp_time costmodel.py:161-163):
//
//   mode F (row-grouped, K fixed):  C[rows_g, N] = A[rows_g, K] . B_slot(g)          (fwd, dgrad)
//   mode W (K-grouped,  M,N fixed):  C_slot(g)[M, N] (+)= A[K_g, M]^T . B[K_g, N]     (wgrad)
//
// Roles (192 threads, 1 CTA per SM):
//   warp 0      TMA producer  (one lane): A/B tiles -> smem ring (SWIZZLE_128B)
//   warp 1      MMA issuer    (one lane): tcgen05.mma 128xBNx16 into TMEM, commit -> mbarriers;
//                                         also owns TMEM alloc/dealloc (512 columns = 2 accumulators)
//   warps 2..5  epilogue      (128 thr):  tcgen05.ld -> fused epilogue -> global
// Tiles are BM=128 x BN, BK=64. The tile list is (group, m-block, n-block) with n fastest,
// distributed round-robin over the persistent CTAs.
#pragma once
#include <cuda.h>
#include "sm100_ptx.cuh"

namespace mb {

enum GemmEpi : int {
  EPI_STORE_BF16 = 0,  // C = bf16(acc)
  EPI_SWIGLU = 1,      // C = bf16(acc) (H, gate|up blocks of BN/2), C2 = bf16(silu(g)*u)
                       //   (pair family with rscale: C2 = bf16(gate * silu(g)*u), 0 on pad rows)
  EPI_DSWIGLU = 2,     // acc = dAct; aux = H; C = dH (gate|up blocks of 2*BN)
  EPI_ACC_F32 = 3,     // C_slot (+)= acc (fp32)
  EPI_DSWIGLU_GATED = 4,  // acc = dout.W2 (unscaled); aux = H; rscale = gate per row:
                          //   C = dH of gate*acc, C2 (optional) = gate*act (feeds dW2),
                          //   rpart[row][N/64] = partial <acc, act> (dgate = <dout, Y>)
};

// Per-group descriptor (device memory, written by the dispatch-plan tables).
struct GemmGroup {
  int32_t rows;       // F: rows of the group (multiple of 128). W: total K rows (multiple of 16).
  int32_t a0;         // F: first row in A (and C). W: first token row in A and B (single segment).
  int32_t slot;       // F: weight slot index in the selected B tensor. W: output slot.
  int32_t flags;      // bit0: accumulate into C (W). bit1: B from tensor map 1 (replica slots).
  int32_t seg_begin;  // W: first entry in the segment table (K split over micro-batches)
  int32_t seg_count;  // W: number of segments; 0 means the single segment (a0, rows)
  int32_t rows_real;  // F: rows holding tokens (the rest of `rows` is padding); used by gated epilogues
  int32_t kblocks;    // W: sum over segments of ceil(rows / 64); 0 = ceil(rows / 64) (single segment)
};
// W-mode K segment: `rows` token rows (multiple of 16) starting at token row `a0`.  The last
// k-block of a segment may be partial: its TMA box reads past the segment (harmless rows of the
// next slot, or zero fill past the tensor end) and only ceil(rest / 16) K16 MMAs are issued.
struct GemmSeg {
  int32_t a0, rows;
};

constexpr int kMaxGroups = 256;
constexpr int BM = 128;
constexpr int BK = 64;

// Walks the k-blocks of a W-mode group over its K segments (one per micro-batch).
struct KWalker {
  const GemmSeg* segs;
  int next, row, left;
  __device__ __forceinline__ KWalker(const GemmGroup& gg, const GemmSeg* s)
      : segs(s), next(gg.seg_begin), row(gg.a0), left(gg.seg_count ? 0 : gg.rows) {}
  // token row of the next k-block; nk16 = K16 steps it holds (1..4)
  __device__ __forceinline__ int step(int& nk16) {
    while (left <= 0) {
      const GemmSeg g = segs[next++];
      row = g.a0;
      left = g.rows;
    }
    const int krow = row;
    nk16 = left >= BK ? BK / 16 : (left + 15) >> 4;
    row += BK;
    left -= BK;
    return krow;
  }
};

__device__ __forceinline__ int w_kblocks(const GemmGroup& gg) {
  return gg.kblocks ? gg.kblocks : (gg.rows + BK - 1) / BK;
}

struct GemmParams {
  CUtensorMap tmA;
  CUtensorMap tmB0;
  CUtensorMap tmB1;
  CUtensorMap tmC;   // epilogue TMA store maps (CTA-pair kernel): output C (box 32 rows x 128 B)
  CUtensorMap tmC2;  // secondary output C2
  CUtensorMap tmAux; // epilogue TMA load map of the auxiliary input (H for the dSwiGLU epilogues)
  CUtensorMap tmAh;  // CTA-pair tail tiles: 64-row boxes of A (K-major) and B (K-major)
  CUtensorMap tmB0h;
  CUtensorMap tmB1h;
  const GemmGroup* groups;
  const GemmSeg* segs;
  int num_groups;
  int M, N, K;          // F: N, K used; W: M, N used
  void* C;
  int64_t ldc;          // elements
  int64_t c_slot_stride;  // W: elements per output slot
  void* C2;
  int64_t ldc2;
  const void* aux;
  int64_t ld_aux;
  const float* rscale;  // per-row scale (gate) for EPI_DSWIGLU_GATED and (optional) EPI_SWIGLU
  float* rpart;         // per-row partial sums [rows][N/64] for EPI_DSWIGLU_GATED
  unsigned long long* prof;  // optional wait-cycle counters (MB_GEMM_PROF): producer/MMA/epilogue
  int* tile_counter;    // CTA-pair kernel: zeroed counter for dynamic tile scheduling (nullptr = static)
  int M2, N2;           // W mode, groups with flag 4: the second problem (A = tmAh, B = tmB0h, C = tmC2)
  int debug;            // bit0: skip the epilogue (TMEM drained, nothing stored); 128 / 256: dSwiGLU
                        // epilogue without its H loads / dH stores -- profiling only
};

template <int BN>
struct GemmCfg {
  static constexpr int kStages = (BN == 256) ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMetaBytes = 10240;  // barriers + tile starts + group table
  static constexpr int kSmemBytes = kStages * kStageBytes + kMetaBytes + 1024;  // +1024 alignment slack
};

struct TileCoord {
  int g, mb, nb, kblocks;
};

template <bool kW, int BN>
__device__ __forceinline__ TileCoord decode_tile(int t, const int* tile_start, const GemmGroup* sg, int ng,
                                                 const GemmParams& p) {
  // binary search over tile_start[0..ng]
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  TileCoord c;
  c.g = lo;
  const int local = t - tile_start[lo];
  const int n_tiles = p.N / BN;
  c.mb = local / n_tiles;
  c.nb = local - c.mb * n_tiles;
  c.kblocks = kW ? w_kblocks(sg[lo]) : (p.K / BK);
  return c;
}

template <bool kW, bool kAmn, bool kBmn, int BN, int kEpi>
__global__ void __launch_bounds__(192, 1) grouped_gemm_kernel(const __grid_constant__ GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* meta = smem + S * Cfg::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* tile_start = reinterpret_cast<int*>(meta + 256);                      // kMaxGroups+1 ints
  GemmGroup* sg = reinterpret_cast<GemmGroup*>(meta + 256 + 4 * (kMaxGroups + 8));

  const int warp = warp_id();
  const int lane = lane_id();
  const int ng = p.num_groups;

  // group table -> smem
  for (int i = threadIdx.x; i < ng; i += blockDim.x) sg[i] = p.groups[i];
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.tmA);
    tma_prefetch_desc(&p.tmB0);
    tma_prefetch_desc(&p.tmB1);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 128);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of tiles per group (warp-parallel, chunks of 32)
    const int n_tiles = p.N / BN;
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      int i = base + lane;
      int cnt = 0;
      if (i < ng) {
        const GemmGroup gg = sg[i];
        if (kW) cnt = (gg.rows > 0) ? (p.M / BM) * n_tiles : 0;
        else cnt = (gg.rows / BM) * n_tiles;
      }
      int incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (i < ng) tile_start[i] = carry + incl - cnt;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tile_start[ng] = carry;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tile_start[ng];

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const TileCoord tc = decode_tile<kW, BN>(t, tile_start, sg, ng, p);
        const GemmGroup gg = sg[tc.g];
        const CUtensorMap* tmB = (gg.flags & 2) ? &p.tmB1 : &p.tmB0;
        // W mode: walk the K segments (one per micro-batch); F mode: a single implicit segment
        KWalker kw(gg, p.segs);
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          int nk16 = BK / 16;
          const int krow = kW ? kw.step(nk16) : 0;  // W: token row of this k-block
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          if (!kAmn) {
            // A K-major: rows of the group, 64 K-columns
            tma_load_2d(a_dst, &p.tmA, &full_bar[stage], kb * BK, gg.a0 + tc.mb * BM);
          } else {
            // A MN-major (W): inner = M, outer = token rows
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a_dst + j * 8192, &p.tmA, &full_bar[stage], tc.mb * BM + j * 64, krow);
          }
          if (!kBmn) {
            tma_load_2d(b_dst, tmB, &full_bar[stage], kb * BK, gg.slot * p.N + tc.nb * BN);
          } else {
            const int row0 = kW ? krow : (gg.slot * p.K + kb * BK);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(b_dst + j * 8192, tmB, &full_bar[stage], tc.nb * BN + j * 64, row0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, kAmn ? 1u : 0u, kBmn ? 1u : 0u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
        const TileCoord tc = decode_tile<kW, BN>(t, tile_start, sg, ng, p);
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        KWalker kw(sg[tc.g], p.segs);
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          int nk16 = BK / 16;
          if (kW) kw.step(nk16);
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if (k >= nk16) break;
            const uint64_t adesc = kAmn ? make_sw128_desc(a_addr + k * 2048, 8192, 1024)
                                        : make_sw128_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bdesc = kBmn ? make_sw128_desc(b_addr + k * 2048, 8192, 1024)
                                        : make_sw128_desc(b_addr + k * 32, 16, 1024);
            umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;             // TMEM lane quarter accessible to this warp
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const TileCoord tc = decode_tile<kW, BN>(t, tile_start, sg, ng, p);
      const GemmGroup gg = sg[tc.g];
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_acc = tmem_base + lane_off + acc * 256;

      if constexpr (kEpi == EPI_STORE_BF16) {
        const int64_t row = gg.a0 + tc.mb * BM + row_in_tile;
        __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + tc.nb * BN;
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_acc + ch * 32, r);
          tmem_ld_wait();
          uint4* dst = reinterpret_cast<uint4*>(crow + ch * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            dst[v] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1])),
                                pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3])),
                                pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5])),
                                pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7])));
        }
      } else if constexpr (kEpi == EPI_SWIGLU) {
        // tile columns [0, BN/2) are gate, [BN/2, BN) are up (interleaved weight layout)
        const int64_t row = gg.a0 + tc.mb * BM + row_in_tile;
        __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + tc.nb * BN;
        __nv_bfloat16* arow = reinterpret_cast<__nv_bfloat16*>(p.C2) + row * p.ldc2 + tc.nb * (BN / 2);
#pragma unroll 1
        for (int ch = 0; ch < BN / 64; ++ch) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_acc + ch * 32, g);
          tmem_ld_32x32b_x32(t_acc + BN / 2 + ch * 32, u);
          tmem_ld_wait();
          uint4* dg = reinterpret_cast<uint4*>(hrow + ch * 32);
          uint4* du = reinterpret_cast<uint4*>(hrow + BN / 2 + ch * 32);
          uint4* da = reinterpret_cast<uint4*>(arow + ch * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint32_t pg[4], pu[4], pa[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const float g0 = __uint_as_float(g[8 * v + 2 * w]), g1 = __uint_as_float(g[8 * v + 2 * w + 1]);
              const float u0 = __uint_as_float(u[8 * v + 2 * w]), u1 = __uint_as_float(u[8 * v + 2 * w + 1]);
              pg[w] = pack_bf16x2(g0, g1);
              pu[w] = pack_bf16x2(u0, u1);
              const float a0 = g0 / (1.0f + __expf(-g0)) * u0;
              const float a1 = g1 / (1.0f + __expf(-g1)) * u1;
              pa[w] = pack_bf16x2(a0, a1);
            }
            dg[v] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
            du[v] = make_uint4(pu[0], pu[1], pu[2], pu[3]);
            da[v] = make_uint4(pa[0], pa[1], pa[2], pa[3]);
          }
        }
      } else if constexpr (kEpi == EPI_DSWIGLU) {
        // acc = dAct tile (BN columns of h'); H / dH rows hold gate|up blocks of 2*BN
        const int64_t row = gg.a0 + tc.mb * BM + row_in_tile;
        const __nv_bfloat16* hrow = reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ld_aux + tc.nb * (2 * BN);
        __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + tc.nb * (2 * BN);
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t d[32];
          tmem_ld_32x32b_x32(t_acc + ch * 32, d);
          const uint4* hg = reinterpret_cast<const uint4*>(hrow + ch * 32);
          const uint4* hu = reinterpret_cast<const uint4*>(hrow + BN + ch * 32);
          uint4 hgv[4], huv[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) { hgv[v] = hg[v]; huv[v] = hu[v]; }
          tmem_ld_wait();
          uint4* og = reinterpret_cast<uint4*>(drow + ch * 32);
          uint4* ou = reinterpret_cast<uint4*>(drow + BN + ch * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint32_t gw[4] = {hgv[v].x, hgv[v].y, hgv[v].z, hgv[v].w};
            const uint32_t uw[4] = {huv[v].x, huv[v].y, huv[v].z, huv[v].w};
            uint32_t rg[4], ru[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              float dg2[2], du2[2];
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const float gv = h2 ? bf16hi(gw[w]) : bf16lo(gw[w]);
                const float uv = h2 ? bf16hi(uw[w]) : bf16lo(uw[w]);
                const float da = __uint_as_float(d[8 * v + 2 * w + h2]);
                const float s = 1.0f / (1.0f + __expf(-gv));
                du2[h2] = da * gv * s;
                dg2[h2] = da * uv * s * (1.0f + gv * (1.0f - s));
              }
              rg[w] = pack_bf16x2(dg2[0], dg2[1]);
              ru[w] = pack_bf16x2(du2[0], du2[1]);
            }
            og[v] = make_uint4(rg[0], rg[1], rg[2], rg[3]);
            ou[v] = make_uint4(ru[0], ru[1], ru[2], ru[3]);
          }
        }
      } else {  // EPI_ACC_F32
        const bool accumulate = (gg.flags & 1) != 0;
        float* crow = reinterpret_cast<float*>(p.C) + gg.slot * p.c_slot_stride +
                      static_cast<int64_t>(tc.mb * BM + row_in_tile) * p.ldc + tc.nb * BN;
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_acc + ch * 32, r);
          float4* dst = reinterpret_cast<float4*>(crow + ch * 32);
          float4 old[8];
          if (accumulate) {
#pragma unroll
            for (int v = 0; v < 8; ++v) old[v] = dst[v];
          }
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            float4 o = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                   __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
            if (accumulate) { o.x += old[v].x; o.y += old[v].y; o.z += old[v].z; o.w += old[v].w; }
            dst[v] = o;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace mb
