// K4 (CTA-pair variant): the grouped GEMM of grouped_gemm.cuh on 2-SM clusters.
//
// A cluster of two CTAs owns a 256 x 256 output tile.  Each CTA stages its 128-row half of A
// and its 128-wide half of B per k-block (32 KB instead of 48 KB), so the shared-memory port
// of each SM carries half the B operand traffic of the 1-CTA kernel; the leader CTA issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16) reading both CTAs' smem and writing both
// CTAs' TMEM (128 lanes each), and commits multicast to both CTAs' mbarriers.  Both CTAs run
// the epilogue on their own TMEM half.  Roles per CTA as in the 1-CTA kernel:
//   warp 0 TMA producer (both CTAs; bytes complete on the leader's full barrier)
//   warp 1 MMA issuer (leader only) + TMEM allocator (both, cta_group::2)
//   warps 2..9 epilogue (both; two warps per TMEM lane quarter split the columns; release the
//              accumulator on the leader's tmem_empty barrier)
#pragma once
#include "grouped_gemm.cuh"

namespace mb {

struct PairCfg {
  static constexpr int kStages = 6;
  static constexpr int kABytes = 128 * BK * 2;  // this CTA's 128 rows of A
  static constexpr int kBBytes = 128 * BK * 2;  // this CTA's 128 columns of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMetaBytes = 10240;
  static constexpr int kSmemBytes = kStages * kStageBytes + kMetaBytes + 1024;
  static constexpr int TM = 256, TN = 256;
};

template <bool kW>
__device__ __forceinline__ TileCoord decode_tile_pair(int t, const int* tile_start, const GemmGroup* sg, int ng,
                                                      const GemmParams& p) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  TileCoord c;
  c.g = lo;
  const int local = t - tile_start[lo];
  const int n_tiles = p.N / PairCfg::TN;
  c.mb = local / n_tiles;
  c.nb = local - c.mb * n_tiles;
  c.kblocks = kW ? (sg[lo].rows / BK) : (p.K / BK);
  return c;
}

template <bool kW, bool kAmn, bool kBmn, int kEpi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ GemmParams p) {
  using Cfg = PairCfg;
  constexpr int S = Cfg::kStages;
  constexpr int TM = Cfg::TM, TN = Cfg::TN;
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
  int* tile_start = reinterpret_cast<int*>(meta + 256);
  GemmGroup* sg = reinterpret_cast<GemmGroup*>(meta + 256 + 4 * (kMaxGroups + 8));

  const int warp = warp_id();
  const int lane = lane_id();
  const int ng = p.num_groups;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

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
      mbar_init(&tempty_bar[i], 16);  // 8 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  __syncthreads();
  if (warp == 0) {
    const int n_tiles = p.N / TN;
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      int i = base + lane;
      int cnt = 0;
      if (i < ng) {
        const GemmGroup gg = sg[i];
        if (kW) cnt = (gg.rows > 0) ? (p.M / TM) * n_tiles : 0;
        else cnt = ((gg.rows + TM - 1) / TM) * n_tiles;
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tile_start[ng];

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < total_tiles; t += nclusters) {
        const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
        const GemmGroup gg = sg[tc.g];
        const CUtensorMap* tmB = (gg.flags & 2) ? &p.tmB1 : &p.tmB0;
        int seg = 0, seg_row = gg.a0, seg_left = kW ? (gg.seg_count ? 0 : gg.rows / BK) : tc.kblocks;
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          if (kW) {
            while (seg_left == 0) {
              const GemmSeg sgm = p.segs[gg.seg_begin + seg++];
              seg_row = sgm.a0;
              seg_left = sgm.rows / BK;
            }
            --seg_left;
          }
          const int krow = seg_row;
          if (kW) seg_row += BK;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t lbar = mapa_shared(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          if (!kAmn) {
            tma_load_2d_pair(a_dst, &p.tmA, lbar, kb * BK, gg.a0 + tc.mb * TM + rank * 128);
          } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d_pair(a_dst + j * 8192, &p.tmA, lbar, tc.mb * TM + rank * 128 + j * 64, krow);
          }
          if (!kBmn) {
            tma_load_2d_pair(b_dst, tmB, lbar, kb * BK, gg.slot * p.N + tc.nb * TN + rank * 128);
          } else {
            const int row0 = kW ? krow : (gg.slot * p.K + kb * BK);
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d_pair(b_dst + j * 8192, tmB, lbar, tc.nb * TN + rank * 128 + j * 64, row0);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(TM, TN, kAmn ? 1u : 0u, kBmn ? 1u : 0u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cluster; t < total_tiles; t += nclusters, ++it) {
        const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc = kAmn ? make_sw128_desc(a_addr + k * 2048, 8192, 1024)
                                        : make_sw128_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bdesc = kBmn ? make_sw128_desc(b_addr + k * 2048, 8192, 1024)
                                        : make_sw128_desc(b_addr + k * 32, 16, 1024);
            umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_pair(&empty_bar[stage], 0x3);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull_bar[acc], 0x3);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // 8 warps: warp w reads TMEM lane quarter (w & 3) and column half ch2 = (w - 2) / 4.
    const int q = warp & 3;
    const int ch2 = (warp - 2) >> 2;
    const int row_in_cta = q * 32 + lane;               // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tempty_bar[1]), 0);
    int it = 0;
    for (int t = cluster; t < total_tiles; t += nclusters, ++it) {
      const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
      const GemmGroup gg = sg[tc.g];
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_acc = tmem_base + lane_off + acc * 256;
      const int tile_row = tc.mb * TM + static_cast<int>(rank) * 128 + row_in_cta;  // row inside the group / M
      const bool valid = kW || tile_row < gg.rows;

      if constexpr (kEpi == EPI_STORE_BF16) {
        const int64_t row = gg.a0 + tile_row;
        __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + tc.nb * TN + ch2 * 128;
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + ch * 32, r);
          tmem_ld_wait();
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(crow + ch * 32);
#pragma unroll
            for (int v = 0; v < 4; ++v)
              dst[v] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1])),
                                  pack_bf16x2(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3])),
                                  pack_bf16x2(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5])),
                                  pack_bf16x2(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7])));
          }
        }
      } else if constexpr (kEpi == EPI_SWIGLU) {
        // gate columns [0,128), up columns [128,256); this warp owns gate/up columns [ch2*64, ch2*64+64)
        const int64_t row = gg.a0 + tile_row;
        __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + tc.nb * TN;
        __nv_bfloat16* arow = reinterpret_cast<__nv_bfloat16*>(p.C2) + row * p.ldc2 + tc.nb * (TN / 2);
#pragma unroll 1
        for (int cc = 0; cc < 2; ++cc) {
          const int ch = ch2 * 2 + cc;
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(t_acc + ch * 32, g);
          tmem_ld_32x32b_x32(t_acc + TN / 2 + ch * 32, u);
          tmem_ld_wait();
          if (!valid) continue;
          uint4* dg = reinterpret_cast<uint4*>(hrow + ch * 32);
          uint4* du = reinterpret_cast<uint4*>(hrow + TN / 2 + ch * 32);
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
              pa[w] = pack_bf16x2(__fdividef(g0, 1.0f + __expf(-g0)) * u0, __fdividef(g1, 1.0f + __expf(-g1)) * u1);
            }
            dg[v] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
            du[v] = make_uint4(pu[0], pu[1], pu[2], pu[3]);
            da[v] = make_uint4(pa[0], pa[1], pa[2], pa[3]);
          }
        }
      } else if constexpr (kEpi == EPI_DSWIGLU) {
        // dAct columns [ch2*128, ch2*128+128) = interleave block (2*nb + ch2): gate|up 256 cols of H/dH
        const int64_t row = gg.a0 + tile_row;
        const int64_t hcol = static_cast<int64_t>(tc.nb * 2 + ch2) * 256;
        const __nv_bfloat16* hrow = reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ld_aux + hcol;
        __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + hcol;
        uint4 hgv[4], huv[4], ngv[4], nuv[4];
        if (valid) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            hgv[v] = reinterpret_cast<const uint4*>(hrow)[v];
            huv[v] = reinterpret_cast<const uint4*>(hrow + 128)[v];
          }
        }
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t d[32];
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + ch * 32, d);
          if (valid && ch + 1 < 4) {  // prefetch H of the next chunk
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              ngv[v] = reinterpret_cast<const uint4*>(hrow + (ch + 1) * 32)[v];
              nuv[v] = reinterpret_cast<const uint4*>(hrow + 128 + (ch + 1) * 32)[v];
            }
          }
          tmem_ld_wait();
          if (valid) {
            uint4* og = reinterpret_cast<uint4*>(drow + ch * 32);
            uint4* ou = reinterpret_cast<uint4*>(drow + 128 + ch * 32);
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
                  const float dav = __uint_as_float(d[8 * v + 2 * w + h2]);
                  const float s = __fdividef(1.0f, 1.0f + __expf(-gv));
                  du2[h2] = dav * gv * s;
                  dg2[h2] = dav * uv * s * (1.0f + gv * (1.0f - s));
                }
                rg[w] = pack_bf16x2(dg2[0], dg2[1]);
                ru[w] = pack_bf16x2(du2[0], du2[1]);
              }
              og[v] = make_uint4(rg[0], rg[1], rg[2], rg[3]);
              ou[v] = make_uint4(ru[0], ru[1], ru[2], ru[3]);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) { hgv[v] = ngv[v]; huv[v] = nuv[v]; }
          }
        }
      } else if constexpr (kEpi == EPI_DSWIGLU_GATED) {
        // acc = dout.W2 (the dout rows arrive unscaled); block b = 2*nb + ch2 of H / dH / Act
        const int64_t row = gg.a0 + tile_row;
        const bool real = valid && tile_row < gg.rows_real;
        const int blk = tc.nb * 2 + ch2;
        const int64_t hcol = static_cast<int64_t>(blk) * 256;
        const __nv_bfloat16* hrow = reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ld_aux + hcol;
        __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + hcol;
        __nv_bfloat16* arow = reinterpret_cast<__nv_bfloat16*>(p.C2) + row * p.ldc2 + static_cast<int64_t>(blk) * 128;
        const float gate = real ? p.rscale[row] : 0.0f;
        float part = 0.0f;
        uint4 hgv[4], huv[4], ngv[4], nuv[4];
        if (real) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            hgv[v] = reinterpret_cast<const uint4*>(hrow)[v];
            huv[v] = reinterpret_cast<const uint4*>(hrow + 128)[v];
          }
        }
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t d[32];
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + ch * 32, d);
          if (real && ch + 1 < 4) {
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              ngv[v] = reinterpret_cast<const uint4*>(hrow + (ch + 1) * 32)[v];
              nuv[v] = reinterpret_cast<const uint4*>(hrow + 128 + (ch + 1) * 32)[v];
            }
          }
          tmem_ld_wait();
          if (!valid) continue;
          uint4* og = reinterpret_cast<uint4*>(drow + ch * 32);
          uint4* ou = reinterpret_cast<uint4*>(drow + 128 + ch * 32);
          uint4* oa = reinterpret_cast<uint4*>(arow + ch * 32);
          if (!real) {  // padding rows: zero dH and gate*act so the wgrad sees exact zeros
#pragma unroll
            for (int v = 0; v < 4; ++v) og[v] = ou[v] = oa[v] = make_uint4(0, 0, 0, 0);
            continue;
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const uint32_t gw[4] = {hgv[v].x, hgv[v].y, hgv[v].z, hgv[v].w};
            const uint32_t uw[4] = {huv[v].x, huv[v].y, huv[v].z, huv[v].w};
            uint32_t rg[4], ru[4], ra[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              float dg2[2], du2[2], ag2[2];
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const float gv = h2 ? bf16hi(gw[w]) : bf16lo(gw[w]);
                const float uv = h2 ? bf16hi(uw[w]) : bf16lo(uw[w]);
                const float raw = __uint_as_float(d[8 * v + 2 * w + h2]);
                const float s = __fdividef(1.0f, 1.0f + __expf(-gv));
                const float act = gv * s * uv;
                part += raw * act;
                const float dav = gate * raw;
                du2[h2] = dav * gv * s;
                dg2[h2] = dav * uv * s * (1.0f + gv * (1.0f - s));
                ag2[h2] = gate * act;
              }
              rg[w] = pack_bf16x2(dg2[0], dg2[1]);
              ru[w] = pack_bf16x2(du2[0], du2[1]);
              ra[w] = pack_bf16x2(ag2[0], ag2[1]);
            }
            og[v] = make_uint4(rg[0], rg[1], rg[2], rg[3]);
            ou[v] = make_uint4(ru[0], ru[1], ru[2], ru[3]);
            oa[v] = make_uint4(ra[0], ra[1], ra[2], ra[3]);
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) { hgv[v] = ngv[v]; huv[v] = nuv[v]; }
        }
        if (real) p.rpart[row * (p.N / 128) + blk] = part;
      } else {  // EPI_ACC_F32
        const bool accumulate = (gg.flags & 1) != 0;
        float* crow = reinterpret_cast<float*>(p.C) + gg.slot * p.c_slot_stride +
                      static_cast<int64_t>(tile_row) * p.ldc + tc.nb * TN + ch2 * 128;
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + ch * 32, r);
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
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty_bar[acc]);
        else mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace mb
