// K4 (CTA-pair variant): the grouped GEMM of grouped_gemm.cuh on 2-SM clusters.
//
// A cluster of two CTAs owns a 256 x 256 output tile.  Each CTA stages its 128-row half of A
// and its 128-wide half of B per k-block (32 KB instead of 48 KB), so the shared-memory port
// of each SM carries half the B operand traffic of the 1-CTA kernel; the leader CTA issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16) reading both CTAs' smem and writing both
// CTAs' TMEM (128 lanes each), and commits multicast to both CTAs' mbarriers.
//
// Epilogue: every output leaves through TMA.  An epilogue warp drains 32 TMEM lanes x 32 or
// 64 columns, applies the fused math, writes one 32-row x 128-byte box into a 128B-swizzled
// staging buffer (double-buffered per warp) and one lane issues cp.async.bulk.tensor (store,
// or reduce-add for the fp32 gradient accumulation, so the L2 does the read-modify-write).
// Row-per-thread global stores were the measured bottleneck of every variant (the mainloop
// alone runs at 1.4-1.9 PFLOP/s).
//
// Roles per CTA:
//   warp 0     TMA producer (both CTAs; bytes complete on the leader's full barrier)
//   warp 1     MMA issuer (leader only) + TMEM allocator (both, cta_group::2)
//   warps 2..9 epilogue (both; two warps per TMEM lane quarter split the columns; release the
//              accumulator on the leader's tmem_empty barrier)
#pragma once
#include "grouped_gemm.cuh"

namespace mb {

struct PairTile {
  static constexpr int TM = 256, TN = 256;
  static constexpr int kBoxBytes = 32 * 128;  // one 32-row x 128-byte TMA box
};

#ifndef MB_PAIR_EPI_WARPS
#define MB_PAIR_EPI_WARPS 8     // two per TMEM lane quarter (4 measured 3-25% slower beside the comm kernels)
#endif
#ifndef MB_PAIR_STAGES
#define MB_PAIR_STAGES 6        // operand ring depth (the MMA warp starved 9-19% of the time with 4-5)
#endif
// Shared memory: MB_PAIR_STAGES x 32 KB operand stages, one 4 KB staging area per epilogue warp
// (light epilogues: one 32-row x 128-byte output box; dSwiGLU epilogues: two 32-row x 64-byte
// boxes -- 32 features of gate and of up -- that carry H in and dH / gate*act out), and a small
// meta block (barriers + tile starts; the group table is read from global memory).
#ifndef MB_PAIR_LIGHT_BOXES
#define MB_PAIR_LIGHT_BOXES 1
#endif
#ifndef MB_W_EVICT_LAST
#define MB_W_EVICT_LAST 0       // wgrad operand loads with an L2 evict_last hint (A/B)
#endif
#ifndef MB_HEAVY_DBUF
#define MB_HEAVY_DBUF 0
#endif
#ifndef MB_SINGLE_STAGES
#define MB_SINGLE_STAGES 4      // single-CTA variant: 48 KB stages (A 128 rows + all 256 columns of B)
#endif
// kPair = false: the single-CTA (cta_group::1) variant for the 128-row tail blocks of odd groups:
// a 128 x 256 tile per CTA at full tensor-core efficiency (M=128 N=256 MMAs), the same roles,
// epilogues and tile scheduler, no cluster.
template <int kEpi, bool kPair = true>
struct PairCfg : PairTile {
  static constexpr bool kHeavy = kEpi == EPI_DSWIGLU || kEpi == EPI_DSWIGLU_GATED;
  static constexpr int kEpiWarps = MB_PAIR_EPI_WARPS;
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr int TM = kPair ? 256 : 128;  // tile rows (per cluster)
  // MB_PAIR_LIGHT_BOXES=2: light epilogues double-buffer their output box (one operand stage less)
  static constexpr int kOutBoxes = (kPair && !kHeavy) ? MB_PAIR_LIGHT_BOXES : 1;
  // MB_HEAVY_DBUF: the dSwiGLU epilogues of the pair kernel double-buffer their H boxes (one
  // operand stage less), so the next 32-feature chunk's H loads while this one computes
  static constexpr bool kHDbuf = kPair && kHeavy && MB_HEAVY_DBUF;
  static constexpr int kStages = kPair ? MB_PAIR_STAGES - (kOutBoxes - 1) - (kHDbuf ? 1 : 0) : MB_SINGLE_STAGES;
  static constexpr int kABytes = 128 * BK * 2;  // this CTA's 128 rows of A
  static constexpr int kBBytes = (kPair ? 128 : 256) * BK * 2;  // this CTA's columns of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kWarpBoxes = kHDbuf ? 2 : kOutBoxes;   // 4 KB staging boxes per epilogue warp
  static constexpr int kStagingBytes = kEpiWarps * kBoxBytes * kWarpBoxes;
  static constexpr int kMetaBytes = 512 + 4 * (kMaxGroups + 8);
  static constexpr int kSmemBytes = kStages * kStageBytes + kStagingBytes + kMetaBytes + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static_assert(2 * kStages * 8 + 4 * 8 + 4 <= 256 && 256 + 8 * kEpiWarps <= 320, "meta layout");
};

// Tile scheduling: the leader CTA's producer hands every tile id of its cluster, in order, to all
// roles of both CTAs through a small ring in shared memory (ids written into both CTAs' rings,
// full barriers completed with cluster-scope releases; the consumers -- leader MMA warp, both
// CTAs' epilogue warps and the peer's producer -- free a slot on the leader's empty barrier).
// Each cluster's first tile is its index; later ids come from a global atomic counter (dynamic:
// a cluster that started late, or whose tiles were cheap, takes fewer tiles -- the GEMM adapts
// to SMs the comm kernels hold) or, without a counter, from the static stride.
constexpr int kTileRing = 8;
constexpr int kTileConsumers = 2 + 2 * MB_PAIR_EPI_WARPS;

template <bool kW>
__device__ __forceinline__ TileCoord decode_tile_pair(int t, const int* tile_start, const GemmGroup* __restrict__ sg,
                                                      int ng, const GemmParams& p) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  TileCoord c;
  c.g = lo;
  const int local = t - tile_start[lo];
  const int n_tiles = (kW && (sg[lo].flags & 4) ? p.N2 : p.N) / PairTile::TN;
  c.mb = local / n_tiles;
  c.nb = local - c.mb * n_tiles;
  c.kblocks = kW ? w_kblocks(sg[lo]) : (p.K / BK);
  return c;
}

// F-mode tail tile (pair kernel): the last 128 padded rows of a group whose row count is an odd multiple of 128.
// It runs as M=128 cta_group::2 MMAs (64 rows per CTA) issued twice with N=128 (the two 128-wide
// column blocks of the 256-wide tile), so no tensor-core work is spent on a half-empty pair tile.
// TMEM layout of such an MMA (the "2x2" datapath layout): lanes 0-63 hold columns [0, 64) and
// lanes 64-127 hold columns [64, 128) of the CTA's 64 rows; block j lands at TMEM column j*64.
__device__ __forceinline__ bool half_tile(const GemmGroup& gg, const TileCoord& tc, int debug) {
  return gg.rows - tc.mb * PairTile::TM <= 128 && !(debug & 16);  // debug 16: full tiles only (A/B)
}

// Per-warp double-buffered TMA store staging: 2 boxes of 32 rows x 128 B, 128B swizzle.
template <int kBufs>
struct BoxStager {
  uint8_t* base;
  int buf = 0;
  int lane;
  int debug = 0;
  // write this lane's 128-byte row of the next box (words lo[0..15] then hi[0..15]) and issue the store
  template <bool kReduce>
  __device__ __forceinline__ void put(const uint32_t (&w)[32], const CUtensorMap* map, int32_t c0, int32_t c1) {
    put2<kReduce>(w, w + 16, map, c0, c1);
  }
  template <bool kReduce>
  __device__ __forceinline__ void put2(const uint32_t* lo, const uint32_t* hi, const CUtensorMap* map, int32_t c0,
                                       int32_t c1) {
    uint8_t* b = base + buf * PairTile::kBoxBytes;
    if (lane == 0) bulk_wait_read<kBufs - 1>();  // the store that last used this buffer has read it
    __syncwarp();
    uint4* row = reinterpret_cast<uint4*>(b + lane * 128);
    if (!(debug & 4)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) row[j ^ (lane & 7)] = make_uint4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        row[(4 + j) ^ (lane & 7)] = make_uint4(hi[4 * j], hi[4 * j + 1], hi[4 * j + 2], hi[4 * j + 3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (debug & 2) return;
    if (lane == 0) {
      const uint64_t pol = (debug & 8) ? l2_evict_last_policy() : l2_evict_first_policy();
      if (kReduce) tma_reduce_add_2d(map, b, c0, c1, pol);
      else tma_store_2d(map, b, c0, c1, pol);
      bulk_commit();
    }
    if (kBufs > 1) buf ^= 1;
  }
};

__device__ __forceinline__ void pack_bf16_words(const uint32_t (&a)[32], const uint32_t (&b)[32], uint32_t (&w)[32]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = pack_bf16x2(__uint_as_float(a[2 * i]), __uint_as_float(a[2 * i + 1]));
#pragma unroll
  for (int i = 0; i < 16; ++i) w[16 + i] = pack_bf16x2(__uint_as_float(b[2 * i]), __uint_as_float(b[2 * i + 1]));
}

template <bool kW, bool kAmn, bool kBmn, int kEpi, bool kPair>
__device__ __forceinline__ void grouped_gemm_body(const GemmParams& p) {
  using Cfg = PairCfg<kEpi, kPair>;
  constexpr int S = Cfg::kStages;
  constexpr int TM = Cfg::TM, TN = Cfg::TN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* sStage = smem + S * Cfg::kStageBytes;
  uint8_t* meta = sStage + Cfg::kStagingBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* hbar_base = reinterpret_cast<uint64_t*>(meta + 256);  // one per epilogue warp (H tile loads)
  int* ring = reinterpret_cast<int*>(meta + 320);                   // tile ids [kTileRing]
  uint64_t* tr_full = reinterpret_cast<uint64_t*>(meta + 352);      // [kTileRing], count 1
  uint64_t* tr_empty = reinterpret_cast<uint64_t*>(meta + 416);     // [kTileRing] (leader), kTileConsumers
  int* tile_start = reinterpret_cast<int*>(meta + 512);
  const GemmGroup* __restrict__ sg = p.groups;   // group table: global memory (L1-cached), read per tile

  const int warp = warp_id();
  const int lane = lane_id();
  const int ng = p.num_groups;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int cluster = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int nclusters = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.tmA);
    tma_prefetch_desc(&p.tmB0);
    tma_prefetch_desc(&p.tmB1);
    tma_prefetch_desc(&p.tmC);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], (kPair ? 2 : 1) * Cfg::kEpiWarps);  // every epilogue warp of the cluster
    }
    for (int i = 0; i < Cfg::kEpiWarps; ++i) mbar_init(&hbar_base[i], 1);
    for (int i = 0; i < kTileRing; ++i) {
      mbar_init(&tr_full[i], 1);
      mbar_init(&tr_empty[i], kPair ? kTileConsumers : 1 + Cfg::kEpiWarps);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) {
    if constexpr (kPair) tmem_alloc_pair<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  __syncthreads();
  if (warp == 0) {
    const int n_tiles = p.N / TN;
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      int i = base + lane;
      int cnt = 0;
      if (i < ng) {
        const GemmGroup gg = sg[i];
        if (kW) cnt = (gg.rows > 0) ? ((gg.flags & 4) ? (p.M2 / TM) * (p.N2 / TN) : (p.M / TM) * n_tiles) : 0;
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
  if constexpr (kPair) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tile_start[ng];
  // i-th tile id of this cluster (consumer side); the caller's lane 0 frees the slot
  auto take_tile = [&](int i) -> int {
    const int slot = i % kTileRing;
    if constexpr (kPair) mbar_wait_cluster(&tr_full[slot], (i / kTileRing) & 1);
    else mbar_wait(&tr_full[slot], (i / kTileRing) & 1);
    const int t = *reinterpret_cast<volatile int*>(&ring[slot]);
    __syncwarp();
    if (lane == 0) {
      if (leader) mbar_arrive(&tr_empty[slot]);
      else mbar_arrive_cluster(mapa_shared(smem_u32(&tr_empty[slot]), 0));
    }
    return t;
  };
#ifdef MB_GEMM_PROFILE
  constexpr bool kProf = true;   // build with -DMB_GEMM_PROFILE: per-role wait-cycle counters
#else
  constexpr bool kProf = false;
#endif
  long long w_empty = 0, w_full = 0, w_tempty = 0, w_tfull = 0;
  const long long t_kernel0 = kProf ? clock64() : 0;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int t_next = cluster;
      for (int i = 0;; ++i) {
        int t;
        if (leader) {   // publish the i-th tile id to both CTAs
          t = t_next;
          const int slot = i % kTileRing;
          mbar_wait(&tr_empty[slot], ((i / kTileRing) & 1) ^ 1);
          if constexpr (kPair) {
            st_shared_cluster_u32(mapa_shared(smem_u32(&ring[slot]), 0), static_cast<uint32_t>(t));
            st_shared_cluster_u32(mapa_shared(smem_u32(&ring[slot]), 1), static_cast<uint32_t>(t));
            mbar_arrive_cluster(mapa_shared(smem_u32(&tr_full[slot]), 0));
            mbar_arrive_cluster(mapa_shared(smem_u32(&tr_full[slot]), 1));
          } else {
            *reinterpret_cast<volatile int*>(&ring[slot]) = t;
            mbar_arrive(&tr_full[slot]);   // release.cta: orders the id store for this CTA's roles
          }
          if (t >= total_tiles) break;
          t_next = p.tile_counter ? nclusters + atomicAdd(p.tile_counter, 1) : t + nclusters;  // fetched early
        } else {
          const int slot = i % kTileRing;
          mbar_wait_cluster(&tr_full[slot], (i / kTileRing) & 1);
          t = *reinterpret_cast<volatile int*>(&ring[slot]);
          mbar_arrive_cluster(mapa_shared(smem_u32(&tr_empty[slot]), 0));
          if (t >= total_tiles) break;
        }
        const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
        const GemmGroup gg = sg[tc.g];
        const CUtensorMap* tmB = (gg.flags & 2) ? &p.tmB1 : ((kW && (gg.flags & 4)) ? &p.tmB0h : &p.tmB0);
        const CUtensorMap* tmBh = (gg.flags & 2) ? &p.tmB1h : &p.tmB0h;
        const bool half = kPair && !kW && half_tile(gg, tc, p.debug);
        const int bytes = !kPair ? Cfg::kStageBytes : half ? 2 * (Cfg::kABytes / 2 + Cfg::kBBytes) : 2 * Cfg::kStageBytes;
        KWalker kw(gg, p.segs);
        // wgrad operands are re-read by every tile of the expert's other dimension: keep them in L2
        const uint64_t w_policy = (kW && MB_W_EVICT_LAST) ? l2_evict_last_policy() : 0;
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          int nk16 = BK / 16;
          const int krow = kW ? kw.step(nk16) : 0;
          {
            const long long t0 = kProf ? clock64() : 0;
            mbar_wait(&empty_bar[stage], phase ^ 1);
            if (kProf) w_empty += clock64() - t0;
          }
          const uint32_t lbar = kPair ? mapa_shared(smem_u32(&full_bar[stage]), 0) : smem_u32(&full_bar[stage]);
          if (p.debug & 32) {  // profiling only: no operand loads (MMAs read stale smem)
            if (leader) mbar_arrive(&full_bar[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
            continue;
          }
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          // pair: bytes complete on the leader's barrier (cta_group::2 form); single: own barrier
          auto load2d = [&](void* dst, const CUtensorMap* map, int32_t c0, int32_t c1) {
            if constexpr (kPair && kW && MB_W_EVICT_LAST) tma_load_2d_pair_hint(dst, map, lbar, c0, c1, w_policy);
            else if constexpr (kPair) tma_load_2d_pair(dst, map, lbar, c0, c1);
            else tma_load_2d(dst, map, &full_bar[stage], c0, c1);
          };
          if (!kAmn) {
            if (half) load2d(a_dst, &p.tmAh, kb * BK, gg.a0 + tc.mb * TM + rank * 64);
            else load2d(a_dst, &p.tmA, (p.debug & 64) ? 0 : kb * BK,
                        (p.debug & 64) ? rank * 128 : gg.a0 + tc.mb * TM + rank * 128);
          } else {
            const CUtensorMap* tmA_w = (kW && (gg.flags & 4)) ? &p.tmAh : &p.tmA;   // W: second problem
#pragma unroll
            for (int j = 0; j < 2; ++j) load2d(a_dst + j * 8192, tmA_w, tc.mb * TM + rank * 128 + j * 64, krow);
          }
          if (!kBmn) {
            if (half) {
              // this CTA's 64-column halves of both 128-column blocks
#pragma unroll
              for (int j = 0; j < 2; ++j)
                load2d(b_dst + j * 8192, tmBh, kb * BK, gg.slot * p.N + tc.nb * TN + j * 128 + rank * 64);
            } else {
              // pair: this CTA's 128 columns; single: all 256 (two 128-row boxes)
#pragma unroll
              for (int j = 0; j < (kPair ? 1 : 2); ++j)
                load2d(b_dst + j * 16384, tmB, kb * BK, gg.slot * p.N + tc.nb * TN + rank * 128 + j * 128);
            }
          } else {
            const int row0 = (p.debug & 64) ? 0 : (kW ? krow : (gg.slot * p.K + kb * BK));
#pragma unroll
            for (int j = 0; j < (kPair ? 2 : 4); ++j) {
              const int col = (p.debug & 64) ? rank * 128 + j * 64
                              : half ? tc.nb * TN + j * 128 + rank * 64 : tc.nb * TN + rank * 128 + j * 64;
              load2d(b_dst + j * 8192, tmB, col, row0);
            }
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
      constexpr uint32_t idesc_h = make_idesc_bf16(128, 128, kAmn ? 1u : 0u, kBmn ? 1u : 0u);
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int slot = it % kTileRing;
        if constexpr (kPair) mbar_wait_cluster(&tr_full[slot], (it / kTileRing) & 1);
        else mbar_wait(&tr_full[slot], (it / kTileRing) & 1);
        const int t = *reinterpret_cast<volatile int*>(&ring[slot]);
        mbar_arrive(&tr_empty[slot]);
        if (t >= total_tiles) break;
        const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
        const int acc = it & 1;
        {
          const long long t0 = kProf ? clock64() : 0;
          mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
          if (kProf) w_tempty += clock64() - t0;
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        const GemmGroup gg = sg[tc.g];
        const bool half = kPair && !kW && half_tile(gg, tc, p.debug);
        KWalker kw(gg, p.segs);
        for (int kb = 0; kb < tc.kblocks; ++kb) {
          int nk16 = BK / 16;
          if (kW) kw.step(nk16);
          {
            const long long t0 = kProf ? clock64() : 0;
            mbar_wait(&full_bar[stage], phase);
            if (kProf) w_full += clock64() - t0;
          }
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if (k >= nk16) break;
            const uint32_t accum = (kb | k) != 0 ? 1u : 0u;
            const uint64_t adesc = kAmn ? make_sw128_desc(a_addr + k * 2048, 8192, 1024)
                                        : make_sw128_desc(a_addr + k * 32, 16, 1024);
            if (!half) {
              const uint64_t bdesc = kBmn ? make_sw128_desc(b_addr + k * 2048, 8192, 1024)
                                          : make_sw128_desc(b_addr + k * 32, 16, 1024);
              if constexpr (kPair) umma_bf16_pair(d_tmem, adesc, bdesc, idesc, accum);
              else umma_bf16(d_tmem, adesc, bdesc, idesc, accum);
            } else {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint64_t bdesc = kBmn ? make_sw128_desc(b_addr + j * 8192 + k * 2048, 8192, 1024)
                                            : make_sw128_desc(b_addr + j * 8192 + k * 32, 16, 1024);
                umma_bf16_pair(d_tmem + j * 64, adesc, bdesc, idesc_h, accum);
              }
            }
          }
          if constexpr (kPair) umma_commit_pair(&empty_bar[stage], 0x3);
          else umma_commit(&empty_bar[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if constexpr (kPair) umma_commit_pair(&tfull_bar[acc], 0x3);
        else umma_commit(&tfull_bar[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // warp w reads TMEM lane quarter (w & 3); with 8 epilogue warps column half ch2 = (w - 2) / 4,
    // with 4 each warp makes two passes, one per column half
    constexpr int kPasses = 8 / Cfg::kEpiWarps;
    const int q = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t tempty_leader0 = kPair ? mapa_shared(smem_u32(&tempty_bar[0]), 0) : 0u;
    const uint32_t tempty_leader1 = kPair ? mapa_shared(smem_u32(&tempty_bar[1]), 0) : 0u;
    BoxStager<Cfg::kOutBoxes> st{sStage + (warp - 2) * Cfg::kWarpBoxes * Cfg::kBoxBytes, 0, lane, p.debug};
    uint64_t* hbar = hbar_base + (warp - 2);
    uint32_t hphase = 0;
    for (int it = 0;; ++it) {
      const int t = take_tile(it);
      if (t >= total_tiles) break;
      const TileCoord tc = decode_tile_pair<kW>(t, tile_start, sg, ng, p);
      const GemmGroup gg = sg[tc.g];
      const int acc = it & 1;
      {
        const long long t0 = kProf ? clock64() : 0;
        mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
        if (kProf) w_tfull += clock64() - t0;
      }
      tc_fence_after();
      const uint32_t t_acc = tmem_base + lane_off + acc * 256;
      bool released = false;
      // hand the accumulator back to the MMA warp as soon as this warp holds all its columns
      auto release_now = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty_bar[acc]);
          else mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
        }
        released = true;
      };
#pragma unroll 1
      for (int pass = 0; pass < kPasses; ++pass) {
      const int ch2 = kPasses == 1 ? (warp - 2) >> 2 : pass;
      auto release = [&]() {
        if (pass == kPasses - 1) release_now();
      };
      // full tile: this warp owns rows q*32.. of the CTA's 128 and columns [ch2*128, +128);
      // tail tile (half_tile): rows (q&1)*32.. of the CTA's 64; lane group q>>1 holds columns
      // [(q>>1)*64, +64) of both 128-column blocks; the ch2 = 1 warps have nothing to do
      const bool half = kPair && !kW && half_tile(gg, tc, p.debug);
      const int warp_row0 = half ? tc.mb * TM + static_cast<int>(rank) * 64 + (q & 1) * 32
                                 : tc.mb * TM + static_cast<int>(rank) * 128 + q * 32;
      const int tile_row = warp_row0 + lane;
      // 64-column segment s of this warp: TMEM column and output column (within the 256-wide tile)
      auto tcol = [&](int s) { return half ? s * 64 : ch2 * 128 + s * 64; };
      auto ocol = [&](int s) { return half ? s * 128 + (q >> 1) * 64 : ch2 * 128 + s * 64; };
      // tail tiles: the two warps of a lane quarter split the two 64-column segments (store and
      // dSwiGLU epilogues); the SwiGLU epilogue needs gate and up of a feature in one warp, so
      // there the ch2 = 1 warps idle
      const bool valid = (kW || warp_row0 < gg.rows) && !(half && ch2 && kEpi == EPI_SWIGLU);
      const int32_t out_row0 = kW ? gg.slot * ((gg.flags & 4) ? p.M2 : p.M) + warp_row0 : gg.a0 + warp_row0;

      if (p.debug & 1) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_acc + ch2 * 128, r);
        tmem_ld_wait();
        if (r[0] == 0x7fffffffu && r[31] == 0x7fffffffu) p.rpart[0] = 0.0f;  // keep the load alive
      } else if (valid) {
        if constexpr (kEpi == EPI_STORE_BF16) {
          uint32_t a0[32], a1[32], b0[32], b1[32], w[32];
          if (half) {  // this warp's one segment
            tmem_ld_32x32b_x32(t_acc + tcol(ch2), a0);
            tmem_ld_32x32b_x32(t_acc + tcol(ch2) + 32, a1);
            tmem_ld_wait();
            release();
            pack_bf16_words(a0, a1, w);
            st.template put<false>(w, &p.tmC, tc.nb * TN + ocol(ch2), out_row0);
          } else {
            tmem_ld_32x32b_x32(t_acc + tcol(0), a0);
            tmem_ld_32x32b_x32(t_acc + tcol(0) + 32, a1);
            tmem_ld_32x32b_x32(t_acc + tcol(1), b0);
            tmem_ld_32x32b_x32(t_acc + tcol(1) + 32, b1);
            tmem_ld_wait();
            release();
            pack_bf16_words(a0, a1, w);
            st.template put<false>(w, &p.tmC, tc.nb * TN + ocol(0), out_row0);
            pack_bf16_words(b0, b1, w);
            st.template put<false>(w, &p.tmC, tc.nb * TN + ocol(1), out_row0);
          }
        } else if constexpr (kEpi == EPI_SWIGLU) {
          // gate columns [0,128), up columns [128,256); this warp owns gate/up features [f0, +64)
          // (tail tile: gate block at TMEM [0,64), up block at [64,128))
          const int f0 = half ? (q >> 1) * 64 : ch2 * 64;
          const int tg = half ? 0 : ch2 * 64, tu = half ? 64 : 128 + ch2 * 64;
          uint32_t g0[32], g1[32], u0[32], u1[32], w[32];
          tmem_ld_32x32b_x32(t_acc + tg, g0);
          tmem_ld_32x32b_x32(t_acc + tg + 32, g1);
          tmem_ld_32x32b_x32(t_acc + tu, u0);
          tmem_ld_32x32b_x32(t_acc + tu + 32, u1);
          tmem_ld_wait();
          release();
          // pack H in place (word i of each half from values 2i, 2i+1); the activation is
          // computed from the bf16-rounded H, exactly what the backward pass recomputes
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            g0[i] = pack_bf16x2(__uint_as_float(g0[2 * i]), __uint_as_float(g0[2 * i + 1]));
            u0[i] = pack_bf16x2(__uint_as_float(u0[2 * i]), __uint_as_float(u0[2 * i + 1]));
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            g1[i] = pack_bf16x2(__uint_as_float(g1[2 * i]), __uint_as_float(g1[2 * i + 1]));
            u1[i] = pack_bf16x2(__uint_as_float(u1[2 * i]), __uint_as_float(u1[2 * i + 1]));
          }
          st.template put2<false>(g0, g1, &p.tmC, tc.nb * TN + f0, out_row0);
          st.template put2<false>(u0, u1, &p.tmC, tc.nb * TN + 128 + f0, out_row0);
          // with rscale: the activation leaves pre-scaled by the row's gate (0 on pad rows), so the
          // down GEMM yields gate*Y for the combine and dW2 reads gate*act without a rewrite
          const float gs = p.rscale ? (tile_row < gg.rows_real ? p.rscale[gg.a0 + tile_row] : 0.0f) : 1.0f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t gw = i < 16 ? g0[i] : g1[i - 16];
            const uint32_t uw = i < 16 ? u0[i] : u1[i - 16];
            const float a0 = bf16lo(gw), a1 = bf16hi(gw), b0 = bf16lo(uw), b1 = bf16hi(uw);
            w[i] = pack_bf16x2(gs * (__fdividef(a0, 1.0f + __expf(-a0)) * b0),
                               gs * (__fdividef(a1, 1.0f + __expf(-a1)) * b1));
          }
          st.template put<false>(w, &p.tmC2, tc.nb * (TN / 2) + f0, out_row0);
        } else if constexpr (kEpi == EPI_DSWIGLU || kEpi == EPI_DSWIGLU_GATED) {
          // dAct columns of 64-column segment hh = features [fo, +64) of interleave block blk,
          // processed as two 32-feature chunks: the chunk's H gate / up columns come in through
          // TMA into the warp's two 2 KB staging boxes (32 rows x 64 B, 64B swizzle), are read
          // back row per lane, and the same boxes then carry dH (gate / up) and gate*act out.
          constexpr bool kGated = kEpi == EPI_DSWIGLU_GATED;
          constexpr int kHalfBox = PairTile::kBoxBytes / 2;
          const int64_t row = gg.a0 + tile_row;
          const bool real = !kGated || tile_row < gg.rows_real;
          const float gate = kGated ? (real ? p.rscale[row] : 0.0f) : 1.0f;
          const int sw = (lane >> 1) & 3;   // 64B swizzle: 16-byte chunk j of row r sits at j ^ ((r >> 1) & 3)
          // the warp's chunks: i = 0 .. n-1 -> segment hh = hh0 + i / 2, chunk c = i % 2
          const int hh0 = half ? ch2 : 0;
          const int n = half ? 2 : 4;
          auto chunk_cols = [&](int i, int& blk, int& f) {
            const int hh = hh0 + (i >> 1);
            blk = tc.nb * 2 + ocol(hh) / 128;
            f = ocol(hh) % 128 + (i & 1) * 32;   // first feature of the chunk within the block
          };
          // box set of chunk i: with kHDbuf two sets alternate, so chunk i+1's H loads while chunk
          // i computes; otherwise one set (load, wait, compute, store per chunk)
          auto set_base = [&](int i) { return st.base + (Cfg::kHDbuf ? (i & 1) * PairTile::kBoxBytes : 0); };
          auto issue_h = [&](int i) {   // lane 0: H gate / up columns of chunk i into its box set
            int blk, f;
            chunk_cols(i, blk, f);
            uint8_t* b = set_base(i);
            bulk_wait_read<0>();  // earlier stores have drained that set
            if (p.debug & 128) {  // profiling only: no H loads (the boxes' stale contents are used)
              mbar_arrive(hbar);
              return;
            }
            mbar_arrive_expect_tx(hbar, PairTile::kBoxBytes);
            tma_load_2d(b, &p.tmAux, hbar, blk * 256 + f, out_row0);
            tma_load_2d(b + kHalfBox, &p.tmAux, hbar, blk * 256 + 128 + f, out_row0);
          };
          if (lane == 0) issue_h(0);
          float part = 0.0f;
#pragma unroll 1
          for (int i = 0; i < n; ++i) {
            int blk, f;
            chunk_cols(i, blk, f);
            const int hh = hh0 + (i >> 1);
            uint8_t* bufA = set_base(i);
            uint8_t* bufB = bufA + kHalfBox;
            uint4* rowA = reinterpret_cast<uint4*>(bufA + lane * 64);
            uint4* rowB = reinterpret_cast<uint4*>(bufB + lane * 64);
            if (!Cfg::kHDbuf && i > 0 && lane == 0) issue_h(i);
            uint32_t d[32];
            tmem_ld_32x32b_x32(t_acc + tcol(hh) + (i & 1) * 32, d);
            mbar_wait(hbar, hphase);
            hphase ^= 1;
            uint4 hg[4], hu[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              hg[v] = rowA[v ^ sw];
              hu[v] = rowB[v ^ sw];
            }
            tmem_ld_wait();
            __syncwarp();  // every lane holds its H row before the boxes are rewritten
            if (Cfg::kHDbuf && i + 1 < n && lane == 0) issue_h(i + 1);  // only one load in flight per barrier
            uint32_t wa[16];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const uint32_t gw[4] = {hg[v].x, hg[v].y, hg[v].z, hg[v].w};
              const uint32_t uw[4] = {hu[v].x, hu[v].y, hu[v].z, hu[v].w};
              uint32_t og[4], ou[4];
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                float dg2[2], du2[2], ag2[2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                  const int col = v * 8 + x * 2 + h2;  // 0..31 within this chunk
                  const float gv = h2 ? bf16hi(gw[x]) : bf16lo(gw[x]);
                  const float uv = h2 ? bf16hi(uw[x]) : bf16lo(uw[x]);
                  const float raw = __uint_as_float(d[col]);
                  const float s = __fdividef(1.0f, 1.0f + __expf(-gv));
                  const float act = gv * s * uv;
                  if (kGated) part += raw * act;
                  const float dav = gate * raw;
                  du2[h2] = real ? dav * gv * s : 0.0f;
                  dg2[h2] = real ? dav * uv * s * (1.0f + gv * (1.0f - s)) : 0.0f;
                  ag2[h2] = real ? gate * act : 0.0f;
                }
                og[x] = pack_bf16x2(dg2[0], dg2[1]);
                ou[x] = pack_bf16x2(du2[0], du2[1]);
                wa[v * 4 + x] = pack_bf16x2(ag2[0], ag2[1]);
              }
              rowA[v ^ sw] = make_uint4(og[0], og[1], og[2], og[3]);
              rowB[v ^ sw] = make_uint4(ou[0], ou[1], ou[2], ou[3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !(p.debug & 256)) {  // (debug 256, profiling only: no dH stores)
              const uint64_t pol = l2_evict_first_policy();
              tma_store_2d(&p.tmC, bufA, blk * 256 + f, out_row0, pol);
              tma_store_2d(&p.tmC, bufB, blk * 256 + 128 + f, out_row0, pol);
              bulk_commit();
            }
            if (kGated && p.C2) {  // gate*act over Act (unless the forward wrote it pre-scaled)
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 4; ++j) rowA[j ^ sw] = make_uint4(wa[4 * j], wa[4 * j + 1], wa[4 * j + 2], wa[4 * j + 3]);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&p.tmC2, bufA, blk * 128 + f, out_row0, l2_evict_first_policy());
                bulk_commit();
              }
            }
            // partial <dAct, act> over the segment's 64 features: rpart[row][N/64]
            if (i & 1) {
              if (kGated && real) p.rpart[row * (p.N / 64) + blk * 2 + (f - 32) / 64] = part;
              part = 0.0f;
            }
          }
        } else {  // EPI_ACC_F32: fp32 boxes of 32 columns, reduce-add into the accumulator or store
          const bool accumulate = (gg.flags & 1) != 0;
          const CUtensorMap* tmCw = (gg.flags & 4) ? &p.tmC2 : &p.tmC;   // second wgrad problem
          uint32_t r0[32], r1[32], r2[32], r3[32];
          tmem_ld_32x32b_x32(t_acc + ch2 * 128, r0);
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + 32, r1);
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + 64, r2);
          tmem_ld_32x32b_x32(t_acc + ch2 * 128 + 96, r3);
          tmem_ld_wait();
          release();
          const int32_t c0 = tc.nb * TN + ch2 * 128;
          if (accumulate) {
            st.template put<true>(r0, tmCw, c0, out_row0);
            st.template put<true>(r1, tmCw, c0 + 32, out_row0);
            st.template put<true>(r2, tmCw, c0 + 64, out_row0);
            st.template put<true>(r3, tmCw, c0 + 96, out_row0);
          } else {
            st.template put<false>(r0, tmCw, c0, out_row0);
            st.template put<false>(r1, tmCw, c0 + 32, out_row0);
            st.template put<false>(r2, tmCw, c0 + 64, out_row0);
            st.template put<false>(r3, tmCw, c0 + 96, out_row0);
          }
        }
      }
      }  // passes
      if (!released) release_now();
    }
    if (lane == 0) bulk_wait<0>();  // every TMA store of this warp has completed
    __syncwarp();
  }
  if (kProf && p.prof && lane == 0 && leader) {
    if (warp == 0) { atomicAdd(&p.prof[0], (unsigned long long)w_empty); atomicAdd(&p.prof[4], (unsigned long long)(clock64() - t_kernel0)); }
    if (warp == 1) { atomicAdd(&p.prof[1], (unsigned long long)w_full); atomicAdd(&p.prof[2], (unsigned long long)w_tempty); }
    if (warp == 2) atomicAdd(&p.prof[3], (unsigned long long)w_tfull);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

template <bool kW, bool kAmn, bool kBmn, int kEpi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<kEpi>::kThreads, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ GemmParams p) {
  grouped_gemm_body<kW, kAmn, kBmn, kEpi, true>(p);
}

template <bool kW, bool kAmn, bool kBmn, int kEpi>
__global__ void __launch_bounds__(PairCfg<kEpi, false>::kThreads, 1)
    grouped_gemm_single_kernel(const __grid_constant__ GemmParams p) {
  grouped_gemm_body<kW, kAmn, kBmn, kEpi, false>(p);
}

}  // namespace mb
