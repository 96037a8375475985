// On-device per-micro-batch dispatch tables: the integer split of every replicated expert's
// tokens over its copies (replicate.round_split, replicate.py:501-525) and, from it, every GPU's
// receive layout, the route table each source uses to place its (token, choice) rows and the
// executed flow matrix (costmodel.flow_matrix, costmodel.py:91-108, with integer splits).
// Bit-identical to the host planner's mbp_round_split + mbp_dispatch_plan
// (csrc/planner/replicate.cpp, dispatch_plan.cpp): the same fp64 products, floors and
// half-to-even rounding, the same stable largest-remainder order and the same slot order
// (home experts ascending, then replicated experts ascending; sources ascending inside a slot).
// One block per micro-batch; the split fractions come from the token-split LP on the host.
#include "capi_common.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

struct TabArgs {
  int G, E, n_rep, pad, maxc, max_slots;
  const int32_t* x;           // [G][E] routing counts of this micro-batch
  const int32_t* home;        // [E]
  const int32_t* rep_experts; // [n_rep] replicated experts in placement order
  const int32_t* rep_ptr;     // [n_rep + 1] CSR into rep_gpus (copy order)
  const int32_t* rep_gpus;
  const double* frac;         // per replicated expert: [G][1 + R_e] fractions, concatenated
  int64_t* counts;            // out: per replicated expert: [G][1 + R_e] integer split
  int32_t* route_tab;         // out: [G][E][maxc][4] {cum_end, dst_gpu, dst_row_base, 0}
  int32_t* ncopies;           // out: [E]
  int32_t* slot_tab;          // out: [G][max_slots][4] {row_begin, rows_real, rows_pad, expert}
  int32_t* slot_w;            // out: [G][max_slots][2] {weight slot, replica}
  int32_t* nslots;            // out: [G]
  int64_t* total_rows;        // out: [G]
  int64_t* flow;              // out: [G][G]
  int32_t* error;             // out: nonzero on inconsistent input
};

__device__ __forceinline__ int64_t tab_cnt(const TabArgs& a, const int* rep_of, int j, int e, int c) {
  const int i = rep_of[e];
  if (i < 0) return c == 0 ? a.x[j * a.E + e] : 0;
  const int k = 1 + a.rep_ptr[i + 1] - a.rep_ptr[i];
  return a.counts[static_cast<int64_t>(a.G) * (a.rep_ptr[i] + i) + j * k + c];
}

__device__ __forceinline__ int tab_copy_gpu(const TabArgs& a, const int* rep_of, int e, int c) {
  return c == 0 ? a.home[e] : a.rep_gpus[a.rep_ptr[rep_of[e]] + c - 1];
}

__device__ __forceinline__ int tab_ncop(const TabArgs& a, const int* rep_of, int e) {
  const int i = rep_of[e];
  return i < 0 ? 1 : 1 + a.rep_ptr[i + 1] - a.rep_ptr[i];
}

__global__ void __launch_bounds__(1024) dispatch_tables_kernel(const TabArgs a) {
  extern __shared__ int rep_of[];   // [E]: index into the replica list, -1 = single copy
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int G = a.G, E = a.E;
  for (int e = tid; e < E; e += nt) rep_of[e] = -1;
  __syncthreads();
  for (int i = tid; i < a.n_rep; i += nt) rep_of[a.rep_experts[i]] = i;
  __syncthreads();
  // ---- round_split per (replicated expert, source): largest remainder
  for (int p = tid; p < a.n_rep * G; p += nt) {
    const int i = p / G, j = p - i * G;
    const int e = a.rep_experts[i];
    const int k = 1 + a.rep_ptr[i + 1] - a.rep_ptr[i];
    const int64_t off = static_cast<int64_t>(G) * (a.rep_ptr[i] + i) + j * k;
    const double target = static_cast<double>(a.x[j * E + e]);
    double raw[16], rem[16];
    int64_t fl[16];
    int64_t fsum = 0;
    for (int c = 0; c < k; ++c) {
      raw[c] = __dmul_rn(a.frac[off + c], target);
      fl[c] = target > 0 ? static_cast<int64_t>(floor(raw[c])) : 0;
      fsum += fl[c];
    }
    if (target > 0) {
      const int64_t shortfall = static_cast<int64_t>(rint(__dsub_rn(target, static_cast<double>(fsum))));
      if (shortfall > 0) {
        for (int c = 0; c < k; ++c) rem[c] = __dsub_rn(raw[c], static_cast<double>(fl[c]));
        // stable order by descending remainder; the first `shortfall` copies get one more token
        for (int64_t q = 0; q < shortfall && q < k; ++q) {
          int best = -1;
          for (int c = 0; c < k; ++c) {
            if (rem[c] < -1.0) continue;   // chosen in an earlier round
            if (best < 0 || -rem[c] < -rem[best]) best = c;   // strict: ties keep the lower copy index
          }
          fl[best] += 1;
          rem[best] = -2.0;   // mark taken (remainders lie in [0, 1))
        }
      }
    }
    int64_t s = 0;
    for (int c = 0; c < k; ++c) {
      a.counts[off + c] = fl[c];
      s += fl[c];
      if (fl[c] < 0) atomicOr(a.error, 1);
    }
    if (s != a.x[j * E + e]) atomicOr(a.error, 1);
  }
  // ---- clear the outputs
  for (int64_t q = tid; q < static_cast<int64_t>(G) * E * a.maxc * 4; q += nt) a.route_tab[q] = 0;
  for (int q = tid; q < G * a.max_slots * 4; q += nt) a.slot_tab[q] = 0;
  for (int q = tid; q < G * a.max_slots * 2; q += nt) a.slot_w[q] = 0;
  for (int e = tid; e < E; e += nt) {
    const int k = tab_ncop(a, rep_of, e);
    a.ncopies[e] = k;
    if (k > a.maxc) atomicOr(a.error, 2);
  }
  __syncthreads();
  // ---- receive layout of GPU d: one warp per destination, lanes over experts, warp scans
  for (int d = warp; d < G; d += nw) {
    int ns = 0, nhome = 0, nrep = 0;
    int64_t row = 0;
    for (int pass = 0; pass < 2; ++pass) {          // 0: home experts, 1: replicas
      for (int e0 = 0; e0 < E; e0 += 32) {
        const int e = e0 + lane;
        int c = -1;
        if (e < E) {
          if (pass == 0) {
            if (a.home[e] == d) c = 0;
          } else {
            const int k = tab_ncop(a, rep_of, e);
            for (int cc = 1; cc < k; ++cc)
              if (tab_copy_gpu(a, rep_of, e, cc) == d) c = cc;
          }
        }
        int64_t real = 0;
        if (c >= 0)
          for (int j = 0; j < G; ++j) real += tab_cnt(a, rep_of, j, e, c);
        const int64_t padded = c >= 0 ? (real + a.pad - 1) / a.pad * a.pad : 0;
        const unsigned flags = __ballot_sync(0xffffffffu, c >= 0);
        const int before = __popc(flags & ((1u << lane) - 1u));
        int64_t incl = padded;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int64_t v = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += v;
        }
        if (c >= 0) {
          const int slot = ns + before;
          const int64_t begin = row + incl - padded;
          if (slot < a.max_slots) {
            int32_t* st = a.slot_tab + (static_cast<int64_t>(d) * a.max_slots + slot) * 4;
            st[0] = static_cast<int32_t>(begin);
            st[1] = static_cast<int32_t>(real);
            st[2] = static_cast<int32_t>(padded);
            st[3] = e;
            int32_t* sw = a.slot_w + (static_cast<int64_t>(d) * a.max_slots + slot) * 2;
            sw[0] = (pass == 0 ? nhome : nrep) + before;
            sw[1] = pass;
          } else {
            atomicOr(a.error, 4);
          }
          int64_t src_base = begin;
          for (int j = 0; j < G; ++j) {
            int32_t* rt = a.route_tab + ((static_cast<int64_t>(j) * E + e) * a.maxc + c) * 4;
            rt[1] = d;
            rt[2] = static_cast<int32_t>(src_base);
            src_base += tab_cnt(a, rep_of, j, e, c);
          }
        }
        const int cnt = __popc(flags);
        ns += cnt;
        if (pass == 0) nhome += cnt; else nrep += cnt;
        row += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) {
      a.nslots[d] = ns;
      a.total_rows[d] = row;
      if (row > 0x7fffffffLL) atomicOr(a.error, 8);
    }
  }
  // ---- executed flow and cumulative split ends per (source, expert)
  for (int p = tid; p < G * G; p += nt) {
    const int j = p / G, d = p - j * G;
    int64_t f = 0;
    for (int e = 0; e < E; ++e) {
      const int k = tab_ncop(a, rep_of, e);
      for (int c = 0; c < k; ++c)
        if (tab_copy_gpu(a, rep_of, e, c) == d) f += tab_cnt(a, rep_of, j, e, c);
    }
    a.flow[p] = f;
  }
  __syncthreads();   // the layout loop wrote route_tab[..][1..2]; cum_end goes into [0]
  for (int p = tid; p < G * E; p += nt) {
    const int j = p / E, e = p - j * E;
    const int k = tab_ncop(a, rep_of, e);
    int64_t cum = 0;
    for (int c = 0; c < k && c < a.maxc; ++c) {
      cum += tab_cnt(a, rep_of, j, e, c);
      a.route_tab[((static_cast<int64_t>(j) * E + e) * a.maxc + c) * 4] = static_cast<int32_t>(cum);
    }
  }
}

}  // namespace mb

using namespace mb;

extern "C" int mb_dispatch_tables(int32_t G, int32_t E, const int32_t* x, const int32_t* home, int32_t n_rep,
                                  const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus,
                                  const double* frac, int32_t pad, int32_t maxc, int32_t max_slots, int64_t* counts,
                                  int32_t* route_tab, int32_t* ncopies, int32_t* slot_tab, int32_t* slot_w,
                                  int32_t* nslots, int64_t* total_rows, int64_t* flow, int32_t* error, void* stream) {
  MB_CHECK_ARG(G >= 1 && G <= 32 && E >= 1 && E <= 4096 && pad >= 1 && maxc >= 1 && maxc <= 16 && max_slots >= 1 &&
                   n_rep >= 0 && n_rep <= E,
               "bad dispatch table dimensions (G=%d E=%d maxc=%d)", G, E, maxc);
  MB_CHECK_ARG(x && home && route_tab && ncopies && slot_tab && slot_w && nslots && total_rows && flow && error &&
                   (n_rep == 0 || (rep_experts && rep_ptr && rep_gpus && frac && counts)),
               "null dispatch table operand");
  TabArgs a{G, E, n_rep, pad, maxc, max_slots, x, home, rep_experts, rep_ptr, rep_gpus, frac, counts, route_tab,
            ncopies, slot_tab, slot_w, nslots, total_rows, flow, error};
  dispatch_tables_kernel<<<1, 1024, static_cast<size_t>(E) * sizeof(int), reinterpret_cast<cudaStream_t>(stream)>>>(a);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}
