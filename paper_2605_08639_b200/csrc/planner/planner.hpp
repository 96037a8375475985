// Internal declarations of the host planners (C-ABI wrappers live in capi.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "common.hpp"
#include "costmodel.hpp"

namespace mbp {

// ReplicaPlacement (replicate.py:48-69): home per expert plus replica GPUs in copy order;
// `order` keeps the dict insertion order of experts that have replicas.
struct Placement {
  std::vector<int64_t> home;
  std::vector<int> order;
  std::vector<std::vector<int>> reps;  // [E]
  explicit Placement(const int64_t* h = nullptr, int E = 0) : home(h, h + E), reps(E) {}
  void add(int e, int g) {
    if (reps[e].empty()) order.push_back(e);
    reps[e].push_back(g);
  }
  std::vector<int> copies(int e) const {
    std::vector<int> c{int(home[e])};
    c.insert(c.end(), reps[e].begin(), reps[e].end());
    return c;
  }
  std::vector<int> slot_usage(int G) const {
    std::vector<int> u(G, 0);
    for (int e : order)
      for (int g : reps[e]) ++u[g];
    return u;
  }
  std::vector<int> serving(int gpu) const {
    const int E = int(home.size());
    std::vector<int> out;
    for (int e = 0; e < E; ++e) {
      bool on = home[e] == gpu;
      for (int g : reps[e]) on = on || g == gpu;
      if (on) out.push_back(e);
    }
    return out;
  }
};

// SplitPlan (replicate.py:72-87): fractions[e] is [G][1+R_e], insertion order in `order`.
struct SplitFr {
  std::vector<int> order;
  std::vector<std::vector<double>> frac;  // [E]
  explicit SplitFr(int E = 0) : frac(E) {}
  std::vector<SplitEntry> to_map(const Placement& p) const {
    std::vector<SplitEntry> m;
    for (int e : order) {
      SplitEntry s;
      s.e = e;
      s.gpus = p.copies(e);
      s.frac = frac[e];
      m.push_back(std::move(s));
    }
    return m;
  }
};

void static_plan(int E, int G, int64_t* out);
void lpt_initial(const double* x, int G, int E, int64_t* out);
int anneal_samples(const Topo& t, int E, int L, int MB, int S, const double* counts, const int32_t* mb_of,
                   const int64_t* source, const double* tokens, const int64_t* plans, int64_t h, int64_t hp,
                   const Hw& hw, const uint64_t* seeds, int nseeds, double cooling, double eps_frac, double term_eps,
                   double beta, double band, int greedy_only, int threads, int64_t* out);
int anneal_reorder(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, const uint64_t* seeds,
                   int nseeds, double cooling, double eps_frac, double term_eps, double beta, const int64_t* extra,
                   int nextra, int threads, int64_t* out, int64_t* iters_total);
int anneal_prepare(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, double beta,
                   const uint64_t* seeds, int nseeds, int64_t* base_out, double* contrib_out, double* consts_out,
                   uint64_t* rng_out);
int anneal_select(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, double beta,
                  const int64_t* cands, int ncand, int64_t* out);

std::vector<int> candidate_gpus(int e, const std::vector<int64_t>& home, const Topo& t);
int greedy_replicate(const double* x, int E, const int64_t* home, const Topo& t, int64_t h, int64_t hp, const Hw& hw,
                     int slots, Placement& pl, SplitFr& sp, double* objective);
int solve_token_split(const double* x, int E, const Placement& pl, const Topo& t, int64_t h, int64_t hp, const Hw& hw,
                      SplitFr& sp);
void round_split(const double* x, int G, int E, const Placement& pl, const SplitFr& sp, std::vector<std::vector<int64_t>>& counts);
void eplb_replication(const double* loads, int E, const int64_t* home, const Topo& t, int slots, int max_rep,
                      Placement& pl);

struct DispatchOut {
  int32_t* route_tab;   // [G][E][maxc][4] {cum_end, dst_gpu, dst_row_base, 0}
  int32_t* ncopies;     // [E]
  int32_t* slot_tab;    // [G][max_slots][4] {row_begin, rows_real, rows_pad, expert}
  int32_t* slot_w;      // [G][max_slots][2] {weight slot, is_replica}
  int32_t* nslots;      // [G]
  int64_t* total_rows;  // [G]
  int64_t* flow;        // [G][G]
};
int dispatch_plan(int G, int E, const int64_t* x, const int64_t* home, const std::vector<std::vector<int>>& reps,
                  const std::vector<std::vector<int64_t>>& counts, int pad, int maxc, int max_slots,
                  const DispatchOut& o);

}  // namespace mbp
