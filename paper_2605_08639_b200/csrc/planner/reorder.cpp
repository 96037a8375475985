// Inter-batch expert reordering: static blocks, LPT greedy and swap-based simulated
// annealing.  C++ restatement of moebalance.reorder (reorder.py:92-362); the chains of one
// layer run in parallel (OpenMP, one chain per thread, results gathered in seed order), the
// paper's "one thread per (layer, seed)" solver.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

#include "costmodel.hpp"
#include "pcg64.hpp"
#include "planner.hpp"

namespace mbp {

void static_plan(int E, int G, int64_t* out) {
  const int M = E / G;
  for (int e = 0; e < E; ++e) out[e] = e / M;
}

// lpt_initial (reorder.py:265-288)
void lpt_initial(const double* x, int G, int E, int64_t* out) {
  const int cap = E / G;
  std::vector<double> loads(E, 0.0);
  for (int e = 0; e < E; ++e) {
    double s = 0.0;
    for (int j = 0; j < G; ++j) s += x[size_t(j) * E + e];
    loads[e] = s;
  }
  std::vector<int> order(E);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return -loads[a] < -loads[b]; });
  std::vector<double> gload(G, 0.0);
  std::vector<int> gcount(G, 0);
  for (int e : order) {
    int target = -1;
    for (int g = 0; g < G; ++g) {
      if (gcount[g] >= cap) continue;
      if (target < 0 || gload[g] < gload[target]) target = g;
    }
    out[e] = target;
    gload[target] += loads[e];
    gcount[target] += 1;
  }
}

// _dest_contrib (reorder.py:92-125): (5,G) load of serving per-source masses `col` at `host`.
static void dest_contrib(const double* col, int host, const Topo& t, double* out) {
  const int G = t.G;
  std::fill(out, out + 5 * G, 0.0);
  std::vector<double> nv(G), sr(G), cr(G), bins(G);
  out[0 * G + host] = np_sum(col, G);
  for (int j = 0; j < G; ++j) {
    const uint8_t c = t.c(j, host);
    nv[j] = c == NV ? col[j] : 0.0;
    sr[j] = c == SR ? col[j] : 0.0;
    cr[j] = c == CR ? col[j] : 0.0;
  }
  const double nv_sum = np_sum(nv.data(), G), sr_sum = np_sum(sr.data(), G), cr_sum = np_sum(cr.data(), G);
  double* o1 = out + 1 * G;
  double* o2 = out + 2 * G;
  double* o3 = out + 3 * G;
  double* o4 = out + 4 * G;
  for (int j = 0; j < G; ++j) o1[j] += nv[j] + cr[j];
  o2[host] += nv_sum;
  for (int j = 0; j < G; ++j) o3[j] += sr[j];
  o4[host] += sr_sum + cr_sum;
  std::fill(bins.begin(), bins.end(), 0.0);
  for (int j = 0; j < G; ++j) bins[t.r(j, host)] += cr[j];
  for (int g = 0; g < G; ++g) o2[g] += bins[g];
  for (int g = 0; g < G; ++g) o3[g] += bins[g];
  o1[host] += nv_sum + cr_sum;
  for (int j = 0; j < G; ++j) o2[j] += nv[j];
  o3[host] += sr_sum;
  for (int j = 0; j < G; ++j) o4[j] += sr[j] + cr[j];
  std::fill(bins.begin(), bins.end(), 0.0);
  for (int j = 0; j < G; ++j) bins[t.r(host, j)] += cr[j];
  for (int g = 0; g < G; ++g) o2[g] += bins[g];
  for (int g = 0; g < G; ++g) o3[g] += bins[g];
}

// Contribution tensor shared by every chain of one layer (AnnealState.__init__, reorder.py:179-194).
struct AnnealShared {
  const Topo* t;
  int E, G;
  double beta, comp_unit, row_units[4];
  std::vector<double> contrib;  // [E][G][5][G]
  AnnealShared(const double* x, int E_, const Topo& topo, int64_t h, int64_t hp, const Hw& hw, double beta_)
      : t(&topo), E(E_), G(topo.G), beta(beta_), contrib(size_t(E_) * topo.G * 5 * topo.G) {
    std::vector<double> col(G);
    for (int e = 0; e < E; ++e) {
      for (int j = 0; j < G; ++j) col[j] = x[size_t(j) * E + e];
      for (int hst = 0; hst < G; ++hst) dest_contrib(col.data(), hst, topo, &contrib[(size_t(e) * G + hst) * 5 * G]);
    }
    comp_unit = 6.0 * double(h) * double(hp) / hw.flops;
    row_units[0] = row_units[1] = hw.bpt / hw.bw_nv;
    row_units[2] = row_units[3] = hw.bpt / hw.bw_rd;
  }
  const double* c(int e, int host) const { return &contrib[(size_t(e) * G + host) * 5 * G]; }
};

struct AnnealChainState {
  const AnnealShared* sh;
  std::vector<int64_t> assign;
  std::vector<double> loads5, tmp5, scratch, comp_t, rows_t;
  int swaps_since_refresh = 0;
  static constexpr int kRefreshEvery = 4096;  // REFRESH_EVERY (reorder.py:27)

  AnnealChainState(const AnnealShared& s, const int64_t* a)
      : sh(&s), assign(a, a + s.E), loads5(size_t(5) * s.G), tmp5(size_t(5) * s.G), scratch(size_t(4) * s.G),
        comp_t(s.G), rows_t(size_t(4) * s.G) {
    refresh();
  }
  void refresh() {
    // contrib[arange(E), assignment].sum(axis=0): sequential over experts
    std::fill(loads5.begin(), loads5.end(), 0.0);
    for (int e = 0; e < sh->E; ++e) {
      const double* c = sh->c(e, int(assign[e]));
      for (size_t i = 0; i < loads5.size(); ++i) loads5[i] += c[i];
    }
    swaps_since_refresh = 0;
  }
  void swap_delta(int a, int b, double* d) const {
    const int ga = int(assign[a]), gb = int(assign[b]);
    const double *aga = sh->c(a, ga), *agb = sh->c(a, gb), *bga = sh->c(b, ga), *bgb = sh->c(b, gb);
    for (int i = 0; i < 5 * sh->G; ++i) d[i] = agb[i] - aga[i] + bga[i] - bgb[i];
  }
  void times(const double* l5) {
    const int G = sh->G;
    for (int g = 0; g < G; ++g) comp_t[g] = l5[g] * sh->comp_unit;
    for (int r = 0; r < 4; ++r)
      for (int g = 0; g < G; ++g) rows_t[size_t(r) * G + g] = l5[size_t(r + 1) * G + g] * sh->row_units[r];
  }
  double smoothed(const double* l5) {
    times(l5);
    const int G = sh->G;
    return lse(comp_t.data(), G, sh->beta, scratch.data()) + lse(rows_t.data(), 4 * G, sh->beta, scratch.data());
  }
  double exact(const double* l5) {
    times(l5);
    return vmax(comp_t.data(), sh->G) + vmax(rows_t.data(), 4 * sh->G);
  }
  void apply_swap(int a, int b, const double* d) {
    for (size_t i = 0; i < loads5.size(); ++i) loads5[i] += d[i];
    std::swap(assign[a], assign[b]);
    if (++swaps_since_refresh >= kRefreshEvery) refresh();
  }
};

// _run_chain (reorder.py:299-326)
static void run_chain(const AnnealShared& sh, const int64_t* a0, double cooling, double eps_frac, double term_eps,
                      uint64_t seed, int64_t* best_out, int64_t* iters_out) {
  AnnealChainState st(sh, a0);
  const int E = sh.E;
  PCG64 rng{SeedSequence(seed)};
  double t_cur = st.smoothed(st.loads5.data());
  double theta = t_cur > 0 ? t_cur : 1.0;
  const double eps = term_eps > 0 ? term_eps : eps_frac * theta;
  std::copy(st.assign.begin(), st.assign.end(), best_out);
  double best_t = t_cur;
  int64_t iters = 0;
  if (sh.G < 2 || E < 2) {
    if (iters_out) *iters_out = 0;
    return;
  }
  std::vector<double> delta(size_t(5) * sh.G), cand(size_t(5) * sh.G);
  while (theta > eps) {
    int ea, eb;
    while (true) {
      ea = int(rng.bounded(uint32_t(E)));
      eb = int(rng.bounded(uint32_t(E)));
      if (ea != eb && st.assign[ea] != st.assign[eb]) break;
    }
    st.swap_delta(ea, eb, delta.data());
    for (size_t i = 0; i < cand.size(); ++i) cand[i] = st.loads5[i] + delta[i];
    const double t_new = st.smoothed(cand.data());
    const double diff = t_new - t_cur;
    bool accept = diff < 0;
    if (!accept) accept = rng.random() < std::exp(-std::min(diff / theta, 745.0));
    if (accept) {
      st.apply_swap(ea, eb, delta.data());
      t_cur = t_new;
      if (t_cur < best_t) {
        best_t = t_cur;
        std::copy(st.assign.begin(), st.assign.end(), best_out);
      }
    }
    theta *= cooling;
    ++iters;
  }
  if (iters_out) *iters_out = iters;
}

// anneal_reorder (reorder.py:329-362)
int anneal_reorder(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, const uint64_t* seeds,
                   int nseeds, double cooling, double eps_frac, double term_eps, double beta, const int64_t* extra,
                   int nextra, int threads, int64_t* out, int64_t* iters_total) {
  const int G = t.G;
  if (E % G != 0) return fail(kInvalid, "%d experts not divisible by %d GPUs", E, G);
  std::vector<int64_t> base(E);
  lpt_initial(x, G, E, base.data());
  AnnealShared sh(x, E, t, h, hp, hw, beta);
  const int ncand = 1 + nextra + nseeds;
  std::vector<int64_t> cands(size_t(ncand) * E);
  std::copy(base.begin(), base.end(), cands.begin());
  for (int i = 0; i < nextra; ++i) std::copy(extra + size_t(i) * E, extra + size_t(i + 1) * E, &cands[size_t(1 + i) * E]);
  std::vector<int64_t> iters(nseeds, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1) if (threads != 1)
  for (int s = 0; s < nseeds; ++s)
    run_chain(sh, base.data(), cooling, eps_frac, term_eps, seeds[s], &cands[size_t(1 + nextra + s) * E], &iters[s]);
  int best = 0;
  double best_t = std::numeric_limits<double>::infinity();
  for (int c = 0; c < ncand; ++c) {
    AnnealChainState st(sh, &cands[size_t(c) * E]);
    const double tt = st.exact(st.loads5.data());
    if (tt < best_t) {
      best_t = tt;
      best = c;
    }
  }
  std::copy(&cands[size_t(best) * E], &cands[size_t(best + 1) * E], out);
  if (iters_total) {
    int64_t s = 0;
    for (auto v : iters) s += v;
    *iters_total = s;
  }
  return kOk;
}

// Device-chain support (mb_anneal_chains in the sm_100a library runs _run_chain, one GPU thread
// per seed): the inputs every chain shares -- LPT start, contribution tensor, time units -- and
// each seed's PCG64 state, computed exactly as anneal_reorder does on the host.
int anneal_prepare(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, double beta,
                   const uint64_t* seeds, int nseeds, int64_t* base_out, double* contrib_out, double* consts_out,
                   uint64_t* rng_out) {
  const int G = t.G;
  if (E % G != 0) return fail(kInvalid, "%d experts not divisible by %d GPUs", E, G);
  lpt_initial(x, G, E, base_out);
  AnnealShared sh(x, E, t, h, hp, hw, beta);
  std::copy(sh.contrib.begin(), sh.contrib.end(), contrib_out);
  consts_out[0] = sh.comp_unit;
  for (int r = 0; r < 4; ++r) consts_out[1 + r] = sh.row_units[r];
  for (int s = 0; s < nseeds; ++s) PCG64{SeedSequence(seeds[s])}.raw(rng_out + size_t(4) * s);
  return kOk;
}

// anneal_reorder's final choice: first minimum of the exact T_MoE over the candidate plans
// (LPT, extra plans, chains in seed order; reorder.py:352-362).
int anneal_select(const double* x, const Topo& t, int E, int64_t h, int64_t hp, const Hw& hw, double beta,
                  const int64_t* cands, int ncand, int64_t* out) {
  if (ncand < 1) return fail(kInvalid, "no candidate plans");
  AnnealShared sh(x, E, t, h, hp, hw, beta);
  int best = 0;
  double best_t = std::numeric_limits<double>::infinity();
  for (int c = 0; c < ncand; ++c) {
    AnnealChainState st(sh, &cands[size_t(c) * E]);
    const double tt = st.exact(st.loads5.data());
    if (tt < best_t) {
      best_t = tt;
      best = c;
    }
  }
  std::copy(&cands[size_t(best) * E], &cands[size_t(best + 1) * E], out);
  return kOk;
}

}  // namespace mbp
