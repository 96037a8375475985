// Data-locality sample placement: a second annealing round that moves whole samples between
// source GPUs (inside each micro-batch's +/- band of the mean token count) under fixed expert
// plans.  C++ restatement of moebalance.reorder (reorder.py:365-564): greedy longest-first
// initial placement, then swap SA chains (one per seed, in parallel) on the smoothed MoE time
// summed over every (micro-batch, layer); the result is the first minimum of the exact time over
// [greedy, chains in seed order].  Loads are integer-valued, so the incremental bookkeeping is
// exact in any order; the LSE uses the same operation order as reorder._lse.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <set>

#include "pcg64.hpp"
#include "planner.hpp"

namespace mbp {

namespace {

// _source_contrib (reorder.py:128-158): (5, G) loads of source `src` sending mass[g] to each GPU
void source_contrib(const double* mass, int src, const Topo& t, double* out, double* nv, double* sr, double* cr,
                    double* bins) {
  const int G = t.G;
  std::fill(out, out + 5 * G, 0.0);
  for (int g = 0; g < G; ++g) out[g] += mass[g];
  for (int g = 0; g < G; ++g) {
    const uint8_t c = t.c(src, g);
    nv[g] = c == NV ? mass[g] : 0.0;
    sr[g] = c == SR ? mass[g] : 0.0;
    cr[g] = c == CR ? mass[g] : 0.0;
  }
  const double nv_sum = np_sum(nv, G), sr_sum = np_sum(sr, G), cr_sum = np_sum(cr, G);
  double* o1 = out + 1 * G;
  double* o2 = out + 2 * G;
  double* o3 = out + 3 * G;
  double* o4 = out + 4 * G;
  // dispatch: src -> destinations
  o1[src] += nv_sum + cr_sum;
  for (int g = 0; g < G; ++g) o2[g] += nv[g];
  o3[src] += sr_sum;
  for (int g = 0; g < G; ++g) o4[g] += sr[g] + cr[g];
  std::fill(bins, bins + G, 0.0);
  for (int g = 0; g < G; ++g) bins[t.r(src, g)] += cr[g];
  for (int g = 0; g < G; ++g) o2[g] += bins[g];
  for (int g = 0; g < G; ++g) o3[g] += bins[g];
  // combine: destinations -> src
  for (int g = 0; g < G; ++g) o1[g] += nv[g] + cr[g];
  o2[src] += nv_sum;
  for (int g = 0; g < G; ++g) o3[g] += sr[g];
  o4[src] += sr_sum + cr_sum;
  std::fill(bins, bins + G, 0.0);
  for (int g = 0; g < G; ++g) bins[t.r(g, src)] += cr[g];
  for (int g = 0; g < G; ++g) o2[g] += bins[g];
  for (int g = 0; g < G; ++g) o3[g] += bins[g];
}

struct SampleProblem {
  const Topo* t;
  int G, L, MB, S;
  std::vector<double> dst_mass;  // [S][L][G]
  std::vector<int> mb_of;
  std::vector<double> tokens;
  std::vector<double> mean;      // [MB]
  double comp_unit, row_units[4], beta, band;
};

// _SampleState (reorder.py:369-435)
struct SampleState {
  const SampleProblem* P;
  std::vector<double> loads5;  // [MB][L][5][G]
  std::vector<double> totals;  // [MB][G]
  std::vector<int64_t> placement;
  std::vector<double> c5, nv, sr, cr, bins, comp_t, rows_t, scratch;

  SampleState(const SampleProblem& p, const int64_t* place, bool apply_all = true)
      : P(&p), loads5(size_t(p.MB) * p.L * 5 * p.G, 0.0), totals(size_t(p.MB) * p.G, 0.0),
        placement(place, place + p.S), c5(size_t(5) * p.G), nv(p.G), sr(p.G), cr(p.G), bins(p.G), comp_t(p.G),
        rows_t(size_t(4) * p.G), scratch(size_t(4) * p.G) {
    if (apply_all)
      for (int i = 0; i < p.S; ++i) apply(i, int(placement[i]), 1.0);
  }
  void apply(int i, int gpu, double sign) {
    const int G = P->G, mb = P->mb_of[i];
    for (int l = 0; l < P->L; ++l) {
      source_contrib(&P->dst_mass[(size_t(i) * P->L + l) * G], gpu, *P->t, c5.data(), nv.data(), sr.data(),
                     cr.data(), bins.data());
      double* dst = &loads5[((size_t(mb) * P->L + l) * 5) * G];
      for (int q = 0; q < 5 * G; ++q) dst[q] += sign * c5[q];
    }
    totals[size_t(mb) * G + gpu] += sign * P->tokens[i];
  }
  void move(int i, int gpu) {
    apply(i, int(placement[i]), -1.0);
    apply(i, gpu, 1.0);
    placement[i] = gpu;
  }
  void times(int mb, int l) {
    const int G = P->G;
    const double* l5 = &loads5[((size_t(mb) * P->L + l) * 5) * G];
    for (int g = 0; g < G; ++g) comp_t[g] = l5[g] * P->comp_unit;
    for (int r = 0; r < 4; ++r)
      for (int g = 0; g < G; ++g) rows_t[size_t(r) * G + g] = l5[size_t(r + 1) * G + g] * P->row_units[r];
  }
  double entry_smoothed(int mb) {
    double total = 0.0;
    for (int l = 0; l < P->L; ++l) {
      times(mb, l);
      total += lse(comp_t.data(), P->G, P->beta, scratch.data()) + lse(rows_t.data(), 4 * P->G, P->beta, scratch.data());
    }
    return total;
  }
  double entry_exact(int mb) {
    double total = 0.0;
    for (int l = 0; l < P->L; ++l) {
      times(mb, l);
      total += vmax(comp_t.data(), P->G) + vmax(rows_t.data(), 4 * P->G);
    }
    return total;
  }
  double entry_comm(int mb) {
    double total = 0.0;
    for (int l = 0; l < P->L; ++l) {
      times(mb, l);
      total += vmax(rows_t.data(), 4 * P->G);
    }
    return total;
  }
  double smoothed_total() {
    double s = 0.0;
    for (int mb = 0; mb < P->MB; ++mb) s += entry_smoothed(mb);
    return s;
  }
  double exact_total() {
    double s = 0.0;
    for (int mb = 0; mb < P->MB; ++mb) s += entry_exact(mb);
    return s;
  }
};

// greedy_sample_initial (reorder.py:457-487)
void greedy_initial(const SampleProblem& p, const int64_t* source, int64_t* out) {
  SampleState st(p, source);
  for (int i = 0; i < p.S; ++i) st.apply(i, int(st.placement[i]), -1.0);
  std::vector<int> order(p.S);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return -p.tokens[a] < -p.tokens[b]; });
  const int G = p.G;
  for (int i : order) {
    const int mb = p.mb_of[i];
    const double hi = (1.0 + p.band) * p.mean[mb];
    std::vector<int> fits;
    for (int g = 0; g < G; ++g)
      if (st.totals[size_t(mb) * G + g] + p.tokens[i] <= hi + 1e-9) fits.push_back(g);
    if (fits.empty()) {
      int a = 0;
      for (int g = 1; g < G; ++g)
        if (st.totals[size_t(mb) * G + g] < st.totals[size_t(mb) * G + a]) a = g;
      fits.push_back(a);
    }
    int best_gpu = fits[0];
    double best_obj = std::numeric_limits<double>::infinity();
    for (int g : fits) {
      st.apply(i, g, 1.0);
      const double obj = st.entry_comm(mb);
      st.apply(i, g, -1.0);
      if (obj < best_obj - 1e-15) {
        best_obj = obj;
        best_gpu = g;
      }
    }
    st.apply(i, best_gpu, 1.0);
    out[i] = best_gpu;
    st.placement[i] = best_gpu;
  }
}

// _run_sample_chain (reorder.py:498-534)
void run_sample_chain(const SampleProblem& p, const int64_t* initial, double cooling, double eps_frac,
                      double term_eps, uint64_t seed, int64_t* best_out) {
  SampleState st(p, initial);
  PCG64 rng{SeedSequence(seed)};
  double t_cur = st.smoothed_total();
  double theta = t_cur > 0 ? t_cur : 1.0;
  const double eps = term_eps > 0 ? term_eps : eps_frac * theta;
  std::copy(st.placement.begin(), st.placement.end(), best_out);
  double best_t = t_cur;
  const int G = p.G;
  while (theta > eps) {
    const int i = int(rng.bounded(uint32_t(p.S)));
    const int j = int(rng.bounded(uint32_t(p.S)));
    const int gi = int(st.placement[i]), gj = int(st.placement[j]);
    if (i == j || gi == gj) {
      theta *= cooling;
      continue;
    }
    const int mbi = p.mb_of[i], mbj = p.mb_of[j];
    const double before = st.entry_smoothed(mbi) + (mbj != mbi ? st.entry_smoothed(mbj) : 0.0);
    st.move(i, gj);
    st.move(j, gi);
    bool in_band = true;
    const std::set<std::pair<int, int>> cells{{mbi, gi}, {mbi, gj}, {mbj, gi}, {mbj, gj}};
    for (const auto& [mb, g] : cells) {
      const double lo = (1.0 - p.band) * p.mean[mb], hi = (1.0 + p.band) * p.mean[mb];
      const double tot = st.totals[size_t(mb) * G + g];
      if (!(lo - 1e-9 <= tot && tot <= hi + 1e-9)) in_band = false;
    }
    const double after = st.entry_smoothed(mbi) + (mbj != mbi ? st.entry_smoothed(mbj) : 0.0);
    const double diff = after - before;
    bool accept = false;
    if (in_band) {
      accept = diff < 0;
      if (!accept) accept = rng.random() < std::exp(-std::min(std::max(diff, 0.0) / theta, 745.0));
    }
    if (accept) {
      t_cur += diff;
      if (t_cur < best_t) {
        best_t = t_cur;
        std::copy(st.placement.begin(), st.placement.end(), best_out);
      }
    } else {
      st.move(i, gi);
      st.move(j, gj);
    }
    theta *= cooling;
  }
}

SampleProblem make_problem(const Topo& t, int E, int L, int MB, int S, const double* counts, const int32_t* mb_of,
                           const double* tokens, const int64_t* plans, int64_t h, int64_t hp, const Hw& hw,
                           double beta, double band) {
  SampleProblem p;
  p.t = &t;
  p.G = t.G;
  p.L = L;
  p.MB = MB;
  p.S = S;
  p.beta = beta;
  p.band = band;
  p.comp_unit = 6.0 * double(h) * double(hp) / hw.flops;
  p.row_units[0] = p.row_units[1] = hw.bpt / hw.bw_nv;
  p.row_units[2] = p.row_units[3] = hw.bpt / hw.bw_rd;
  p.mb_of.assign(mb_of, mb_of + S);
  p.tokens.assign(tokens, tokens + S);
  // dst_mass[i, l] = bincount(plans[l], weights=counts[i, l], minlength=G)
  p.dst_mass.assign(size_t(S) * L * p.G, 0.0);
  for (int i = 0; i < S; ++i)
    for (int l = 0; l < L; ++l) {
      double* d = &p.dst_mass[(size_t(i) * L + l) * p.G];
      const double* c = counts + (size_t(i) * L + l) * E;
      for (int e = 0; e < E; ++e) d[plans[size_t(l) * E + e]] += c[e];
    }
  // _mb_means (reorder.py:490-495): integer token sum per micro-batch / G
  p.mean.assign(MB, 0.0);
  std::vector<int64_t> tsum(MB, 0);
  for (int i = 0; i < S; ++i) tsum[mb_of[i]] += int64_t(tokens[i]);
  for (int mb = 0; mb < MB; ++mb) p.mean[mb] = double(tsum[mb]) / double(p.G);
  return p;
}

}  // namespace

// anneal_sample_placement (reorder.py:537-568); greedy_only -> greedy_sample_initial
int anneal_samples(const Topo& t, int E, int L, int MB, int S, const double* counts, const int32_t* mb_of,
                   const int64_t* source, const double* tokens, const int64_t* plans, int64_t h, int64_t hp,
                   const Hw& hw, const uint64_t* seeds, int nseeds, double cooling, double eps_frac, double term_eps,
                   double beta, double band, int greedy_only, int threads, int64_t* out) {
  for (int i = 0; i < S; ++i) {
    if (mb_of[i] < 0 || mb_of[i] >= MB) return fail(kInvalid, "sample micro_batch out of range");
    if (source[i] < 0 || source[i] >= t.G) return fail(kInvalid, "sample source_gpu out of range");
  }
  for (int64_t q = 0; q < int64_t(L) * E; ++q)
    if (plans[q] < 0 || plans[q] >= t.G) return fail(kInvalid, "plan assigns an expert outside [0, G)");
  const SampleProblem p = make_problem(t, E, L, MB, S, counts, mb_of, tokens, plans, h, hp, hw, beta, band);
  std::vector<int64_t> initial(S);
  greedy_initial(p, source, initial.data());
  if (greedy_only) {
    std::copy(initial.begin(), initial.end(), out);
    return kOk;
  }
  const int nchains = (t.G >= 2 && S >= 2) ? nseeds : 0;
  std::vector<int64_t> cands(size_t(1 + nchains) * S);
  std::copy(initial.begin(), initial.end(), cands.begin());
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1) if (threads != 1)
  for (int c = 0; c < nchains; ++c)
    run_sample_chain(p, initial.data(), cooling, eps_frac, term_eps, seeds[c], &cands[size_t(1 + c) * S]);
  int best = 0;
  double best_exact = 0.0;
  for (int c = 0; c <= nchains; ++c) {
    SampleState st(p, &cands[size_t(c) * S]);
    const double ex = st.exact_total();
    if (c == 0 || ex < best_exact) {
      best_exact = ex;
      best = c;
    }
  }
  std::copy(&cands[size_t(best) * S], &cands[size_t(best + 1) * S], out);
  return kOk;
}

}  // namespace mbp
