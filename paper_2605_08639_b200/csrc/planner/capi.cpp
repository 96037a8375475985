// extern "C" wrappers of the host planners (see include/mb_planner.h).  No C++ exception
// crosses the ABI; every failure becomes a status code plus a thread-local message.
#include <dlfcn.h>

#include <exception>
#include <string>

#include "../../../include/mb_planner.h"
#include "planner.hpp"
#include "simplex.hpp"

#include <algorithm>

using namespace mbp;

#define GUARD(...)                                            \
  try {                                                        \
    __VA_ARGS__                                                    \
  } catch (const std::exception& ex) {                         \
    return fail(kInvalid, "planner exception: %s", ex.what());   \
  }

static int check_topo(int nodes, int gpn) {
  if (nodes < 1 || gpn < 1) return fail(kInvalid, "topology needs at least one node and one GPU per node");
  return kOk;
}

static Placement placement_from_csr(const int64_t* home, int E, int n_rep, const int32_t* rep_experts,
                                    const int32_t* rep_ptr, const int32_t* rep_gpus) {
  Placement p(home, E);
  for (int i = 0; i < n_rep; ++i)
    for (int q = rep_ptr[i]; q < rep_ptr[i + 1]; ++q) p.add(rep_experts[i], rep_gpus[q]);
  return p;
}

static void placement_to_csr(const Placement& p, int32_t* n_rep, int32_t* rep_experts, int32_t* rep_ptr,
                             int32_t* rep_gpus) {
  *n_rep = int32_t(p.order.size());
  int q = 0;
  rep_ptr[0] = 0;
  for (size_t i = 0; i < p.order.size(); ++i) {
    rep_experts[i] = p.order[i];
    for (int g : p.reps[p.order[i]]) rep_gpus[q++] = g;
    rep_ptr[i + 1] = q;
  }
}

extern "C" const char* mbp_last_error(void) { return g_err.c_str(); }

extern "C" int mbp_use_numpy_blas(const char* path, const char* prefix) {
  if (!path) {
    numpy_blas() = NumpyBlas();
    return kOk;
  }
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(kInvalid, "dlopen(%s) failed: %s", path, dlerror());
  const std::string p = prefix ? prefix : "";
  NumpyBlas b;
  b.dgemm = reinterpret_cast<NumpyBlas::dgemm_t>(dlsym(h, (p + "cblas_dgemm64_").c_str()));
  b.dgemv = reinterpret_cast<NumpyBlas::dgemv_t>(dlsym(h, (p + "cblas_dgemv64_").c_str()));
  b.ddot = reinterpret_cast<NumpyBlas::ddot_t>(dlsym(h, (p + "cblas_ddot64_").c_str()));
  if (!b.ok()) return fail(kInvalid, "%s lacks ILP64 %scblas_{dgemm,dgemv,ddot}64_", path, p.c_str());
  numpy_blas() = b;
  return kOk;
}

extern "C" int mbp_numpy_blas_active(void) { return numpy_blas().ok() ? 1 : 0; }

extern "C" int mbp_static_plan(int32_t E, int32_t G, int64_t* assignment) {
  if (G < 1 || E % G != 0) return fail(kInvalid, "%d experts not divisible by %d GPUs", E, G);
  static_plan(E, G, assignment);
  return kOk;
}

extern "C" int mbp_lpt_initial(const double* x, int32_t G, int32_t E, int64_t* assignment) {
  if (G < 1 || E % G != 0) return fail(kInvalid, "%d experts not divisible by %d GPUs", E, G);
  GUARD(lpt_initial(x, G, E, assignment); return kOk;)
}

extern "C" int mbp_anneal_reorder(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden,
                                  int64_t inter, double flops, double bw_nv, double bw_rd, double bpt,
                                  const uint64_t* seeds, int32_t nseeds, double cooling, double eps_frac,
                                  double term_eps, double beta, const int64_t* extra, int32_t nextra, int32_t threads,
                                  int64_t* assignment, int64_t* iterations) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  if (nseeds < 1) return fail(kInvalid, "need at least one annealing seed");
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt};
        return anneal_reorder(x, t, E, hidden, inter, hw, seeds, nseeds, cooling, eps_frac, term_eps, beta, extra,
                              nextra, threads, assignment, iterations);)
}

extern "C" int mbp_anneal_prepare(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden,
                                  int64_t inter, double flops, double bw_nv, double bw_rd, double bpt, double beta,
                                  const uint64_t* seeds, int32_t nseeds, int64_t* base, double* contrib,
                                  double* consts, uint64_t* rng) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  if (nseeds < 0) return fail(kInvalid, "bad seed count");
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt};
        return anneal_prepare(x, t, E, hidden, inter, hw, beta, seeds, nseeds, base, contrib, consts, rng);)
}

extern "C" int mbp_anneal_select(const double* x, int32_t nodes, int32_t gpn, int32_t E, int64_t hidden,
                                 int64_t inter, double flops, double bw_nv, double bw_rd, double bpt, double beta,
                                 const int64_t* cands, int32_t ncand, int64_t* assignment) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt};
        return anneal_select(x, t, E, hidden, inter, hw, beta, cands, ncand, assignment);)
}

extern "C" int mbp_sample_placement(int32_t nodes, int32_t gpn, int32_t E, int32_t L, int32_t MB, int32_t S,
                                    const double* counts, const int32_t* micro_batch, const int64_t* source_gpu,
                                    const double* tokens, const int64_t* plans, int64_t hidden, int64_t inter,
                                    double flops, double bw_nv, double bw_rd, double bpt, const uint64_t* seeds,
                                    int32_t nseeds, double cooling, double eps_frac, double term_eps, double beta,
                                    double band, int32_t greedy_only, int32_t threads, int64_t* placement) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  if (S < 0 || L < 1 || MB < 1 || E < 1) return fail(kInvalid, "bad sample-placement dimensions");
  if (!greedy_only && nseeds < 1) return fail(kInvalid, "need at least one annealing seed");
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt};
        return anneal_samples(t, E, L, MB, S, counts, micro_batch, source_gpu, tokens, plans, hidden, inter, hw, seeds,
                              nseeds, cooling, eps_frac, term_eps, beta, band, greedy_only, threads, placement);)
}

extern "C" int mbp_compute_loads(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* placement,
                                 int32_t nsplit, const int32_t* split_expert, const int32_t* split_ptr,
                                 const int32_t* split_gpus, const double* split_frac, double* loads, double* flow) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  GUARD(Topo t(nodes, gpn); const int G = t.G; std::vector<SplitEntry> splits; size_t foff = 0;
        for (int i = 0; i < nsplit; ++i) {
          SplitEntry s;
          s.e = split_expert[i];
          for (int q = split_ptr[i]; q < split_ptr[i + 1]; ++q) s.gpus.push_back(split_gpus[q]);
          const size_t n = size_t(G) * s.gpus.size();
          s.frac.assign(split_frac + foff, split_frac + foff + n);
          foff += n;
          splits.push_back(std::move(s));
        } std::vector<double> fl;
        const Loads L = compute_loads(x, E, placement, t, splits, flow ? &fl : nullptr);
        for (int g = 0; g < G; ++g) {
          loads[0 * G + g] = L.comp[g];
          loads[1 * G + g] = L.nvtx[g];
          loads[2 * G + g] = L.nvrx[g];
          loads[3 * G + g] = L.rdtx[g];
          loads[4 * G + g] = L.rdrx[g];
        } if (flow) std::copy(fl.begin(), fl.end(), flow);
        return kOk;)
}

extern "C" int mbp_greedy_replicate(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home,
                                    int64_t hidden, int64_t inter, double flops, double bw_nv, double bw_rd,
                                    double bpt, int32_t slots, int32_t* n_rep, int32_t* rep_experts, int32_t* rep_ptr,
                                    int32_t* rep_gpus, double* frac, double* objective) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  if (slots < 0) return fail(kInvalid, "slots_per_gpu must be >= 0");
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt}; Placement pl; SplitFr sp;
        int rc = greedy_replicate(x, E, home, t, hidden, inter, hw, slots, pl, sp, objective); if (rc) return rc;
        placement_to_csr(pl, n_rep, rep_experts, rep_ptr, rep_gpus); size_t off = 0;
        for (int e : pl.order) {
          std::copy(sp.frac[e].begin(), sp.frac[e].end(), frac + off);
          off += sp.frac[e].size();
        } return kOk;)
}

extern "C" int mbp_solve_token_split(const double* x, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home,
                                     int64_t hidden, int64_t inter, double flops, double bw_nv, double bw_rd,
                                     double bpt, int32_t n_rep, const int32_t* rep_experts, const int32_t* rep_ptr,
                                     const int32_t* rep_gpus, int32_t* out_experts, double* frac) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  GUARD(Topo t(nodes, gpn); Hw hw{flops, bw_nv, bw_rd, bpt};
        Placement pl = placement_from_csr(home, E, n_rep, rep_experts, rep_ptr, rep_gpus);
        for (int e : pl.order) {
          const std::vector<int> cands = candidate_gpus(e, pl.home, t);
          for (size_t a = 0; a < pl.reps[e].size(); ++a) {
            const int g = pl.reps[e][a];
            if (std::find(cands.begin(), cands.end(), g) == cands.end())
              return fail(kInvalid, "replica of expert %d on GPU %d leaves its home node or duplicates home", e, g);
            for (size_t b = 0; b < a; ++b)
              if (pl.reps[e][b] == g) return fail(kInvalid, "duplicate replica GPUs for expert %d", e);
          }
        } SplitFr sp;
        int rc = solve_token_split(x, E, pl, t, hidden, inter, hw, sp); if (rc) return rc; size_t off = 0;
        for (size_t i = 0; i < sp.order.size(); ++i) {
          const int e = sp.order[i];
          out_experts[i] = e;
          std::copy(sp.frac[e].begin(), sp.frac[e].end(), frac + off);
          off += sp.frac[e].size();
        } return kOk;)
}

extern "C" int mbp_round_split(const double* x, int32_t G, int32_t E, const int64_t* home, int32_t n_rep,
                               const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus,
                               const double* frac, int64_t* counts) {
  GUARD(Placement pl = placement_from_csr(home, E, n_rep, rep_experts, rep_ptr, rep_gpus); SplitFr sp(E);
        size_t off = 0;
        for (int i = 0; i < n_rep; ++i) {
          const int e = rep_experts[i];
          const size_t n = size_t(G) * (1 + pl.reps[e].size());
          sp.frac[e].assign(frac + off, frac + off + n);
          sp.order.push_back(e);
          off += n;
        } std::vector<std::vector<int64_t>> out;
        round_split(x, G, E, pl, sp, out); off = 0;
        for (int i = 0; i < n_rep; ++i) {
          const int e = rep_experts[i];
          std::copy(out[e].begin(), out[e].end(), counts + off);
          off += out[e].size();
        } return kOk;)
}

extern "C" int mbp_eplb_replication(const double* loads, int32_t nodes, int32_t gpn, int32_t E, const int64_t* home,
                                    int32_t slots, int32_t max_rep, int32_t* n_rep, int32_t* rep_experts,
                                    int32_t* rep_ptr, int32_t* rep_gpus) {
  if (int rc = check_topo(nodes, gpn)) return rc;
  GUARD(Topo t(nodes, gpn); Placement pl; eplb_replication(loads, E, home, t, slots, max_rep, pl);
        placement_to_csr(pl, n_rep, rep_experts, rep_ptr, rep_gpus); return kOk;)
}

extern "C" int mbp_uniform_matrices(const uint32_t* in, int64_t rows, int32_t E, uint32_t* out) {
  if (E < 1) return fail(kInvalid, "need at least one expert");
  for (int64_t r = 0; r < rows; ++r) {
    int64_t s = 0;
    for (int e = 0; e < E; ++e) s += in[r * E + e];
    const int64_t base = s / E, extra = s - base * E;
    for (int e = 0; e < E; ++e) out[r * E + e] = uint32_t(base + (e < extra ? 1 : 0));
  }
  return kOk;
}

extern "C" int mbp_dispatch_plan(int32_t G, int32_t E, const int64_t* x, const int64_t* home, int32_t n_rep,
                                 const int32_t* rep_experts, const int32_t* rep_ptr, const int32_t* rep_gpus,
                                 const int64_t* counts, int32_t pad, int32_t maxc, int32_t max_slots,
                                 int32_t* route_tab, int32_t* ncopies, int32_t* slot_tab, int32_t* slot_w,
                                 int32_t* nslots, int64_t* total_rows, int64_t* flow) {
  if (G < 1 || E < 1 || pad < 1 || maxc < 1 || max_slots < 1) return fail(kInvalid, "bad dispatch plan dimensions");
  GUARD(std::vector<std::vector<int>> reps(E); std::vector<std::vector<int64_t>> cnts(E); size_t off = 0;
        for (int i = 0; i < n_rep; ++i) {
          const int e = rep_experts[i];
          if (e < 0 || e >= E) return fail(kInvalid, "replicated expert %d out of range", e);
          for (int q = rep_ptr[i]; q < rep_ptr[i + 1]; ++q) reps[e].push_back(rep_gpus[q]);
          const size_t n = size_t(G) * (1 + reps[e].size());
          cnts[e].assign(counts + off, counts + off + n);
          off += n;
        } DispatchOut o{route_tab, ncopies, slot_tab, slot_w, nslots, total_rows, flow};
        return dispatch_plan(G, E, x, home, reps, cnts, pad, maxc, max_slots, o);)
}
