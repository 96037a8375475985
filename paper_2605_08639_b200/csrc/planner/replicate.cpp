// Intra-batch expert replication: token-split LP, greedy replication, integer splitting and
// the oracle-load EPLB baseline.  C++ restatement of moebalance.replicate
// (replicate.py:104-437, 501-525) and sim._eplb_replication (sim.py:142-194).
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <set>
#include <tuple>

#include "planner.hpp"
#include "simplex.hpp"

namespace mbp {

std::vector<int> candidate_gpus(int e, const std::vector<int64_t>& home, const Topo& t) {
  const int h = int(home[e]);
  std::vector<int> out;
  const int n = t.node_of(h);
  for (int g = n * t.gpn; g < (n + 1) * t.gpn; ++g)
    if (g != h) out.push_back(g);
  return out;
}

// TokenSplitLP (replicate.py:147-302)
class TokenSplitLP {
 public:
  static constexpr int kAux = 4;  // pc, qc, pm, qm
  TokenSplitLP(const double* x, int E, const std::vector<int64_t>& home, const Topo& t, int64_t h, int64_t hp,
               const Hw& hw)
      : x_(x), E_(E), G_(t.G), home_(home), t_(&t), reps_(E) {
    comp_unit_ = 6.0 * double(h) * double(hp) / hw.flops;
    u_nv_ = hw.bpt / hw.bw_nv;
    u_rd_ = hw.bpt / hw.bw_rd;
    const Loads base = compute_loads(x, E, home.data(), t, {});
    TimeModel tm(h, hp, hw);
    std::vector<double> comp_c(G_), rows(size_t(4) * G_);
    for (int g = 0; g < G_; ++g) comp_c[g] = tm.comp_time(base.comp[g]);
    tm.comm_rows(base, G_, rows.data());
    t0_comp_ = vmax(comp_c.data(), G_);
    t0_comm_ = vmax(rows.data(), 4 * G_);
    const int m = 5 * G_;
    std::vector<double> A(size_t(m) * kAux, 0.0), b(m);
    for (int i = 0; i < G_; ++i) A[size_t(i) * kAux + 0] = -1.0, A[size_t(i) * kAux + 1] = 1.0;
    for (int i = G_; i < m; ++i) A[size_t(i) * kAux + 2] = -1.0, A[size_t(i) * kAux + 3] = 1.0;
    for (int i = 0; i < G_; ++i) b[i] = t0_comp_ - comp_c[i];
    for (int i = 0; i < 4 * G_; ++i) b[G_ + i] = t0_comm_ - rows[i];
    solver_ = DenseSimplex({1.0, -1.0, 1.0, -1.0}, A, b, m, kAux);
  }

  const std::vector<int>& order() const { return order_; }
  const std::vector<int>& reps(int e) const { return reps_[e]; }

  int add_replica(int e, int gpu) {
    std::vector<int>& prior = reps_[e];
    for (int g : prior)
      if (g == gpu) return fail(kInvalid, "expert %d already has a copy on GPU %d", e, gpu);
    if (gpu == home_[e]) return fail(kInvalid, "expert %d already has a copy on GPU %d", e, gpu);
    const bool had_prior = !prior.empty();
    if (!had_prior) order_.push_back(e);
    prior.push_back(gpu);
    std::vector<int> sources;
    for (int j = 0; j < G_; ++j)
      if (x_[size_t(j) * E_ + e] > 0) sources.push_back(j);
    if (sources.empty()) return kOk;
    if (had_prior && !rows_built_.count(e)) {
      for (int j : sources) {
        const int pos = col_pos_.at(std::make_tuple(j, e, prior[0]));
        int rc = solver_.add_row({{pos, 1.0}}, 1.0);
        if (rc) return rc;
        sum_rows_[{j, e}] = solver_.num_rows() - 1;
      }
      rows_built_.insert(e);
    }
    const int m = solver_.num_rows();
    const int s = int(sources.size());
    std::vector<double> cols(size_t(m) * s, 0.0);
    for (int q = 0; q < s; ++q) {
      const int j = sources[q];
      const std::vector<double>& cg = pair_charge(j, gpu);
      const std::vector<double>& ch = pair_charge(j, int(home_[e]));
      const double xe = x_[size_t(j) * E_ + e];
      for (int r = 0; r < 5 * G_; ++r) cols[size_t(r) * s + q] = xe * (cg[r] - ch[r]);
      if (rows_built_.count(e)) cols[size_t(sum_rows_.at({j, e})) * s + q] = 1.0;
      col_pos_[std::make_tuple(j, e, gpu)] = kAux + int(var_meta_.size());
      var_meta_.push_back(std::make_tuple(j, e, gpu));
    }
    solver_.add_columns(cols, s, std::vector<double>(s, 0.0), std::vector<double>(s, 1.0));
    return kOk;
  }

  int solve(double* obj) {
    double o = 0.0;
    int rc = solver_.solve(&o);
    if (rc) return rc;
    *obj = t0_comp_ + t0_comm_ + o;
    return kOk;
  }

  // split_plan (replicate.py:283-302)
  SplitFr split_plan() const {
    SplitFr sp(E_);
    const std::vector<double> values = solver_.solution();
    for (int e : order_) {
      const int k = 1 + int(reps_[e].size());
      sp.frac[e].assign(size_t(G_) * k, 0.0);
      for (int j = 0; j < G_; ++j) sp.frac[e][size_t(j) * k] = 1.0;
      sp.order.push_back(e);
    }
    for (size_t v = 0; v < var_meta_.size(); ++v) {
      const int j = std::get<0>(var_meta_[v]), e = std::get<1>(var_meta_[v]), gpu = std::get<2>(var_meta_[v]);
      const int k = 1 + int(reps_[e].size());
      int col = 0;
      if (gpu != home_[e])
        for (int c = 0; c < int(reps_[e].size()); ++c)
          if (reps_[e][c] == gpu) {
            col = c + 1;
            break;
          }
      sp.frac[e][size_t(j) * k + col] = values[kAux + v];
    }
    for (int e : order_) {
      const int k = 1 + int(reps_[e].size());
      std::vector<double>& f = sp.frac[e];
      std::vector<int> routed;
      for (int j = 0; j < G_; ++j)
        if (x_[size_t(j) * E_ + e] > 0) routed.push_back(j);
      for (int j : routed) {
        double s = 0.0;
        for (int c = 1; c < k; ++c) s += f[size_t(j) * k + c];
        f[size_t(j) * k] = 1.0 - s;
      }
      for (double& v : f) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      for (int j : routed) {
        double s = 0.0;
        for (int c = 0; c < k; ++c) s += f[size_t(j) * k + c];
        for (int c = 0; c < k; ++c) f[size_t(j) * k + c] /= s;
      }
    }
    return sp;
  }

 private:
  const double* x_;
  int E_, G_;
  std::vector<int64_t> home_;
  const Topo* t_;
  double comp_unit_, u_nv_, u_rd_, t0_comp_, t0_comm_;
  DenseSimplex solver_;
  std::vector<std::tuple<int, int, int>> var_meta_;
  std::map<std::tuple<int, int, int>, int> col_pos_;
  std::map<std::pair<int, int>, int> sum_rows_;
  std::set<int> rows_built_;
  std::vector<std::vector<int>> reps_;
  std::vector<int> order_;
  std::map<std::pair<int, int>, std::vector<double>> charge_cache_;

  // _pair_charge (replicate.py:194-222)
  const std::vector<double>& pair_charge(int j, int g) {
    auto key = std::make_pair(j, g);
    auto it = charge_cache_.find(key);
    if (it != charge_cache_.end()) return it->second;
    std::vector<double> v(size_t(5) * G_, 0.0);
    v[g] += comp_unit_;
    auto comm = [&](int d, int gpu, double unit) { v[G_ + d * G_ + gpu] += unit; };
    const uint8_t c = t_->c(j, g);
    if (c == NV) {
      comm(0, j, u_nv_); comm(1, g, u_nv_);
      comm(0, g, u_nv_); comm(1, j, u_nv_);
    } else if (c == SR) {
      comm(2, j, u_rd_); comm(3, g, u_rd_);
      comm(2, g, u_rd_); comm(3, j, u_rd_);
    } else if (c == CR) {
      const int rj = t_->r(j, g), rg = t_->r(g, j);
      comm(0, j, u_nv_); comm(1, rj, u_nv_); comm(2, rj, u_rd_); comm(3, g, u_rd_);
      comm(0, g, u_nv_); comm(1, rg, u_nv_); comm(2, rg, u_rd_); comm(3, j, u_rd_);
    }
    return charge_cache_.emplace(key, std::move(v)).first->second;
  }
};

static double exact_objective(const double* x, int E, const Placement& pl, const SplitFr& sp, const Topo& t,
                              const TimeModel& tm, std::vector<double>* comp_t = nullptr,
                              std::vector<double>* comm_t = nullptr) {
  const Loads L = compute_loads(x, E, pl.home.data(), t, sp.to_map(pl));
  std::vector<double> ct(t.G), mt(t.G);
  const double v = tm.moe_time(L, t.G, ct.data(), mt.data());
  if (comp_t) *comp_t = ct;
  if (comm_t) *comm_t = mt;
  return v;
}

// _served_tokens (replicate.py:339-344)
static double served_tokens(const double* x, int G, int E, const Placement& pl, const SplitFr& sp, int e, int gpu) {
  std::vector<double> v(G);
  if (!sp.frac[e].empty()) {
    const std::vector<int> cp = pl.copies(e);
    const int k = int(cp.size());
    int col = int(std::find(cp.begin(), cp.end(), gpu) - cp.begin());
    for (int j = 0; j < G; ++j) v[j] = x[size_t(j) * E + e] * sp.frac[e][size_t(j) * k + col];
    return np_sum(v.data(), G);
  }
  if (pl.home[e] != gpu) return 0.0;
  for (int j = 0; j < G; ++j) v[j] = x[size_t(j) * E + e];
  return np_sum(v.data(), G);
}

// _bottleneck_candidates (replicate.py:350-362)
static std::vector<int> bottleneck_candidates(const std::vector<double>& comp_t, const std::vector<double>& comm_t) {
  const int G = int(comp_t.size());
  std::set<int> cands;
  for (const std::vector<double>* v : {&comp_t, &comm_t}) {
    const double top = vmax(v->data(), G);
    for (int g = 0; g < G; ++g)
      if ((*v)[g] >= top * (1.0 - 1e-9)) cands.insert(g);
  }
  std::vector<int> ranked(cands.begin(), cands.end());
  std::vector<double> score(G);
  for (int g = 0; g < G; ++g) score[g] = comp_t[g] + comm_t[g];
  std::sort(ranked.begin(), ranked.end(), [&](int a, int b) {
    if (-score[a] != -score[b]) return -score[a] < -score[b];
    return a < b;
  });
  if (ranked.size() > 8) ranked.resize(8);
  return ranked;
}

// greedy_replicate (replicate.py:365-437)
int greedy_replicate(const double* x, int E, const int64_t* home, const Topo& t, int64_t h, int64_t hp, const Hw& hw,
                     int slots, Placement& pl, SplitFr& sp, double* objective) {
  const int G = t.G;
  pl = Placement(home, E);
  sp = SplitFr(E);
  TimeModel tm(h, hp, hw);
  double total = np_sum(x, int64_t(G) * E);
  if (slots == 0 || total == 0.0) {
    if (objective) *objective = exact_objective(x, E, pl, sp, t, tm);
    return kOk;
  }
  TokenSplitLP lp(x, E, pl.home, t, h, hp, hw);
  double best = exact_objective(x, E, pl, sp, t, tm);
  std::vector<int> used = pl.slot_usage(G);
  auto any_free = [&]() {
    for (int g = 0; g < G; ++g)
      if (used[g] < slots) return true;
    return false;
  };
  while (any_free()) {
    std::vector<double> comp_t, comm_t;
    exact_objective(x, E, pl, sp, t, tm, &comp_t, &comm_t);
    std::vector<double> score(G);
    for (int g = 0; g < G; ++g) score[g] = comp_t[g] + comm_t[g];
    bool accepted = false;
    for (int gb : bottleneck_candidates(comp_t, comm_t)) {
      std::vector<std::pair<int, double>> served;
      for (int e : pl.serving(gb)) served.emplace_back(e, served_tokens(x, G, E, pl, sp, e, gb));
      std::stable_sort(served.begin(), served.end(), [](const std::pair<int, double>& a, const std::pair<int, double>& b) {
        if (-a.second != -b.second) return -a.second < -b.second;
        return a.first < b.first;
      });
      int e_star = -1, g_t = -1;
      for (auto& es : served) {
        const int e = es.first;
        int best_g = -1;
        for (int g : candidate_gpus(e, pl.home, t)) {
          bool present = false;
          for (int rg : pl.reps[e]) present = present || rg == g;
          if (present || used[g] >= slots) continue;
          if (best_g < 0 || score[g] < score[best_g] || (score[g] == score[best_g] && g < best_g)) best_g = g;
        }
        if (best_g >= 0) {
          e_star = e;
          g_t = best_g;
          break;
        }
      }
      if (e_star < 0) continue;
      TokenSplitLP snap = lp;
      int rc = lp.add_replica(e_star, g_t);
      if (rc) return rc;
      double lp_obj;
      rc = lp.solve(&lp_obj);
      if (rc) return fail(kSolver, "token-split LP failed (%s)", g_err.c_str());
      Placement trial(home, E);
      for (int e : lp.order())
        for (int g : lp.reps(e)) trial.add(e, g);
      SplitFr tsp = lp.split_plan();
      const double tobj = exact_objective(x, E, trial, tsp, t, tm);
      if (tobj < best * (1.0 - 1e-9)) {
        pl = trial;
        sp = tsp;
        best = tobj;
        used = pl.slot_usage(G);
        accepted = true;
        break;
      }
      lp = snap;
    }
    if (!accepted) break;
  }
  if (objective) *objective = best;
  return kOk;
}

// solve_token_split_lp (replicate.py:305-321): replicas added in ascending expert order
int solve_token_split(const double* x, int E, const Placement& pl, const Topo& t, int64_t h, int64_t hp, const Hw& hw,
                      SplitFr& sp) {
  TokenSplitLP lp(x, E, pl.home, t, h, hp, hw);
  std::vector<int> es(pl.order);
  std::sort(es.begin(), es.end());
  for (int e : es)
    for (int g : pl.reps[e]) {
      int rc = lp.add_replica(e, g);
      if (rc) return rc;
    }
  double o;
  int rc = lp.solve(&o);
  if (rc) return rc;
  sp = lp.split_plan();
  return kOk;
}

// round_split (replicate.py:501-525): largest remainder per (source, expert)
void round_split(const double* x, int G, int E, const Placement& pl, const SplitFr& sp,
                 std::vector<std::vector<int64_t>>& counts) {
  counts.assign(E, {});
  for (int e : sp.order) {
    const int k = 1 + int(pl.reps[e].size());
    std::vector<int64_t>& out = counts[e];
    out.assign(size_t(G) * k, 0);
    std::vector<double> raw(k), rem(k);
    std::vector<int64_t> fl(k);
    std::vector<int> ord(k);
    for (int j = 0; j < G; ++j) {
      const double target = x[size_t(j) * E + e];
      if (target <= 0) continue;
      int64_t fsum = 0;
      for (int c = 0; c < k; ++c) {
        raw[c] = sp.frac[e][size_t(j) * k + c] * target;
        fl[c] = static_cast<int64_t>(std::floor(raw[c]));
        fsum += fl[c];
      }
      const double d = target - double(fsum);
      const int64_t shortfall = static_cast<int64_t>(std::nearbyint(d));
      if (shortfall > 0) {
        for (int c = 0; c < k; ++c) rem[c] = raw[c] - double(fl[c]);
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return -rem[a] < -rem[b]; });
        for (int64_t q = 0; q < shortfall && q < k; ++q) fl[ord[q]] += 1;
      }
      for (int c = 0; c < k; ++c) out[size_t(j) * k + c] = fl[c];
    }
  }
}

// sim._eplb_replication (sim.py:142-194)
void eplb_replication(const double* loads, int E, const int64_t* home, const Topo& t, int slots, int max_rep,
                      Placement& pl) {
  const int gpn = t.gpn;
  pl = Placement(home, E);
  std::vector<int> copies(E, 1);
  std::vector<int64_t> node_slots(t.nodes, int64_t(slots) * gpn);
  while (true) {
    int best_e = -1;
    double best_pc = 0.0;
    for (int e = 0; e < E; ++e) {
      if (loads[e] <= 0 || copies[e] >= gpn) continue;
      if (max_rep >= 0 && copies[e] - 1 >= max_rep) continue;
      if (node_slots[t.node_of(int(home[e]))] <= 0) continue;
      const double pc = loads[e] / copies[e];
      if (best_e < 0 || pc > best_pc + 1e-15) {
        best_pc = pc;
        best_e = e;
      }
    }
    if (best_e < 0) break;
    copies[best_e] += 1;
    node_slots[t.node_of(int(home[best_e]))] -= 1;
  }
  std::vector<double> gload(t.G, 0.0);
  for (int e = 0; e < E; ++e) gload[home[e]] += loads[e] / copies[e];
  std::vector<int> slot_used(t.G, 0);
  struct Share { double v; int e, i; };
  std::vector<Share> shares;
  for (int e = 0; e < E; ++e)
    for (int i = 0; i < copies[e] - 1; ++i) shares.push_back({loads[e] / copies[e], e, i});
  std::stable_sort(shares.begin(), shares.end(), [](const Share& a, const Share& b) {
    if (-a.v != -b.v) return -a.v < -b.v;
    if (a.e != b.e) return a.e < b.e;
    return a.i < b.i;
  });
  for (const Share& s : shares) {
    int gt = -1;
    for (int g : candidate_gpus(s.e, pl.home, t)) {
      if (slot_used[g] >= slots) continue;
      bool present = false;
      for (int rg : pl.reps[s.e]) present = present || rg == g;
      if (present) continue;
      if (gt < 0 || gload[g] < gload[gt] || (gload[g] == gload[gt] && g < gt)) gt = g;
    }
    if (gt < 0) continue;
    pl.add(s.e, gt);
    gload[gt] += s.v;
    slot_used[gt] += 1;
  }
}

}  // namespace mbp
