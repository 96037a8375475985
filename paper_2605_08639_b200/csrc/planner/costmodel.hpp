// Load accounting and MoE-time model: C++ restatement of moebalance.costmodel
// (costmodel.py:64-213) with numpy's exact reduction order:
//   ndarray.sum(axis=1) on a C-order (G,G) -> pairwise per row (np_sum)
//   ndarray.sum(axis=0)                    -> sequential over rows
//   np.bincount(weights=...)               -> sequential in ravel order
#pragma once
#include <vector>
#include "common.hpp"

namespace mbp {

// One replicated expert's split (SplitMap entry, costmodel.py:21-24): serving GPUs in copy order
// and fractions [G][k] row-major.
struct SplitEntry {
  int e = 0;
  std::vector<int> gpus;
  std::vector<double> frac;
};

struct Loads {
  std::vector<double> comp, nvtx, nvrx, rdtx, rdrx;
  explicit Loads(int G = 0) : comp(G, 0.0), nvtx(G, 0.0), nvrx(G, 0.0), rdtx(G, 0.0), rdrx(G, 0.0) {}
};

// flow_matrix (costmodel.py:91-108): flow[src][serving gpu]
inline void flow_matrix(const double* x, int G, int E, const int64_t* placement, const std::vector<SplitEntry>& splits,
                        std::vector<double>& flow) {
  flow.assign(size_t(G) * G, 0.0);
  std::vector<char> is_split(E, 0);
  for (const auto& s : splits) is_split[s.e] = 1;
  std::vector<int> cols;
  std::vector<double> tmp;
  for (int dst = 0; dst < G; ++dst) {
    cols.clear();
    for (int e = 0; e < E; ++e)
      if (placement[e] == dst && !is_split[e]) cols.push_back(e);
    if (cols.empty()) continue;
    tmp.resize(cols.size());
    for (int j = 0; j < G; ++j) {
      for (size_t c = 0; c < cols.size(); ++c) tmp[c] = x[size_t(j) * E + cols[c]];
      flow[size_t(j) * G + dst] += np_sum(tmp.data(), int64_t(cols.size()));
    }
  }
  for (const auto& s : splits) {
    const int k = int(s.gpus.size());
    for (int j = 0; j < G; ++j)
      for (int c = 0; c < k; ++c) flow[size_t(j) * G + s.gpus[c]] += x[size_t(j) * E + s.e] * s.frac[size_t(j) * k + c];
  }
}

// _accumulate_direction (costmodel.py:64-88) for flow F (F[a][b] = mass a -> b); `transposed`
// reads F as its transpose (the mirrored combine pass).
inline void accumulate_direction(const std::vector<double>& F, bool transposed, const Topo& t, Loads& L) {
  const int G = t.G;
  auto at = [&](int a, int b) { return transposed ? F[size_t(b) * G + a] : F[size_t(a) * G + b]; };
  std::vector<double> m(size_t(G) * G), row(G);
  auto masked = [&](uint8_t cls) {
    for (int a = 0; a < G; ++a)
      for (int b = 0; b < G; ++b) m[size_t(a) * G + b] = (t.c(a, b) == cls) ? at(a, b) : 0.0;
  };
  auto add_rowsums = [&](std::vector<double>& acc) {
    for (int a = 0; a < G; ++a) acc[a] += np_sum(&m[size_t(a) * G], G);
  };
  auto add_colsums = [&](std::vector<double>& acc) {
    for (int b = 0; b < G; ++b) {
      double s = 0.0;
      for (int a = 0; a < G; ++a) s += m[size_t(a) * G + b];
      acc[b] += s;
    }
  };
  masked(NV);
  add_rowsums(L.nvtx);
  add_colsums(L.nvrx);
  masked(SR);
  add_rowsums(L.rdtx);
  add_colsums(L.rdrx);
  masked(CR);
  add_rowsums(L.nvtx);
  add_colsums(L.rdrx);
  std::vector<double> bins(G, 0.0);
  for (int a = 0; a < G; ++a)
    for (int b = 0; b < G; ++b) bins[t.r(a, b)] += m[size_t(a) * G + b];
  for (int g = 0; g < G; ++g) L.nvrx[g] += bins[g];
  for (int g = 0; g < G; ++g) L.rdtx[g] += bins[g];
}

// compute_loads (costmodel.py:127-158)
inline Loads compute_loads(const double* x, int E, const int64_t* placement, const Topo& t,
                           const std::vector<SplitEntry>& splits, std::vector<double>* flow_out = nullptr) {
  const int G = t.G;
  std::vector<double> flow;
  flow_matrix(x, G, E, placement, splits, flow);
  Loads L(G);
  for (int b = 0; b < G; ++b) {
    double s = 0.0;
    for (int a = 0; a < G; ++a) s += flow[size_t(a) * G + b];
    L.comp[b] = s;
  }
  accumulate_direction(flow, false, t, L);
  accumulate_direction(flow, true, t, L);
  if (flow_out) *flow_out = std::move(flow);
  return L;
}

struct TimeModel {
  double comp_c;        // 6.0*h*h' (evaluated left to right as numpy does)
  Hw hw;
  TimeModel(int64_t h, int64_t hp, Hw w) : comp_c(6.0 * double(h) * double(hp)), hw(w) {}
  double comp_time(double load) const { return comp_c * load / hw.flops; }
  // comm_row_times (costmodel.py:166-171): (4,G) seconds
  void comm_rows(const Loads& L, int G, double* rows) const {
    for (int g = 0; g < G; ++g) {
      rows[0 * G + g] = L.nvtx[g] * hw.bpt / hw.bw_nv;
      rows[1 * G + g] = L.nvrx[g] * hw.bpt / hw.bw_nv;
      rows[2 * G + g] = L.rdtx[g] * hw.bpt / hw.bw_rd;
      rows[3 * G + g] = L.rdrx[g] * hw.bpt / hw.bw_rd;
    }
  }
  // moe_time (costmodel.py:202-213): comp_times, comm_times and t_moe
  double moe_time(const Loads& L, int G, double* comp_t, double* comm_t) const {
    std::vector<double> rows(size_t(4) * G);
    comm_rows(L, G, rows.data());
    for (int g = 0; g < G; ++g) {
      comp_t[g] = comp_time(L.comp[g]);
      double m = rows[g];
      for (int d = 1; d < 4; ++d)
        if (rows[size_t(d) * G + g] > m) m = rows[size_t(d) * G + g];
      comm_t[g] = m;
    }
    return vmax(comp_t, G) + vmax(comm_t, G);
  }
};

}  // namespace mbp
