// Per-(micro-batch, layer) integer tables that drive the data plane: receive layout of every
// GPU, the route table every source needs to place its (token, choice) rows, and the integer
// flow matrix (the executed counterpart of costmodel.flow_matrix, costmodel.py:91-108, with
// the split fractions replaced by round_split integers, replicate.py:501-525).
//
// Receive layout of GPU d: slots = home experts of d ascending, then experts replicated onto d
// ascending; inside a slot rows are ordered by source GPU, then by the stable rank of the
// (token, choice) entry on that source; every slot is padded to a multiple of `pad` rows.
#include <algorithm>

#include "planner.hpp"

namespace mbp {


int dispatch_plan(int G, int E, const int64_t* x, const int64_t* home, const std::vector<std::vector<int>>& reps,
                  const std::vector<std::vector<int64_t>>& counts, int pad, int maxc, int max_slots,
                  const DispatchOut& o) {
  auto ncop = [&](int e) { return 1 + int(reps[e].size()); };
  auto cnt = [&](int j, int e, int c) -> int64_t {
    if (reps[e].empty()) return c == 0 ? x[size_t(j) * E + e] : 0;
    return counts[e][size_t(j) * ncop(e) + c];
  };
  auto copy_gpu = [&](int e, int c) { return c == 0 ? int(home[e]) : reps[e][c - 1]; };
  for (int e = 0; e < E; ++e) {
    if (ncop(e) > maxc) return fail(kInvalid, "expert %d has %d copies > maxc %d", e, ncop(e), maxc);
    if (!reps[e].empty() && counts[e].size() != size_t(G) * ncop(e))
      return fail(kInvalid, "split counts of expert %d have the wrong shape", e);
    for (int j = 0; j < G; ++j) {
      int64_t s = 0;
      for (int c = 0; c < ncop(e); ++c) {
        if (cnt(j, e, c) < 0) return fail(kInvalid, "negative split count (src %d, expert %d)", j, e);
        s += cnt(j, e, c);
      }
      if (s != x[size_t(j) * E + e])
        return fail(kInvalid, "split counts of (src %d, expert %d) sum to %lld, routing has %lld", j, e, (long long)s,
                    (long long)x[size_t(j) * E + e]);
    }
  }
  std::fill(o.flow, o.flow + size_t(G) * G, 0);
  std::fill(o.route_tab, o.route_tab + size_t(G) * E * maxc * 4, 0);
  std::fill(o.slot_tab, o.slot_tab + size_t(G) * max_slots * 4, 0);
  std::fill(o.slot_w, o.slot_w + size_t(G) * max_slots * 2, 0);
  for (int e = 0; e < E; ++e) o.ncopies[e] = ncop(e);
  // slot_of[e][c] = slot index of copy c of e on its GPU
  std::vector<std::vector<int>> slot_of(E);
  for (int e = 0; e < E; ++e) slot_of[e].assign(ncop(e), -1);
  for (int d = 0; d < G; ++d) {
    int ns = 0, nhome = 0, nrep = 0;
    int64_t row = 0;
    auto add_slot = [&](int e, int c, bool replica) -> int {
      if (ns >= max_slots) return fail(kInvalid, "GPU %d needs more than %d slots", d, max_slots);
      int64_t real = 0;
      for (int j = 0; j < G; ++j) real += cnt(j, e, c);
      const int64_t padded = (real + pad - 1) / pad * pad;
      int32_t* st = o.slot_tab + (size_t(d) * max_slots + ns) * 4;
      st[0] = int32_t(row);
      st[1] = int32_t(real);
      st[2] = int32_t(padded);
      st[3] = e;
      int32_t* sw = o.slot_w + (size_t(d) * max_slots + ns) * 2;
      sw[0] = replica ? nrep++ : nhome++;
      sw[1] = replica ? 1 : 0;
      // route entries for every source
      int64_t src_base = row;
      for (int j = 0; j < G; ++j) {
        int32_t* rt = o.route_tab + ((size_t(j) * E + e) * maxc + c) * 4;
        rt[1] = d;
        rt[2] = int32_t(src_base);
        src_base += cnt(j, e, c);
        o.flow[size_t(j) * G + d] += cnt(j, e, c);
      }
      slot_of[e][c] = ns;
      row += padded;
      ++ns;
      return kOk;
    };
    for (int e = 0; e < E; ++e)
      if (home[e] == d)
        if (int rc = add_slot(e, 0, false)) return rc;
    for (int e = 0; e < E; ++e)
      for (int c = 1; c < ncop(e); ++c)
        if (copy_gpu(e, c) == d)
          if (int rc = add_slot(e, c, true)) return rc;
    if (row > 0x7fffffffLL) return fail(kInvalid, "GPU %d receive layout exceeds 2^31 rows", d);
    o.nslots[d] = ns;
    o.total_rows[d] = row;
  }
  // cumulative ends per (source, expert, copy)
  for (int j = 0; j < G; ++j)
    for (int e = 0; e < E; ++e) {
      int64_t cum = 0;
      for (int c = 0; c < ncop(e); ++c) {
        cum += cnt(j, e, c);
        o.route_tab[((size_t(j) * E + e) * maxc + c) * 4 + 0] = int32_t(cum);
      }
    }
  return kOk;
}

}  // namespace mbp
