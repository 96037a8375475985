// Shared host-planner infrastructure: status/error reporting across the C-ABI, the
// rail-optimised topology (class and relay matrices), and reductions that reproduce
// numpy's float64 summation order bit for bit.
//
// Compiled with -ffp-contract=off so that no multiply-add is fused: the reference
// evaluates every product and sum as separately rounded numpy float64 operations.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

namespace mbp {

enum Status : int { kOk = 0, kInvalid = 1, kSolver = 5, kLimit = 6 };

inline thread_local std::string g_err;
inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

struct Error {
  int code;
  std::string msg;
};

// TrafficClass (topology.py:20-27)
enum Cls : uint8_t { LOC = 0, NV = 1, SR = 2, CR = 3 };

// ClusterTopology (topology.py:50-115): node-major ids, class and relay matrices.
struct Topo {
  int nodes = 1, gpn = 1, G = 1;
  std::vector<uint8_t> cls;    // [G][G]
  std::vector<int32_t> relay;  // [G][G]
  Topo() = default;
  Topo(int n, int p) : nodes(n), gpn(p), G(n * p), cls(size_t(G) * G), relay(size_t(G) * G) {
    for (int j = 0; j < G; ++j)
      for (int g = 0; g < G; ++g) {
        const bool same_node = j / gpn == g / gpn, same_rail = j % gpn == g % gpn;
        uint8_t c = CR;
        if (!same_node && same_rail) c = SR;
        if (same_node) c = NV;
        if (j == g) c = LOC;
        cls[size_t(j) * G + g] = c;
        relay[size_t(j) * G + g] = (j / gpn) * gpn + (g % gpn);
      }
  }
  int node_of(int g) const { return g / gpn; }
  uint8_t c(int j, int g) const { return cls[size_t(j) * G + g]; }
  int r(int j, int g) const { return relay[size_t(j) * G + g]; }
};

struct Hw {
  double flops, bw_nv, bw_rd, bpt;
};

// numpy pairwise_sum for a contiguous float64 vector (np.add.reduce / ndarray.sum()).
inline double np_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_sum(a, n2) + np_sum(a + n2, n - n2);
}

inline double vmax(const double* a, int64_t n) {
  double m = a[0];
  for (int64_t i = 1; i < n; ++i)
    if (a[i] > m || std::isnan(a[i])) m = a[i];
  return m;
}

// reorder._lse (reorder.py:171-173): m + log(sum(exp(beta*(v-m)))) / beta
inline double lse(const double* v, int64_t n, double beta, double* scratch) {
  const double m = vmax(v, n);
  for (int64_t i = 0; i < n; ++i) scratch[i] = std::exp(beta * (v[i] - m));
  return m + std::log(np_sum(scratch, n)) / beta;
}

}  // namespace mbp
