// Bounded-variable dense primal simplex (min c.x s.t. A x <= b, 0 <= x <= u, b >= 0):
// C++ restatement of moebalance.lp.DenseSimplex (lp.py:29-254) with the same pivot rules
// (Dantzig pricing, Bland after 64 stalled pivots, ratio-test ties broken toward the lowest
// basic index, tolerances 1e-9) and the same warm-start operations (append columns through
// B^-1, append a row expressed in the current basis).  Value-semantics: copying the object is
// the snapshot, assigning it back is the restore.
#pragma once
#include <cmath>
#include <limits>
#include <utility>
#include <vector>

#include "common.hpp"

namespace mbp {

// Optional: the BLAS that numpy itself links (numpy.libs/libscipy_openblas64_*.so, ILP64 CBLAS).
// When loaded (mbp_use_numpy_blas), the three products of the reference's warm start
// (lp.py:79-80 and the dot in lp.py:100) are issued exactly as numpy's matmul dispatch issues
// them, so LP vertices and fractions are bit-identical to the reference on the same host;
// otherwise plain loops are used (objective-equal, last-ULP differences possible).
struct NumpyBlas {
  typedef void (*dgemm_t)(int, int, int, int64_t, int64_t, int64_t, double, const double*, int64_t, const double*,
                          int64_t, double, double*, int64_t);
  typedef void (*dgemv_t)(int, int, int64_t, int64_t, double, const double*, int64_t, const double*, int64_t, double,
                          double*, int64_t);
  typedef double (*ddot_t)(int64_t, const double*, int64_t, const double*, int64_t);
  dgemm_t dgemm = nullptr;
  dgemv_t dgemv = nullptr;
  ddot_t ddot = nullptr;
  bool ok() const { return dgemm && dgemv && ddot; }
};
inline NumpyBlas& numpy_blas() {
  static NumpyBlas b;
  return b;
}
enum { kRowMajor = 101, kColMajor = 102, kNoTrans = 111, kTrans = 112 };

// numpy's float(a @ b) for 1-D float64 vectors: 0.0 + cblas_ddot
inline double np_dot(const double* a, const double* b, int64_t n) {
  const NumpyBlas& B = numpy_blas();
  if (B.ok()) return 0.0 + B.ddot(n, a, 1, b, 1);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

class DenseSimplex {
 public:
  static constexpr double kPivotTol = 1e-9, kCostTol = 1e-9;
  static constexpr int kStallLimit = 64;

  DenseSimplex() = default;
  // A is m x n row-major.
  DenseSimplex(const std::vector<double>& c, const std::vector<double>& A, const std::vector<double>& b, int m, int n)
      : m_(m), nc_(n + m) {
    tab_.assign(size_t(m_) * nc_, 0.0);
    for (int i = 0; i < m; ++i) {
      for (int j = 0; j < n; ++j) tab_[size_t(i) * nc_ + j] = A[size_t(i) * n + j];
      tab_[size_t(i) * nc_ + n + i] = 1.0;
    }
    rhs_ = b;
    cost_.assign(nc_, 0.0);
    for (int j = 0; j < n; ++j) cost_[j] = c[j];
    red_ = cost_;
    upper_.assign(nc_, kInf);
    at_upper_.assign(nc_, 0);
    for (int j = 0; j < n; ++j) struct_idx_.push_back(j);
    for (int i = 0; i < m; ++i) slack_idx_.push_back(n + i), basis_.push_back(n + i);
  }

  int num_rows() const { return m_; }
  int num_struct() const { return int(struct_idx_.size()); }
  double objective() const { return objective_; }

  // add_columns (lp.py:68-87): cols is m x s row-major
  void add_columns(const std::vector<double>& cols, int s, const std::vector<double>& c_new,
                   const std::vector<double>& upper_new) {
    // transformed = B^-1 @ cols, B^-1 = tab[:, slack_idx].  numpy's fancy index on axis 1 yields
    // an F-contiguous copy, i.e. the row-major buffer of (B^-1)^T: keep that buffer (binvT).
    std::vector<double> binv(size_t(m_) * m_), binvT(size_t(m_) * m_);
    for (int i = 0; i < m_; ++i)
      for (int l = 0; l < m_; ++l) {
        const double v = tab_[size_t(i) * nc_ + slack_idx_[l]];
        binv[size_t(i) * m_ + l] = v;
        binvT[size_t(l) * m_ + i] = v;
      }
    std::vector<double> costb(m_);
    for (int i = 0; i < m_; ++i) costb[i] = cost_[basis_[i]];
    std::vector<double> tr(size_t(m_) * s, 0.0), red_new(s);
    const NumpyBlas& B = numpy_blas();
    if (B.ok()) {
      // numpy matmul dispatch for an F-ordered left operand:
      //   (m,m)@(m,1) -> gemv(RowMajor, Trans, lda=m); (m,m)@(m,s) -> gemm(RowMajor, Trans, NoTrans)
      if (s == 1)
        B.dgemv(kRowMajor, kTrans, m_, m_, 1.0, binvT.data(), m_, cols.data(), 1, 0.0, tr.data(), 1);
      else
        B.dgemm(kRowMajor, kTrans, kNoTrans, m_, s, m_, 1.0, binvT.data(), m_, cols.data(), s, 0.0, tr.data(), s);
      // (m,)@(m,1) -> dot; (m,)@(m,s) -> gemv(RowMajor, Trans)
      if (s == 1) {
        red_new[0] = c_new[0] - np_dot(costb.data(), tr.data(), m_);
      } else {
        std::vector<double> tmp(s);
        B.dgemv(kRowMajor, kTrans, m_, s, 1.0, tr.data(), s, costb.data(), 1, 0.0, tmp.data(), 1);
        for (int q = 0; q < s; ++q) red_new[q] = c_new[q] - tmp[q];
      }
    } else {
      for (int i = 0; i < m_; ++i)
        for (int q = 0; q < s; ++q) {
          double acc = 0.0;
          for (int l = 0; l < m_; ++l) acc += binv[size_t(i) * m_ + l] * cols[size_t(l) * s + q];
          tr[size_t(i) * s + q] = acc;
        }
      for (int q = 0; q < s; ++q) {
        double acc = 0.0;
        for (int i = 0; i < m_; ++i) acc += costb[i] * tr[size_t(i) * s + q];
        red_new[q] = c_new[q] - acc;
      }
    }
    const int start = nc_;
    grow_cols(s);
    for (int i = 0; i < m_; ++i)
      for (int q = 0; q < s; ++q) tab_[size_t(i) * nc_ + start + q] = tr[size_t(i) * s + q];
    for (int q = 0; q < s; ++q) {
      cost_[start + q] = c_new[q];
      red_[start + q] = red_new[q];
      upper_[start + q] = upper_new[q];
      at_upper_[start + q] = 0;
      struct_idx_.push_back(start + q);
    }
  }


  // add_row (lp.py:89-120): one <= row over structural positions {pos: coef}
  int add_row(const std::vector<std::pair<int, double>>& coefs, double b_new) {
    std::vector<double> orig(nc_, 0.0);
    for (auto& pc : coefs) orig[struct_idx_[pc.first]] = pc.second;
    const std::vector<double> xnow = full_solution();
    const double slack = b_new - np_dot(orig.data(), xnow.data(), nc_);
    if (slack < -kPivotTol) return fail(kSolver, "new row is violated at the current point");
    std::vector<double> trow = orig;
    for (int i = 0; i < m_; ++i) {
      const double coef = orig[basis_[i]];
      if (coef != 0.0)
        for (int j = 0; j < nc_; ++j) trow[j] -= coef * tab_[size_t(i) * nc_ + j];
    }
    const int newcol = nc_;
    grow_cols(1);
    tab_.resize(size_t(m_ + 1) * nc_, 0.0);
    for (int j = 0; j < newcol; ++j) tab_[size_t(m_) * nc_ + j] = trow[j];
    tab_[size_t(m_) * nc_ + newcol] = 1.0;
    rhs_.push_back(slack > 0.0 ? slack : 0.0);
    cost_[newcol] = 0.0;
    red_[newcol] = 0.0;
    upper_[newcol] = kInf;
    at_upper_[newcol] = 0;
    slack_idx_.push_back(newcol);
    basis_.push_back(newcol);
    ++m_;
    return kOk;
  }

  // solve (lp.py:201-223); returns status, objective in *obj
  int solve(double* obj) {
    const int64_t max_iter = 200LL * (m_ + num_struct()) + 2000;
    int stall = 0;
    double last = objective_;
    std::vector<char> mask;
    for (int64_t it = 0; it < max_iter; ++it) {
      eligible(mask);
      int col = -1;
      double best = -1.0;
      for (int j = 0; j < nc_; ++j) {
        if (!mask[j]) continue;
        if (stall >= kStallLimit) {
          col = j;
          break;
        }
        const double a = std::fabs(red_[j]);
        if (col < 0 || a > best) {
          col = j;
          best = a;
        }
      }
      if (col < 0) {
        *obj = objective_;
        return kOk;
      }
      int rc = step(col);
      if (rc) return rc;
      if (objective_ < last - 1e-12 * (1.0 + std::fabs(last))) {
        stall = 0;
        last = objective_;
      } else {
        ++stall;
      }
    }
    return fail(kSolver, "simplex exceeded %lld iterations (m=%d, n=%d)", (long long)max_iter, m_, num_struct());
  }

  std::vector<double> full_solution() const {
    std::vector<double> x(nc_, 0.0);
    for (int j = 0; j < nc_; ++j)
      if (at_upper_[j]) x[j] = upper_[j];
    for (int i = 0; i < m_; ++i) x[basis_[i]] = rhs_[i];
    return x;
  }
  // structural values in the order added (lp.py:225-227)
  std::vector<double> solution() const {
    const std::vector<double> x = full_solution();
    std::vector<double> out(struct_idx_.size());
    for (size_t i = 0; i < struct_idx_.size(); ++i) out[i] = x[struct_idx_[i]];
    return out;
  }

 private:
  static constexpr double kInf = std::numeric_limits<double>::infinity();
  int m_ = 0, nc_ = 0;
  std::vector<double> tab_, rhs_, cost_, red_, upper_;
  std::vector<char> at_upper_;
  std::vector<int> struct_idx_, slack_idx_, basis_;
  double objective_ = 0.0;
  int64_t pivots_ = 0;

  void grow_cols(int s) {
    const int nn = nc_ + s;
    std::vector<double> t(size_t(m_) * nn, 0.0);
    for (int i = 0; i < m_; ++i)
      for (int j = 0; j < nc_; ++j) t[size_t(i) * nn + j] = tab_[size_t(i) * nc_ + j];
    tab_.swap(t);
    nc_ = nn;
    cost_.resize(nn, 0.0);
    red_.resize(nn, 0.0);
    upper_.resize(nn, kInf);
    at_upper_.resize(nn, 0);
  }

  void eligible(std::vector<char>& mask) const {
    mask.assign(nc_, 0);
    for (int j = 0; j < nc_; ++j) {
      const bool lo = !at_upper_[j] && red_[j] < -kCostTol;
      const bool up = at_upper_[j] && red_[j] > kCostTol;
      mask[j] = lo || up;
    }
    for (int i = 0; i < m_; ++i) mask[basis_[i]] = 0;
  }

  // _step (lp.py:138-199)
  int step(int col) {
    const bool from_upper = at_upper_[col] != 0;
    std::vector<double> dir(m_);
    for (int i = 0; i < m_; ++i) {
      const double d = tab_[size_t(i) * nc_ + col];
      dir[i] = from_upper ? -d : d;
    }
    double t_best = upper_[col];
    int block_row = -1;
    bool block_to_upper = false;
    // basics decreasing toward zero
    {
      double best = kInf;
      bool any = false;
      for (int i = 0; i < m_; ++i)
        if (dir[i] > kPivotTol) {
          const double r = rhs_[i] / dir[i];
          if (!any || r < best) best = r;
          any = true;
        }
      if (any && best < t_best - kPivotTol * (1.0 + std::fabs(best))) {
        const double lim = best + kPivotTol * (1.0 + std::fabs(best));
        int pick = -1;
        for (int i = 0; i < m_; ++i)
          if (dir[i] > kPivotTol && rhs_[i] / dir[i] <= lim && (pick < 0 || basis_[i] < basis_[pick])) pick = i;
        block_row = pick;
        block_to_upper = false;
        t_best = best > 0.0 ? best : 0.0;
      }
    }
    // basics increasing toward a finite upper bound
    {
      double best = kInf;
      bool any = false;
      for (int i = 0; i < m_; ++i)
        if (dir[i] < -kPivotTol && std::isfinite(upper_[basis_[i]])) {
          const double gap = (upper_[basis_[i]] - rhs_[i]) / (-dir[i]);
          if (!any || gap < best) best = gap;
          any = true;
        }
      if (any && best < t_best - kPivotTol * (1.0 + std::fabs(best))) {
        const double lim = best + kPivotTol * (1.0 + std::fabs(best));
        int pick = -1;
        for (int i = 0; i < m_; ++i)
          if (dir[i] < -kPivotTol && std::isfinite(upper_[basis_[i]]) &&
              (upper_[basis_[i]] - rhs_[i]) / (-dir[i]) <= lim && (pick < 0 || basis_[i] < basis_[pick]))
            pick = i;
        block_row = pick;
        block_to_upper = true;
        t_best = best > 0.0 ? best : 0.0;
      }
    }
    if (!std::isfinite(t_best)) return fail(kSolver, "LP is unbounded (no blocking bound)");
    const double t = t_best;
    for (int i = 0; i < m_; ++i) rhs_[i] -= t * dir[i];
    objective_ += red_[col] * (from_upper ? -t : t);
    if (block_row < 0) {
      at_upper_[col] = from_upper ? 0 : 1;
      return kOk;
    }
    const int leaving = basis_[block_row];
    if (block_to_upper) at_upper_[leaving] = 1;
    const double piv = tab_[size_t(block_row) * nc_ + col];
    if (std::fabs(piv) < kPivotTol) return fail(kSolver, "numerically singular pivot");
    const double entering = from_upper ? upper_[col] - t : t;
    double* prow = &tab_[size_t(block_row) * nc_];
    for (int j = 0; j < nc_; ++j) prow[j] /= piv;
    std::vector<double> factors(m_);
    for (int i = 0; i < m_; ++i) factors[i] = tab_[size_t(i) * nc_ + col];
    factors[block_row] = 0.0;
    for (int i = 0; i < m_; ++i) {
      const double f = factors[i];
      double* row = &tab_[size_t(i) * nc_];
      for (int j = 0; j < nc_; ++j) row[j] -= f * prow[j];
    }
    const double rfac = red_[col];
    for (int j = 0; j < nc_; ++j) red_[j] -= rfac * prow[j];
    basis_[block_row] = col;
    at_upper_[col] = 0;
    rhs_[block_row] = entering;
    ++pivots_;
    return kOk;
  }
};

}  // namespace mbp
