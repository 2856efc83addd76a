// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
#include "linalg.hpp"

#include <algorithm>
#include <thread>

namespace oracle {

namespace {
// static-partition parallel loop over [lo, hi) (the image has no libgomp)
template <class F>
void parallel_for(int lo, int hi, F&& f, int grain = 64) {
  const int n = hi - lo;
  const int workers = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), n / grain));
  if (workers <= 1) {
    for (int i = lo; i < hi; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (int i = lo + w; i < hi; i += workers) f(i);
    });
  for (auto& t : pool) t.join();
}
}  // namespace

// Right-looking Cholesky B = L L^T (lower, in place), then X = L^-T L^-1.
//
// Blocked for the 1k-7k node grids, with every element receiving exactly the
// same floating-point operations in the same order as the unblocked
// column-by-column algorithm (so results are bit-identical to it):
//   * factor: a panel of kPanel columns is factored unblocked, then each
//     trailing column j >= panel end takes the panel's updates k = k0..k1-1 in
//     increasing k (threads over trailing columns; each column stays in cache
//     while the panel streams);
//   * inverse: groups of kRhs unit right-hand sides are solved together
//     (row-major n x kRhs scratch), so L is streamed once per group instead of
//     once per column.
bool spd_inverse(const Mat& b, Mat& x) {
  const int n = b.rows;
  Mat l = b;
  double max_diag = 0.0;
  for (int i = 0; i < n; ++i) max_diag = std::max(max_diag, std::abs(b(i, i)));
  constexpr int kPanel = 48;
  for (int k0 = 0; k0 < n; k0 += kPanel) {
    const int k1 = std::min(n, k0 + kPanel);
    // unblocked factorization of the panel columns k0..k1-1 (rows k..n-1)
    for (int k = k0; k < k1; ++k) {
      double d = l(k, k);
      if (!(d > 1e-13 * max_diag)) return false;
      d = std::sqrt(d);
      l(k, k) = d;
      double* ck = l.col(k);
      for (int i = k + 1; i < n; ++i) ck[i] /= d;
      for (int j = k + 1; j < k1; ++j) {
        const double f = ck[j];
        if (f == 0.0) continue;
        double* cj = l.col(j);
        for (int i = j; i < n; ++i) cj[i] -= ck[i] * f;
      }
    }
    // trailing columns: the panel's updates in increasing k
    auto update = [&](int j) {
      double* cj = l.col(j);
      for (int k = k0; k < k1; ++k) {
        const double* ck = l.col(k);
        const double f = ck[j];
        if (f == 0.0) continue;
        for (int i = j; i < n; ++i) cj[i] -= ck[i] * f;
      }
    };
    if (n - k1 > 256) {
      parallel_for(k1, n, update);
    } else {
      for (int j = k1; j < n; ++j) update(j);
    }
  }
  // X = L^-T L^-1: solve L Y = I, then L^T X = Y, kRhs columns at a time.
  x = Mat(n, n);
  constexpr int kRhs = 16;
  const int groups = (n + kRhs - 1) / kRhs;
  parallel_for(0, groups, [&](int gi) {
    const int c0 = gi * kRhs;
    const int nc = std::min(kRhs, n - c0);
    std::vector<double> y(static_cast<std::size_t>(n) * kRhs, 0.0);  // y[i * kRhs + r]
    for (int r = 0; r < nc; ++r) y[static_cast<std::size_t>(c0 + r) * kRhs + r] = 1.0;
    // forward: column r's solve starts at k = c0 + r (entries above are 0 and
    // the unblocked solve skips zero pivots' updates)
    for (int k = c0; k < n; ++k) {
      const double dk = l(k, k);
      double* yk = &y[static_cast<std::size_t>(k) * kRhs];
      double v[kRhs];
      bool any = false;
      for (int r = 0; r < kRhs; ++r) {
        if (r < nc && k >= c0 + r) yk[r] /= dk;
        v[r] = (r < nc && k >= c0 + r) ? yk[r] : 0.0;
        any |= v[r] != 0.0;
      }
      if (!any) continue;
      const double* lk = l.col(k);
      for (int i = k + 1; i < n; ++i) {
        double* yi = &y[static_cast<std::size_t>(i) * kRhs];
        const double li = lk[i];
        for (int r = 0; r < kRhs; ++r)
          if (v[r] != 0.0) yi[r] -= li * v[r];
      }
    }
    for (int k = n - 1; k >= 0; --k) {
      const double* lk = l.col(k);
      double s[kRhs];
      double* yk = &y[static_cast<std::size_t>(k) * kRhs];
      for (int r = 0; r < kRhs; ++r) s[r] = yk[r];
      for (int i = k + 1; i < n; ++i) {
        const double li = lk[i];
        const double* yi = &y[static_cast<std::size_t>(i) * kRhs];
        for (int r = 0; r < kRhs; ++r) s[r] -= li * yi[r];
      }
      const double dk = l(k, k);
      for (int r = 0; r < kRhs; ++r) yk[r] = s[r] / dk;
    }
    for (int r = 0; r < nc; ++r) {
      double* xc = x.col(c0 + r);
      for (int i = 0; i < n; ++i) xc[i] = y[static_cast<std::size_t>(i) * kRhs + r];
    }
  }, 2);
  // symmetrize to remove rounding asymmetry (X is symmetric in exact arithmetic)
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i) {
      const double v = 0.5 * (x(i, j) + x(j, i));
      x(i, j) = v;
      x(j, i) = v;
    }
  return true;
}

}  // namespace oracle
