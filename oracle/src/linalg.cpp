// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
#include "linalg.hpp"

#include <algorithm>
#include <thread>

namespace oracle {

namespace {
// static-partition parallel loop over [lo, hi) (the image has no libgomp)
template <class F>
void parallel_for(int lo, int hi, F&& f) {
  const int n = hi - lo;
  const int workers = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), n / 64));
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
// Threads over independent columns keep the 1k-7k node grids tractable.
bool spd_inverse(const Mat& b, Mat& x) {
  const int n = b.rows;
  Mat l = b;
  double max_diag = 0.0;
  for (int i = 0; i < n; ++i) max_diag = std::max(max_diag, std::abs(b(i, i)));
  for (int k = 0; k < n; ++k) {
    double d = l(k, k);
    if (!(d > 1e-13 * max_diag)) return false;
    d = std::sqrt(d);
    l(k, k) = d;
    double* ck = l.col(k);
    for (int i = k + 1; i < n; ++i) ck[i] /= d;
    auto update = [&](int j) {
      const double f = ck[j];
      if (f == 0.0) return;
      double* cj = l.col(j);
      for (int i = j; i < n; ++i) cj[i] -= ck[i] * f;
    };
    if (n - k > 512) {
      parallel_for(k + 1, n, update);
    } else {
      for (int j = k + 1; j < n; ++j) update(j);
    }
  }
  // X = L^-T L^-1: solve L Y = I column by column, then L^T X = Y.
  x = Mat(n, n);
  parallel_for(0, n, [&](int c) {
    Vec y(n, 0.0);
    y[c] = 1.0;
    for (int k = c; k < n; ++k) {
      y[k] /= l(k, k);
      const double v = y[k];
      if (v == 0.0) continue;
      const double* lk = l.col(k);
      for (int i = k + 1; i < n; ++i) y[i] -= lk[i] * v;
    }
    for (int k = n - 1; k >= 0; --k) {
      const double* lk = l.col(k);
      double s = y[k];
      for (int i = k + 1; i < n; ++i) s -= lk[i] * y[i];
      y[k] = s / l(k, k);
    }
    double* xc = x.col(c);
    for (int i = 0; i < n; ++i) xc[i] = y[i];
  });
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
