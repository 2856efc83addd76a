// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Minimal dense linear algebra replacing the reference's Eigen3 calls, keeping
// each call site's DECISION RULE:
//   * FullPivLU with complete pivoting and Eigen's rank rule
//     (|pivot| > threshold * max|pivot|), used for the Woodbury capacitance
//     (dc_engine.cpp:248-263, setThreshold(1e-10)).
//   * Singular values by one-sided Jacobi, used for the sigma_min < 1e-8 test of
//     the flow-compensation matrix (dc_engine.cpp:346-349).
//   * Base inverse X = B_red^-1 (dc_engine.cpp:107-110, importer.cpp:377): the
//     reference uses FullPivLU().inverse(); B_red of a grid is symmetric positive
//     definite iff the grid is connected, so the oracle factors it by Cholesky
//     (backward stable, same singular/non-singular decision, O(n^3/3) instead of
//     O(2n^3/3) with full pivoting) and reports singularity on a non-positive pivot.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;

// Column-major dense matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<std::size_t>(j) * rows + i]; }
  double operator()(int i, int j) const { return a[static_cast<std::size_t>(j) * rows + i]; }
  double* col(int j) { return a.data() + static_cast<std::size_t>(j) * rows; }
  const double* col(int j) const { return a.data() + static_cast<std::size_t>(j) * rows; }
};

// Complete-pivoting LU with Eigen's FullPivLU rank semantics.
class FullPivLU {
 public:
  void compute(const Mat& m) {
    lu_ = m;
    n_ = m.rows;
    row_perm_.resize(n_);
    col_perm_.resize(n_);
    for (int i = 0; i < n_; ++i) row_perm_[i] = col_perm_[i] = i;
    max_pivot_ = 0.0;
    nonzero_pivots_ = n_;
    for (int k = 0; k < n_; ++k) {
      // largest magnitude in the trailing corner, first hit in column-major order
      int br = k, bc = k;
      double big = -1.0;
      for (int j = k; j < n_; ++j)
        for (int i = k; i < n_; ++i) {
          double v = std::abs(lu_(i, j));
          if (v > big) {
            big = v;
            br = i;
            bc = j;
          }
        }
      if (big == 0.0) {
        nonzero_pivots_ = k;
        break;
      }
      if (big > max_pivot_) max_pivot_ = big;
      if (br != k) {
        for (int j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(br, j));
        std::swap(row_perm_[k], row_perm_[br]);
      }
      if (bc != k) {
        for (int i = 0; i < n_; ++i) std::swap(lu_(i, k), lu_(i, bc));
        std::swap(col_perm_[k], col_perm_[bc]);
      }
      const double piv = lu_(k, k);
      for (int i = k + 1; i < n_; ++i) lu_(i, k) /= piv;
      for (int j = k + 1; j < n_; ++j) {
        const double r = lu_(k, j);
        if (r == 0.0) continue;
        for (int i = k + 1; i < n_; ++i) lu_(i, j) -= lu_(i, k) * r;
      }
    }
  }
  void set_threshold(double t) { threshold_ = t; }
  int rank() const {
    const double cut = std::abs(max_pivot_) * threshold_;
    int r = 0;
    for (int i = 0; i < nonzero_pivots_; ++i)
      if (std::abs(lu_(i, i)) > cut) ++r;
    return r;
  }
  bool invertible() const { return rank() == n_; }
  // x = A^-1 b for an invertible A
  Vec solve(const Vec& b) const {
    Vec y(n_);
    for (int i = 0; i < n_; ++i) y[i] = b[row_perm_[i]];
    for (int i = 0; i < n_; ++i)
      for (int k = 0; k < i; ++k) y[i] -= lu_(i, k) * y[k];
    for (int i = n_ - 1; i >= 0; --i) {
      for (int k = i + 1; k < n_; ++k) y[i] -= lu_(i, k) * y[k];
      y[i] /= lu_(i, i);
    }
    Vec x(n_);
    for (int i = 0; i < n_; ++i) x[col_perm_[i]] = y[i];
    return x;
  }
  int size() const { return n_; }

 private:
  Mat lu_;
  int n_ = 0;
  std::vector<int> row_perm_, col_perm_;
  double max_pivot_ = 0.0;
  int nonzero_pivots_ = 0;
  double threshold_ = 1e-10;
};

// Singular values (descending) of a small square matrix, one-sided Jacobi.
inline Vec singular_values(const Mat& m) {
  Mat u = m;
  const int n = m.cols, r = m.rows;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < r; ++i) {
          alpha += u(i, p) * u(i, p);
          beta += u(i, q) * u(i, q);
          gamma += u(i, p) * u(i, q);
        }
        if (gamma == 0.0) continue;
        off = std::max(off, std::abs(gamma) / std::sqrt(alpha * beta));
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < r; ++i) {
          const double up = u(i, p), uq = u(i, q);
          u(i, p) = c * up - s * uq;
          u(i, q) = s * up + c * uq;
        }
      }
    if (off < 1e-15) break;
  }
  Vec sv(n);
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < r; ++i) s += u(i, j) * u(i, j);
    sv[j] = std::sqrt(s);
  }
  std::sort(sv.begin(), sv.end(), [](double a, double b) { return a > b; });
  return sv;
}

// Inverse of a symmetric positive definite matrix via Cholesky.
// Returns false when a pivot is not positive (singular / disconnected grid).
bool spd_inverse(const Mat& b, Mat& x);

}  // namespace oracle
