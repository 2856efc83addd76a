// Base factorization and base-case tables on the device.
// Replaces the DcContext constructor's dense inverse and base solve
// (dc_engine.cpp:88-116) and build_ptdf's gather (importer.cpp:358-401).
#include "engine.cuh"

namespace tgb {

namespace {

__global__ void k_gj_pivot(const double* a, int n, int k, double* row, double* col, double tol, int* bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    col[i] = a[static_cast<size_t>(k) * n + i];
    row[i] = a[static_cast<size_t>(i) * n + k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double p = a[static_cast<size_t>(k) * n + k];
    if (!(p > tol)) *bad = 1;
  }
}

// One Gauss-Jordan elimination step on the column-major matrix.
__global__ void k_gj_update(double* a, int n, int k, const double* row, const double* col) {
  const double p = row[k];
  const double ip = 1.0 / p;
  const size_t total = static_cast<size_t>(n) * n;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx / n), i = static_cast<int>(idx % n);
    double v;
    if (i == k && j == k)
      v = ip;
    else if (i == k)
      v = row[j] * ip;
    else if (j == k)
      v = -col[i] * ip;
    else
      v = fma(-col[i] * ip, row[j], a[idx]);
    a[idx] = v;
  }
}

__global__ void k_max_diag(const double* a, int n, double* out) {
  __shared__ double s[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(a[static_cast<size_t>(i) * n + i]));
  s[threadIdx.x] = m;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

__global__ void k_symmetrize(double* a, int n) {
  const size_t total = static_cast<size_t>(n) * n;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx / n), i = static_cast<int>(idx % n);
    if (i < j) {
      const double v = 0.5 * (a[idx] + a[static_cast<size_t>(i) * n + j]);
      a[idx] = v;
      a[static_cast<size_t>(i) * n + j] = v;
    }
  }
}

__device__ __forceinline__ double xat(const DevGrid& g, int r, int c) {
  return (r < 0 || c < 0) ? 0.0 : g.X[static_cast<size_t>(c) * g.Nr + r];
}

__global__ void k_theta(DevGrid g, const double* p_red, double* theta) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.Nr; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < g.Nr; ++j) acc = fma(g.X[static_cast<size_t>(j) * g.Nr + i], p_red[j], acc);
    theta[i] = acc;
  }
}

__global__ void k_row_static(DevGrid g, const double* f0, double4* out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.E; e += gridDim.x * blockDim.x)
    out[e] = make_double4(f0[e], g.br_b[e], g.br_lim[e], g.br_on[e] ? 1.0 : 0.0);
}

__global__ void k_branch_base(DevGrid g, const double* theta, double* f0, double* tdiag) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < g.E; e += gridDim.x * blockDim.x) {
    const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
    const double b = g.br_b[e];
    const double ti = ri >= 0 ? theta[ri] : 0.0, tj = rj >= 0 ? theta[rj] : 0.0;
    f0[e] = g.br_on[e] ? b * (ti - tj) : 0.0;
    tdiag[e] = b * (xat(g, ri, ri) - 2.0 * xat(g, ri, rj) + xat(g, rj, rj));
  }
}

// T_base[e, k] = b_e a_e^T X a_beta(k), stored in sweep tiles [k / W][e][k % W]
// (W = sweep_tile_k()) so one pipeline stage of the sweep is one contiguous block.
// The diagonal (e = beta(k), the outaged branch itself) is stored as 0: its
// element is never scored (dc_engine.cpp:328-343 removes the branch; every
// sweep excludes e == beta(k)), and its LODF value f_c / (1 - T_ee) would
// otherwise dominate the skip records of row e in its own tile (at cfg4 it
// made ~90 % of the blocks that passed the bounds). The true diagonal stays in
// Tdiag for alpha.
__global__ void k_tk(DevGrid g, double* tk, int W) {
  const size_t total = static_cast<size_t>(g.E) * g.Kpad;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int kk = static_cast<int>(idx % W);
    const size_t rest = idx / W;
    const int e = static_cast<int>(rest % g.E), k = static_cast<int>(rest / g.E) * W + kk;
    double v = 0.0;
    if (k < g.Ks && g.br_on[e] && g.ks_branch[k] != e) {
      const int beta = g.ks_branch[k];
      const int fk = g.red[g.br_from[beta]], tk2 = g.red[g.br_to[beta]];
      const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
      v = g.br_b[e] * ((xat(g, ri, fk) - xat(g, ri, tk2)) - (xat(g, rj, fk) - xat(g, rj, tk2)));
    }
    tk[idx] = v;
  }
}

// alpha0[k] = f0[beta] / (1 - Tdiag[beta]): the contingency's flow factor in
// the unchanged topology (0 for padding).
__global__ void k_alpha0(DevGrid g, double* alpha0) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < g.Kpad; k += gridDim.x * blockDim.x) {
    double a = 0.0;
    if (k < g.Ks) {
      const int beta = g.ks_branch[k];
      const double den = 1.0 - g.Tdiag[beta];
      a = fabs(den) >= 1e-8 ? g.f0[beta] / den : 0.0;
    }
    alpha0[k] = a;
  }
}

// Skip record [tile][e][kRec]: max_k |T_base[e, k]| over each sub-tile, then
// max_k and min_k of T_base[e, k] * alpha0[k] over the tile (the unchanged
// topology's post-contingency flow change on e).
__global__ void k_tmax(DevGrid g, const double* tk, const double* alpha0, float* tmax, int W, int ld) {
  const int ntiles = g.Kpad / W;
  const int total = ntiles * g.E;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int tile = idx / g.E, e = idx % g.E;
    const double* row = tk + (static_cast<size_t>(tile) * g.E + e) * W;
    const double* a0 = alpha0 + static_cast<size_t>(tile) * W;
    float* rec = tmax + (static_cast<size_t>(tile) * ld + e) * kRec;
    const int sw = W / kTmaxSub;
    double dmax = 0.0, dmin = 0.0;
    for (int s = 0; s < kTmaxSub; ++s) {
      double m = 0.0;
      for (int k = s * sw; k < (s + 1) * sw; ++k) {
        m = fmax(m, fabs(row[k]));
        const double d = row[k] * a0[k];
        dmax = fmax(dmax, d);
        dmin = fmin(dmin, d);
      }
      rec[s] = __double2float_ru(m);  // rounded up: the bound stays rigorous
    }
    *reinterpret_cast<double2*>(rec + kTmaxSub) = make_double2(dmax, dmin);  // exact (read as FP64)
  }
}

// Skip records over all profiles: the sub-tile maxima of |T_base| are
// profile-independent, max / min of T_base * alpha0_t over the profiles.
__global__ void k_rec_combine(const float* recs, size_t rec_floats, int n_t, float* out) {
  const size_t n = rec_floats / kRec;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float* r0 = recs + i * kRec;
    float* o = out + i * kRec;
    for (int j = 0; j < kTmaxSub; ++j) o[j] = r0[j];
    double2 d = *reinterpret_cast<const double2*>(r0 + kTmaxSub);
    for (int t = 1; t < n_t; ++t) {
      const double2 dt = *reinterpret_cast<const double2*>(recs + static_cast<size_t>(t) * rec_floats + i * kRec + kTmaxSub);
      d.x = fmax(d.x, dt.x);
      d.y = fmin(d.y, dt.y);
    }
    *reinterpret_cast<double2*>(o + kTmaxSub) = d;
  }
}

// Base N-1 headroom of every branch row: lim_e - max_k |f0_e + T_base[e,k] alpha0_k|
// over the single-branch contingencies (own outage excluded), one warp per row.
// Used once at context creation to order the sweep rows (near-overloaded rows
// last). X is symmetric: x(r_e, c) is read along row r_e (contiguous).
__global__ void k_row_headroom(DevGrid g, double* h) {
  const int lane = threadIdx.x & 31;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < g.E; e += (gridDim.x * blockDim.x) >> 5) {
    const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
    const double b = g.br_b[e], fe = g.f0[e];
    const double* xi = ri >= 0 ? g.X + static_cast<size_t>(ri) * g.Nr : nullptr;
    const double* xj = rj >= 0 ? g.X + static_cast<size_t>(rj) * g.Nr : nullptr;
    double m = fabs(fe);
    for (int k = lane; k < g.Ks && g.br_on[e]; k += 32) {
      const int beta = g.ks_branch[k];
      if (beta == e) continue;
      const int fk = g.red[g.br_from[beta]], tk = g.red[g.br_to[beta]];
      const double ai = xi ? (fk >= 0 ? xi[fk] : 0.0) - (tk >= 0 ? xi[tk] : 0.0) : 0.0;
      const double aj = xj ? (fk >= 0 ? xj[fk] : 0.0) - (tk >= 0 ? xj[tk] : 0.0) : 0.0;
      const double den = 1.0 - g.Tdiag[beta];
      const double a0 = fabs(den) >= 1e-8 ? g.f0[beta] / den : 0.0;
      m = fmax(m, fabs(fe + b * (ai - aj) * a0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) h[e] = g.br_lim[e] - m;
  }
}

// Chunk record per (tile, 32-row chunk), one thread each: the chunk-level
// relaxation of the row records. For every row e of the chunk and element k of
// the tile, |f1| <= max(f0_e + D0max, -(f0_e + D0min)) + |f_c - f0|_e + w_e, so
// a chunk whose rows all satisfy  max|f_c - f0| + max w < min_e headroom_e
// cannot overload (sweep.cu, chunked sweep). Writing the base term as
// |f0_e| + d_e, the same inequality also holds when
//   max_e (|f_c - f0|_e - (lim_e - |f0_e|)) + max_e d_e + max w < 0,
// which ties each row's flow change to its own static headroom; the record
// carries max_e d_e for that second test. The headroom is lowered by
// 1e-9 (lim + |f0| + |D0max| + |D0min|) over the chunk: far more than the
// rounding of any computed f1 (FP64, a few ulps).
__global__ void k_chunk_rec(DevGrid g, float* crec, int W, int ld) {
  const int ntiles = g.Kpad / W, nch = (g.E + kChunkRows - 1) / kChunkRows;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ntiles * nch; idx += gridDim.x * blockDim.x) {
    const int tile = idx / nch, ch = idx % nch;
    float tm[kTmaxSub];
    for (int q = 0; q < kTmaxSub; ++q) tm[q] = 0.0f;
    double h = CUDART_INF, sl = 0.0, dm = 0.0;
    for (int e = ch * kChunkRows; e < min(g.E, (ch + 1) * kChunkRows); ++e) {
      const float* rec = g.Tmax + (static_cast<size_t>(tile) * ld + e) * kRec;
      for (int q = 0; q < kTmaxSub; ++q) tm[q] = fmaxf(tm[q], rec[q]);
      const double2 d0 = *reinterpret_cast<const double2*>(rec + kTmaxSub);
      const double f = g.f0[e], lim = g.br_lim[e];
      const double base = fmax(f + d0.x, -(f + d0.y));  // max_k |f0_e + T_base[e,k] alpha0_k| over the tile
      h = fmin(h, lim - base);
      dm = fmax(dm, base - fabs(f));
      sl = fmax(sl, fabs(lim) + fabs(f) + fabs(d0.x) + fabs(d0.y));
    }
    float* out = crec + static_cast<size_t>(idx) * kRec;
    for (int q = 0; q < kTmaxSub; ++q) out[q] = tm[q];
    // second double: the tile's largest base flow change over |f0| in the chunk,
    // raised by the same rounding margin (the row-coupled test of the chunked sweep)
    *reinterpret_cast<double2*>(out + kTmaxSub) = make_double2(h - 1e-9 * sl, dm + 1e-9 * sl);
  }
}

// Branch-space columns (DevGrid::PhiA / PsiD): one CTA per column, columns
// [0, A) the actions' split columns u_a (moved base-active branch ends, the
// U-column terms of topo.cuh analyze for a split whose moved branches are all
// live), [A, A + D) the disconnectables' removal columns a_d. Row e holds
// (X u)[from_e] - (X u)[to_e] with X u evaluated by build_z's term formula.
__global__ void k_phi_cols(DevGrid g, double* phiA, int* act_nmv, double* psiD) {
  __shared__ int tidx[kMaxTerms];
  __shared__ double tcoef[kMaxTerms];
  __shared__ int nt_s;
  const int col = blockIdx.x;
  if (threadIdx.x == 0) {
    int nt = 0;
    if (col < g.A) {
      const int a = col, s = g.act_station[a], t0 = g.st_term_ptr[s], nterm = g.st_term_ptr[s + 1] - t0;
      const uint8_t* grp = g.act_group + g.act_group_ptr[a];
      int nmv = 0;
      for (int q = 0; q < nterm; ++q) {
        const int kind = g.term_kind[t0 + q], el = g.term_elem[t0 + q];
        if (!grp[q] || kind == 2 || !g.br_on[el]) continue;
        ++nmv;
        const double coef = g.br_b[el] * (kind == 0 ? 1.0 : -1.0);
        const int ri = g.red[g.br_from[el]], rj = g.red[g.br_to[el]];
        if (nt + 2 > kMaxTerms) {
          nt = -1;
          break;
        }
        if (ri >= 0) tidx[nt] = ri, tcoef[nt++] = coef;
        if (rj >= 0) tidx[nt] = rj, tcoef[nt++] = -coef;
      }
      act_nmv[a] = nt < 0 ? -1 : nmv;
    } else {
      const int e = g.disc[col - g.A];
      const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
      if (ri >= 0) tidx[nt] = ri, tcoef[nt++] = 1.0;
      if (rj >= 0) tidx[nt] = rj, tcoef[nt++] = -1.0;
    }
    nt_s = nt;
  }
  __syncthreads();
  const int nt = nt_s;
  if (nt < 0) return;
  double* out = col < g.A ? phiA + static_cast<size_t>(col) * g.E : psiD + static_cast<size_t>(col - g.A) * g.E;
  for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
    const int rf = g.red[g.br_from[e]], rt = g.red[g.br_to[e]];
    double zf = 0.0, zt = 0.0;
    if (rf >= 0)
      for (int p = 0; p < nt; ++p) zf = fma(tcoef[p], g.X[static_cast<size_t>(tidx[p]) * g.Nr + rf], zf);
    if (rt >= 0)
      for (int p = 0; p < nt; ++p) zt = fma(tcoef[p], g.X[static_cast<size_t>(tidx[p]) * g.Nr + rt], zt);
    out[e] = zf - zt;
  }
}

}  // namespace

void launch_phi_columns(const DevGrid& g, double* phiA, int* act_nmv, double* psiD, cudaStream_t stream) {
  if (g.A + g.D > 0) k_phi_cols<<<g.A + g.D, 256, 0, stream>>>(g, phiA, act_nmv, psiD);
}

void launch_chunk_records(const DevGrid& g, float* crec, cudaStream_t stream) {
  const int n = (g.Kpad / sweep_tile_k()) * ((g.E + kChunkRows - 1) / kChunkRows);
  if (n > 0) k_chunk_rec<<<(n + 255) / 256, 256, 0, stream>>>(g, crec, sweep_tile_k(), g.E + sweep_chunk());
}

void launch_row_headroom(const DevGrid& g, const double* p_red, double* theta0, double* f0, double* tdiag, double* h,
                         cudaStream_t stream) {
  k_theta<<<(g.Nr + 255) / 256 + 1, 256, 0, stream>>>(g, p_red, theta0);
  DevGrid g2 = g;
  g2.theta0 = theta0;
  k_branch_base<<<(g.E + 255) / 256 + 1, 256, 0, stream>>>(g2, theta0, f0, tdiag);
  g2.f0 = f0;
  g2.Tdiag = tdiag;
  k_row_headroom<<<148 * 8, 256, 0, stream>>>(g2, h);
}

void launch_rec_combine(const float* recs, size_t rec_floats, int n_t, float* out, cudaStream_t stream) {
  k_rec_combine<<<1024, 256, 0, stream>>>(recs, rec_floats, n_t, out);
}

// PTDF of importer.cpp:358-401: row e = b_e (X[red(from_e), :] - X[red(to_e), :])
// over the full node index (slack column zero), 0 rows for out-of-service
// branches; out is [E][N] row-major.
__global__ void k_ptdf(int N, int E, int Nr, const int* red, const int* from, const int* to, const double* b,
                       const uint8_t* on, const double* X, double* out) {
  const size_t total = static_cast<size_t>(E) * N;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int e = static_cast<int>(idx / N), v = static_cast<int>(idx % N);
    const int rv = red[v], i = red[from[e]], j = red[to[e]];
    double val = 0.0;
    if (on[e] && rv >= 0) {
      const double xi = i >= 0 ? X[static_cast<size_t>(rv) * Nr + i] : 0.0;  // X symmetric
      const double xj = j >= 0 ? X[static_cast<size_t>(rv) * Nr + j] : 0.0;
      val = b[e] * (xi - xj);
    }
    out[idx] = val;
  }
}

void launch_ptdf(int N, int E, int Nr, const int* red, const int* from, const int* to, const double* b,
                 const uint8_t* on, const double* X, double* out, cudaStream_t stream) {
  const size_t total = static_cast<size_t>(E) * N;
  if (total == 0) return;
  k_ptdf<<<static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16)), 256, 0, stream>>>(N, E, Nr, red, from, to,
                                                                                                  b, on, X, out);
}

bool device_spd_inverse(double* a, int n, cudaStream_t stream) {
  if (n == 0) return true;
  double *row = nullptr, *col = nullptr, *dmax = nullptr;
  int* bad = nullptr;
  cudaMalloc(&row, n * sizeof(double));
  cudaMalloc(&col, n * sizeof(double));
  cudaMalloc(&dmax, sizeof(double));
  cudaMalloc(&bad, sizeof(int));
  cudaMemsetAsync(bad, 0, sizeof(int), stream);
  k_max_diag<<<1, 256, 0, stream>>>(a, n, dmax);
  double hmax = 0.0;
  cudaMemcpyAsync(&hmax, dmax, sizeof(double), cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  const double tol = 1e-13 * hmax;
  const size_t total = static_cast<size_t>(n) * n;
  const int upd_blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
  for (int k = 0; k < n; ++k) {
    k_gj_pivot<<<(n + 255) / 256, 256, 0, stream>>>(a, n, k, row, col, tol, bad);
    k_gj_update<<<upd_blocks, 256, 0, stream>>>(a, n, k, row, col);
  }
  k_symmetrize<<<upd_blocks, 256, 0, stream>>>(a, n);
  int hbad = 0;
  cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  cudaFree(row);
  cudaFree(col);
  cudaFree(dmax);
  cudaFree(bad);
  return hbad == 0;
}

void launch_row_static(const DevGrid& g, const double* f0, double4* out, cudaStream_t stream) {
  if (g.E > 0) k_row_static<<<(g.E + 255) / 256, 256, 0, stream>>>(g, f0, out);
}

void launch_base_tables(const DevGrid& g, const double* p_red, double* theta0, double* f0, double* tdiag, double* tk,
                        float* tmax, double* alpha0, cudaStream_t stream) {
  k_theta<<<(g.Nr + 255) / 256 + 1, 256, 0, stream>>>(g, p_red, theta0);
  DevGrid g2 = g;
  g2.theta0 = theta0;
  k_branch_base<<<(g.E + 255) / 256 + 1, 256, 0, stream>>>(g2, theta0, f0, tdiag);
  const size_t total = static_cast<size_t>(g.E) * g.Kpad;
  if (total > 0) {
    k_tk<<<static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 32)), 256, 0, stream>>>(g2, tk, sweep_tile_k());
    g2.f0 = f0;
    g2.Tdiag = tdiag;
    k_alpha0<<<(g.Kpad + 255) / 256 + 1, 256, 0, stream>>>(g2, alpha0);
    k_tmax<<<static_cast<int>(std::min<size_t>((total / sweep_tile_k() + 255) / 256 + 1, 148 * 32)), 256, 0, stream>>>(
        g2, tk, alpha0, tmax, sweep_tile_k(), g.E + sweep_chunk());
  }
}

}  // namespace tgb
