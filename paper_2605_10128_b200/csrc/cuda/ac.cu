// Batched AC Newton-Raphson cases (see ac.cuh). One CTA per case; the
// reference's per-case algorithm (ac_validator.cpp:37-272) with the case's
// dense Ybus / Jacobian in the CTA's workspace.
#include <cfloat>

#include "ac.cuh"

namespace tgb {

namespace {

constexpr double kBaseMva = 100.0;  // ac_validator.cpp:14

// Workspace of one case (offsets in bytes, 16-byte aligned sections).
struct AcWs {
  double *J, *Gd, *Bd, *vm, *va, *P, *Q, *psp, *qsp, *vset, *dx, *lm, *red;
  double *yb, *sc;  // [2E] y_ft of each live branch; [2 * 2E] sin / cos per branch-end slot of the grid CSR
  int *bus_of, *node_of, *ang, *mag, *ang_pos, *mag_pos, *pv, *reach, *ired;
  uint8_t* live;
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline size_t ws_layout(int n_bus, int nu, int E, unsigned char* base, AcWs* w) {
  size_t off = 0;
  auto take_d = [&](size_t n) {
    double* p = reinterpret_cast<double*>(base + off);
    off = align16(off + n * sizeof(double));
    return p;
  };
  auto take_i = [&](size_t n) {
    int* p = reinterpret_cast<int*>(base + off);
    off = align16(off + n * sizeof(int));
    return p;
  };
  const size_t nb = static_cast<size_t>(n_bus), nn = static_cast<size_t>(nu);
  AcWs t{};
  t.J = take_d(nn * nn);
  t.Gd = take_d(nb);
  t.Bd = take_d(nb);
  t.vm = take_d(nb);
  t.va = take_d(nb);
  t.P = take_d(nb);
  t.Q = take_d(nb);
  t.psp = take_d(nb);
  t.qsp = take_d(nb);
  t.vset = take_d(nb);
  t.dx = take_d(nn);
  t.lm = take_d(nn);
  t.red = take_d(64);
  t.yb = take_d(2 * static_cast<size_t>(E));
  t.sc = take_d(4 * static_cast<size_t>(E));
  t.bus_of = take_i(nb);
  t.node_of = take_i(nb);
  t.ang = take_i(nn);
  t.mag = take_i(nn);
  t.ang_pos = take_i(nb);
  t.mag_pos = take_i(nb);
  t.pv = take_i(nb);
  t.reach = take_i(nb);
  t.ired = take_i(64);
  t.live = reinterpret_cast<uint8_t*>(base + off);
  off = align16(off + static_cast<size_t>(E));
  if (w) *w = t;
  return off;
}

// ---- block reductions (every thread calls; deterministic order) -----------
template <int NT>
__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < NT / 32; ++i) r = fmax(r, red[i]);
  return r;
}

template <int NT>
__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < NT / 32; ++i) r += red[i];
  return r;
}

template <int NT>
__device__ int block_sum_int(int v, int* ired) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ired[w] = v;
  __syncthreads();
  int r = 0;
  for (int i = 0; i < NT / 32; ++i) r += ired[i];
  return r;
}

// first index of the largest value (values < 0 never win: the caller passes -1
// for no candidate)
template <int NT>
__device__ int block_argmax(double v, int idx, double* red, int* ired) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) v = ov, idx = oi;
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v, ired[w] = idx;
  __syncthreads();
  double bv = red[0];
  int bi = ired[0];
  for (int i = 1; i < NT / 32; ++i)
    if (red[i] > bv || (red[i] == bv && ired[i] < bi)) bv = red[i], bi = ired[i];
  return bi;
}

// block_argmax for the LU's column loop: the LU's own barriers already order
// the previous column's reads of red / ired before this write, and the
// per-warp winners are reduced by shuffles (one total order on (value, index),
// so the result is block_argmax's)
template <int NT>
__device__ int lu_argmax(double v, int idx, double* red, int* ired) {
  // (value, index) as an ordered key: v is -1 (no candidate) or some |a_ik|
  // (never NaN), whose bit pattern orders like the value; + 1 puts 0.0 above
  // "no candidate". The largest key, then the smallest index among its
  // holders: three REDUX steps per warp (the shuffle butterfly's result).
  const unsigned long long key = v >= 0.0 ? static_cast<unsigned long long>(__double_as_longlong(v)) + 1ull : 0ull;
  auto warp_pick = [](unsigned long long k, unsigned i, unsigned long long& wk) {
    const unsigned hi = static_cast<unsigned>(k >> 32), lo = static_cast<unsigned>(k);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    wk = (static_cast<unsigned long long>(mhi) << 32) | mlo;
    return __reduce_min_sync(0xffffffffu, hi == mhi && lo == mlo ? i : 0xffffffffu);
  };
  unsigned long long wk;
  unsigned wi = warp_pick(key, static_cast<unsigned>(idx), wk);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = NT / 32;
  static_assert(NW >= 2 && (NW & (NW - 1)) == 0, "warps per CTA: a power of two");
  unsigned long long* rk = reinterpret_cast<unsigned long long*>(red);
  if (lane == 0) rk[w] = wk, ired[w] = static_cast<int>(wi);
  __syncthreads();
  // every group of NW lanes holds a full copy of the per-warp winners
  wi = warp_pick(rk[lane & (NW - 1)], static_cast<unsigned>(ired[lane & (NW - 1)]), wk);
  return static_cast<int>(wi);
}

__device__ __forceinline__ bool in_list(const int* lo, const int* hi, int x) {
  for (const int* p = lo; p < hi; ++p)
    if (*p == x) return true;
  return false;
}

// Series and shunt admittances of branch e in the pi model with the tap on the
// from side: yff = (ys + j bc/2) / t^2, yft = ytf = -ys / t, ytt = ys + j bc/2
// (ac_validator.cpp:123-133).
struct BranchY {
  double ffr, ffi, ftr, fti, ttr, tti;
};
__device__ __forceinline__ BranchY branch_y(const AcGrid& g, int e) {
  const double r = g.br_r[e], x = g.br_x[e], t = g.br_tap[e];
  const double d = r * r + x * x;
  const double ysr = r / d, ysi = -x / d;  // 1 / (r + j x)
  const double shi = g.br_bc[e] / 2.0;
  BranchY y;
  y.ffr = ysr / (t * t);
  y.ffi = (ysi + shi) / (t * t);
  y.ftr = -ysr / t;
  y.fti = -ysi / t;
  y.ttr = ysr;
  y.tti = ysi + shi;
  return y;
}

// LU with row partial pivoting of the nu x nu row-major J, solving J x = dx in
// place (dx <- x). Eigen::PartialPivLU's pivot rule (first largest |a_ik|);
// a zero pivot leaves non-finite entries, tested by the caller like the
// reference's step.allFinite() (ac_validator.cpp:239-241).
template <int NT>
__device__ __forceinline__ void lu_solve(double* J, double* dx, double* lm, int nu, double* red, int* ired) {
  const int tid = threadIdx.x;
  for (int k = 0; k < nu; ++k) {
    double best = -1.0;
    int bi = nu;
    for (int i = k + tid; i < nu; i += NT) {
      const double a = fabs(J[static_cast<size_t>(i) * nu + k]);
      if (a > best) best = a, bi = i;
    }
    int p = lu_argmax<NT>(best, bi, red, ired);
    if (p >= nu) p = k;
    if (p != k) {
      for (int j = k + tid; j < nu; j += NT) {
        const double t = J[static_cast<size_t>(k) * nu + j];
        J[static_cast<size_t>(k) * nu + j] = J[static_cast<size_t>(p) * nu + j];
        J[static_cast<size_t>(p) * nu + j] = t;
      }
      if (tid == 0) {
        const double t = dx[k];
        dx[k] = dx[p];
        dx[p] = t;
      }
    }
    __syncthreads();
    const double piv = J[static_cast<size_t>(k) * nu + k];
    const double bk = dx[k];
    for (int i = k + 1 + tid; i < nu; i += NT) {
      const double l = J[static_cast<size_t>(i) * nu + k] / piv;
      lm[i] = l;
      dx[i] -= l * bk;
    }
    __syncthreads();
    // trailing update: warps over rows, lanes over columns (row-major J, so a
    // warp touches consecutive words)
    // (two rows per warp: each pivot-row element is loaded once for both)
    const double* rk = J + static_cast<size_t>(k) * nu;
    for (int i = k + 1 + 2 * (tid >> 5); i < nu; i += 2 * (NT / 32)) {
      const bool two = i + 1 < nu;
      const double l0 = lm[i], l1 = two ? lm[i + 1] : 0.0;
      if (l0 == 0.0 && l1 == 0.0) continue;
      double* r0 = J + static_cast<size_t>(i) * nu;
      double* r1 = r0 + nu;
      if constexpr (NT >= 256) {
        // four column groups per pass, all loads issued before the stores (the
        // rows may alias as far as the compiler knows, so a plain loop would wait
        // out each load's latency: the scratch path's rows live in L1 / L2)
        for (int jb = k + 1 + (tid & 31); jb < nu; jb += 4 * 32) {
          double x[4], a0[4], a1[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = jb + 32 * u;
            x[u] = j < nu ? rk[j] : 0.0;
            a0[u] = j < nu ? r0[j] : 0.0;
            a1[u] = two && j < nu ? r1[j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = jb + 32 * u;
            if (j >= nu) break;
            if (l0 != 0.0) {
              a0[u] -= l0 * x[u];
              r0[j] = a0[u];
            }
            if (l1 != 0.0) {
              a1[u] -= l1 * x[u];
              r1[j] = a1[u];
            }
          }
        }
      } else {
        for (int j = k + 1 + (tid & 31); j < nu; j += 32) {
          const double x = rk[j];
          if (l0 != 0.0) r0[j] -= l0 * x;
          if (l1 != 0.0) r1[j] -= l1 * x;
        }
      }
    }
    __syncthreads();
  }
  for (int i = nu - 1; i >= 0; --i) {
    if (tid == 0) dx[i] = dx[i] / J[static_cast<size_t>(i) * nu + i];
    __syncthreads();
    const double xi = dx[i];
    for (int r = tid; r < i; r += NT) dx[r] -= J[static_cast<size_t>(r) * nu + i] * xi;
    __syncthreads();
  }
}

// The Ybus off-diagonal terms of bus i as a sum over its live branches
// (sparse form of ac_validator.cpp:117-141; parallel branches add up like the
// dense matrix's entries): fn(k, g_ik, b_ik) for every branch to bus k. The
// candidates are the base node's incident branches (a split section's: the
// station node's), kept if one of their current ends is bus i's node.
template <class F>
__device__ __forceinline__ void for_each_branch_of_bus(const AcGrid& g, const AcWs& w, const int* ef, const int* et,
                                                       const int* split_node, int i, F&& fn) {
  const int v = w.node_of[i];
  const int base = v < g.N ? v : split_node[v - g.N];
  for (int p = g.node_ptr[base]; p < g.node_ptr[base + 1]; ++p) {
    const int e = g.node_br[p];
    if (!w.live[e]) continue;
    const int a = ef[e], b = et[e];
    if (a != v && b != v) continue;  // this end moved to another section
    fn(w.bus_of[a == v ? b : a], w.yb[2 * e], w.yb[2 * e + 1], p);  // y_ft = y_tf
  }
}

template <int NT>
__device__ void solve_case(const AcGrid& g, const AcTopo& tp, const AcCases& io, const AcSolver& sv, int c,
                           const AcWs& w) {
  const int tid = threadIdx.x;
  const int E = g.E, I = g.I;
  const int gi = io.genome[c], ci = io.cont[c];
  const int nnew = tp.n_new[gi];
  const int nbus = g.N + nnew;
  const int* ef = tp.from + static_cast<size_t>(gi) * E;
  const int* et = tp.to + static_cast<size_t>(gi) * E;
  const uint8_t* rem = tp.removed + static_cast<size_t>(gi) * E;
  const int* inode = tp.inj_node + static_cast<size_t>(gi) * I;
  const int* split_node = tp.split_node + static_cast<size_t>(gi) * tp.split_stride;
  const int* cb0 = ci >= 0 ? g.cont_br + g.cont_br_ptr[ci] : nullptr;
  const int* cb1 = ci >= 0 ? g.cont_br + g.cont_br_ptr[ci + 1] : nullptr;
  const int* cj0 = ci >= 0 ? g.cont_inj + g.cont_inj_ptr[ci] : nullptr;
  const int* cj1 = ci >= 0 ? g.cont_inj + g.cont_inj_ptr[ci + 1] : nullptr;
  const bool fold = io.fold != nullptr && io.fold_case != nullptr && io.fold_case[c];

  // live branches (ac_validator.cpp:45-49) and reachability from the slack
  // (52-73) by label propagation over the live edges
  for (int e = tid; e < E; e += NT) w.live[e] = g.br_on[e] && !rem[e] && !in_list(cb0, cb1, e);
  for (int v = tid; v < nbus; v += NT) w.reach[v] = v == g.slack;
  __syncthreads();
  for (;;) {
    bool changed = false;
    for (int e = tid; e < E; e += NT) {
      if (!w.live[e]) continue;
      const int a = ef[e], b = et[e];
      if (w.reach[a] != w.reach[b]) {
        w.reach[a] = 1;
        w.reach[b] = 1;
        changed = true;
      }
    }
    if (!__syncthreads_or(changed)) break;
  }
  // a live component without the slack, or a stranded nonzero injection:
  // not converged after zero iterations (ac_validator.cpp:74-82)
  bool bad = false;
  for (int e = tid; e < E; e += NT)
    if (w.live[e] && !w.reach[ef[e]]) bad = true;
  for (int i = tid; i < I; i += NT)
    if ((g.inj_p[i] != 0.0 || g.inj_q[i] != 0.0) && !w.reach[inode[i]] && !in_list(cj0, cj1, i)) bad = true;
  const bool floating = __syncthreads_or(bad);

  int* sh = w.ired + 32;  // n, slack bus, n angles, n magnitudes
  if (!floating) {
    // bus numbering, specified injections, PV buses (ac_validator.cpp:84-115),
    // Ybus in branch order (117-141), flat start and unknown order (143-156)
    if (tid == 0) {
      int n = 0;
      for (int v = 0; v < nbus; ++v) {
        w.bus_of[v] = w.reach[v] ? n : -1;
        if (w.reach[v]) w.node_of[n++] = v;
      }
      for (int b = 0; b < n; ++b) w.psp[b] = 0.0, w.qsp[b] = 0.0, w.vset[b] = 1.0, w.pv[b] = 0;
      for (int i = 0; i < I; ++i) {
        if (in_list(cj0, cj1, i)) continue;
        const int b = w.bus_of[inode[i]];
        if (b < 0) continue;
        if (g.inj_gen[i]) {
          w.psp[b] += g.inj_p[i] / kBaseMva;
          if (g.inj_has_vset[i]) {
            if (!w.pv[b]) w.vset[b] = g.inj_vset[i];
            w.pv[b] = 1;
          } else {
            w.qsp[b] += g.inj_q[i] / kBaseMva;
          }
        } else {
          w.psp[b] -= g.inj_p[i] / kBaseMva;
          w.qsp[b] -= g.inj_q[i] / kBaseMva;
        }
      }
      // Ybus diagonal in branch order (the off-diagonal terms are summed per bus
      // over its branches, for_each_branch_of_bus)
      for (int b = 0; b < n; ++b) w.Gd[b] = 0.0, w.Bd[b] = 0.0;
      for (int e = 0; e < E; ++e) {
        if (!w.live[e]) continue;
        const BranchY y = branch_y(g, e);
        const int f = w.bus_of[ef[e]], t = w.bus_of[et[e]];
        w.Gd[f] += y.ffr, w.Bd[f] += y.ffi;
        w.Gd[t] += y.ttr, w.Bd[t] += y.tti;
      }
      for (int v = 0; v < g.N; ++v)
        if (w.bus_of[v] >= 0 && g.node_shunt[v] != 0.0) w.Bd[w.bus_of[v]] += g.node_shunt[v];
      const int sl = w.bus_of[g.slack];
      int na = 0, nm = 0;
      for (int b = 0; b < n; ++b) {
        w.vm[b] = (w.pv[b] || b == sl) ? w.vset[b] : 1.0;
        w.va[b] = 0.0;
        w.ang_pos[b] = -1;
        w.mag_pos[b] = -1;
        if (b == sl) continue;
        w.ang_pos[b] = na;
        w.ang[na++] = b;
      }
      for (int b = 0; b < n; ++b)
        if (b != sl && !w.pv[b]) w.mag_pos[b] = nm, w.mag[nm++] = b;
      sh[0] = n, sh[1] = sl, sh[2] = na, sh[3] = nm;
    }
    __syncthreads();
  }
  const int n = floating ? 0 : sh[0];
  const int na = floating ? 0 : sh[2], nm = floating ? 0 : sh[3], nu = na + nm;

  bool ok = false;
  int iters = 0;
  if (!floating) {
    // the live branches' y_ft, formed once per case (the Newton loop reads them
    // twice per iteration)
    for (int e = tid; e < E; e += NT) {
      if (!w.live[e]) continue;
      const BranchY y = branch_y(g, e);
      w.yb[2 * e] = y.ftr;
      w.yb[2 * e + 1] = y.fti;
    }
    __syncthreads();
    for (int it = 1; it <= sv.max_iter; ++it) {  // ac_validator.cpp:175-244
      // bus injections (159-173)
      for (int i = tid; i < n; i += NT) {
        const double vi = w.vm[i], ai = w.va[i];
        double p = vi * vi * w.Gd[i], q = -vi * vi * w.Bd[i];
        for_each_branch_of_bus(g, w, ef, et, split_node, i, [&](int k, double gik, double bik, int slot) {
          double s, co;
          sincos(ai - w.va[k], &s, &co);
          w.sc[2 * slot] = s;  // reused by the Jacobian (same angles)
          w.sc[2 * slot + 1] = co;
          p += vi * w.vm[k] * (gik * co + bik * s);
          q += vi * w.vm[k] * (gik * s - bik * co);
        });
        w.P[i] = p;
        w.Q[i] = q;
      }
      __syncthreads();
      double wl = 0.0;
      for (int r = tid; r < nu; r += NT) {
        const double m = r < na ? w.psp[w.ang[r]] - w.P[w.ang[r]] : w.qsp[w.mag[r - na]] - w.Q[w.mag[r - na]];
        w.dx[r] = m;
        wl = fmax(wl, fabs(m));  // std::max(worst, |m|): a NaN mismatch is skipped, like the reference
      }
      const double worst = block_max<NT>(wl, w.red);
      iters = it;
      if (!isfinite(worst) || worst > 1e8) break;
      if (worst < sv.tol) {
        ok = true;
        break;
      }
      if (it == sv.max_iter) break;
      // Jacobian (186-236): zeroed, then each bus fills its own rows (diagonal
      // terms, and one term per branch for the neighbour's columns)
      for (int idx = tid; idx < nu * nu; idx += NT) w.J[idx] = 0.0;
      __syncthreads();
      for (int i = tid; i < n; i += NT) {
        const int rp = w.ang_pos[i], rq = w.mag_pos[i] >= 0 ? na + w.mag_pos[i] : -1;
        if (rp < 0 && rq < 0) continue;  // the slack bus has no row
        const double vi = w.vm[i], gii = w.Gd[i], bii = w.Bd[i];
        double* JP = rp >= 0 ? w.J + static_cast<size_t>(rp) * nu : nullptr;
        double* JQ = rq >= 0 ? w.J + static_cast<size_t>(rq) * nu : nullptr;
        if (JP) {
          JP[rp] = -w.Q[i] - bii * vi * vi;
          if (rq >= 0) JP[rq] = w.P[i] / vi + gii * vi;
        }
        if (JQ) {
          if (rp >= 0) JQ[rp] = w.P[i] - gii * vi * vi;
          JQ[rq] = w.Q[i] / vi - bii * vi;
        }
        for_each_branch_of_bus(g, w, ef, et, split_node, i, [&](int k, double gik, double bik, int slot) {
          const int ct = w.ang_pos[k], cv = w.mag_pos[k] >= 0 ? na + w.mag_pos[k] : -1;
          const double s = w.sc[2 * slot], co = w.sc[2 * slot + 1];  // sincos(va_i - va_k) of the injections
          const double vk = w.vm[k];
          if (JP) {
            if (ct >= 0) JP[ct] += vi * vk * (gik * s - bik * co);
            if (cv >= 0) JP[cv] += vi * (gik * co + bik * s);
          }
          if (JQ) {
            if (ct >= 0) JQ[ct] += -vi * vk * (gik * co + bik * s);
            if (cv >= 0) JQ[cv] += vi * (gik * s - bik * co);
          }
        });
      }
      __syncthreads();
      lu_solve<NT>(w.J, w.dx, w.lm, nu, w.red, w.ired);
      // step.allFinite() (ac_validator.cpp:239-241) tested with the update's
      // barrier: a non-finite step ends the case unconverged, whose voltages
      // are never reported, so applying it first changes no output
      bool fin = true;
      for (int r = tid; r < nu; r += NT) {
        const double d = w.dx[r];
        fin = fin && isfinite(d);
        if (r < na)
          w.va[w.ang[r]] += d;
        else
          w.vm[w.mag[r - na]] += d;
      }
      if (!__syncthreads_and(fin)) break;
    }
  }

  // outputs (ac_validator.cpp:246-272, 274-288)
  if (io.vm)
    for (int v = tid; v < io.vm_stride; v += NT) {
      const int b = ok && v < nbus ? w.bus_of[v] : -1;
      io.vm[static_cast<size_t>(c) * io.vm_stride + v] = b >= 0 ? w.vm[b] : 0.0;
      io.va[static_cast<size_t>(c) * io.vm_stride + v] = b >= 0 ? w.va[b] : 0.0;
    }
  double en = 0.0;
  int cr = 0;
  for (int e = tid; e < E; e += NT) {
    double load = 0.0;
    if (ok && w.live[e]) {
      const BranchY y = branch_y(g, e);
      const int f = w.bus_of[ef[e]], t = w.bus_of[et[e]];
      double sf, cf, st, ct;
      sincos(w.va[f], &sf, &cf);
      sincos(w.va[t], &st, &ct);
      const double vfr = w.vm[f] * cf, vfi = w.vm[f] * sf, vtr = w.vm[t] * ct, vti = w.vm[t] * st;
      // I_f = yff V_f + yft V_t, I_t = ytf V_f + ytt V_t; S = V conj(I)
      const double ifr = y.ffr * vfr - y.ffi * vfi + y.ftr * vtr - y.fti * vti;
      const double ifi = y.ffr * vfi + y.ffi * vfr + y.ftr * vti + y.fti * vtr;
      const double itr = y.ftr * vfr - y.fti * vfi + y.ttr * vtr - y.tti * vti;
      const double iti = y.ftr * vfi + y.fti * vfr + y.ttr * vti + y.tti * vtr;
      const double sfr = vfr * ifr + vfi * ifi, sfi = vfi * ifr - vfr * ifi;
      const double str = vtr * itr + vti * iti, sti = vti * itr - vtr * iti;
      load = fmax(hypot(sfr, sfi), hypot(str, sti)) * kBaseMva;
    }
    if (io.loading) io.loading[static_cast<size_t>(c) * E + e] = load;
    if (ok) {
      const double d = load - g.br_lim[e];
      en += d > 0.0 ? d : 0.0;
      cr += load > g.br_lim[e];
    }
    if (fold && ok) atomicMax(io.fold + static_cast<size_t>(gi) * E + e, static_cast<unsigned long long>(__double_as_longlong(load)));
  }
  const double energy = block_sum<NT>(en, w.red);
  const int crit = block_sum_int<NT>(cr, w.ired);
  if (tid == 0) {
    io.converged[c] = ok;
    io.iterations[c] = iters;
    if (io.energy) io.energy[c] = ok ? energy : 0.0;
    if (io.critical) io.critical[c] = ok ? crit : 0;
    if (fold && !ok && io.nonconverged) atomicAdd(io.nonconverged + gi, 1);
  }
  __syncthreads();
}

// the workspace sections at base, from the layout's offsets (rel = the layout
// at address 0, computed on the host: a kernel parameter, so the section
// pointers cost one add wherever the compiler rematerializes them)
__device__ __forceinline__ AcWs rebase(const AcWs& rel, unsigned char* base) {
  auto d = [&](double* p) { return reinterpret_cast<double*>(base + reinterpret_cast<size_t>(p)); };
  auto i = [&](int* p) { return reinterpret_cast<int*>(base + reinterpret_cast<size_t>(p)); };
  AcWs w;
  w.J = d(rel.J), w.Gd = d(rel.Gd), w.Bd = d(rel.Bd), w.vm = d(rel.vm), w.va = d(rel.va), w.P = d(rel.P);
  w.Q = d(rel.Q), w.psp = d(rel.psp), w.qsp = d(rel.qsp), w.vset = d(rel.vset), w.dx = d(rel.dx);
  w.lm = d(rel.lm), w.red = d(rel.red), w.yb = d(rel.yb), w.sc = d(rel.sc);
  w.bus_of = i(rel.bus_of), w.node_of = i(rel.node_of), w.ang = i(rel.ang), w.mag = i(rel.mag);
  w.ang_pos = i(rel.ang_pos), w.mag_pos = i(rel.mag_pos), w.pv = i(rel.pv), w.reach = i(rel.reach);
  w.ired = i(rel.ired);
  w.live = base + reinterpret_cast<size_t>(rel.live);
  return w;
}

// SMEM: the workspace is the dynamic shared memory (a separate instantiation,
// so every workspace pointer is provably shared: LDS / STS with 32-bit
// addresses instead of generic loads), else the CTA's HBM scratch slot
template <int NT, bool SMEM>
__global__ void __launch_bounds__(NT, NT == 512 ? 2 : (NT == 256 ? (SMEM ? 2 : 4) : 16))
    k_ac_case(AcGrid g, AcTopo tp, AcCases io, AcSolver sv, AcWs rel) {
  extern __shared__ __align__(16) unsigned char ac_smem[];
  // (the scratch instantiation keeps the runtime choice: its generic-pointer
  // code measured faster on the 118-bus case than a provably global base)
  unsigned char* base =
      SMEM || sv.in_smem ? ac_smem : sv.scratch + static_cast<size_t>(blockIdx.x) * sv.ws_bytes;
  const AcWs w = rebase(rel, base);
  if (SMEM || sv.next_case == nullptr) {
    // shared-memory workspace: one CTA per case (the block scheduler balances
    // the uneven Newton runs)
    for (int c = blockIdx.x; c < io.n; c += gridDim.x) solve_case<NT>(g, tp, io, sv, c, w);
  } else {
    // scratch slots (one per resident CTA): cases claimed dynamically
    __shared__ int next_s;
    for (;;) {
      if (threadIdx.x == 0) next_s = static_cast<int>(atomicAdd(sv.next_case, 1u));
      __syncthreads();
      const int c = next_s;
      __syncthreads();
      if (c >= io.n) break;
      solve_case<NT>(g, tp, io, sv, c, w);
    }
  }
}

// apply_genome (genome.cpp:76-110): base endpoints, disconnections removed,
// then each split slot in order moves its group's terminals to node N + j.
__global__ void k_ac_topo(AcGrid g, const int* genomes, int n_a, int n_d, AcTopo t) {
  const int gi = blockIdx.x, E = g.E, I = g.I;
  const int* gen = genomes + static_cast<size_t>(gi) * (n_a + n_d);
  int* from = t.from + static_cast<size_t>(gi) * E;
  int* to = t.to + static_cast<size_t>(gi) * E;
  uint8_t* rem = t.removed + static_cast<size_t>(gi) * E;
  int* inode = t.inj_node + static_cast<size_t>(gi) * I;
  for (int e = threadIdx.x; e < E; e += blockDim.x) from[e] = g.br_from[e], to[e] = g.br_to[e], rem[e] = 0;
  for (int i = threadIdx.x; i < I; i += blockDim.x) inode[i] = g.inj_node[i];
  __syncthreads();
  if (threadIdx.x < n_d) {
    const int d = gen[n_a + threadIdx.x];
    if (d >= 0) rem[g.disc[d]] = 1;
  }
  int nn = 0;
  for (int s = 0; s < n_a; ++s) {
    const int a = gen[s];
    if (a < 0) continue;
    const int st = g.act_station[a];
    const int t0 = g.st_term_ptr[st], nt = g.st_term_ptr[st + 1] - t0;
    if (threadIdx.x == 0) t.split_node[static_cast<size_t>(gi) * t.split_stride + nn] = g.st_node[st];
    const uint8_t* grp = g.act_group + g.act_group_ptr[a];
    const int node = g.N + nn;
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
      if (!grp[k]) continue;
      const int kind = g.term_kind[t0 + k], el = g.term_elem[t0 + k];
      if (kind == 2)
        inode[el] = node;
      else if (kind == 0)
        from[el] = node;
      else
        to[el] = node;
    }
    ++nn;
  }
  if (threadIdx.x == 0) t.n_new[gi] = nn;
}

// one warp per genome: lambda_o and critical count over the folded maxima
// (ac_validator.cpp:451-456); lane partial sums then a fixed shuffle tree
__global__ void k_ac_fold_finish(AcGrid g, const unsigned long long* fold, int n, double* lambda_o, int* critical) {
  const int gi = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (gi >= n) return;
  double s = 0.0;
  int cnt = 0;
  for (int e = lane; e < g.E; e += 32) {
    const double m = __longlong_as_double(static_cast<long long>(fold[static_cast<size_t>(gi) * g.E + e]));
    const double d = m - g.br_lim[e];
    s += d > 0.0 ? d : 0.0;
    cnt += m > g.br_lim[e];
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (lane == 0) lambda_o[gi] = s, critical[gi] = cnt;
}

}  // namespace

size_t ac_workspace_bytes(int n_bus, int nu, int E) { return ws_layout(n_bus, nu, E, nullptr, nullptr); }

int ac_threads(int nu) { return nu <= 48 ? 64 : (nu <= 160 ? 256 : 512); }

void ac_launch_topo(const AcGrid& g, const int* genomes, int n_genomes, int n_a, int n_d, const AcTopo& t,
                    cudaStream_t s) {
  if (n_genomes > 0) k_ac_topo<<<n_genomes, 128, 0, s>>>(g, genomes, n_a, n_d, t);
}

void ac_launch_cases(const AcGrid& g, const AcTopo& t, const AcCases& c, const AcSolver& sv, int ctas,
                     cudaStream_t s) {
  if (c.n <= 0) return;
  const size_t smem = sv.in_smem ? sv.ws_bytes : 0;
  AcWs rel;
  ws_layout(sv.n_bus, sv.nu, g.E, nullptr, &rel);
  auto launch = [&](auto kern, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<ctas, nt, smem, s>>>(g, t, c, sv, rel);
  };
  // scratch: four 256-thread CTAs per SM at 64 registers (cases claimed from a
  // counter; 4 x 256 measured 719 /s on the 118-bus case, 2 x 512: 525, 8 x 128: 679)
  switch (sv.in_smem ? ac_threads(sv.nu) : 256) {
    case 64:
      if (sv.in_smem)
        launch(k_ac_case<64, true>, 64);
      else
        launch(k_ac_case<64, false>, 64);
      break;
    case 256:
      if (sv.in_smem)
        launch(k_ac_case<256, true>, 256);
      else
        launch(k_ac_case<256, false>, 256);
      break;
    default:
      if (sv.in_smem)
        launch(k_ac_case<512, true>, 512);
      else
        launch(k_ac_case<512, false>, 512);
      break;
  }
}

void ac_launch_fold_finish(const AcGrid& g, const unsigned long long* fold, int n_genomes, double* lambda_o,
                           int* critical, cudaStream_t s) {
  if (n_genomes > 0) k_ac_fold_finish<<<(n_genomes + 3) / 4, 128, 0, s>>>(g, fold, n_genomes, lambda_o, critical);
}

}  // namespace tgb
