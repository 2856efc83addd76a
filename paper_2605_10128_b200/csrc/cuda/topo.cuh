// Per-candidate topology analysis and low-rank (Schur + Woodbury) solve.
//
// Replaces the reference's node-space Woodbury operator (dc_engine.cpp:154-283)
// with a flow-space form whose rank is the number of live splits plus removed
// branches plus grounded dead busbars:
//
//   z = (theta, psi), psi_j = theta(s'_j) - theta(s_j) for the new node of split j
//   K = [[B, U], [U^T, W]] + V Delta V^T
//     U = sum_{active moved l} b_l a_l c_l^T,  W = sum b_l c_l c_l^T
//     V = [a_d (removed branches) | e_v (dead busbars, ground 1.0)], Delta = diag(-b_d | +1)
//   S = W - U^T X U                       (Schur complement of the split block)
//   C = Delta^-1 + V^T X V + Phi^T S^-1 Phi,  Phi = U^T X V
//   branch e: phi_e = U^T X a_e - c_e,  rho_e = V^T X a_e + Phi^T S^-1 phi_e
//   T_cand[e,k] = T_base[e,k] + b_e (phi_e^T S^-1 phi_k - rho_e^T C^-1 rho_k)
//   f_cand[e]   = f0'[e]      + b_e (phi_e^T S^-1 phi_p - rho_e^T C^-1 rho_p)
//
// Islanding keeps the reference's decision rule (dc_engine.cpp:172-199, 257-262):
// a dead node hosting a nonzero injection, a dead slack, or a singular S / C
// (a live component without the slack) islands the topology. Dead busbars
// without injection are grounded exactly like the reference's placeholder.
#pragma once

#include "common.cuh"

namespace tgb {

// Result of the topology analysis (thread-serial, shared memory). k_analyze
// stores it per candidate so k_prep reloads it with a cooperative copy.
struct alignas(16) TopoCore {
  int islanded;
  int n_new;                        // non-empty action slots (new node index j)
  int action_of_new[kMaxSplits];
  int q_of_new[kMaxSplits];         // psi index of new node j, -1 when the split is dropped
  int node_of_q[kMaxSplits];        // psi index -> new node j
  int ns, nv;                       // live splits, V columns
  // moved branch ends: branch, coefficient per new node
  int nmv;
  int mv_branch[kMaxMoved];
  signed char mv_c[kMaxMoved][kMaxSplits];
  // injections moved to new nodes
  int ninj;
  int inj_id[kMaxInjMoved];
  int inj_new[kMaxInjMoved];
  // removed in-service branches (genome + outage) and grounded dead nodes
  int nrem;
  int rem[kMaxRemoved];
  int ng;
  int ground[kMaxGround];           // base node id
  // omitted injections
  int nom;
  int omit[kMaxPMod];
  // sparse columns of [U | V] in reduced node space
  int col_ptr[kMaxCols + 1];
  int term_idx[kMaxTerms];
  double term_coef[kMaxTerms];
  double W[kMaxSplits * kMaxSplits];
  double dinv[kMaxCols];            // 1/delta of V columns
  double ppsi[kMaxSplits];          // net injection moved to each live split
  double thresh_scale;
};

struct Topo : TopoCore {
  // small-solve results (Sinv, Y, Cinv contiguous: copied as one block of kTopoSol doubles)
  alignas(16) double Sinv[kMaxSplits * kMaxSplits];
  double Y[kMaxSplits * kMaxCols];  // S^-1 Phi  (ns x nv), row-major
  double Cinv[kMaxCols * kMaxCols];
  double Rp[kMaxSplits + kMaxCols]; // [S^-1 phi_p ; -C^-1 rho_p]
};
static_assert(sizeof(Topo::Sinv) + sizeof(Topo::Y) + sizeof(Topo::Cinv) == kTopoSol * sizeof(double) &&
                  (kTopoSol * 8) % 16 == 0,
              "the small-solve factors are one 16-byte multiple block");

// Cooperative copy of a 16-byte aligned block by the threads [0, nthreads).
__device__ __forceinline__ void copy_block(void* dst, const void* src, size_t bytes, int tid, int nthreads) {
  uint4* d = static_cast<uint4*>(dst);
  const uint4* q = static_cast<const uint4*>(src);
  for (size_t i = tid; i < bytes / 16; i += nthreads) d[i] = q[i];
}

__device__ __forceinline__ bool bit_get(const uint32_t* bits, int i) { return (bits[i >> 5] >> (i & 31)) & 1u; }
__device__ __forceinline__ void bit_set(uint32_t* bits, int i) { bits[i >> 5] |= 1u << (i & 31); }

__device__ inline int moved_slot(const TopoCore& t, const uint32_t* mv_bits, int e) {
  if (!bit_get(mv_bits, e)) return -1;
  for (int i = 0; i < t.nmv; ++i)
    if (t.mv_branch[i] == e) return i;
  return -1;
}

__device__ inline bool active_branch(const DevGrid& g, const uint32_t* rm_bits, int e) {
  return g.br_on[e] && !bit_get(rm_bits, e);
}

__device__ inline bool omitted(const TopoCore& t, int inj) {
  for (int i = 0; i < t.nom; ++i)
    if (t.omit[i] == inj) return true;
  return false;
}

// Candidate endpoint ids: base node, or N + j for the new node of split j.
__device__ inline int cand_end(const DevGrid& g, const TopoCore& t, const uint32_t* mv_bits, int e, bool from_end) {
  const int s = moved_slot(t, mv_bits, e);
  if (s >= 0)
    for (int j = 0; j < t.n_new; ++j)
      if (t.mv_c[s][j] == (from_end ? 1 : -1)) return g.N + j;
  return from_end ? g.br_from[e] : g.br_to[e];
}

// split j whose station node is v, or -1
__device__ inline int split_at_node(const DevGrid& g, const TopoCore& t, int v) {
  for (int j = 0; j < t.n_new; ++j)
    if (g.st_node[g.act_station[t.action_of_new[j]]] == v) return j;
  return -1;
}

// Live branches incident to a candidate node (base or new), optionally ignoring one branch.
__device__ inline int cand_degree(const DevGrid& g, const TopoCore& t, const uint32_t* mv_bits, const uint32_t* rm_bits,
                                  int node) {
  int deg = 0;
  if (node >= g.N) {
    const int j = node - g.N;
    for (int i = 0; i < t.nmv; ++i)
      if (t.mv_c[i][j] != 0 && active_branch(g, rm_bits, t.mv_branch[i])) ++deg;
    return deg;
  }
  for (int p = g.node_ptr[node]; p < g.node_ptr[node + 1]; ++p) {
    const int e = g.node_br[p];
    if (!active_branch(g, rm_bits, e)) continue;
    // an end moved away from this station node no longer touches it
    if ((g.br_from[e] == node && cand_end(g, t, mv_bits, e, true) != node) ||
        (g.br_to[e] == node && cand_end(g, t, mv_bits, e, false) != node))
      continue;
    ++deg;
  }
  return deg;
}

__device__ inline bool inj_moved_to(const TopoCore& t, int inj, int* j_out) {
  for (int i = 0; i < t.ninj; ++i)
    if (t.inj_id[i] == inj) {
      *j_out = t.inj_new[i];
      return true;
    }
  return false;
}

// Nonzero, non-omitted injection at a candidate node.
__device__ inline bool cand_hosts_injection(const DevGrid& g, const TopoCore& t, int node) {
  if (node >= g.N) {
    const int j = node - g.N;
    for (int i = 0; i < t.ninj; ++i)
      if (t.inj_new[i] == j && g.inj_net[t.inj_id[i]] != 0.0 && !omitted(t, t.inj_id[i])) return true;
    return false;
  }
  for (int p = g.node_inj_ptr[node]; p < g.node_inj_ptr[node + 1]; ++p) {
    const int i = g.node_inj[p];
    int j;
    if (inj_moved_to(t, i, &j)) continue;
    if (g.inj_net[i] != 0.0 && !omitted(t, i)) return true;
  }
  return false;
}

// Net injection moved onto each live split node (the only part of the
// analysis that depends on the injection values, not just their zero
// pattern: recomputed per injection profile).
__device__ inline void moved_injections(const DevGrid& g, TopoCore& t) {
  for (int q = 0; q < t.ns; ++q) t.ppsi[q] = 0.0;
  for (int i = 0; i < t.ninj; ++i) {
    const int q = t.q_of_new[t.inj_new[i]];
    if (q >= 0 && !omitted(t, t.inj_id[i])) t.ppsi[q] += g.inj_net[t.inj_id[i]];
  }
}

// Thread-0 analysis of one topology: genome slots plus an optional outage
// (extra removed branches, omitted injections). Bitmaps must be zeroed.
__device__ inline void analyze(const DevGrid& g, TopoCore& t, uint32_t* mv_bits, uint32_t* rm_bits, const int* slots,
                               int n_a, int n_d, const int* extra_rem, int n_extra, const int* omit_inj,
                               int n_omit) {
  t.islanded = 0;
  t.n_new = 0;
  t.nmv = 0;
  t.ninj = 0;
  t.nrem = 0;
  t.ng = 0;
  t.nom = 0;
  t.thresh_scale = 0.0;
  auto add_removed = [&](int e) {
    if (!g.br_on[e] || bit_get(rm_bits, e)) return;
    if (t.nrem >= kMaxRemoved) {
      t.islanded = 2;  // capacity exceeded: reported as an error by the host
      return;
    }
    bit_set(rm_bits, e);
    t.rem[t.nrem++] = e;
  };
  for (int k = 0; k < n_d; ++k) {
    const int d = slots[n_a + k];
    if (d >= 0) add_removed(g.disc[d]);
  }
  for (int k = 0; k < n_extra; ++k) add_removed(extra_rem[k]);
  if (n_omit > kMaxPMod) {
    t.islanded = 2;  // capacity exceeded (never truncated)
    return;
  }
  for (int k = 0; k < n_omit; ++k) t.omit[t.nom++] = omit_inj[k];

  // splits: one new node per non-empty action slot, in slot order (genome.cpp:90-108)
  for (int k = 0; k < n_a; ++k) {
    const int a = slots[k];
    if (a < 0) continue;
    const int j = t.n_new++;
    t.action_of_new[j] = a;
    const int s = g.act_station[a];
    const int t0 = g.st_term_ptr[s], nt = g.st_term_ptr[s + 1] - t0;
    const uint8_t* grp = g.act_group + g.act_group_ptr[a];
    for (int q = 0; q < nt; ++q) {
      if (!grp[q]) continue;
      const int kind = g.term_kind[t0 + q], el = g.term_elem[t0 + q];
      if (kind == 2) {
        if (t.ninj >= kMaxInjMoved) {
          t.islanded = 2;  // capacity exceeded (never truncated)
          return;
        }
        t.inj_id[t.ninj] = el;
        t.inj_new[t.ninj++] = j;
        continue;
      }
      int slot = moved_slot(t, mv_bits, el);
      if (slot < 0) {
        if (t.nmv >= kMaxMoved) {
          t.islanded = 2;
          return;
        }
        slot = t.nmv++;
        t.mv_branch[slot] = el;
        for (int jj = 0; jj < kMaxSplits; ++jj) t.mv_c[slot][jj] = 0;
        bit_set(mv_bits, el);
      }
      t.mv_c[slot][j] = kind == 0 ? 1 : -1;
    }
  }

  auto add_ground = [&](int v) {
    for (int i = 0; i < t.ng; ++i)
      if (t.ground[i] == v) return;
    if (t.ng >= kMaxGround) {
      t.islanded = 2;
      return;
    }
    t.ground[t.ng++] = v;
  };

  // dead busbars of split stations (dc_engine.cpp:181-229)
  t.ns = 0;
  for (int j = 0; j < t.n_new; ++j) {
    const int a = t.action_of_new[j];
    const int vs = g.st_node[g.act_station[a]];
    const bool live1 = cand_degree(g, t, mv_bits, rm_bits, g.N + j) > 0;
    const bool live0 = cand_degree(g, t, mv_bits, rm_bits, vs) > 0;
    t.q_of_new[j] = -1;
    if (!live1 && cand_hosts_injection(g, t, g.N + j)) {
      t.islanded = 1;
      return;
    }
    if (!live0) {
      if (vs == g.slack || cand_hosts_injection(g, t, vs)) {
        t.islanded = 1;
        return;
      }
      add_ground(vs);
    }
    if (live1) {
      t.q_of_new[j] = t.ns;
      t.node_of_q[t.ns++] = j;
    }
  }
  // dead busbars created by removals at unsplit nodes
  for (int i = 0; i < t.nrem; ++i) {
    const int e = t.rem[i];
    for (int side = 0; side < 2; ++side) {
      const int w = side == 0 ? g.br_from[e] : g.br_to[e];
      if (split_at_node(g, t, w) >= 0) continue;  // handled above
      if (cand_degree(g, t, mv_bits, rm_bits, w) > 0) continue;
      if (w == g.slack || cand_hosts_injection(g, t, w)) {
        t.islanded = 1;
        return;
      }
      add_ground(w);
    }
  }

  // sparse columns: U (live splits), then V (removals, grounds)
  int nt = 0;
  int col = 0;
  double wmax = 0.0;
  for (int q = 0; q < t.ns; ++q) {
    const int j = t.node_of_q[q];
    t.col_ptr[col++] = nt;
    for (int q2 = 0; q2 < t.ns; ++q2) t.W[q * kMaxSplits + q2] = 0.0;
    for (int i = 0; i < t.nmv; ++i) {
      const int e = t.mv_branch[i];
      const int cj = t.mv_c[i][j];
      if (cj == 0 || !active_branch(g, rm_bits, e)) continue;
      const double coef = g.br_b[e] * cj;
      const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
      if (nt + 2 > kMaxTerms) {
        t.islanded = 2;
        return;
      }
      if (ri >= 0) t.term_idx[nt] = ri, t.term_coef[nt++] = coef;
      if (rj >= 0) t.term_idx[nt] = rj, t.term_coef[nt++] = -coef;
      for (int q2 = 0; q2 < t.ns; ++q2) t.W[q * kMaxSplits + q2] += g.br_b[e] * cj * t.mv_c[i][t.node_of_q[q2]];
    }
    wmax = fmax(wmax, t.W[q * kMaxSplits + q]);
  }
  t.nv = 0;
  for (int i = 0; i < t.nrem; ++i) {
    const int e = t.rem[i];
    t.col_ptr[col++] = nt;
    const int ri = g.red[g.br_from[e]], rj = g.red[g.br_to[e]];
    if (ri >= 0) t.term_idx[nt] = ri, t.term_coef[nt++] = 1.0;
    if (rj >= 0) t.term_idx[nt] = rj, t.term_coef[nt++] = -1.0;
    t.dinv[t.nv++] = -1.0 / g.br_b[e];
  }
  for (int i = 0; i < t.ng; ++i) {
    t.col_ptr[col++] = nt;
    t.term_idx[nt] = g.red[t.ground[i]];
    t.term_coef[nt++] = 1.0;
    t.dinv[t.nv++] = 1.0;
  }
  t.col_ptr[col] = nt;
  t.thresh_scale = wmax;  // S pivots are compared with the moved susceptance sum

  moved_injections(g, t);
}

// In-place inverse of a small dense matrix (row-major, leading dim ld) by
// Gauss-Jordan with complete pivoting. Returns false when a pivot falls below
// rel * scale (numerically singular: the topology islands).
__device__ inline bool small_inverse(double* a, int n, int ld, double scale, double rel) {
  int piv_r[kMaxCols], piv_c[kMaxCols];
  for (int k = 0; k < n; ++k) {
    int br = k, bc = k;
    double best = -1.0;
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j) {
        double v = fabs(a[i * ld + j]);
        if (v > best) best = v, br = i, bc = j;
      }
    if (!(best > rel * scale)) return false;
    piv_r[k] = br;
    piv_c[k] = bc;
    if (br != k)
      for (int j = 0; j < n; ++j) {
        double tmp = a[k * ld + j];
        a[k * ld + j] = a[br * ld + j];
        a[br * ld + j] = tmp;
      }
    if (bc != k)
      for (int i = 0; i < n; ++i) {
        double tmp = a[i * ld + k];
        a[i * ld + k] = a[i * ld + bc];
        a[i * ld + bc] = tmp;
      }
    const double p = 1.0 / a[k * ld + k];
    a[k * ld + k] = 1.0;
    for (int j = 0; j < n; ++j) a[k * ld + j] *= p;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[i * ld + k];
      if (f == 0.0) continue;
      a[i * ld + k] = 0.0;
      for (int j = 0; j < n; ++j) a[i * ld + j] -= f * a[k * ld + j];
    }
  }
  // undo permutations: inverse of P A Q is Q^T A^-1 P^T
  for (int k = n - 1; k >= 0; --k) {
    if (piv_c[k] != k)
      for (int j = 0; j < n; ++j) {
        double tmp = a[k * ld + j];
        a[k * ld + j] = a[piv_c[k] * ld + j];
        a[piv_c[k] * ld + j] = tmp;
      }
    if (piv_r[k] != k)
      for (int i = 0; i < n; ++i) {
        double tmp = a[i * ld + k];
        a[i * ld + k] = a[i * ld + piv_r[k]];
        a[i * ld + piv_r[k]] = tmp;
      }
  }
  return true;
}

// Z = X [U | V]: row v of Z at zrow (stride ldz), all threads of the block.
__device__ inline void build_z(const DevGrid& g, const TopoCore& t, double* zbuf, int ldz) {
  const int ncol = t.ns + t.nv;
  for (int v = threadIdx.x; v < g.Nr; v += blockDim.x) {
    double* zr = zbuf + static_cast<size_t>(v) * ldz;
    for (int c = 0; c < ncol; ++c) {
      double acc = 0.0;
      for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p)
        acc = fma(t.term_coef[p], g.X[static_cast<size_t>(t.term_idx[p]) * g.Nr + v], acc);
      zr[c] = acc;
    }
  }
}

__device__ __forceinline__ double zget(const DevGrid& g, const double* zbuf, int ldz, int node, int c) {
  const int r = g.red[node];
  return r < 0 ? 0.0 : zbuf[static_cast<size_t>(r) * ldz + c];
}

// column^T y for a Z column (y = Z[:, c2]) or a base vector
__device__ inline double col_dot_z(const TopoCore& t, int c, const double* zbuf, int ldz, int c2) {
  double acc = 0.0;
  for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p)
    acc = fma(t.term_coef[p], zbuf[static_cast<size_t>(t.term_idx[p]) * ldz + c2], acc);
  return acc;
}

// theta' = theta0 + sum_omitted (-net_i) X[:, red(node_i)] at reduced index r
__device__ inline double theta_mod(const DevGrid& g, const TopoCore& t, int r) {
  double th = g.theta0[r];
  for (int i = 0; i < t.nom; ++i) {
    const int rv = g.red[g.inj_node[t.omit[i]]];
    if (rv >= 0) th -= g.inj_net[t.omit[i]] * g.X[static_cast<size_t>(rv) * g.Nr + r];
  }
  return th;
}

// All threads of the block, after build_z: the Gram entries G = [U|V]^T Z
// (ncol x ncol, row stride ldg) and th[c] = [U|V]_c^T theta'.
__device__ inline void gram_terms(const DevGrid& g, const TopoCore& t, const double* zbuf, int ldz, double* G, int ldg,
                                  double* th) {
  const int ncol = t.ns + t.nv;
  for (int i = threadIdx.x; i < ncol * ncol + ncol; i += blockDim.x) {
    if (i < ncol * ncol) {
      const int c = i / ncol, c2 = i % ncol;
      G[c * ldg + c2] = col_dot_z(t, c, zbuf, ldz, c2);
    } else {
      const int c = i - ncol * ncol;
      double acc = 0.0;
      for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p) acc = fma(t.term_coef[p], theta_mod(g, t, t.term_idx[p]), acc);
      th[c] = acc;
    }
  }
}

__device__ inline void small_rhs(Topo& t, const double* th);

// th[c] = [U|V]_c^T theta' (thread 0; no Z needed).
__device__ inline void theta_terms(const DevGrid& g, const TopoCore& t, double* th) {
  for (int c = 0; c < t.ns + t.nv; ++c) {
    double acc = 0.0;
    for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p) acc = fma(t.term_coef[p], theta_mod(g, t, t.term_idx[p]), acc);
    th[c] = acc;
  }
}

// Thread-0 small solve on the Gram entries (block-synchronized by the caller).
// Sets t.islanded = 1 when S or C is singular.
__device__ inline void small_solve(Topo& t, const double* G, int ldg, const double* th) {
  const int ns = t.ns, nv = t.nv;
  constexpr double kRel = 1e-10;  // dc_engine.cpp:258 threshold
  double* S = t.Sinv;
  for (int q = 0; q < ns; ++q)
    for (int q2 = 0; q2 < ns; ++q2) S[q * kMaxSplits + q2] = t.W[q * kMaxSplits + q2] - G[q * ldg + q2];
  // symmetrize against rounding (S is symmetric in exact arithmetic)
  for (int q = 0; q < ns; ++q)
    for (int q2 = q + 1; q2 < ns; ++q2) {
      const double m = 0.5 * (S[q * kMaxSplits + q2] + S[q2 * kMaxSplits + q]);
      S[q * kMaxSplits + q2] = S[q2 * kMaxSplits + q] = m;
    }
  if (ns > 0 && !small_inverse(S, ns, kMaxSplits, t.thresh_scale, kRel)) {
    t.islanded = 1;
    return;
  }
  // Phi = U^T X V (ns x nv) = G[q][ns + m];  Y = S^-1 Phi
  for (int q = 0; q < ns; ++q)
    for (int m = 0; m < nv; ++m) {
      double acc = 0.0;
      for (int q2 = 0; q2 < ns; ++q2) acc += S[q * kMaxSplits + q2] * G[q2 * ldg + ns + m];
      t.Y[q * kMaxCols + m] = acc;
    }
  // C = Delta^-1 + V^T X V + Phi^T Y
  double* C = t.Cinv;
  double cscale = 0.0;
  for (int m = 0; m < nv; ++m) {
    for (int m2 = 0; m2 < nv; ++m2) {
      double v = G[(ns + m) * ldg + ns + m2];
      for (int q = 0; q < ns; ++q) v += G[q * ldg + ns + m] * t.Y[q * kMaxCols + m2];
      C[m * kMaxCols + m2] = v + (m == m2 ? t.dinv[m] : 0.0);
    }
    cscale = fmax(cscale, fabs(t.dinv[m]));
  }
  for (int m = 0; m < nv; ++m)
    for (int m2 = m + 1; m2 < nv; ++m2) {
      const double a = 0.5 * (C[m * kMaxCols + m2] + C[m2 * kMaxCols + m]);
      C[m * kMaxCols + m2] = C[m2 * kMaxCols + m] = a;
    }
  if (nv > 0 && !small_inverse(C, nv, kMaxCols, cscale, kRel)) {
    t.islanded = 1;
    return;
  }
  small_rhs(t, th);
}

// Injection side of the small solve (the only part that depends on the
// injection profile): phi_p = U^T theta' - p_psi, rho_p = V^T theta' + Y^T phi_p,
// Rp = [S^-1 phi_p ; -C^-1 rho_p].
__device__ inline void small_rhs_into(const Topo& t, const double* th, const double* ppsi, double* Rp) {
  const int ns = t.ns, nv = t.nv;
  const double* S = t.Sinv;
  const double* C = t.Cinv;
  double php[kMaxSplits], rhp[kMaxCols];
  for (int c = 0; c < ns + nv; ++c) {
    if (c < ns)
      php[c] = th[c] - ppsi[c];
    else
      rhp[c - ns] = th[c];
  }
  for (int m = 0; m < nv; ++m)
    for (int q = 0; q < ns; ++q) rhp[m] += t.Y[q * kMaxCols + m] * php[q];
  for (int q = 0; q < ns; ++q) {
    double acc = 0.0;
    for (int q2 = 0; q2 < ns; ++q2) acc += S[q * kMaxSplits + q2] * php[q2];
    Rp[q] = acc;
  }
  for (int m = 0; m < nv; ++m) {
    double acc = 0.0;
    for (int m2 = 0; m2 < nv; ++m2) acc += C[m * kMaxCols + m2] * rhp[m2];
    Rp[ns + m] = -acc;
  }
}
__device__ inline void small_rhs(Topo& t, const double* th) { small_rhs_into(t, th, t.ppsi, t.Rp); }

// Branch features phi_e (ns) and rho_e (nv); returns false for inactive e.
__device__ inline bool branch_features(const DevGrid& g, const Topo& t, const uint32_t* mv_bits,
                                       const uint32_t* rm_bits, const double* zbuf, int ldz, int e, double* phi,
                                       double* rho) {
  const int ns = t.ns, nv = t.nv;
  const int rf = g.red[g.br_from[e]], rt = g.red[g.br_to[e]];
  const double* zf = rf >= 0 ? zbuf + static_cast<size_t>(rf) * ldz : nullptr;
  const double* zt = rt >= 0 ? zbuf + static_cast<size_t>(rt) * ldz : nullptr;
  for (int c = 0; c < ns + nv; ++c) {
    const double d = (zf ? zf[c] : 0.0) - (zt ? zt[c] : 0.0);
    if (c < ns)
      phi[c] = d;
    else
      rho[c - ns] = d;
  }
  const int s = moved_slot(t, mv_bits, e);
  if (s >= 0)
    for (int q = 0; q < ns; ++q) phi[q] -= t.mv_c[s][t.node_of_q[q]];
  for (int m = 0; m < nv; ++m)
    for (int q = 0; q < ns; ++q) rho[m] += t.Y[q * kMaxCols + m] * phi[q];
  return active_branch(g, rm_bits, e);
}

// ---- precomputed branch-space columns (no per-candidate Z) -------------------
// With DevGrid::PhiA / PsiD a column of [U | V] is read in branch space: the
// split column of action a (all its base-active moved ends) is PhiA[a], a
// removed disconnectable d is PsiD[d]; any other column (a split whose moved
// branch is also removed, a grounded dead node) is evaluated from its sparse
// node-space terms by X gathers. Same values as build_z + branch_features
// (up to the summation order of the terms).

// Z value of column c at reduced node v: sum_p coef_p X[term_p, v] (build_z's row formula).
__device__ __forceinline__ double zval(const DevGrid& g, const TopoCore& t, int c, int v) {
  double acc = 0.0;
  for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p)
    acc = fma(t.term_coef[p], g.X[static_cast<size_t>(t.term_idx[p]) * g.Nr + v], acc);
  return acc;
}

// Gram entries G = [U|V]^T X [U|V] and th = [U|V]^T theta' from X gathers
// (all threads of the block; gram_terms without Z).
__device__ inline void gram_terms_x(const DevGrid& g, const TopoCore& t, double* G, int ldg, double* th) {
  const int ncol = t.ns + t.nv;
  for (int i = threadIdx.x; i < ncol * ncol + ncol; i += blockDim.x) {
    if (i < ncol * ncol) {
      const int c = i / ncol, c2 = i % ncol;
      double acc = 0.0;
      for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p) acc = fma(t.term_coef[p], zval(g, t, c2, t.term_idx[p]), acc);
      G[c * ldg + c2] = acc;
    } else {
      const int c = i - ncol * ncol;
      double acc = 0.0;
      for (int p = t.col_ptr[c]; p < t.col_ptr[c + 1]; ++p) acc = fma(t.term_coef[p], theta_mod(g, t, t.term_idx[p]), acc);
      th[c] = acc;
    }
  }
}

// Branch-space source of each column (thread 0): PhiA / PsiD row, or null
// for the gather path.
__device__ inline void column_sources(const DevGrid& g, const TopoCore& t, const uint32_t* rm_bits,
                                      const double** base) {
  for (int q = 0; q < t.ns; ++q) {
    const int j = t.node_of_q[q], a = t.action_of_new[j];
    int cnt = 0;
    for (int i = 0; i < t.nmv; ++i) cnt += t.mv_c[i][j] != 0 && active_branch(g, rm_bits, t.mv_branch[i]);
    base[q] = g.act_nmv[a] == cnt ? g.PhiA + static_cast<size_t>(a) * g.E : nullptr;
  }
  for (int m = 0; m < t.nv; ++m) {
    const int d = m < t.nrem ? g.disc_of_br[t.rem[m]] : -1;
    base[t.ns + m] = d >= 0 ? g.PsiD + static_cast<size_t>(d) * g.E : nullptr;
  }
}

// branch_features with the branch-space column sources.
__device__ inline bool branch_features_pc(const DevGrid& g, const Topo& t, const uint32_t* mv_bits,
                                          const uint32_t* rm_bits, const double* const* base, int e, double* phi,
                                          double* rho) {
  const int ns = t.ns, nv = t.nv;
  const int rf = g.red[g.br_from[e]], rt = g.red[g.br_to[e]];
  for (int c = 0; c < ns + nv; ++c) {
    double d;
    if (base[c]) {
      d = base[c][e];
    } else {
      d = (rf >= 0 ? zval(g, t, c, rf) : 0.0) - (rt >= 0 ? zval(g, t, c, rt) : 0.0);
    }
    if (c < ns)
      phi[c] = d;
    else
      rho[c - ns] = d;
  }
  const int s = moved_slot(t, mv_bits, e);
  if (s >= 0)
    for (int q = 0; q < ns; ++q) phi[q] -= t.mv_c[s][t.node_of_q[q]];
  for (int m = 0; m < nv; ++m)
    for (int q = 0; q < ns; ++q) rho[m] += t.Y[q * kMaxCols + m] * phi[q];
  return active_branch(g, rm_bits, e);
}

// Base flow of e under the (possibly omitted-injection) base injections.
__device__ inline double base_flow_mod(const DevGrid& g, const TopoCore& t, int e) {
  double f = g.f0[e];
  if (t.nom == 0) return f;
  const int rf = g.red[g.br_from[e]], rt = g.red[g.br_to[e]];
  for (int i = 0; i < t.nom; ++i) {
    const int rv = g.red[g.inj_node[t.omit[i]]];
    if (rv < 0) continue;
    const double* xc = g.X + static_cast<size_t>(rv) * g.Nr;
    f -= g.inj_net[t.omit[i]] * g.br_b[e] * ((rf >= 0 ? xc[rf] : 0.0) - (rt >= 0 ? xc[rt] : 0.0));
  }
  return f;
}

// Candidate flow on e given its features (0 for inactive branches).
__device__ inline double cand_flow(const DevGrid& g, const Topo& t, int e, const double* phi, const double* rho,
                                   bool active) {
  if (!active) return 0.0;
  double acc = 0.0;
  for (int q = 0; q < t.ns; ++q) acc = fma(phi[q], t.Rp[q], acc);
  for (int m = 0; m < t.nv; ++m) acc = fma(rho[m], t.Rp[t.ns + m], acc);
  return base_flow_mod(g, t, e) + g.br_b[e] * acc;
}

}  // namespace tgb
