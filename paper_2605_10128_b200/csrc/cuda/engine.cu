// DC N-1 evaluation kernels: candidate prep (K2), rank bucketing, fused N-1
// sweep (K3), special outages (K4), score finish (K5).
//
// Reference path replaced: DcContext::evaluate_batch -> evaluate ->
// apply_topology / screen_contingencies / compute_scores
// (dc_engine.cpp:147-468). See topo.cuh for the low-rank formulation.
#include "engine.cuh"
#include "topo.cuh"

namespace tgb {

namespace {

constexpr int kPrepThreads = 256;

// ---------------------------------------------------------------- K2a analysis
// Topology analysis (one warp-sized CTA per candidate, thread 0 serial, so a
// whole batch runs in one wave): rank of the low-rank update and structural
// islanding, so the sweep's candidate groups can be formed before the rows are
// written (k_prep writes straight into them). The analysis and its bitmaps are
// stored for k_prep.
constexpr int kAnalyzeThreads = 32;

__global__ void __launch_bounds__(kAnalyzeThreads) k_analyze(DevGrid g, Batch b, int n_a, int n_d) {
  extern __shared__ uint32_t bits[];
  __shared__ TopoCore t;
  const int words = (g.E + 31) >> 5;
  for (int c = blockIdx.x; c < b.n; c += gridDim.x) {
    for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) bits[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
      analyze(g, t, bits, bits + words, b.genomes + static_cast<size_t>(c) * (n_a + n_d), n_a, n_d, nullptr, 0,
              nullptr, 0);
      if (!t.islanded && t.ns + t.nv > kSweepRank) t.islanded = 2;
      b.status[c] = t.islanded;
      b.rank[c] = t.islanded ? -1 : t.ns + t.nv;
    }
    __syncthreads();
    if (!t.islanded) {
      copy_block(b.topo + c, &t, sizeof(TopoCore), threadIdx.x, blockDim.x);
      uint32_t* tb = b.tbits + static_cast<size_t>(c) * 2 * words;
      for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) tb[i] = bits[i];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2 prep
// One CTA per candidate (grid-stride over candidates; Z scratch per CTA slot).
__global__ void __launch_bounds__(kPrepThreads) k_prep(DevGrid g, Batch b, int n_a, int n_d, double* zscratch,
                                                       int zslots) {
  extern __shared__ uint32_t bits[];
  __shared__ Topo t;
  __shared__ double gram[kSweepRank * kSweepRank];
  __shared__ double thv[kSweepRank];
  const int words = (g.E + 31) >> 5;
  uint32_t* mv_bits = bits;
  uint32_t* rm_bits = bits + words;
  double* zbuf = zscratch + static_cast<size_t>(blockIdx.x) * g.Nr * kStride;
  for (int c = blockIdx.x; c < b.n; c += gridDim.x) {
    const int slot = b.slot[c];
    if (slot < 0) continue;  // islanded (or over capacity) by the analysis: status already set
    copy_block(static_cast<TopoCore*>(&t), b.topo + c, sizeof(TopoCore), threadIdx.x, blockDim.x);
    const uint32_t* tb = b.tbits + static_cast<size_t>(c) * 2 * words;
    for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) bits[i] = tb[i];
    __syncthreads();
    build_z(g, t, zbuf, kStride);
    __syncthreads();
    gram_terms(g, t, zbuf, kStride, gram, kSweepRank, thv);
    __syncthreads();
    if (threadIdx.x == 0) small_solve(t, gram, kSweepRank, thv);
    __syncthreads();
    if (t.islanded) {
      if (threadIdx.x == 0) {
        b.status[c] = t.islanded;
        b.rank[c] = -1;
      }
      __syncthreads();
      continue;
    }
    const int ns = t.ns, nv = t.nv, r = ns + nv, rs = row_stride(r);
    // branch rows: [f_c, b_e*phi_e, b_e*rho_e, 0...]
    for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
      double phi[kMaxSplits], rho[kMaxCols];
      const bool on = branch_features(g, t, mv_bits, rm_bits, zbuf, kStride, e, phi, rho);
      double row[kStride];
#pragma unroll
      for (int i = 0; i < kStride; ++i) row[i] = 0.0;
      row[0] = cand_flow(g, t, e, phi, rho, on);
      if (on) {
        const double be = g.br_b[e];
        for (int q = 0; q < ns; ++q) row[1 + q] = be * phi[q];
        for (int m = 0; m < nv; ++m) row[1 + ns + m] = be * rho[m];
      }
      double2* dst = reinterpret_cast<double2*>(b.feat + feat_index(slot, b.nchunks, e, r));
#pragma unroll
      for (int i = 0; i < kStride / 2; ++i)
        if (2 * i < rs) dst[i] = make_double2(row[2 * i], row[2 * i + 1]);
    }
    __syncthreads();
    // contingency rows: [alpha_k, R[:,k] * alpha_k, 0...], flag
    double* kd = b.kdat + static_cast<size_t>(c) * g.Kpad * kStride;
    uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad;
    for (int k = threadIdx.x; k < g.Kpad; k += blockDim.x) {
      double row[kStride];
#pragma unroll
      for (int i = 0; i < kStride; ++i) row[i] = 0.0;
      uint8_t flag = 2;  // padding
      if (k < g.Ks) {
        const int beta = g.ks_branch[k];
        double phi[kMaxSplits], rho[kMaxCols];
        const bool on = branch_features(g, t, mv_bits, rm_bits, zbuf, kStride, beta, phi, rho);
        flag = 0;
        if (on) {
          double rk[kSweepRank];
          double lr = 0.0;
          for (int q = 0; q < ns; ++q) {
            double acc = 0.0;
            for (int q2 = 0; q2 < ns; ++q2) acc += t.Sinv[q * kMaxSplits + q2] * phi[q2];
            rk[q] = acc;
            lr += phi[q] * acc;
          }
          for (int m = 0; m < nv; ++m) {
            double acc = 0.0;
            for (int m2 = 0; m2 < nv; ++m2) acc += t.Cinv[m * kMaxCols + m2] * rho[m2];
            rk[ns + m] = -acc;
            lr -= rho[m] * acc;
          }
          const double tkk = g.Tdiag[beta] + g.br_b[beta] * lr;
          const double den = 1.0 - tkk;
          if (fabs(den) < 1e-8) {
            // bridge under the candidate topology (dc_engine.cpp:346-349 -> rebuild):
            // only a dead stub (degree 1, no injection, not the slack) keeps flows
            bool stub = false;
            for (int side = 0; side < 2 && !stub; ++side) {
              const int w = cand_end(g, t, mv_bits, beta, side == 0);
              stub = w != g.slack && cand_degree(g, t, mv_bits, rm_bits, w) == 1 && !cand_hosts_injection(g, t, w);
            }
            flag = stub ? 0 : 1;
          } else {
            const double alpha = b.feat[feat_index(slot, b.nchunks, beta, r)] / den;
            row[0] = alpha;
            for (int i = 0; i < r; ++i) row[1 + i] = rk[i] * alpha;
          }
        }
        if (flag == 1) b.energy[static_cast<size_t>(c) * g.Kall + g.ks_cont[k]] = b.params.penalty;
      }
      double2* dst = reinterpret_cast<double2*>(kd + static_cast<size_t>(k) * rs);
#pragma unroll
      for (int i = 0; i < kStride / 2; ++i)
        if (2 * i < rs) dst[i] = make_double2(row[2 * i], row[2 * i + 1]);
      kf[k] = flag;
    }
    if (threadIdx.x == 0) {
      b.status[c] = 0;
      b.rank[c] = r;
      int* rem = b.removed + static_cast<size_t>(c) * kMaxRemovedSweep;
      for (int i = 0; i < kMaxRemovedSweep; ++i) rem[i] = i < t.nrem ? t.rem[i] : -1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K4 special outages
// Multi-branch / injection contingencies and busbar outages: the outage is
// folded into the topology (extra removals, omitted injections) and the flows
// are solved directly, which equals the reference's compensation when it is
// regular and its rebuild when it is singular (dc_engine.cpp:303-356).
__global__ void __launch_bounds__(kPrepThreads) k_special(DevGrid g, Batch b, int n_a, int n_d, int full,
                                                          double* zscratch) {
  extern __shared__ uint32_t bits[];
  __shared__ Topo t;
  __shared__ int extra[kMaxRemoved];
  __shared__ int omit[kMaxPMod];
  __shared__ int n_extra, n_omit, skip;
  __shared__ double red_sum[kPrepThreads / 32];
  __shared__ double gram[kMaxCols * kMaxCols];
  __shared__ double thv[kMaxCols];
  const int words = (g.E + 31) >> 5;
  uint32_t* mv_bits = bits;
  uint32_t* rm_bits = bits + words;
  double* zbuf = zscratch + static_cast<size_t>(blockIdx.x) * g.Nr * kMaxCols;
  const int n_cases = g.Kx + g.Kb;
  const long total = static_cast<long>(b.n) * n_cases;
  for (long w = blockIdx.x; w < total; w += gridDim.x) {
    const int c = static_cast<int>(w / n_cases), cs = static_cast<int>(w % n_cases);
    const int* slots = b.genomes + static_cast<size_t>(c) * (n_a + n_d);
    if (threadIdx.x == 0) {
      skip = b.status[c] != 0;
      n_extra = 0;
      n_omit = 0;
      if (!skip) {
        if (cs < g.Kx) {
          for (int p = g.kx_br_ptr[cs]; p < g.kx_br_ptr[cs + 1] && n_extra < kMaxRemoved; ++p) extra[n_extra++] = g.kx_br[p];
          for (int p = g.kx_inj_ptr[cs]; p < g.kx_inj_ptr[cs + 1] && n_omit < kMaxPMod; ++p) {
            // injection outages only matter when the injection carries power
            omit[n_omit++] = g.kx_inj[p];
          }
        } else {
          // busbar outage: implied set of the station's action or the default (dc_engine.cpp:373-379)
          const int bo = cs - g.Kx;
          const int st = g.bo_station[bo];
          int act = -1;
          for (int k = 0; k < n_a; ++k)
            if (slots[k] >= 0 && g.act_station[slots[k]] == st) act = slots[k];
          int lo, hi;
          const int* src;
          if (act >= 0) {
            const int idx = g.act_bb_ptr[act] + g.bo_busbar[bo];
            lo = g.act_imp_ptr[idx];
            hi = g.act_imp_ptr[idx + 1];
            src = g.act_imp;
          } else {
            lo = g.bo_def_ptr[bo];
            hi = g.bo_def_ptr[bo + 1];
            src = g.bo_def;
          }
          for (int p = lo; p < hi && n_extra < kMaxRemoved; ++p) extra[n_extra++] = src[p];
        }
      }
    }
    __syncthreads();
    if (skip) {
      __syncthreads();
      continue;
    }
    for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) bits[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) analyze(g, t, mv_bits, rm_bits, slots, n_a, n_d, extra, n_extra, omit, n_omit);
    __syncthreads();
    if (!t.islanded) {
      build_z(g, t, zbuf, kMaxCols);
      __syncthreads();
      gram_terms(g, t, zbuf, kMaxCols, gram, kMaxCols, thv);
      __syncthreads();
      if (threadIdx.x == 0) small_solve(t, gram, kMaxCols, thv);
      __syncthreads();
    }
    const bool is_bus = cs >= g.Kx;
    if (t.islanded) {
      if (threadIdx.x == 0) {
        if (t.islanded == 2) b.status[c] = 3;  // capacity overflow: surfaced as an error
        if (is_bus) {
          atomicAdd(b.isl_bus + c, 1);
        } else {
          atomicAdd(b.isl_out + c, 1);
          b.energy[static_cast<size_t>(c) * g.Kall + g.kx_cont[cs]] = b.params.penalty;
        }
      }
      __syncthreads();
      continue;
    }
    unsigned long long* fold = (is_bus ? b.fbus : b.fmax) + static_cast<size_t>(c) * g.E;
    double part = 0.0;
    for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
      double phi[kMaxSplits], rho[kMaxCols];
      const bool on = branch_features(g, t, mv_bits, rm_bits, zbuf, kMaxCols, e, phi, rho);
      const double a = fabs(cand_flow(g, t, e, phi, rho, on));
      const double lim = g.br_lim[e];
      if (a > lim) part += a - lim;
      if (full ? a > 0.0 : a > lim) atomic_max_pos(fold + e, a);
    }
    if (!is_bus) {
      // fixed-order block reduction (deterministic)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if ((threadIdx.x & 31) == 0) red_sum[threadIdx.x >> 5] = part;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kPrepThreads / 32; ++i) s += red_sum[i];
        b.energy[static_cast<size_t>(c) * g.Kall + g.kx_cont[cs]] = s;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K5 finish
// dc_engine.cpp:390-437: metric sums, fitness, worst-k list; islanded genomes
// get the sentinel score with lambda_d/s/r filled.
__global__ void __launch_bounds__(256) k_finish(DevGrid g, Batch b, int n_a, int n_d) {
  __shared__ double s_o[8], s_b[8];
  __shared__ int s_c[8], s_c0[8], s_isl[8];
  __shared__ double best_v[8];
  __shared__ int best_i[8];
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int* slots = b.genomes + static_cast<size_t>(c) * (n_a + n_d);
  int ld = 0, ls = 0, lr = 0;
  for (int k = 0; k < n_d; ++k) ld += slots[n_a + k] >= 0;
  for (int k = 0; k < n_a; ++k)
    if (slots[k] >= 0) ++ls, lr += g.act_lambda_r[slots[k]];
  Scores& o = b.out;
  const int st = b.status[c];
  if (st != 0) {
    if (threadIdx.x == 0) {
      o.lambda_o[c] = 0.0;
      o.lambda_c[c] = 0;
      o.lambda_c0[c] = 0;
      o.lambda_b[c] = 0.0;
      o.lambda_d[c] = ld;
      o.lambda_s[c] = ls;
      o.lambda_r[c] = lr;
      o.fitness[c] = -CUDART_INF;
      o.islanded[c] = st == 1 ? 1 : 0;
      o.error[c] = st == 1 ? 0 : st;
      o.worst_n[c] = 0;
      o.isl_out[c] = 0;
      o.isl_bus[c] = 0;
    }
    return;
  }
  const int slot = b.slot[c];
  const unsigned long long* fm = b.fmax + static_cast<size_t>(c) * g.E;
  const unsigned long long* fb = b.fbus + static_cast<size_t>(c) * g.E;
  double so = 0.0, sb = 0.0;
  int nc = 0, nc0 = 0;
  for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
    const double lim = g.br_lim[e];
    const double m = __longlong_as_double(static_cast<long long>(fm[e]));
    const double mb = __longlong_as_double(static_cast<long long>(fb[e]));
    if (m > lim) so += m - lim, ++nc;
    if (fabs(b.feat[feat_index(slot, b.nchunks, e, b.rank[c])]) > lim) ++nc0;
    if (mb > lim) sb += mb - lim;
  }
  int isl = 0;
  const uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad;
  for (int k = threadIdx.x; k < g.Ks; k += blockDim.x) isl += kf[k] == 1;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    so += __shfl_xor_sync(0xffffffffu, so, d);
    sb += __shfl_xor_sync(0xffffffffu, sb, d);
    nc += __shfl_xor_sync(0xffffffffu, nc, d);
    nc0 += __shfl_xor_sync(0xffffffffu, nc0, d);
    isl += __shfl_xor_sync(0xffffffffu, isl, d);
  }
  if (lane == 0) s_o[wid] = so, s_b[wid] = sb, s_c[wid] = nc, s_c0[wid] = nc0, s_isl[wid] = isl;
  __syncthreads();
  const double* en = b.energy + static_cast<size_t>(c) * g.Kall;
  if (threadIdx.x == 0) {
    double lo = 0.0, lb = 0.0;
    int lc = 0, lc0 = 0, iso = b.isl_out[c];
    for (int w = 0; w < 8; ++w) lo += s_o[w], lb += s_b[w], lc += s_c[w], lc0 += s_c0[w], iso += s_isl[w];
    const int isb = b.isl_bus[c];
    lo += b.params.penalty * iso;
    lb += b.params.penalty * isb;
    double fit = -(lo + b.params.weight_c0 * lc0 + b.params.weight_c * lc);
    if (b.params.variant == 2) fit -= fmax(lb - b.params.lambda_b_pre, 0.0);
    o.lambda_o[c] = lo;
    o.lambda_c[c] = lc;
    o.lambda_c0[c] = lc0;
    o.lambda_b[c] = lb;
    o.lambda_d[c] = ld;
    o.lambda_s[c] = ls;
    o.lambda_r[c] = lr;
    o.fitness[c] = fit;
    o.islanded[c] = 0;
    o.error[c] = 0;
    o.isl_out[c] = iso;
    o.isl_bus[c] = isb;
  }
  // worst-k: repeated block argmax under the order (energy desc, index asc)
  double pv = CUDART_INF;
  int pi = -1;
  int nsel = 0;
  for (int round = 0; round < b.params.worst_k; ++round) {
    double bv = 0.0;
    int bi = -1;
    for (int k = threadIdx.x; k < g.Kall; k += blockDim.x) {
      const double v = en[k];
      if (!(v > 0.0)) continue;
      const bool after = v < pv || (v == pv && k > pi);
      if (!after) continue;
      if (bi < 0 || v > bv || (v == bv && k < bi)) bv = v, bi = k;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
      if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) bv = ov, bi = oi;
    }
    if (lane == 0) best_v[wid] = bv, best_i[wid] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      int i = -1;
      for (int w = 0; w < 8; ++w)
        if (best_i[w] >= 0 && (i < 0 || best_v[w] > v || (best_v[w] == v && best_i[w] < i))) v = best_v[w], i = best_i[w];
      best_v[0] = v;
      best_i[0] = i;
    }
    __syncthreads();
    pv = best_v[0];
    pi = best_i[0];
    __syncthreads();
    if (pi < 0) break;
    if (threadIdx.x == 0) {
      o.worst_idx[static_cast<size_t>(c) * b.params.worst_k + round] = pi;
      o.worst_val[static_cast<size_t>(c) * b.params.worst_k + round] = pv;
    }
    ++nsel;
  }
  if (threadIdx.x == 0) o.worst_n[c] = nsel;
}

// Dense copy of the candidate base flows (f_c) for callers that ask for them.
__global__ void k_extract_base(DevGrid g, Batch b, double* out) {
  const size_t total = static_cast<size_t>(b.n) * g.E;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t c = i / g.E;
    const int e = static_cast<int>(i % g.E);
    out[i] = b.status[c] == 0 ? b.feat[feat_index(b.slot[c], b.nchunks, e, b.rank[c])] : 0.0;
  }
}

__global__ void k_bits_to_double(const unsigned long long* in, double* out, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = __longlong_as_double(static_cast<long long>(in[i]));
}

}  // namespace

size_t topo_core_bytes() { return sizeof(TopoCore); }

// ---------------------------------------------------------------- launcher
void launch_evaluate(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                     cudaStream_t stream, int* kernels, cudaEvent_t sweep_begin, cudaEvent_t sweep_end) {
  int launched = 0;
  const int words = (g.E + 31) >> 5;
  const size_t bits_bytes = 2 * static_cast<size_t>(words) * sizeof(uint32_t);
  cudaMemsetAsync(b.fmax, 0, static_cast<size_t>(b.n) * g.E * sizeof(unsigned long long), stream);
  cudaMemsetAsync(b.fbus, 0, static_cast<size_t>(b.n) * g.E * sizeof(unsigned long long), stream);
  cudaMemsetAsync(b.energy, 0, static_cast<size_t>(b.n) * g.Kall * sizeof(double), stream);
  cudaMemsetAsync(b.isl_out, 0, b.n * sizeof(int), stream);
  cudaMemsetAsync(b.isl_bus, 0, b.n * sizeof(int), stream);
  static bool carveout = false;
  if (!carveout) {  // one wave of warp-sized analysis CTAs needs the full shared-memory carveout
    cudaFuncSetAttribute(k_analyze, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carveout = true;
  }
  k_analyze<<<b.n < 65535 ? b.n : 65535, kAnalyzeThreads, bits_bytes, stream>>>(g, b, n_a, n_d);
  ++launched;
  launch_bucket(b, stream, &launched);
  const int prep_grid = b.n < s.zslots ? b.n : s.zslots;
  k_prep<<<prep_grid, kPrepThreads, bits_bytes, stream>>>(g, b, n_a, n_d, s.zprep, s.zslots);
  ++launched;
  if (g.Ks > 0) launch_sweep(g, b, full, stream, sweep_begin, sweep_end, &launched);
  if (g.Kx + g.Kb > 0) {
    const long total = static_cast<long>(b.n) * (g.Kx + g.Kb);
    const int grid = static_cast<int>(total < s.zslots_special ? total : s.zslots_special);
    k_special<<<grid, kPrepThreads, bits_bytes, stream>>>(g, b, n_a, n_d, full ? 1 : 0, s.zspecial);
    ++launched;
  }
  k_finish<<<b.n, 256, 0, stream>>>(g, b, n_a, n_d);
  ++launched;
  if (kernels) *kernels = launched;
}

void launch_extract(const DevGrid& g, Batch& b, double* base_out, double* fmax_out, double* fbus_out,
                    cudaStream_t stream) {
  const size_t n = static_cast<size_t>(b.n) * g.E;
  if (base_out) k_extract_base<<<512, 256, 0, stream>>>(g, b, base_out);
  if (fmax_out) k_bits_to_double<<<512, 256, 0, stream>>>(b.fmax, fmax_out, n);
  if (fbus_out) k_bits_to_double<<<512, 256, 0, stream>>>(b.fbus, fbus_out, n);
}


}  // namespace tgb
