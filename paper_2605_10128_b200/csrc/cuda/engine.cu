// DC N-1 evaluation kernels: candidate prep (K2), rank bucketing, fused N-1
// sweep (K3), special outages (K4), score finish (K5).
//
// Reference path replaced: DcContext::evaluate_batch -> evaluate ->
// apply_topology / screen_contingencies / compute_scores
// (dc_engine.cpp:147-468). See topo.cuh for the low-rank formulation.
#include <algorithm>
#include <cstdlib>

#include "engine.cuh"
#include "topo.cuh"

namespace tgb {

namespace {

constexpr int kPrepThreads = 256;
constexpr int kPrepCta = 512;  // k_prep block size (a multiple of 128: the timestep bound folds)

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
// One CTA per candidate (grid-stride over candidates). Z = X [U | V] lives in
// the CTA's global scratch slot (row stride row_stride(r); L2-resident at cfg2:
// keeping it in shared memory measured slower, 2 CTAs per SM either way).
// Warp-wide maximum of a chunk summary, one REDUX per slot: floats compared
// through an order-preserving unsigned key (non-negative floats are their bit
// patterns; the last slot may be negative or -inf).
__device__ __forceinline__ void warp_max_summary(float (&v)[kCsum]) {
#pragma unroll
  for (int q = 0; q < kCsum; ++q) {
    const unsigned b = __float_as_uint(v[q]);
    const unsigned key = (b >> 31) ? ~b : (b | 0x80000000u);
    const unsigned m = __reduce_max_sync(0xffffffffu, key);
    v[q] = __uint_as_float((m >> 31) ? (m & 0x7fffffffu) : ~m);
  }
}

__global__ void __launch_bounds__(kPrepCta) k_prep(DevGrid g, Batch b, int n_a, int n_d, double* zscratch) {
  extern __shared__ __align__(16) uint32_t bits[];
  __shared__ Topo t;
  __shared__ double gram[kSweepRank * kSweepRank];
  __shared__ double thv[kSweepRank];
  __shared__ const double* cbase[kSweepRank];
  __shared__ int nc0_s;
  if (threadIdx.x == 0) nc0_s = 0;
  const int words = (g.E + 31) >> 5;
  uint32_t* mv_bits = bits;
  uint32_t* rm_bits = bits + words;
  double* zglob = zscratch + static_cast<size_t>(blockIdx.x) * g.Nr * kStride;
  for (int c = blockIdx.x; c < b.n; c += gridDim.x) {
    const int slot = b.slot[c];
    if (slot < 0) continue;  // islanded (or over capacity) by the analysis: status already set
    copy_block(static_cast<TopoCore*>(&t), b.topo + c, sizeof(TopoCore), threadIdx.x, blockDim.x);
    const uint32_t* tb = b.tbits + static_cast<size_t>(c) * 2 * words;
    for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) bits[i] = tb[i];
    __syncthreads();
    if (threadIdx.x == 0) moved_injections(g, t);  // this profile's injections (the analysis may be shared)
    double* sol = b.topo_sol ? b.topo_sol + static_cast<size_t>(c) * kTopoSol : nullptr;
    const int ldz = row_stride(t.ns + t.nv);
    double* zbuf = zglob;
    const bool pc = g.PhiA != nullptr;  // branch-space columns: no Z = X [U | V] per candidate
    __syncthreads();
    if (pc) {
      if (threadIdx.x == 0) column_sources(g, t, rm_bits, cbase);
      gram_terms_x(g, t, gram, kSweepRank, thv);
    } else {
      build_z(g, t, zbuf, ldz);
      __syncthreads();
      gram_terms(g, t, zbuf, ldz, gram, kSweepRank, thv);
    }
    __syncthreads();
    if (threadIdx.x == 0) small_solve(t, gram, kSweepRank, thv);
    __syncthreads();
    // the topology factors for k_prep_mt (later injection profiles)
    if (sol && !t.islanded) copy_block(sol, t.Sinv, kTopoSol * sizeof(double), threadIdx.x, blockDim.x);
    if (t.islanded) {
      if (threadIdx.x == 0) {
        b.status[c] = t.islanded;
        b.rank[c] = -1;
      }
      __syncthreads();
      continue;
    }
    const int ns = t.ns, nv = t.nv, r = ns + nv, rs = row_stride(r);
    // branch rows: [f_c, b_e*phi_e, b_e*rho_e, 0...]; lambda_c0 = #(|f_c| > limit)
    // (dc_engine.cpp:397) counted on the way
    int nc0 = 0;
    // a warp covers 32 consecutive rows (one sweep chunk) per pass, so the
    // chunk summaries of the chunked sweep are warp reductions
    float* csum = r <= kChunkedMaxRank ? b.csum + static_cast<size_t>(c) * b.nchunks * kCsum : nullptr;
    for (int e0 = threadIdx.x & ~31; e0 < g.E; e0 += blockDim.x) {
      const int e = e0 + (threadIdx.x & 31);
      double row[kStride];
#pragma unroll
      for (int i = 0; i < kStride; ++i) row[i] = 0.0;
      bool on = false;
      if (e < g.E) {
        double phi[kMaxSplits], rho[kMaxCols];
        on = pc ? branch_features_pc(g, t, mv_bits, rm_bits, cbase, e, phi, rho)
                : branch_features(g, t, mv_bits, rm_bits, zbuf, ldz, e, phi, rho);
        row[0] = cand_flow(g, t, e, phi, rho, on);
        nc0 += fabs(row[0]) > g.br_lim[e];
        if (on) {
          const double be = g.br_b[e];
          for (int q = 0; q < ns; ++q) row[1 + q] = be * phi[q];
          for (int m = 0; m < nv; ++m) row[1 + ns + m] = be * rho[m];
        }
      }
      if (csum) {
        // live rows only: removed / out-of-service rows carry no flow in the
        // exact path (their elements are never scored)
        float v[kCsum];
        v[0] = on ? __double2float_ru(fabs(row[0] - g.f0[e])) : 0.0f;
#pragma unroll
        for (int q = 0; q + 1 < kCsum; ++q) v[1 + q] = on && q < r ? __double2float_ru(fabs(row[1 + q])) : 0.0f;
        if (r + 2 <= kCsum)  // row-coupled chunk test slot, as in prep_branch_chunk
          v[kCsum - 1] = on ? __double2float_ru(fabs(row[0] - g.f0[e]) - (g.br_lim[e] - fabs(g.f0[e]))) : -CUDART_INF_F;
        warp_max_summary(v);
        if ((threadIdx.x & 31) == 0) {
          float4* dst = reinterpret_cast<float4*>(csum + static_cast<size_t>(e0 >> 5) * kCsum);
          dst[0] = make_float4(v[0], v[1], v[2], v[3]);
          dst[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
      }
      if (e >= g.E) continue;
      if (b.feat_mt) {  // multi-timestep bounds (profile 0; k_prep_mt folds the later profiles in)
        unsigned long long* m = reinterpret_cast<unsigned long long*>(b.feat_mt + feat_index(slot, b.nchunks, e, r + 1));
        const unsigned long long key = order_key(row[0]);
        m[0] = key;
        m[1] = key;
        double* l = reinterpret_cast<double*>(m) + 2;
        for (int q = 0; q < r; ++q) l[q] = row[1 + q];
      }
      double2* dst = reinterpret_cast<double2*>(b.feat + feat_index(slot, b.nchunks, e, r));
#pragma unroll
      for (int i = 0; i < kStride / 2; ++i)
        if (2 * i < rs) dst[i] = make_double2(row[2 * i], row[2 * i + 1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nc0 += __shfl_xor_sync(0xffffffffu, nc0, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&nc0_s, nc0);
    __syncthreads();
    if (threadIdx.x == 0) b.nc0[c] = nc0_s, nc0_s = 0;
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
        // phi, rho of the outaged branch from its branch row (written above,
        // L = b_beta [phi; rho]) instead of a second pass over Z
        const double* fr = b.feat + feat_index(slot, b.nchunks, beta, r);
        const bool on = g.br_on[beta] && !bit_get(rm_bits, beta);
        double phi[kMaxSplits], rho[kMaxCols];
        if (on) {
          const double ib = 1.0 / g.br_b[beta];
          for (int q = 0; q < ns; ++q) phi[q] = fr[1 + q] * ib;
          for (int m = 0; m < nv; ++m) rho[m] = fr[1 + ns + m] * ib;
        }
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
            const double alpha = fr[0] / den;
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
      if (b.amx_mt) {
        // multi-timestep bounds per (tile, sub-tile): a warp covers 32
        // consecutive contingencies of one tile (blockDim and tiles are
        // multiples of 128), half a warp one 16-wide sub-tile
        const int ntiles = g.Kpad / 128, tile = k >> 7, sub = (k & 127) >> 4;
        double dl = fabs(row[0] - g.alpha0[k]);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) dl = fmax(dl, __shfl_xor_sync(0xffffffffu, dl, o));
        if ((threadIdx.x & 15) == 0)
          atomicMax(b.amx_mt + (static_cast<size_t>(c) * ntiles + tile) * kTmaxSub + sub, dbits(dl));
        for (int q = 0; q < r; ++q) {
          double rq = fabs(row[1 + q]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) rq = fmax(rq, __shfl_xor_sync(0xffffffffu, rq, o));
          if ((threadIdx.x & 31) == 0)
            atomicMax(b.rmx_mt + (static_cast<size_t>(c) * ntiles + tile) * kStride + 1 + q, dbits(rq));
        }
      }
    }
    if (threadIdx.x == 0) {
      b.rank[c] = r;  // status stays k_analyze's 0 (k_special may run beside this kernel)
      int* rem = b.removed + static_cast<size_t>(c) * kMaxRemovedSweep;
      for (int i = 0; i < kMaxRemovedSweep; ++i) rem[i] = i < t.nrem ? t.rem[i] : -1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2 prep, split form
// With the branch-space columns (DevGrid::PhiA) a candidate's prep splits in
// two kernels with no CTA-wide phases and no Z = X [U | V]:
//   k_prep_solve: one warp per candidate: column sources, Gram entries from X
//     gathers (topo.cuh gram_terms_x), the serial small solve (S^-1, Y, C^-1,
//     Rp), compact factors to Batch::pc;
//   k_prep_rows: one warp per (candidate, 32 branch rows) -- the branch rows
//     [f_c, b_e phi_e, b_e rho_e], the chunk summary (csum) and lambda_c0 --
//     or per (candidate, 32 contingencies) -- [alpha_k, R'_k] and the flag,
//     with phi / rho of the outaged branch read from the same columns.
// Same formulas as k_prep (topo.cuh branch_features / cand_flow); rank R is a
// template parameter so the row vectors live in registers.
__global__ void __launch_bounds__(32) k_prep_solve(DevGrid g, Batch b) {
  __shared__ Topo t;
  __shared__ double gram[kSweepRank * kSweepRank];
  __shared__ double thv[kSweepRank];
  __shared__ const double* cbase[kSweepRank];
  const int words = (g.E + 31) >> 5;
  const int tid = threadIdx.x;
  for (int c = blockIdx.x; c < b.n; c += gridDim.x) {
    if (b.slot[c] < 0) continue;  // islanded (or over capacity) by the analysis: status already set
    copy_block(static_cast<TopoCore*>(&t), b.topo + c, sizeof(TopoCore), tid, 32);
    __syncthreads();
    const uint32_t* rm_bits = b.tbits + static_cast<size_t>(c) * 2 * words + words;
    if (tid == 0) {
      moved_injections(g, t);
      column_sources(g, t, rm_bits, cbase);
    }
    __syncthreads();
    gram_terms_x(g, t, gram, kSweepRank, thv);
    __syncthreads();
    if (tid == 0) small_solve(t, gram, kSweepRank, thv);
    __syncthreads();
    if (t.islanded) {
      if (tid == 0) {
        b.status[c] = t.islanded;
        b.rank[c] = -1;
      }
      __syncthreads();
      continue;
    }
    const int ns = t.ns, nv = t.nv;
    PcFac* f = b.pc + c;
    for (int i = tid; i < kMaxSplits * kMaxSplits; i += 32) f->Sinv[i] = t.Sinv[i];
    for (int i = tid; i < ns * nv; i += 32) f->Y[(i / nv) * kSweepRank + i % nv] = t.Y[(i / nv) * kMaxCols + i % nv];
    for (int i = tid; i < nv * nv; i += 32) f->Cinv[(i / nv) * kSweepRank + i % nv] = t.Cinv[(i / nv) * kMaxCols + i % nv];
    if (tid < ns + nv) {
      f->Rp[tid] = t.Rp[tid];
      f->base[tid] = cbase[tid];
    }
    if (tid == 0) {
      f->ns = ns;
      f->nv = nv;
      b.rank[c] = ns + nv;  // status stays k_analyze's 0 (k_special may run beside this kernel)
      b.nc0[c] = 0;  // k_prep_rows adds its counts
      int* rem = b.removed + static_cast<size_t>(c) * kMaxRemovedSweep;
      for (int i = 0; i < kMaxRemovedSweep; ++i) rem[i] = i < t.nrem ? t.rem[i] : -1;
    }
    __syncthreads();
  }
}

// z = [phi_e ; rho_e] of branch e for a rank-R candidate (branch_features_pc
// with the compact factors); returns whether e is live.
template <int R>
__device__ __forceinline__ bool pc_features(const DevGrid& g, const TopoCore& t, const PcFac& f, const uint32_t* mv_bits,
                                            const uint32_t* rm_bits, int ns, int e, double (&z)[R > 0 ? R : 1]) {
  int rf = -2, rt = -2;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    const double* src = f.base[c];
    if (src) {
      z[c] = __ldg(src + e);
    } else {
      if (rf == -2) rf = g.red[g.br_from[e]], rt = g.red[g.br_to[e]];
      z[c] = (rf >= 0 ? zval(g, t, c, rf) : 0.0) - (rt >= 0 ? zval(g, t, c, rt) : 0.0);
    }
  }
  if (bit_get(mv_bits, e)) {
    const int s = moved_slot(t, mv_bits, e);
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (q < ns) z[q] -= t.mv_c[s][t.node_of_q[q]];
  }
  // rho_m += sum_q Y[q][m] phi_q (rho index m = c - ns)
#pragma unroll
  for (int c = 0; c < R; ++c) {
    if (c < ns) continue;
    double acc = z[c];
#pragma unroll
    for (int q = 0; q < (R < kMaxSplits ? R : kMaxSplits); ++q)
      if (q < ns) acc += f.Y[q * kSweepRank + (c - ns)] * z[q];
    z[c] = acc;
  }
  return g.br_on[e] && !bit_get(rm_bits, e);
}

// candidate flow on a live branch (cand_flow): f0 + b_e (phi . Rp_s + rho . Rp_v)
template <int R>
__device__ __forceinline__ double pc_flow(const DevGrid& g, const PcFac& f, int e, const double (&z)[R > 0 ? R : 1]) {
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < R; ++c) acc = fma(z[c], f.Rp[c], acc);
  return g.f0[e] + g.br_b[e] * acc;
}

template <int R>
__device__ __forceinline__ void prep_branch_chunk(const DevGrid& g, const Batch& b, int c, int slot, int chunk,
                                                  const TopoCore& t, const PcFac& f, const uint32_t* mv_bits,
                                                  const uint32_t* rm_bits) {
  constexpr int RS = row_stride(R);
  const int lane = threadIdx.x & 31, ns = f.ns;
  const int e = chunk * kChunkRows + lane;
  double row[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) row[i] = 0.0;
  bool on = false;
  // the row's static data (f0, b, limit, in service) in one load, issued first
  double4 rs = make_double4(0.0, 0.0, 0.0, 0.0);
  if (e < g.E) {
    const double2* p = reinterpret_cast<const double2*>(g.row_static + e);
    const double2 a = __ldg(p), b2 = __ldg(p + 1);
    rs = make_double4(a.x, a.y, b2.x, b2.y);
  }
  if (e < g.E) {
    double z[R > 0 ? R : 1];
    pc_features<R>(g, t, f, mv_bits, rm_bits, ns, e, z);  // (its live flag: rs.w and rm_bits, below)
    on = rs.w != 0.0 && !bit_get(rm_bits, e);
    if (on) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) acc = fma(z[q], f.Rp[q], acc);
      row[0] = rs.x + rs.y * acc;  // pc_flow
#pragma unroll
      for (int q = 0; q < R; ++q) row[1 + q] = rs.y * z[q];
    }
  }
  const unsigned over = __ballot_sync(0xffffffffu, e < g.E && fabs(row[0]) > rs.z);
  if (lane == 0 && over) atomicAdd(b.nc0 + c, __popc(over));
  if (R <= kChunkedMaxRank) {
    float v[kCsum];
    v[0] = on ? __double2float_ru(fabs(row[0] - rs.x)) : 0.0f;
#pragma unroll
    for (int q = 0; q + 1 < kCsum; ++q) v[1 + q] = on && q < R ? __double2float_ru(fabs(row[1 + (q < R ? q : 0)])) : 0.0f;
    // ranks <= kCsum - 2: the last slot carries max_e (|f_c - f0|_e - (lim_e - |f0_e|))
    // for the row-coupled chunk test (setup.cu k_chunk_rec); dead rows never overload
    if (R + 2 <= kCsum)
      v[kCsum - 1] = on ? __double2float_ru(fabs(row[0] - rs.x) - (rs.z - fabs(rs.x))) : -CUDART_INF_F;
    warp_max_summary(v);
    if (lane == 0) {
      float4* dst = reinterpret_cast<float4*>(b.csum + (static_cast<size_t>(c) * b.nchunks + chunk) * kCsum);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  if (e < g.E) {
    double2* dst = reinterpret_cast<double2*>(b.feat + feat_index(slot, b.nchunks, e, R));
#pragma unroll
    for (int i = 0; i < RS / 2; ++i) __stcs(dst + i, make_double2(row[2 * i], row[2 * i + 1]));  // streaming: read back by the sweep, not by this kernel
  }
}

template <int R>
__device__ __forceinline__ void prep_cont_chunk(const DevGrid& g, const Batch& b, int c, int kchunk, const TopoCore& t,
                                                const PcFac& f, const uint32_t* mv_bits, const uint32_t* rm_bits) {
  constexpr int RS = row_stride(R);
  const int lane = threadIdx.x & 31, ns = f.ns, nv = f.nv;
  const int k = kchunk * 32 + lane;
  double row[RS];
#pragma unroll
  for (int i = 0; i < RS; ++i) row[i] = 0.0;
  uint8_t flag = 2;  // padding
  if (k < g.Ks) {
    const int beta = g.ks_branch[k];
    flag = 0;
    double z[R > 0 ? R : 1];
    if (pc_features<R>(g, t, f, mv_bits, rm_bits, ns, beta, z)) {
      double rk[R > 0 ? R : 1];
      double lr = 0.0;
#pragma unroll
      for (int q = 0; q < (R < kMaxSplits ? R : kMaxSplits); ++q) {
        if (q >= ns) continue;
        double acc = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < (R < kMaxSplits ? R : kMaxSplits); ++q2)
          if (q2 < ns) acc += f.Sinv[q * kMaxSplits + q2] * z[q2];
        rk[q] = acc;
        lr += z[q] * acc;
      }
#pragma unroll
      for (int c2 = 0; c2 < R; ++c2) {
        if (c2 < ns) continue;
        const int m = c2 - ns;
        double acc = 0.0;
#pragma unroll
        for (int c3 = 0; c3 < R; ++c3)
          if (c3 >= ns) acc += f.Cinv[m * kSweepRank + (c3 - ns)] * z[c3];
        rk[c2] = -acc;
        lr -= z[c2] * acc;
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
        const double alpha = pc_flow<R>(g, f, beta, z) / den;
        row[0] = alpha;
#pragma unroll
        for (int i = 0; i < R; ++i) row[1 + i] = rk[i] * alpha;
      }
      (void)nv;
    }
    if (flag == 1) b.energy[static_cast<size_t>(c) * g.Kall + g.ks_cont[k]] = b.params.penalty;
  }
  if (k < g.Kpad) {
    double2* dst = reinterpret_cast<double2*>(b.kdat + static_cast<size_t>(c) * g.Kpad * kStride +
                                              static_cast<size_t>(k) * RS);
#pragma unroll
    for (int i = 0; i < RS / 2; ++i) __stcs(dst + i, make_double2(row[2 * i], row[2 * i + 1]));
    b.kflag[static_cast<size_t>(c) * g.Kpad + k] = flag;
  }
}

// Warp work item = (candidate of the rank class, segment of kPrepSeg
// consecutive 32-row chunks: branch rows, then contingency rows). The
// candidate's factors are staged once per segment in the warp's shared slab.
constexpr int kPrepSeg = 16;
constexpr int kPrepRowWarps = 8;

template <int R>
__device__ __forceinline__ void prep_segment(const DevGrid& g, const Batch& b, int c, int slot, int j0, int j1,
                                             const PcFac& f) {
  const int words = (g.E + 31) >> 5;
  const uint32_t* mv_bits = b.tbits + static_cast<size_t>(c) * 2 * words;
  const TopoCore& t = b.topo[c];
  for (int j = j0; j < j1; ++j) {
    if (j < b.nchunks)
      prep_branch_chunk<R>(g, b, c, slot, j, t, f, mv_bits, mv_bits + words);
    else
      prep_cont_chunk<R>(g, b, c, j - b.nchunks, t, f, mv_bits, mv_bits + words);
  }
}

template <int RLO, int RHI>
__device__ __forceinline__ void prep_segment_dispatch(const DevGrid& g, const Batch& b, int r, int c, int slot, int j0,
                                                      int j1, const PcFac& f) {
  if constexpr (RLO <= RHI) {
    if (r == RLO)
      prep_segment<RLO>(g, b, c, slot, j0, j1, f);
    else
      prep_segment_dispatch<RLO + 1, RHI>(g, b, r, c, slot, j0, j1, f);
  }
}

// Ranks [RLO, RHI] from the rank buckets of k_bucket (one register allocation
// per class; the classes run as separate launches).
template <int RLO, int RHI>
__global__ void __launch_bounds__(32 * kPrepRowWarps, RHI <= 4 ? 4 : (RHI <= 7 ? 3 : 2))
    k_prep_rows(DevGrid g, Batch b, unsigned* ctr) {
  __shared__ PcFac slab[kPrepRowWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PcFac& f = slab[warp];
  const int per = b.nchunks + g.Kpad / 32;
  const int nseg = (per + kPrepSeg - 1) / kPrepSeg;
  const int first = b.wl_start[RLO];
  const int ncand = b.wl_start[RHI] + b.wl_count[RHI] - first;
  const unsigned total = static_cast<unsigned>(ncand) * static_cast<unsigned>(nseg);  // 32-bit: cheap division
  int loaded = -1;
  for (;;) {
    // items claimed from a counter (a static striding leaves the last CTA wave
    // partly filled)
    unsigned w = 0;
    if (lane == 0) w = atomicAdd(ctr, 1u);
    w = __shfl_sync(0xffffffffu, w, 0);
    if (w >= total) break;
    const unsigned ci = w / static_cast<unsigned>(nseg);
    const int c = b.wl_list[first + static_cast<int>(ci)];
    const int sg = static_cast<int>(w - ci * static_cast<unsigned>(nseg));
    if (b.status[c] != 0) continue;  // islanded by the small solve
    if (c != loaded) {
      __syncwarp();
      copy_block(&f, b.pc + c, sizeof(PcFac), lane, 32);
      __syncwarp();
      loaded = c;
    }
    const int j0 = sg * kPrepSeg, j1 = min(per, j0 + kPrepSeg);
    prep_segment_dispatch<RLO, RHI>(g, b, b.rank[c], c, b.slot[c], j0, j1, f);
  }
}

// ---------------------------------------------------------------- K2b prep, profiles 1..n_t-1
// Multi-timestep screening (capi.cu enqueue_evaluate_mt): the topology factors,
// the L rows and the unscaled contingency factors rk are profile-independent,
// only f_c and alpha change with the injections. One CTA per candidate writes
// the compact per-profile arrays in one pass: the per-profile small right-hand
// sides in parallel (one thread per profile), then each thread reads its
// branch's L row once (profile 0, written by k_prep) and emits f_c for all
// profiles, and each contingency's rk row once and its alpha per profile
// (R'_t = rk * alpha_t is formed by the masked sweep); the bounds of the mask
// pass are folded over the profiles in registers (no per-profile atomics).
__global__ void __launch_bounds__(kPrepCta, 2) k_prep_mt(DevGrid g, Batch b, MtProfiles P) {
  extern __shared__ __align__(16) uint32_t bits[];
  __shared__ Topo t;
  constexpr int kRp = kMaxSplits + kMaxCols;
  const int words = (g.E + 31) >> 5;
  uint32_t* rm_bits = bits + words;
  double* rp_all = reinterpret_cast<double*>(bits + ((2 * words + 3) & ~3));
  int* nc0_s = reinterpret_cast<int*>(rp_all + static_cast<size_t>(P.n_t) * kRp);
  const int lane = threadIdx.x & 31;
  const int ntiles = g.Kpad / 128;
  for (int c = blockIdx.x; c < b.n; c += gridDim.x) {
    const int slot = b.slot[c];
    if (slot < 0 || b.status[c] != 0) continue;  // islanded (analysis or profile 0's small solve)
    copy_block(static_cast<TopoCore*>(&t), b.topo + c, sizeof(TopoCore), threadIdx.x, blockDim.x);
    const uint32_t* tb = b.tbits + static_cast<size_t>(c) * 2 * words;
    for (int i = threadIdx.x; i < 2 * words; i += blockDim.x) bits[i] = tb[i];
    copy_block(t.Sinv, b.topo_sol + static_cast<size_t>(c) * kTopoSol, kTopoSol * sizeof(double), threadIdx.x,
               blockDim.x);
    for (int i = threadIdx.x; i < P.n_t; i += blockDim.x) nc0_s[i] = 0;
    __syncthreads();
    const int ns = t.ns, nv = t.nv, r = ns + nv, rs = row_stride(r);
    // injection side of the small solve, one thread per profile
    for (int tt = 1 + threadIdx.x; tt < P.n_t; tt += blockDim.x) {
      double ppsi[kMaxSplits], th[kMaxCols];
      for (int q = 0; q < ns; ++q) ppsi[q] = 0.0;
      for (int i = 0; i < t.ninj; ++i) {
        const int q = t.q_of_new[t.inj_new[i]];
        if (q >= 0 && !omitted(t, t.inj_id[i])) ppsi[q] += P.inj_net[tt][t.inj_id[i]];
      }
      const double* th0 = P.theta0[tt];
      for (int cc = 0; cc < r; ++cc) {
        double acc = 0.0;
        for (int p = t.col_ptr[cc]; p < t.col_ptr[cc + 1]; ++p) acc = fma(t.term_coef[p], th0[t.term_idx[p]], acc);
        th[cc] = acc;
      }
      small_rhs_into(t, th, ppsi, rp_all + static_cast<size_t>(tt) * kRp);
    }
    __syncthreads();
    // f_c of every profile from the L row of profile 0 (compact per-profile
    // arrays [t][n][E]; profile 0's value is its row's)
    const int e_end = (g.E + 31) & ~31;
    for (int e0 = threadIdx.x; e0 < e_end; e0 += blockDim.x) {
      const int e = e0 < g.E ? e0 : g.E - 1;
      const bool valid = e0 < g.E;
      const double* fr0 = b.feat + feat_index(slot, b.nchunks, e, r);
      const double fc0 = fr0[0];
      const bool on = g.br_on[e] && !bit_get(rm_bits, e);
      // phi / rho in registers: unrolled loops with a CTA-uniform exit (ns, nv
      // are the candidate's), so every index is static
      double phi[kMaxSplits], rho[kSweepRank];
      const double be = g.br_b[e], ib = 1.0 / be;
#pragma unroll
      for (int q = 0; q < kMaxSplits; ++q) {
        if (q >= ns) break;
        phi[q] = on ? fr0[1 + q] * ib : 0.0;
      }
#pragma unroll
      for (int m = 0; m < kSweepRank; ++m) {
        if (m >= nv) break;
        rho[m] = on ? fr0[1 + ns + m] * ib : 0.0;
      }
      unsigned long long* mk = reinterpret_cast<unsigned long long*>(b.feat_mt + feat_index(slot, b.nchunks, e, r + 1));
      unsigned long long kmax = 0ull, kmin = ~0ull;
      const double lim = g.br_lim[e];
      if (valid) P.fc[static_cast<size_t>(c) * g.E + e] = fc0;
      for (int tt = 1; tt < P.n_t; ++tt) {
        const double* rp = rp_all + static_cast<size_t>(tt) * kRp;
        double fc = 0.0;
        if (on) {  // cand_flow (topo.cuh) with this profile's base flow and Rp
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < kMaxSplits; ++q) {
            if (q >= ns) break;
            acc = fma(phi[q], rp[q], acc);
          }
#pragma unroll
          for (int m = 0; m < kSweepRank; ++m) {
            if (m >= nv) break;
            acc = fma(rho[m], rp[ns + m], acc);
          }
          fc = P.f0[tt][e] + be * acc;
        }
        const unsigned cnt = __popc(__ballot_sync(0xffffffffu, valid && fabs(fc) > lim));
        if (lane == 0 && cnt) atomicAdd(nc0_s + tt, static_cast<int>(cnt));
        if (valid) {
          const unsigned long long key = order_key(fc);
          kmax = max(kmax, key);
          kmin = min(kmin, key);
          P.fc[static_cast<size_t>(tt) * P.fc_stride + static_cast<size_t>(c) * g.E + e] = fc;
        }
      }
      if (valid) {
        mk[0] = max(mk[0], kmax);
        mk[1] = min(mk[1], kmin);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int tt = 1; tt < P.n_t; ++tt) b.nc0[static_cast<size_t>(tt) * P.nc0_stride + c] = nc0_s[tt];
    // contingencies: the topology part once (rk rows [0, S^-1 phi, -C^-1 rho]
    // at row_stride(r), profile-independent), alpha per profile ([t][n][Kpad])
    for (int k = threadIdx.x; k < g.Kpad; k += blockDim.x) {
      double rks[kMaxSplits], rkv[kSweepRank];  // rk = [S^-1 phi, -C^-1 rho]
      double den = 1.0;
      bool live = false;  // regular contingency with an active outaged branch
      int beta = -1;
      const uint8_t flag = b.kflag[static_cast<size_t>(c) * g.Kpad + k];  // topology-only, from profile 0
      if (k < g.Ks && flag == 0) {
        beta = g.ks_branch[k];
        const bool on = g.br_on[beta] && !bit_get(rm_bits, beta);
        if (on) {
          const double* fr = b.feat + feat_index(slot, b.nchunks, beta, r);
          const double ib = 1.0 / g.br_b[beta];
          double phi[kMaxSplits], rho[kSweepRank];
#pragma unroll
          for (int q = 0; q < kMaxSplits; ++q) {
            if (q >= ns) break;
            phi[q] = fr[1 + q] * ib;
          }
#pragma unroll
          for (int m = 0; m < kSweepRank; ++m) {
            if (m >= nv) break;
            rho[m] = fr[1 + ns + m] * ib;
          }
          double lr = 0.0;
#pragma unroll
          for (int q = 0; q < kMaxSplits; ++q) {
            if (q >= ns) break;
            double acc = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < kMaxSplits; ++q2) {
              if (q2 >= ns) break;
              acc += t.Sinv[q * kMaxSplits + q2] * phi[q2];
            }
            rks[q] = acc;
            lr += phi[q] * acc;
          }
#pragma unroll
          for (int m = 0; m < kSweepRank; ++m) {
            if (m >= nv) break;
            double acc = 0.0;
#pragma unroll
            for (int m2 = 0; m2 < kSweepRank; ++m2) {
              if (m2 >= nv) break;
              acc += t.Cinv[m * kMaxCols + m2] * rho[m2];
            }
            rkv[m] = -acc;
            lr -= rho[m] * acc;
          }
          den = 1.0 - (g.Tdiag[beta] + g.br_b[beta] * lr);
          live = !(fabs(den) < 1e-8);  // a bridge with flag 0 is a dead stub: flows unchanged
        }
      }
      {
        double row[kStride];
#pragma unroll
        for (int i = 0; i < kStride; ++i) row[i] = 0.0;
        if (live) {
#pragma unroll
          for (int q = 0; q < kMaxSplits; ++q) {
            if (q >= ns) break;
            row[1 + q] = rks[q];
          }
#pragma unroll
          for (int m = 0; m < kSweepRank; ++m) {
            if (m >= nv) break;
            row[1 + ns + m] = rkv[m];
          }
        }
        double2* dst = reinterpret_cast<double2*>(P.rk + static_cast<size_t>(c) * g.Kpad * kStride +
                                                  static_cast<size_t>(k) * rs);
#pragma unroll
        for (int i = 0; i < kStride / 2; ++i)
          if (2 * i < rs) dst[i] = make_double2(row[2 * i], row[2 * i + 1]);
      }
      double dlmax = 0.0, rqs[kMaxSplits], rqv[kSweepRank];  // max_t |rk alpha_t| per column
#pragma unroll
      for (int q = 0; q < kMaxSplits; ++q) rqs[q] = 0.0;
#pragma unroll
      for (int m = 0; m < kSweepRank; ++m) rqv[m] = 0.0;
      for (int tt = 0; tt < P.n_t; ++tt) {
        double alpha = 0.0;
        if (live) {
          const double fcb = P.fc[static_cast<size_t>(tt) * P.fc_stride + static_cast<size_t>(c) * g.E + beta];
          alpha = fcb / den;
        }
        P.al[static_cast<size_t>(tt) * P.al_stride + static_cast<size_t>(c) * g.Kpad + k] = alpha;
        if (tt == 0) continue;  // profile 0: penalties and bounds written by k_prep
        if (k < g.Ks && flag == 1)
          b.energy[static_cast<size_t>(tt) * P.energy_stride + static_cast<size_t>(c) * g.Kall + g.ks_cont[k]] =
              b.params.penalty;
        dlmax = fmax(dlmax, fabs(alpha - P.alpha0[tt][k]));
        if (live) {  // (rk is zero otherwise: the maxima stay 0)
#pragma unroll
          for (int q = 0; q < kMaxSplits; ++q) {
            if (q >= ns) break;
            rqs[q] = fmax(rqs[q], fabs(rks[q] * alpha));
          }
#pragma unroll
          for (int m = 0; m < kSweepRank; ++m) {
            if (m >= nv) break;
            rqv[m] = fmax(rqv[m], fabs(rkv[m] * alpha));
          }
        }
      }
      // fold into the bounds profile 0 wrote (tiles of 128: a warp is 32
      // consecutive contingencies of one tile, half a warp one sub-tile)
      const int tile = k >> 7, sub = (k & 127) >> 4;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) dlmax = fmax(dlmax, __shfl_xor_sync(0xffffffffu, dlmax, o));
      if ((threadIdx.x & 15) == 0)
        atomicMax(b.amx_mt + (static_cast<size_t>(c) * ntiles + tile) * kTmaxSub + sub, dbits(dlmax));
      for (int q = 0; q < r; ++q) {
        double rq = 0.0;  // rqmax[q] (static register indices)
#pragma unroll
        for (int i = 0; i < kMaxSplits; ++i)
          if (i == q) rq = rqs[i];
#pragma unroll
        for (int m = 0; m < kSweepRank; ++m)
          if (ns + m == q) rq = rqv[m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rq = fmax(rq, __shfl_xor_sync(0xffffffffu, rq, o));
        if (lane == 0) atomicMax(b.rmx_mt + (static_cast<size_t>(c) * ntiles + tile) * kStride + 1 + q, dbits(rq));
      }
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
  __shared__ int n_extra, n_omit, skip, overflow;
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
      overflow = 0;
      if (!skip) {
        if (cs < g.Kx) {
          // lists longer than the capacities are rejected at context creation;
          // never truncated here (an overflow is a capacity error for the lane)
          if (g.kx_br_ptr[cs + 1] - g.kx_br_ptr[cs] > kMaxRemoved || g.kx_inj_ptr[cs + 1] - g.kx_inj_ptr[cs] > kMaxPMod)
            overflow = 1;
          for (int p = g.kx_br_ptr[cs]; p < g.kx_br_ptr[cs + 1] && n_extra < kMaxRemoved; ++p) extra[n_extra++] = g.kx_br[p];
          for (int p = g.kx_inj_ptr[cs]; p < g.kx_inj_ptr[cs + 1] && n_omit < kMaxPMod; ++p) omit[n_omit++] = g.kx_inj[p];
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
          if (hi - lo > kMaxRemoved) overflow = 1;
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
    if (threadIdx.x == 0) {
      analyze(g, t, mv_bits, rm_bits, slots, n_a, n_d, extra, n_extra, omit, n_omit);
      if (overflow) t.islanded = 2;
    }
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
// get the sentinel score with lambda_d/s/r filled. One warp per candidate
// (warp reductions only). Worst-k (dc_engine.cpp:400-420: energy > 0, sorted
// by energy desc then index asc, first worst_k): the positive energies are
// compacted into the warp's shared list, then worst_k selection rounds run on
// the list (or on all contingencies when it overflows).
constexpr int kFinishWarps = 8;
constexpr int kFinishList = 256;

__device__ __forceinline__ bool worst_before(double v, int k, double u, int j) {
  return v > u || (v == u && k < j);
}

// One warp: the first wk entries with energy > 0 of en[0..K) in the order
// (energy desc, index asc) -- the reference's worst list (dc_engine.cpp:398-419).
// One pass over en: positive energies are appended to the warp's shared list
// (lv, li; kFinishList entries); when the list would overflow it is cut to its
// wk best entries, and from then on only entries ranked before the wk-th best
// seen so far are appended (later indices lose ties, so "before" is a strict
// energy comparison there). Selection rounds then rank the list.
__device__ void warp_select(const double* lv, const int* li, int n, int wk, int lane, int* sel_idx, double* sel_val,
                            int* n_sel, double* last_v, int* last_i) {
  double pv = CUDART_INF;
  int pi = -1, nsel = 0;
  for (int round = 0; round < wk; ++round) {
    double bv = 0.0;
    int bi = -1;
    for (int i = lane; i < n; i += 32) {
      const double v = lv[i];
      const int k = li[i];
      if (!worst_before(pv, pi, v, k)) continue;  // already selected
      if (bi < 0 || worst_before(v, k, bv, bi)) bv = v, bi = k;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
      if (oi >= 0 && (bi < 0 || worst_before(ov, oi, bv, bi))) bv = ov, bi = oi;
    }
    if (bi < 0) break;
    if (sel_idx && lane == 0) sel_idx[round] = bi, sel_val[round] = bv;
    pv = bv;
    pi = bi;
    ++nsel;
  }
  *n_sel = nsel;
  *last_v = pv;
  *last_i = pi;
}

__device__ void warp_worst(const double* en, int K, int wk, double* lv, int* li, int* out_idx, double* out_val,
                           int* out_n, int lane) {
  if (2 * wk > kFinishList) {  // long worst lists: rank the energies in place (no list)
    double pv = CUDART_INF;
    int pi = -1, nsel = 0;
    for (int round = 0; round < wk; ++round) {
      double bv = 0.0;
      int bi = -1;
      for (int k = lane; k < K; k += 32) {
        const double v = en[k];
        if (!(v > 0.0) || !worst_before(pv, pi, v, k)) continue;
        if (bi < 0 || worst_before(v, k, bv, bi)) bv = v, bi = k;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, d);
        if (oi >= 0 && (bi < 0 || worst_before(ov, oi, bv, bi))) bv = ov, bi = oi;
      }
      if (bi < 0) break;
      if (lane == 0) out_idx[round] = bi, out_val[round] = bv;
      pv = bv;
      pi = bi;
      ++nsel;
    }
    if (lane == 0) *out_n = nsel;
    return;
  }
  int npos = 0;
  double tv = 0.0;  // entries must rank before (tv, ti); ti < 0: any positive energy
  int ti = -1;
  for (int k0 = 0; k0 < K; k0 += 128) {
    double vv[4];  // four blocks of 32 in flight
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = k0 + 32 * u + lane < K ? en[k0 + 32 * u + lane] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + 32 * u + lane;
      const double v = vv[u];
      bool take = v > 0.0 && (ti < 0 || worst_before(v, k, tv, ti));
      unsigned m = __ballot_sync(0xffffffffu, take);
      if (npos + __popc(m) > kFinishList) {
        // cut the list to its wk best entries (stable, in place: writes trail reads)
        __syncwarp();
        int ns;
        warp_select(lv, li, npos, wk, lane, nullptr, nullptr, &ns, &tv, &ti);
        int kept = 0;
        for (int i0 = 0; i0 < npos; i0 += 32) {
          const int i = i0 + lane;
          double x = 0.0;
          int xi = 0;
          bool keep = false;
          if (i < npos) {
            x = lv[i];
            xi = li[i];
            keep = ti >= 0 && !worst_before(tv, ti, x, xi);  // ranked at or before the wk-th best
          }
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          if (keep) {
            const int at = kept + __popc(km & ((1u << lane) - 1u));
            lv[at] = x;
            li[at] = xi;
          }
          kept += __popc(km);
        }
        __syncwarp();
        npos = kept;
        if (ti < 0) npos = 0;  // wk == 0: nothing is ever kept
        take = v > 0.0 && ti >= 0 && worst_before(v, k, tv, ti);
        m = __ballot_sync(0xffffffffu, take);
      }
      if (take) {
        const int at = npos + __popc(m & ((1u << lane) - 1u));
        lv[at] = v;
        li[at] = k;
      }
      npos += __popc(m);
    }
  }
  __syncwarp();
  int nsel;
  double lvv;
  int lii;
  warp_select(lv, li, npos, wk, lane, out_idx, out_val, &nsel, &lvv, &lii);
  if (lane == 0) *out_n = nsel;
}

__global__ void __launch_bounds__(32 * kFinishWarps) k_finish(DevGrid g, Batch b, int n_a, int n_d) {
  __shared__ double wl_v[kFinishWarps][kFinishList];
  __shared__ int wl_i[kFinishWarps][kFinishList];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = blockIdx.x * kFinishWarps + wid;
  if (c >= b.n) return;
  const int* slots = b.genomes + static_cast<size_t>(c) * (n_a + n_d);
  int ld = 0, ls = 0, lr = 0;
  for (int k = 0; k < n_d; ++k) ld += slots[n_a + k] >= 0;
  for (int k = 0; k < n_a; ++k)
    if (slots[k] >= 0) ++ls, lr += g.act_lambda_r[slots[k]];
  Scores& o = b.out;
  const int st = b.status[c];
  if (st != 0) {
    if (lane == 0) {
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
      if (st != 1 && b.err_sticky) atomicOr(b.err_sticky, 1);
      o.worst_n[c] = 0;
      o.isl_out[c] = 0;
      o.isl_bus[c] = 0;
    }
    return;
  }
  const unsigned long long* fm = b.fmax + static_cast<size_t>(c) * g.E;
  const unsigned long long* fb = b.fbus + static_cast<size_t>(c) * g.E;
  double so = 0.0, sb = 0.0;
  int nc = 0, nc0 = lane == 0 ? b.nc0[c] : 0;  // counted by k_prep
  // four rows per lane in flight (loads first), summed in branch order per lane
  for (int e0 = lane; e0 < g.E; e0 += 128) {
    double lim[4], m[4], mb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + 32 * u;
      lim[u] = e < g.E ? g.br_lim[e] : CUDART_INF;
      m[u] = e < g.E ? __longlong_as_double(static_cast<long long>(fm[e])) : 0.0;
      mb[u] = e < g.E && g.Kb > 0 ? __longlong_as_double(static_cast<long long>(fb[e])) : 0.0;  // no busbar outages: 0
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (m[u] > lim[u]) so += m[u] - lim[u], ++nc;
      if (mb[u] > lim[u]) sb += mb[u] - lim[u];
    }
  }
  int isl = 0;
  const uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad;
  for (int k = lane; k < g.Ks; k += 32) isl += kf[k] == 1;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    so += __shfl_xor_sync(0xffffffffu, so, d);
    sb += __shfl_xor_sync(0xffffffffu, sb, d);
    nc += __shfl_xor_sync(0xffffffffu, nc, d);
    nc0 += __shfl_xor_sync(0xffffffffu, nc0, d);
    isl += __shfl_xor_sync(0xffffffffu, isl, d);
  }
  if (lane == 0) {
    const int iso = b.isl_out[c] + isl, isb = b.isl_bus[c];
    const double lo = so + b.params.penalty * iso;
    const double lb = sb + b.params.penalty * isb;
    double fit = -(lo + b.params.weight_c0 * nc0 + b.params.weight_c * nc);
    if (b.params.variant == 2) fit -= fmax(lb - b.params.lambda_b_pre, 0.0);
    o.lambda_o[c] = lo;
    o.lambda_c[c] = nc;
    o.lambda_c0[c] = nc0;
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
  if (b.no_worst) {  // one profile of a timestep grid: the worst list is ranked on the summed energies
    if (lane == 0) o.worst_n[c] = 0;
    return;
  }
  warp_worst(b.energy + static_cast<size_t>(c) * g.Kall, g.Kall, b.params.worst_k, wl_v[wid], wl_i[wid],
             o.worst_idx + static_cast<size_t>(c) * b.params.worst_k,
             o.worst_val + static_cast<size_t>(c) * b.params.worst_k, o.worst_n + c, lane);
}

// ---------------------------------------------------------------- timesteps
// Timestep extension (model.hpp): a batch over T injection profiles runs the
// whole pipeline once per timestep (the topology part is recomputed; tables
// indexed by t) and aggregates: lambda_o, lambda_c, lambda_c0, lambda_b and the
// islanded counts summed over t, per-contingency energies summed over t (the
// worst list ranks the sums), islanded if islanded at any t. With T == 1 this
// is exactly the reference's evaluate.
__global__ void k_accum_t(Batch bt, Scores agg, double* agg_energy, int Kall, int first) {
  const size_t n_en = agg_energy ? static_cast<size_t>(bt.n) * Kall : 0;  // null: energies summed by k_sum_profiles
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n_en;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    agg_energy[i] = first ? bt.energy[i] : agg_energy[i] + bt.energy[i];
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < bt.n; c += gridDim.x * blockDim.x) {
    const Scores& o = bt.out;
    if (first) {
      agg.lambda_o[c] = o.lambda_o[c];
      agg.lambda_c[c] = o.lambda_c[c];
      agg.lambda_c0[c] = o.lambda_c0[c];
      agg.lambda_b[c] = o.lambda_b[c];
      agg.lambda_d[c] = o.lambda_d[c];
      agg.lambda_s[c] = o.lambda_s[c];
      agg.lambda_r[c] = o.lambda_r[c];
      agg.islanded[c] = o.islanded[c];
      agg.error[c] = o.error[c];
      agg.isl_out[c] = o.isl_out[c];
      agg.isl_bus[c] = o.isl_bus[c];
    } else {
      agg.lambda_o[c] += o.lambda_o[c];
      agg.lambda_c[c] += o.lambda_c[c];
      agg.lambda_c0[c] += o.lambda_c0[c];
      agg.lambda_b[c] += o.lambda_b[c];
      agg.islanded[c] |= o.islanded[c];
      agg.error[c] = max(agg.error[c], o.error[c]);
      agg.isl_out[c] += o.isl_out[c];
      agg.isl_bus[c] += o.isl_bus[c];
    }
  }
}

// Fitness (dc_engine.cpp:402-410 on the summed metrics) and the worst list of
// the summed energies; one warp per candidate.
__global__ void __launch_bounds__(32 * kFinishWarps) k_finish_agg(Batch b, int Kall) {
  __shared__ double wl_v[kFinishWarps][kFinishList];
  __shared__ int wl_i[kFinishWarps][kFinishList];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = blockIdx.x * kFinishWarps + wid;
  if (c >= b.n) return;
  Scores& o = b.out;
  const int wk = b.params.worst_k;
  if (o.islanded[c] || o.error[c]) {
    if (lane == 0) {
      o.lambda_o[c] = 0.0;
      o.lambda_c[c] = 0;
      o.lambda_c0[c] = 0;
      o.lambda_b[c] = 0.0;
      o.fitness[c] = -CUDART_INF;
      o.worst_n[c] = 0;
      o.isl_out[c] = 0;
      o.isl_bus[c] = 0;
    }
    return;
  }
  if (lane == 0) {
    double fit = -(o.lambda_o[c] + b.params.weight_c0 * o.lambda_c0[c] + b.params.weight_c * o.lambda_c[c]);
    if (b.params.variant == 2) fit -= fmax(o.lambda_b[c] - b.params.lambda_b_pre, 0.0);
    o.fitness[c] = fit;
  }
  warp_worst(b.energy + static_cast<size_t>(c) * Kall, Kall, wk, wl_v[wid], wl_i[wid],
             o.worst_idx + static_cast<size_t>(c) * wk, o.worst_val + static_cast<size_t>(c) * wk, o.worst_n + c,
             lane);
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
// Phases of one evaluation (launch_evaluate runs them in order; the
// multi-timestep path of capi.cu interleaves them across profiles).
int launch_eval_reset(const DevGrid& g, Batch& b, cudaStream_t stream) {
  cudaMemsetAsync(b.fmax, 0, static_cast<size_t>(b.n) * g.E * sizeof(unsigned long long), stream);
  if (g.Kb > 0)  // only busbar outages fold into fbus (k_special); k_finish reads it only then
    cudaMemsetAsync(b.fbus, 0, static_cast<size_t>(b.n) * g.E * sizeof(unsigned long long), stream);
  cudaMemsetAsync(b.energy, 0, static_cast<size_t>(b.n) * g.Kall * sizeof(double), stream);
  cudaMemsetAsync(b.isl_out, 0, b.n * sizeof(int), stream);
  cudaMemsetAsync(b.isl_bus, 0, b.n * sizeof(int), stream);
  return 0;
}

int launch_analyze(const DevGrid& g, Batch& b, int n_a, int n_d, cudaStream_t stream) {
  int launched = 0;
  const size_t bits_bytes = 2 * static_cast<size_t>((g.E + 31) >> 5) * sizeof(uint32_t);
  static std::atomic<unsigned long long> carveout{0};
  if (first_use_on_device(carveout))  // one wave of warp-sized analysis CTAs needs the full shared-memory carveout
    cudaFuncSetAttribute(k_analyze, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_analyze<<<b.n < 65535 ? b.n : 65535, kAnalyzeThreads, bits_bytes, stream>>>(g, b, n_a, n_d);
  ++launched;
  launch_bucket(b, stream, &launched);
  return launched;
}

int launch_prep(const DevGrid& g, Batch& b, int n_a, int n_d, const EvalScratch& s, cudaStream_t stream) {
  // split form (branch-space columns; single-profile batches: the timestep
  // screening keeps k_prep, which also writes its bounds and factors)
  static const bool split_off = std::getenv("TGB_NO_SPLIT_PREP") != nullptr;  // A/B switch
  if (g.PhiA && !b.feat_mt && !b.amx_mt && !b.topo_sol && !split_off) {
    if (b.n == 0) return 0;
    k_prep_solve<<<b.n < 65535 ? b.n : 65535, 32, 0, stream>>>(g, b);
    // grid: the warp work items a class can have at most (small batches launch
    // few CTAs), at most 8 CTAs per SM
    const long seg = (b.nchunks + g.Kpad / 32 + kPrepSeg - 1) / kPrepSeg;
    const int rows_grid = static_cast<int>(std::min<long>(148 * 8, (static_cast<long>(b.n) * seg + 7) / 8));
    cudaMemsetAsync(b.item_ctr + 1, 0, 3 * sizeof(unsigned int), stream);  // the classes' item counters
    k_prep_rows<0, 4><<<rows_grid, 256, 0, stream>>>(g, b, b.item_ctr + 1);
    k_prep_rows<5, kChunkedMaxRank><<<rows_grid, 256, 0, stream>>>(g, b, b.item_ctr + 2);  // without the rank 8-11 registers
    k_prep_rows<kChunkedMaxRank + 1, kSweepRank><<<rows_grid, 256, 0, stream>>>(g, b, b.item_ctr + 3);
    return 4;
  }
  const size_t bits_bytes = 2 * static_cast<size_t>((g.E + 31) >> 5) * sizeof(uint32_t);
  if (bits_bytes > 48 * 1024)  // (per launch: the size depends on the grid)
    cudaFuncSetAttribute(k_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bits_bytes));
  const int prep_grid = b.n < s.zslots ? b.n : s.zslots;
  k_prep<<<prep_grid, kPrepCta, bits_bytes, stream>>>(g, b, n_a, n_d, s.zprep);
  return 1;
}

int launch_prep_mt(const DevGrid& g, Batch& b, const MtProfiles& p, cudaStream_t stream) {
  if (p.n_t < 2 || b.n == 0) return 0;
  const size_t bits_bytes = 2 * static_cast<size_t>((g.E + 31) >> 5) * sizeof(uint32_t);
  const size_t smem = ((bits_bytes + 15) & ~size_t{15}) + static_cast<size_t>(p.n_t) * (kMaxSplits + kMaxCols) * 8 +
                      static_cast<size_t>(p.n_t) * sizeof(int);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_prep_mt, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_prep_mt<<<b.n, kPrepCta, smem, stream>>>(g, b, p);
  return 1;
}

int launch_special(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                   cudaStream_t stream) {
  if (g.Kx + g.Kb == 0 || b.n == 0) return 0;
  const size_t bits_bytes = 2 * static_cast<size_t>((g.E + 31) >> 5) * sizeof(uint32_t);
  const long total = static_cast<long>(b.n) * (g.Kx + g.Kb);
  const int grid = static_cast<int>(total < s.zslots_special ? total : s.zslots_special);
  k_special<<<grid, kPrepThreads, bits_bytes, stream>>>(g, b, n_a, n_d, full ? 1 : 0, s.zspecial);
  return 1;
}

int launch_special_finish(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                          cudaStream_t stream) {
  int launched = launch_special(g, b, n_a, n_d, full, s, stream);
  k_finish<<<(b.n + kFinishWarps - 1) / kFinishWarps, 32 * kFinishWarps, 0, stream>>>(g, b, n_a, n_d);
  ++launched;
  return launched;
}

void launch_evaluate(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                     cudaStream_t stream, int* kernels, cudaEvent_t sweep_begin, cudaEvent_t sweep_end,
                     const SideStream* side) {
  int launched = launch_eval_reset(g, b, stream);
  launched += launch_analyze(g, b, n_a, n_d, stream);
  // the special outages (multi-branch / injection contingencies, busbar
  // outages) only need the analysis: on the side stream they run beside the
  // prep and the sweep (they write their own energies and fold atomically)
  const bool fork = side && side->stream && g.Kx + g.Kb > 0;
  if (fork) {
    cudaEventRecord(side->fork, stream);
    cudaStreamWaitEvent(side->stream, side->fork, 0);
    launched += launch_special(g, b, n_a, n_d, full, s, side->stream);
    cudaEventRecord(side->join, side->stream);
  }
  launched += launch_prep(g, b, n_a, n_d, s, stream);
  if (g.Ks > 0) launch_sweep(g, b, full, stream, sweep_begin, sweep_end, &launched);
  if (fork) {
    cudaStreamWaitEvent(stream, side->join, 0);
    k_finish<<<(b.n + kFinishWarps - 1) / kFinishWarps, 32 * kFinishWarps, 0, stream>>>(g, b, n_a, n_d);
    ++launched;
  } else {
    launched += launch_special_finish(g, b, n_a, n_d, full, s, stream);
  }
  if (kernels) *kernels = launched;
}

int launch_accumulate_timestep(const Batch& bt, Scores& agg, double* agg_energy, int Kall, bool first,
                               cudaStream_t stream) {
  const size_t work = static_cast<size_t>(bt.n) * (Kall > 0 ? Kall : 1);
  const int grid = static_cast<int>(std::min<size_t>((work + 255) / 256, 148 * 8));
  k_accum_t<<<grid, 256, 0, stream>>>(bt, agg, agg_energy, Kall, first ? 1 : 0);
  return 1;
}

// Sum of the per-profile energy arrays in profile order (the same additions as
// k_accum_t's running sum), one pass over all profiles.
__global__ void k_sum_profiles(const double* e, int n_t, size_t stride, size_t n, double* out) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double acc = e[i];
    for (int t = 1; t < n_t; ++t) acc = acc + e[static_cast<size_t>(t) * stride + i];
    out[i] = acc;
  }
}

int launch_sum_profiles(const double* e, int n_t, size_t stride, size_t n, double* out, cudaStream_t stream) {
  const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 8));
  k_sum_profiles<<<grid > 0 ? grid : 1, 256, 0, stream>>>(e, n_t, stride, n, out);
  return 1;
}

int launch_finish_aggregate(Batch& b, int Kall, cudaStream_t stream) {
  k_finish_agg<<<(b.n + kFinishWarps - 1) / kFinishWarps, 32 * kFinishWarps, 0, stream>>>(b, Kall);
  return 1;
}

void launch_extract(const DevGrid& g, Batch& b, double* base_out, double* fmax_out, double* fbus_out,
                    cudaStream_t stream) {
  const size_t n = static_cast<size_t>(b.n) * g.E;
  if (base_out) k_extract_base<<<512, 256, 0, stream>>>(g, b, base_out);
  if (fmax_out) k_bits_to_double<<<512, 256, 0, stream>>>(b.fmax, fmax_out, n);
  if (fbus_out) k_bits_to_double<<<512, 256, 0, stream>>>(b.fbus, fbus_out, n);
}


}  // namespace tgb
