// K3: the fused N-1 contingency sweep (dc_engine.cpp:294-371 for single-branch
// contingencies, all candidates of a batch at once).
//
// For candidate c, monitored branch e and contingency k (branch beta_k):
//   f1[e,k] = f_c[e] + T_base[e,k] * alpha_k + sum_r L[e,r] * R'[r,k]
// (topo.cuh: T_cand = T_base + L R, alpha_k = f_c[beta]/(1 - T_cand[beta,beta]),
// R' = R * alpha). The E x K x B tensor is never written: each element is
// tested against the branch limit in registers; only elements with
// |f1| > limit touch the per-(c,k) energy accumulators (registers, summed in
// branch order) and the per-(c,e) max (atomicMax on the ordered bit pattern).
//
// Dataflow (one CTA = one 128-contingency tile x 8*NC candidates):
//   * T_base tiles ([tile][E][128], 32 branches = 32 KB per stage), the
//     candidates' branch rows (f_c, L) and the branch limits are streamed into
//     shared memory by TMA bulk copies (cp.async.bulk + mbarrier complete_tx),
//     3-stage pipeline, one elected producer thread;
//   * each lane owns 4 contingencies: alpha / R' live in registers for the
//     whole sweep; each warp processes NC candidates so one T load feeds NC
//     candidates' FMAs;
//   * two-stage exact skip: a per-row bound over the whole tile (no element
//     work), then the exact first FMA f_c + T alpha per element with the L R'
//     part bounded; only rows passing both run the remaining R DFMA per
//     element and a 2-op hi-word test; the exact path runs only where |f1| can
//     exceed the limit.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "engine.cuh"

namespace tgb {

namespace {

constexpr int kKpl = 4;                  // contingencies per lane
constexpr int kTileK = 32 * kKpl;        // contingencies per CTA tile
constexpr int kWarps = 16;
constexpr int kThreads = 32 * kWarps;
constexpr int kChunk = 32;               // branches per pipeline stage
constexpr int kStages = 3;
constexpr int kMaxCand = kWarps;         // one candidate per warp
constexpr int kGroupBlock = 8;           // candidate groups per CTA super-block (L2 reuse of T_base tiles)

// candidates per warp for a given rank (register budget)
__host__ __device__ constexpr int nc_for_rank(int) { return 1; }
__host__ __device__ constexpr int cand_per_cta(int r) { return kWarps * nc_for_rank(r); }

constexpr size_t kStageT = static_cast<size_t>(kChunk) * kTileK;           // doubles
constexpr size_t kStageF = static_cast<size_t>(kMaxCand) * kChunk * kStride;  // doubles
constexpr size_t kStageL = kChunk;                                         // doubles
constexpr size_t kStageTm = static_cast<size_t>(kChunk) * kRec;           // skip record per row
constexpr int kSubLanes = 32 / kTmaxSub;                                   // lanes per sub-tile
static_assert(kTileK % kTmaxSub == 0 && kSubLanes * kTmaxSub == 32 && kTmaxSub == kStride, "sub-tile layout");
constexpr size_t kStageDoubles = kStageT + kStageF + kStageL + kStageTm;
static_assert(kMaxCand == kGroupSlots && kChunk == kChunkRows, "sweep tiles must match the row layout");
constexpr size_t kSmemBytes = kStages * kStageDoubles * sizeof(double) + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t hi_abs(double x) {
  return static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu;
}

struct CtaWork {
  int cand[kMaxCand];
  int ncand;
  int group;
};

// Producer: stage `s` <- chunk `i` (T tile rows, candidate rows, limits).
__device__ __forceinline__ void issue_chunk(const DevGrid& g, const Batch& b, const CtaWork& w, int tile, int i,
                                           double* stage, uint64_t* bar) {
  const int e0 = i * kChunk;
  const int rows = min(kChunk, g.E - e0);
  const uint32_t bt = rows * kTileK * sizeof(double);
  const uint32_t bf = kStageF * sizeof(double);  // the group's rows of this chunk: one contiguous block
  const uint32_t bl = ((rows + 1) & ~1) * sizeof(double);
  const uint32_t bm = rows * kRec * sizeof(double);
  mbar_expect_tx(bar, bt + bf + bl + bm);
  bulk_g2s(stage, g.TK + (static_cast<size_t>(tile) * g.E + e0) * kTileK, bt, bar);
  bulk_g2s(stage + kStageT, b.feat + feat_index(w.group * kGroupSlots, b.nchunks, e0), bf, bar);
  bulk_g2s(stage + kStageT + kStageF, g.br_lim + e0, bl, bar);
  bulk_g2s(stage + kStageT + kStageF + kStageL, g.Tmax + (static_cast<size_t>(tile) * (g.E + kChunk) + e0) * kRec,
           bm, bar);
}

template <int R, int NC, bool FULL>
__device__ __forceinline__ void sweep_cta(const DevGrid& g, const Batch& b, const CtaWork& w, int tile, double* smem,
                                          uint64_t* bars, int* release, double* rmax_s, double* amax_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = tile * kTileK + lane * kKpl;
  // per-(candidate, contingency) operands in registers
  double alpha[NC][kKpl], rr[NC][kKpl][R > 0 ? R : 1], energy[NC][kKpl];
  bool kval[NC][kKpl];
  int kbr[kKpl];
  int cid[NC], rem[NC][kMaxRemovedSweep];
#pragma unroll
  for (int i = 0; i < kKpl; ++i) kbr[i] = kb + i < g.Ks ? g.ks_branch[kb + i] : -1;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int slot = warp * NC + j;
    cid[j] = slot < w.ncand ? w.cand[slot] : -1;
    if (cid[j] >= 0 && b.status[cid[j]] != 0) cid[j] = -1;  // islanded by the small solve in k_prep
    const int c = cid[j] >= 0 ? cid[j] : w.cand[0];
    const double* kd = b.kdat + (static_cast<size_t>(c) * g.Kpad + kb) * kStride;
    const uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad + kb;
#pragma unroll
    for (int i = 0; i < kKpl; ++i) {
      alpha[j][i] = kd[i * kStride];
#pragma unroll
      for (int q = 0; q < R; ++q) rr[j][i][q] = kd[i * kStride + 1 + q];
      energy[j][i] = 0.0;
      kval[j][i] = cid[j] >= 0 && kf[i] == 0;
    }
#pragma unroll
    for (int q = 0; q < kMaxRemovedSweep; ++q) rem[j][q] = b.removed[static_cast<size_t>(c) * kMaxRemovedSweep + q];
  }
  // Skip-bound operands in shared memory (invalid contingencies carry alpha 0):
  // max |alpha - alpha0| per sub-tile, asub[j][s] (the candidate's departure
  // from the unchanged topology's flow factors), and the tile max of each
  // |R'_q| as a row weight vector rms[j][slot] (0 for f_c and padding).
  double* rms = rmax_s + warp * NC * kStride;
  double* asub = amax_s + warp * NC * kTmaxSub;
  if (lane < NC * kStride) rms[lane] = 0.0;
  __syncwarp();
  double a0[kKpl];
#pragma unroll
  for (int k = 0; k < kKpl; ++k) a0[k] = g.alpha0[kb + k];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) a = fmax(a, fabs(alpha[j][k] - a0[k]));
#pragma unroll
    for (int o = kSubLanes / 2; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane % kSubLanes == 0) asub[j * kTmaxSub + lane / kSubLanes] = a * (1.0 + 1e-12);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double r = 0.0;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) r = fmax(r, fabs(rr[j][k][q]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (lane == 0) rms[j * kStride + 1 + q] = r * (1.0 + 1e-12);
    }
  }
  __syncwarp();

  const int nchunks = (g.E + kChunk - 1) / kChunk;
  unsigned rows_computed = 0, rows_offered = 0, rows_exact = 0, rows_partial = 0;  // skip statistics, one atomic per warp at the end
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && s < nchunks; ++s)
      issue_chunk(g, b, w, tile, s, smem + s * kStageDoubles, bars + s);

  // exact path for one branch row: energies (registers) and fmax (atomicMax)
  auto exact_row = [&](int e, double lim, const double (&f1)[NC][kKpl]) {
    const unsigned long long lim_bits = static_cast<unsigned long long>(__double_as_longlong(lim));
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      bool skip_row = false;
#pragma unroll
      for (int q = 0; q < kMaxRemovedSweep; ++q) skip_row |= e == rem[j][q];
      unsigned long long m = 0ull;  // max |f1| as the ordered bit pattern of a non-negative double
#pragma unroll
      for (int k = 0; k < kKpl; ++k) {
        if (!kval[j][k] || skip_row || e == kbr[k]) continue;  // the outaged branch carries 0
        const double a = fabs(f1[j][k]);
        if (a > lim) energy[j][k] += a - lim;
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(a)));
      }
      if (cid[j] < 0) continue;
      unsigned long long* fmx = b.fmax + static_cast<size_t>(cid[j]) * g.E;
      if (FULL) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0 && m > 0ull) atomicMax(fmx + e, m);
      } else if (m > lim_bits) {
        atomicMax(fmx + e, m);
      }
    }
  };

  for (int i = 0; i < nchunks; ++i) {
    const int s = i % kStages;
    const double* st = smem + s * kStageDoubles;
    mbar_wait(bars + s, (i / kStages) & 1);
    const int e0 = i * kChunk;
    const int rows = min(kChunk, g.E - e0);
    const double* sT = st + lane * kKpl;
    const double* sF = st + kStageT + static_cast<size_t>(warp) * NC * kChunk * kStride;
    const double* sL = st + kStageT + kStageF;
    // Stage 1 (one lane per row): rows that can reach their limit for one of
    // the warp's candidates. With alpha = alpha0 + delta (alpha0: unchanged
    // topology) every element of the tile satisfies
    //   f1 = f_c + T alpha0 + T delta + L R'  in  [f_c + D0min - w, f_c + D0max + w],
    //   w = max_s max|T_base|_s max|delta|_s + lrb,  lrb = sum_q |L_q| max|R'_q|
    // (D0max / D0min: max / min of T_base * alpha0 over the tile, precomputed;
    // s: sub-tiles; R' maxima over the tile). A relative slack of 1e-12 on
    // every term covers the rounding of the computed f1. For stage 2 each lane
    // keeps, per candidate, the high word of lim (1 - 1e-12) - lrb (0 when that
    // is not positive).
    unsigned need = rows >= 32 ? 0xffffffffu : ((1u << rows) - 1u);
    uint32_t thr_lane[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) thr_lane[j] = 0u;
    if (!FULL) {
      bool hot = false;
      if (lane < rows) {
        const double lim = sL[lane] * (1.0 - 1e-12);
        const double* rec = st + kStageT + kStageF + kStageL + lane * kRec;
        const double2* tmr = reinterpret_cast<const double2*>(rec);
        const double2 d0 = *reinterpret_cast<const double2*>(rec + kTmaxSub);
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          // the row's 4 double2 read in a lane-rotated order (conflict-free),
          // each weighted by its slots' R' maxima
          const double2* fr = reinterpret_cast<const double2*>(sF + (static_cast<size_t>(j) * kChunk + lane) * kStride);
          const double2* wr = reinterpret_cast<const double2*>(rms + j * kStride);
          const double2* ar = reinterpret_cast<const double2*>(asub + j * kTmaxSub);
          double lrb = 0.0, fc = 0.0, ta = 0.0;
#pragma unroll
          for (int i = 0; i < kStride / 2; ++i) {
            const int idx = (i + (lane >> 1)) & (kStride / 2 - 1);
            const double2 p2 = fr[idx];
            const double2 w2 = wr[idx];
            const double2 t2 = tmr[idx];
            const double2 a2 = ar[idx];
            lrb = fma(fabs(p2.x), w2.x, lrb);
            lrb = fma(fabs(p2.y), w2.y, lrb);
            fc = idx == 0 ? p2.x : fc;
            ta = fmax(ta, fmax(t2.x * a2.x, t2.y * a2.y));
          }
          const double thr = lim - lrb;
          thr_lane[j] = thr > 0.0 ? hi_abs(thr) : 0u;
          const double w = ta + lrb;
          const double slack = 1e-12 * (fabs(fc) + fmax(d0.x, -d0.y) + w);
          hot |= (fc + d0.x + w + slack >= lim) || (fc + d0.y - w - slack <= -lim);
        }
      }
      need = __ballot_sync(0xffffffffu, hot);
      rows_partial += __popc(need);
      rows_offered += rows;
    }
    // Stage 2 (two rows per step, loads issued before the FMA chains): the
    // first FMA f_c + T alpha of every element is exact; the row goes on to the
    // remaining R FMAs only when |f_c + T alpha| can reach lim - lrb (tested on
    // high words: hi(|x|) < hi(t) implies |x| < t for non-negative t).
    while (need) {
      int els[2];
      els[0] = __ffs(need) - 1;
      need &= need - 1;
      els[1] = need ? __ffs(need) - 1 : -1;
      if (need) need &= need - 1;
      const int nu = els[1] >= 0 ? 2 : 1;
      double tv[2][kKpl], fc[2][NC], lim[2];
      uint32_t thr[2][NC];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int el = u < nu ? els[u] : els[0];
        const double2 t01 = *reinterpret_cast<const double2*>(sT + el * kTileK);
        const double2 t23 = *reinterpret_cast<const double2*>(sT + el * kTileK + 2);
        tv[u][0] = t01.x, tv[u][1] = t01.y, tv[u][2] = t23.x, tv[u][3] = t23.y;
        lim[u] = sL[el];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          fc[u][j] = sF[(static_cast<size_t>(j) * kChunk + el) * kStride];
          thr[u][j] = __shfl_sync(0xffffffffu, thr_lane[j], el);
        }
      }
      double f1[2][NC][kKpl];
      bool hot[2] = {FULL, FULL && nu == 2};
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          uint32_t m = 0u;
#pragma unroll
          for (int k = 0; k < kKpl; ++k) {
            f1[u][j][k] = fma(tv[u][k], alpha[j][k], fc[u][j]);
            m = max(m, hi_abs(f1[u][j][k]));
          }
          if (!FULL) hot[u] |= m >= thr[u][j];
        }
      if (!FULL) {
        hot[0] = __any_sync(0xffffffffu, hot[0]);
        hot[1] = __any_sync(0xffffffffu, hot[1]) && nu == 2;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!hot[u]) continue;
        ++rows_computed;
        const int el = els[u];
        double fl[NC][R > 0 ? R : 1];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const double* fr = sF + (static_cast<size_t>(j) * kChunk + el) * kStride;
#pragma unroll
          for (int q = 0; q < R; ++q) fl[j][q] = fr[1 + q];
        }
        uint32_t mx = 0u;
#pragma unroll
        for (int j = 0; j < NC; ++j)
#pragma unroll
          for (int k = 0; k < kKpl; ++k) {
            double acc = f1[u][j][k];
#pragma unroll
            for (int q = 0; q < R; ++q) acc = fma(fl[j][q], rr[j][k][q], acc);
            f1[u][j][k] = acc;
            mx = max(mx, hi_abs(acc));
          }
        if (FULL || mx >= hi_abs(lim[u])) {
          exact_row(e0 + el, lim[u], f1[u]);
          ++rows_exact;
        }
      }
    }
    // release the stage; the last warp out refills it (no CTA-wide barrier)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int done = atomicAdd(release + s, 1);
      if (done == kWarps - 1) {
        release[s] = 0;
        __threadfence_block();
        if (i + kStages < nchunks) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_chunk(g, b, w, tile, i + kStages, smem + s * kStageDoubles, bars + s);
        }
      }
    }
  }
  if (!FULL && lane == 0) {
    atomicAdd(b.rows_done, static_cast<unsigned long long>(rows_computed));
    atomicAdd(b.rows_done + 1, static_cast<unsigned long long>(rows_offered));
    atomicAdd(b.rows_done + 2, static_cast<unsigned long long>(rows_exact));
    atomicAdd(b.rows_done + 3, static_cast<unsigned long long>(rows_partial));
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    if (cid[j] < 0) continue;
    double* en = b.energy + static_cast<size_t>(cid[j]) * g.Kall;
#pragma unroll
    for (int k = 0; k < kKpl; ++k)
      if (kval[j][k] && kb + k < g.Ks) en[g.ks_cont[kb + k]] = energy[j][k];
  }
}

// CTA order: super-blocks of `gblock` candidate groups x all tiles, tile-major
// inside a super-block, so the CTAs resident at one time share each T_base
// tile across gblock groups (one HBM read of a tile per super-block instead of
// per group) while the super-block's candidate rows stay in L2 across its tiles.
template <bool FULL>
__global__ void __launch_bounds__(kThreads, 1) k_sweep(DevGrid g, Batch b, int ntiles, int ngroups, int gblock) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CtaWork w;
  __shared__ int r_s;
  __shared__ int release[kStages];
  __shared__ __align__(16) double rmax_s[kWarps * kStride];
  __shared__ __align__(16) double amax_s[kWarps * kTmaxSub];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* smem = reinterpret_cast<double*>(smem_raw + 64);
  const int per_sb = gblock * ntiles;
  const int sb = static_cast<int>(blockIdx.x) / per_sb, rr = static_cast<int>(blockIdx.x) % per_sb;
  const int g0 = sb * gblock, gg = min(gblock, ngroups - g0);
  const int tile = rr / gg, group = g0 + rr % gg;
  if (group >= b.wl_group0[kSweepRank + 1]) return;
  if (threadIdx.x == 0) {
    int r = 0;
    while (r < kSweepRank && group >= b.wl_group0[r + 1]) ++r;
    r_s = r;
    const int per = cand_per_cta(r);
    const int first = (group - b.wl_group0[r]) * per;
    int n = 0;
    for (int j = 0; j < per; ++j)
      if (first + j < b.wl_count[r]) w.cand[n++] = b.wl_list[b.wl_start[r] + first + j];
    w.ncand = n;
    w.group = group;
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1), release[s] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  switch (r_s) {
    case 0: sweep_cta<0, nc_for_rank(0), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 1: sweep_cta<1, nc_for_rank(1), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 2: sweep_cta<2, nc_for_rank(2), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 3: sweep_cta<3, nc_for_rank(3), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 4: sweep_cta<4, nc_for_rank(4), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 5: sweep_cta<5, nc_for_rank(5), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    case 6: sweep_cta<6, nc_for_rank(6), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
    default: sweep_cta<7, nc_for_rank(7), FULL>(g, b, w, tile, smem, bars, release, rmax_s, amax_s); break;
  }
}

// Stable per-rank lists of swept candidates; bucket r is cut into CTA groups
// of cand_per_cta(r), and every swept candidate gets its row slot
// (group * kGroupSlots + position) so k_prep writes straight into the layout
// the sweep streams.
__global__ void k_bucket(Batch b) {
  __shared__ int warp_tot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = threadIdx.x; c < b.n; c += blockDim.x) b.slot[c] = -1;
  __syncthreads();
  int base = 0, group_base = 0;
  for (int r = 0; r <= kSweepRank; ++r) {
    int running = 0;
    for (int c0 = 0; c0 < b.n; c0 += blockDim.x) {
      const int c = c0 + threadIdx.x;
      const bool mine = c < b.n && b.rank[c] == r;
      const unsigned m = __ballot_sync(0xffffffffu, mine);
      if (lane == 0) warp_tot[wid] = __popc(m);
      __syncthreads();
      int off = 0, tot = 0;
      for (int x = 0; x < nw; ++x) {
        if (x < wid) off += warp_tot[x];
        tot += warp_tot[x];
      }
      if (mine) {
        const int pos = running + off + __popc(m & ((1u << lane) - 1));
        b.wl_list[base + pos] = c;
        b.slot[c] = (group_base + pos / cand_per_cta(r)) * kGroupSlots + pos % cand_per_cta(r);
      }
      running += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      b.wl_start[r] = base;
      b.wl_count[r] = running;
      b.wl_group0[r] = group_base;
    }
    base += running;
    group_base += (running + cand_per_cta(r) - 1) / cand_per_cta(r);
  }
  if (threadIdx.x == 0) b.wl_group0[kSweepRank + 1] = group_base;
}

}  // namespace

int sweep_tile_k() { return kTileK; }
int sweep_chunk() { return kChunk; }

void launch_sweep(const DevGrid& g, Batch& b, bool full, cudaStream_t stream, cudaEvent_t ev0, cudaEvent_t ev1,
                  int* launched) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    cudaFuncSetAttribute(k_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    configured = true;
  }
  // group slots: every bucket rounds up to whole groups of >= kWarps candidates
  static const int gblock_env = [] {
    const char* v = std::getenv("TGB_SWEEP_GROUP_BLOCK");
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  const int ntiles = g.Kpad / kTileK, ngroups = max_sweep_groups(b.n);
  const int gblock = std::min(ngroups, gblock_env ? gblock_env : kGroupBlock);
  const unsigned grid = static_cast<unsigned>(ntiles) * ngroups;
  if (ev0) cudaEventRecord(ev0, stream);
  if (full)
    k_sweep<true><<<grid, kThreads, kSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
  else
    k_sweep<false><<<grid, kThreads, kSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
  if (ev1) cudaEventRecord(ev1, stream);
  *launched += 1;
}

void launch_bucket(Batch& b, cudaStream_t stream, int* launched) {
  k_bucket<<<1, 1024, 0, stream>>>(b);
  *launched += 1;
}

}  // namespace tgb
