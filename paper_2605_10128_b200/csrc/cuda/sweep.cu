// K3: the fused N-1 contingency sweep (dc_engine.cpp:294-371 for single-branch
// contingencies, all candidates of a batch at once).
//
// For candidate c, monitored branch e and contingency k (branch beta_k):
//   f1[e,k] = f_c[e] + T_base[e,k] * alpha_k + sum_q L[e,q] * R'[q,k]
// (topo.cuh: T_cand = T_base + L R, alpha_k = f_c[beta]/(1 - T_cand[beta,beta]),
// R' = R * alpha). The E x K x B tensor is never written: each element is
// tested against the branch limit in registers; only elements with
// |f1| > limit touch the per-(c,k) energy accumulators (registers, summed in
// branch order) and the per-(c,e) max (atomicMax on the ordered bit pattern).
//
// One CTA = one 128-contingency tile x one group of 16 candidates of equal
// update rank R (one candidate per warp), or half a group (8 warps, two CTAs
// per SM: k_sweep<..., HALF> on grids up to kHalfMaxRows rows). Each lane owns
// 4 contingencies: alpha / R' live in registers for the whole sweep. Candidate
// rows are row_stride(R) doubles (f_c, L[0..R-1]), contingency rows likewise.
//
// Scores-only kernel (k_sweep<false, kTmSingle, *>, the MapElites path): branch
// rows are streamed in stages of 1-4 chunks of 32 by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a 2-8 stage ring: the group's
// candidate rows, the limits and the per-(tile, row) skip record (sub-tile max
// |T_base| as floats rounded up, extrema of T_base * alpha0 as doubles); warps
// release a stage on its empty mbarrier and thread 0 refills it. T_base itself
// is NOT streamed:
//   stage 1 (one lane per row, no element work): a rigorous bound of |f1|
//     over the whole tile proves most (row, candidate) blocks safe;
//   stage 2 (rows that fail it): the lanes load that row of the T_base tile
//     (1 KB, coalesced, L2) and evaluate the exact first FMA f_c + T alpha per
//     element with the L R' part bounded;
//   stage 3: the remaining R DFMA per element and a hi-word test; the exact
//     path runs only where |f1| can exceed the limit.
// Skipped work cannot change any score (tests/test_gpu_scale.py compares the
// skipping and the dense kernel bit for bit, and both with the oracle).
//
// Flows kernel (k_sweep<true>, FlowResult requested): every element computed,
// T_base tiles streamed with the rows, max |f1| folded for every branch.
// Ranks 8..11 run in the persistent k_sweep_hi (own register allocation).
// Timestep grids: k_sweep<false, kTmMask, *> marks the rows that can overload at
// some injection profile; k_sweep_masked visits only those, 8 profiles per
// launch, keeping a row for a profile only if that profile's own bound fails.
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
constexpr int kMaxCand = kWarps;         // one candidate per warp
constexpr int kGroupBlock = 8;           // candidate groups per CTA super-block (L2 reuse)
constexpr int kMaxStages = 8;
constexpr size_t kStageBudget = 216 * 1024;  // dynamic shared memory for the stage ring (one CTA per SM)
constexpr size_t kHalfBudget = 104 * 1024;   // the same for half-group CTAs (two per SM)
constexpr int kSubLanes = 32 / kTmaxSub;     // lanes per skip sub-tile
static_assert(kTileK % kTmaxSub == 0 && kSubLanes * kTmaxSub == 32, "sub-tile layout");
static_assert(kMaxCand == kGroupSlots && kChunk == kChunkRows, "sweep tiles must match the row layout");

__host__ __device__ constexpr int cand_per_cta(int) { return kWarps; }

// Stage ring geometry for rank R (doubles per stage, number of stages).
// Timestep modes (Batch::t_mode): 0 one profile, 1 mask generation over all
// profiles (k_sweep with rows [max f_c, min f_c, L...], no element work), 2
// masked sweep (k_sweep_masked, launch_sweep_masked: only the rows marked by
// mode 1, kMaskProfiles profiles per launch).
constexpr int kTmSingle = 0, kTmMask = 1;

// Warps (candidates) per sweep CTA: a whole group of 16 at one CTA per SM, or
// (HALF, scores-only kernels on grids with few row chunks) half a group at two
// CTAs per SM, so one CTA's prologue, barrier waits and tail overlap the other's
// rows; on long sweeps the whole-group CTA streams the skip records once.
template <bool HALF>
__host__ __device__ constexpr int cta_warps() { return HALF ? kWarps / 2 : kWarps; }
constexpr int kHalfMaxRows = 4096;  // branch rows up to which the scores-only sweep uses half-group CTAs

template <int R, bool FULL, int TM = kTmSingle, bool HALF = false>
struct Ring {
  static constexpr int S = row_stride(TM == kTmMask ? R + 1 : R);
  static constexpr int H = FULL ? 1 : (S <= 4 ? 4 : (S <= 10 ? 2 : 1));          // 32-row chunks per stage
  static constexpr size_t FH = static_cast<size_t>(cta_warps<HALF>()) * kChunk * S;  // one chunk of candidate rows
  static constexpr size_t T = FULL ? static_cast<size_t>(kChunk) * kTileK : 0;  // T_base tile rows
  static constexpr size_t F = H * FH;                                           // candidate rows
  static constexpr size_t L = H * kChunk;                                       // limits
  static constexpr size_t M = FULL ? 0 : static_cast<size_t>(H) * kChunk * kRec / 2;  // skip records (floats)
  static constexpr size_t doubles = T + F + L + M;
  static constexpr size_t fit = (HALF ? kHalfBudget : kStageBudget) / (doubles * sizeof(double));
  static constexpr int stages = fit < static_cast<size_t>(kMaxStages) ? static_cast<int>(fit) : kMaxStages;
  static_assert(stages >= 2, "stage ring too small");
};
constexpr size_t kSmemBytes = kStageBudget + 128;
constexpr size_t kHalfSmemBytes = kHalfBudget + 128;

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
  int half;  // which part of the group a half-group CTA takes (k_sweep scores-only, k_sweep_masked)
};

// Producer: stage <- stage-chunk i = 32-row chunks [H i, H i + H) (T tile rows
// when FULL, the group's candidate rows, limits, skip records when not FULL).
template <int R, bool FULL, int TM, bool HALF>
__device__ __forceinline__ void issue_chunk(const DevGrid& g, const Batch& b, const CtaWork& w, int tile, int i,
                                           double* stage, uint64_t* bar) {
  using Rg = Ring<R, FULL, TM, HALF>;
  const int e0 = i * Rg::H * kChunk;
  const int rows = min(Rg::H * kChunk, g.E - e0);
  const int nch = (rows + kChunk - 1) / kChunk;
  const uint32_t bt = FULL ? rows * kTileK * sizeof(double) : 0;
  const uint32_t bf = nch * Rg::FH * sizeof(double);
  const uint32_t bl = ((rows + 1) & ~1) * sizeof(double);
  const uint32_t bm = Rg::M ? rows * kRec * sizeof(float) : 0;
  mbar_expect_tx(bar, bt + bf + bl + bm);
  if (FULL) bulk_g2s(stage, g.TK + (static_cast<size_t>(tile) * g.E + e0) * kTileK, bt, bar);
  const double* rows_src = TM == kTmMask ? b.feat_mt : b.feat;
  const int rl = TM == kTmMask ? R + 1 : R, slot0 = w.group * kGroupSlots + w.half * cta_warps<HALF>();
  if (cta_warps<HALF>() == kGroupSlots) {  // the whole group's rows of these chunks: one contiguous block
    bulk_g2s(stage + Rg::T, rows_src + feat_index(slot0, b.nchunks, e0, rl), bf, bar);
  } else {  // half a group: one block per chunk
    for (int h = 0; h < nch; ++h)
      bulk_g2s(stage + Rg::T + h * Rg::FH, rows_src + feat_index(slot0, b.nchunks, e0 + h * kChunk, rl),
               static_cast<uint32_t>(Rg::FH * sizeof(double)), bar);
  }
  bulk_g2s(stage + Rg::T + Rg::F, g.br_lim + e0, bl, bar);
  if (Rg::M)
    bulk_g2s(stage + Rg::T + Rg::F + Rg::L, g.Tmax + (static_cast<size_t>(tile) * (g.E + kChunk) + e0) * kRec, bm,
             bar);
  static_assert(kRec % 4 == 0, "skip records are whole float4");
}

template <int R, bool FULL, int TM = kTmSingle, bool HALF = false>
__device__ __forceinline__ void sweep_cta(const DevGrid& g, const Batch& b, const CtaWork& w, int tile, double* smem,
                                          uint64_t* bars, double* rmax_s, float* amax_s) {
  using Rg = Ring<R, FULL, TM, HALF>;
  constexpr int S = Rg::S, NST = Rg::stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = tile * kTileK + lane * kKpl;
  // per-(candidate, contingency) operands in registers
  double alpha[kKpl], rr[kKpl][R > 0 ? R : 1], energy[kKpl];
  bool kval[kKpl];
  int kbr[kKpl], rem[kMaxRemovedSweep];
  int cid = warp < w.ncand ? w.cand[warp] : -1;
  if (cid >= 0 && b.status[cid] != 0) cid = -1;  // islanded by the small solve in k_prep
  if (TM != kTmMask) {
    const int c = cid >= 0 ? cid : w.cand[0];
    const double* kd = b.kdat + static_cast<size_t>(c) * g.Kpad * kStride + static_cast<size_t>(kb) * S;
    const uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad + kb;
#pragma unroll
    for (int i = 0; i < kKpl; ++i) {
      kbr[i] = kb + i < g.Ks ? g.ks_branch[kb + i] : -1;
      alpha[i] = kd[i * S];
#pragma unroll
      for (int q = 0; q < R; ++q) rr[i][q] = kd[i * S + 1 + q];
      energy[i] = 0.0;
      kval[i] = cid >= 0 && kf[i] == 0;
    }
#pragma unroll
    for (int q = 0; q < kMaxRemovedSweep; ++q) rem[q] = b.removed[static_cast<size_t>(c) * kMaxRemovedSweep + q];
  }
  // Skip-bound operands in shared memory (invalid contingencies carry alpha 0):
  // max |alpha - alpha0| per sub-tile, asub[s] (the candidate's departure from
  // the unchanged topology's flow factors), and the tile max of each |R'_q| as
  // a row weight vector rms[slot] (0 for f_c and padding).
  double* rms = rmax_s + warp * kStride;
  float* asub = amax_s + warp * kTmaxSub;  // rounded up to float: the T_base x delta bound runs in FP32
  const int ntiles = g.Kpad / kTileK;
  if (TM == kTmMask) {
    // bounds over all profiles, folded by k_prep (bit patterns of non-negative doubles)
    const size_t at = (static_cast<size_t>(cid >= 0 ? cid : 0) * ntiles + tile);
    if (lane < kStride)
      rms[lane] = lane >= 1 && lane <= R && cid >= 0 ? __longlong_as_double(b.rmx_mt[at * kStride + lane]) * (1.0 + 1e-12)
                                                     : 0.0;
    if (lane < kTmaxSub)
      asub[lane] = cid >= 0 ? __double2float_ru(__longlong_as_double(b.amx_mt[at * kTmaxSub + lane]) * (1.0 + 1e-12))
                            : 0.0f;
    __syncwarp();
  } else if (!FULL && TM == kTmSingle) {
    if (lane < kStride) rms[lane] = 0.0;
    __syncwarp();
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) a = fmax(a, fabs(alpha[k] - g.alpha0[kb + k]));
#pragma unroll
    for (int o = kSubLanes / 2; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane % kSubLanes == 0) asub[lane / kSubLanes] = __double2float_ru(a * (1.0 + 1e-12));
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double r = 0.0;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) r = fmax(r, fabs(rr[k][q]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (lane == 0) rms[1 + q] = r * (1.0 + 1e-12);
    }
    __syncwarp();
  }
  // small ranks keep the per-warp skip weights in registers (stage 1 then reads
  // only the row data from shared memory)
  constexpr bool kRegW = !FULL && TM == kTmSingle && R <= 3;
  float areg[kRegW ? kTmaxSub : 1];
  double wreg[kRegW ? S : 1];
  if (kRegW) {
#pragma unroll
    for (int q = 0; q < kTmaxSub; ++q) areg[q] = asub[q];
#pragma unroll
    for (int q = 0; q < S; ++q) wreg[q] = rms[q];
  }

  const int nchunks = (g.E + Rg::H * kChunk - 1) / (Rg::H * kChunk);  // stage-chunks
  unsigned rows_computed = 0, rows_offered = 0, rows_exact = 0, rows_partial = 0;  // skip statistics
  if (threadIdx.x == 0)
    for (int s = 0; s < NST && s < nchunks; ++s)
      issue_chunk<R, FULL, TM, HALF>(g, b, w, tile, s, smem + s * Rg::doubles, bars + s);

  // exact path for one branch row: energies (registers) and fmax (atomicMax)
  auto exact_row = [&](int e, double lim, const double (&f1)[kKpl]) {
    bool skip_row = false;
#pragma unroll
    for (int q = 0; q < kMaxRemovedSweep; ++q) skip_row |= e == rem[q];
    unsigned long long m = 0ull;  // max |f1| as the ordered bit pattern of a non-negative double
#pragma unroll
    for (int k = 0; k < kKpl; ++k) {
      if (!kval[k] || skip_row || e == kbr[k]) continue;  // the outaged branch carries 0
      const double a = fabs(f1[k]);
      if (FULL) {
        if (a > lim) energy[k] += a - lim;
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(a)));
      } else if (a > lim) {  // only a max above the limit is folded: track overloaded elements only
        energy[k] += a - lim;
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(a)));
      }
    }
    if (cid < 0) return;
    unsigned long long* fmx = b.fmax + static_cast<size_t>(cid) * g.E;
    if (FULL) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0 && m > 0ull) atomicMax(fmx + e, m);
    } else if (m > static_cast<unsigned long long>(__double_as_longlong(lim))) {
      atomicMax(fmx + e, m);
    }
  };
  // remaining R FMAs of one row (L from shared memory), then the exact path
  // when `test` is off or some |f1| can exceed the limit (hi-word test)
  auto finish_row = [&](int e, double lim, const double* fr, double (&f1)[kKpl], bool test) {
    double fl[R > 0 ? R : 1];
#pragma unroll
    for (int q = 0; q < R; ++q) fl[q] = fr[1 + q];
    uint32_t mx = 0u;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) {
      double acc = f1[k];
#pragma unroll
      for (int q = 0; q < R; ++q) acc = fma(fl[q], rr[k][q], acc);
      f1[k] = acc;
      mx = max(mx, hi_abs(acc));
    }
    if (!test || __any_sync(0xffffffffu, mx >= hi_abs(lim))) {
      exact_row(e, lim, f1);
      return true;
    }
    return false;
  };

  for (int i = 0; i < nchunks; ++i) {
    const int s = i % NST;
    const double* st = smem + s * Rg::doubles;
    mbar_wait(bars + s, (i / NST) & 1);
#pragma unroll 1
    for (int h = 0; h < Rg::H; ++h) {
    const int e0 = (i * Rg::H + h) * kChunk;
    const int rows = min(kChunk, g.E - e0);
    if (rows <= 0) break;
    const double* sF = st + Rg::T + h * Rg::FH + static_cast<size_t>(warp) * kChunk * S;
    const double* sL = st + Rg::T + Rg::F + h * kChunk;
    if (FULL) {
      const double* sT = st + lane * kKpl;
      for (int el = 0; el < rows; ++el) {
        const double2 t01 = *reinterpret_cast<const double2*>(sT + el * kTileK);
        const double2 t23 = *reinterpret_cast<const double2*>(sT + el * kTileK + 2);
        const double tv[kKpl] = {t01.x, t01.y, t23.x, t23.y};
        const double fc = sF[el * S];
        double f1[kKpl];
#pragma unroll
        for (int k = 0; k < kKpl; ++k) f1[k] = fma(tv[k], alpha[k], fc);
        finish_row(e0 + el, sL[el], sF + el * S, f1, false);
      }
    } else {
      // Stage 1 (one lane per row). With alpha = alpha0 + delta (alpha0: the
      // unchanged topology) every element of the tile satisfies
      //   f1 = f_c + T alpha0 + T delta + L R'  in  [f_c + D0min - w, f_c + D0max + w],
      //   w = max_s max|T_base|_s max|delta|_s + lrb,  lrb = sum_q |L_q| max|R'_q|
      // (D0max / D0min: max / min of T_base * alpha0 over the tile, precomputed;
      // s: sub-tiles; R' maxima over the tile). A relative slack of 1e-12 on
      // every term covers the rounding of the computed f1. Stage 2 tests
      // against the high word of lim (1 - 1e-12) - lrb (0 when not positive).
      bool hot = false;
      uint32_t thr_lane = 0u;
      const int chunk32 = i * Rg::H + h;
      if (lane < rows) {
        const double lim = sL[lane] * (1.0 - 1e-12);
        const float4* rec = reinterpret_cast<const float4*>(st + Rg::T + Rg::F + Rg::L) + (h * kChunk + lane) * (kRec / 4);
        const double2* fr = reinterpret_cast<const double2*>(sF + lane * S);
        const double2* wr = reinterpret_cast<const double2*>(rms);
        double l0 = 0.0, l1 = 0.0, fc = 0.0, flo = 0.0;  // two accumulators: half the dependent chain
        if (TM == kTmMask) {
          // rows [key(max_t f_c), key(min_t f_c), L_0..L_{R-1}]; rms slot 1 + q weighs L_q
          const unsigned long long* kr = reinterpret_cast<const unsigned long long*>(fr);
          fc = order_value(kr[0]);
          flo = order_value(kr[1]);
          const double* l = reinterpret_cast<const double*>(fr) + 2;
#pragma unroll
          for (int q = 0; q < R; ++q) {
            if (q & 1)
              l1 = fma(fabs(l[q]), rms[1 + q], l1);
            else
              l0 = fma(fabs(l[q]), rms[1 + q], l0);
          }
        } else {
#pragma unroll
          for (int q = 0; q < S / 2; ++q) {
            const double2 p2 = fr[q];
            const double2 w2 = kRegW ? make_double2(wreg[kRegW ? 2 * q : 0], wreg[kRegW ? 2 * q + 1 : 0]) : wr[q];
            l0 = fma(fabs(p2.x), w2.x, l0);
            l1 = fma(fabs(p2.y), w2.y, l1);
            if (q == 0) fc = p2.x;
          }
          flo = fc;
        }
        const double lrb = l0 + l1;
        // max_s Tmax_s * delta_s in FP32 rounded up (both factors are
        // non-negative upper bounds already rounded up to float)
        const float4* ar = reinterpret_cast<const float4*>(asub);
        float taf = 0.0f;
#pragma unroll
        for (int q = 0; q < kTmaxSub / 4; ++q) {
          const float4 t4 = rec[q];
          const float4 a4 = kRegW ? make_float4(areg[kRegW ? 4 * q : 0], areg[kRegW ? 4 * q + 1 : 0],
                                                areg[kRegW ? 4 * q + 2 : 0], areg[kRegW ? 4 * q + 3 : 0])
                                  : ar[q];
          taf = fmaxf(taf, fmaxf(fmaxf(__fmul_ru(t4.x, a4.x), __fmul_ru(t4.y, a4.y)),
                                 fmaxf(__fmul_ru(t4.z, a4.z), __fmul_ru(t4.w, a4.w))));
        }
        const double2 d0 = reinterpret_cast<const double2*>(rec)[kTmaxSub / 4];
        const double thr = lim - lrb;
        thr_lane = thr > 0.0 ? hi_abs(thr) : 0u;
        // some |f1| of the tile can reach lim only if
        //   fc + D0max + w + slack >= lim  or  flo + D0min - w - slack <= -lim,
        // i.e. w (1 + 1e-12) + s0 >= lim - max(fc + D0max, -(flo + D0min)), with
        // slack = 1e-12 (max(|fc|, |flo|) + |D0max| + |D0min| + w); the gap and
        // s0 do not depend on w (short dependent chain)
        const double gap = lim - fmax(fc + d0.x, -(flo + d0.y));
        const double s0 = 1e-12 * (fmax(fabs(fc), fabs(flo)) + fabs(d0.x) + fabs(d0.y));
        const double wd = static_cast<double>(taf) + lrb;
        hot = fma(wd, 1.0 + 1e-12, s0) >= gap;
      }
      unsigned need = __ballot_sync(0xffffffffu, hot);
      rows_partial += __popc(need);
      rows_offered += rows;
      if (TM == kTmMask) {
        if (lane == 0 && cid >= 0) b.mask[(static_cast<size_t>(cid) * ntiles + tile) * b.nchunks + chunk32] = need;
        continue;  // no element work in mask generation
      }
      // Stage 2: hot rows in batches of NB, T_base row loads issued before use
      constexpr int NB = R >= 6 ? 1 : (R >= 4 ? 2 : 4);  // register budget (128 per thread at 512 threads)
      const double* tk_rows = g.TK + (static_cast<size_t>(tile) * g.E + e0) * kTileK + lane * kKpl;
      while (need) {
        int els[NB];
        int nu = 0;
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          els[u] = need ? __ffs(need) - 1 : -1;
          if (need) need &= need - 1, ++nu;
        }
        double2 t[NB][2];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int el = els[u] >= 0 ? els[u] : els[0];
          const double2* src = reinterpret_cast<const double2*>(tk_rows + static_cast<size_t>(el) * kTileK);
          t[u][0] = __ldg(src);
          t[u][1] = __ldg(src + 1);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          if (u >= nu) break;
          const int el = els[u];
          const double fc = sF[el * S];
          const uint32_t thr = __shfl_sync(0xffffffffu, thr_lane, el);
          const double tv[kKpl] = {t[u][0].x, t[u][0].y, t[u][1].x, t[u][1].y};
          double f1[kKpl];
          uint32_t m = 0u;
#pragma unroll
          for (int k = 0; k < kKpl; ++k) {
            f1[k] = fma(tv[k], alpha[k], fc);
            m = max(m, hi_abs(f1[k]));
          }
          if (!__any_sync(0xffffffffu, m >= thr)) continue;
          ++rows_computed;
          rows_exact += finish_row(e0 + el, sL[el], sF + el * S, f1, true) ? 1u : 0u;
        }
      }
    }
    }  // h
    // release the stage (arrive on its empty barrier, no return value); thread 0
    // refills it once all 16 warps have left it (no CTA-wide barrier)
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + kMaxStages + s);
    if (threadIdx.x == 0 && i + NST < nchunks) {
      mbar_wait(bars + kMaxStages + s, (i / NST) & 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_chunk<R, FULL, TM, HALF>(g, b, w, tile, i + NST, smem + s * Rg::doubles, bars + s);
    }
    __syncwarp();
  }
  if (!FULL && lane == 0) {
    atomicAdd(b.rows_done, static_cast<unsigned long long>(rows_computed));
    atomicAdd(b.rows_done + 1, static_cast<unsigned long long>(rows_offered));
    atomicAdd(b.rows_done + 2, static_cast<unsigned long long>(rows_exact));
    atomicAdd(b.rows_done + 3, static_cast<unsigned long long>(rows_partial));
  }
  if (cid >= 0) {
    double* en = b.energy + static_cast<size_t>(cid) * g.Kall;
#pragma unroll
    for (int k = 0; k < kKpl; ++k)
      if (kval[k] && kb + k < g.Ks) en[g.ks_cont[kb + k]] = energy[k];
  }
}

// Common-rank kernel (ranks 0..kFastRank). CTA order: super-blocks of
// `gblock` candidate groups x all tiles, tile-major inside a super-block, so
// the CTAs resident at one time share each T_base tile across gblock groups
// while the super-block's candidate rows stay in L2 across its tiles.
constexpr int kFastRank = 7;

// CTA setup for (group, half, rank r): the candidate list and fresh stage barriers.
template <bool HALF>
__device__ __forceinline__ void cta_setup(const Batch& b, int group, int half, int r, CtaWork& w, uint64_t* bars) {
  constexpr int W = cta_warps<HALF>();
  const int first = (group - b.wl_group0[r]) * cand_per_cta(r) + half * W;
  int n = 0;
  for (int j = 0; j < W; ++j)
    if (first + j < b.wl_count[r]) w.cand[n++] = b.wl_list[b.wl_start[r] + first + j];
  w.ncand = n;
  w.group = group;
  w.half = half;
  for (int s = 0; s < kMaxStages; ++s) mbar_init(bars + s, 1), mbar_init(bars + kMaxStages + s, W);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

template <bool FULL, int TM, bool HALF>
__global__ void __launch_bounds__(32 * cta_warps<HALF>(), HALF ? 2 : 1)
    k_sweep(DevGrid g, Batch b, int ntiles, int ngroups, int gblock) {
  constexpr int W = cta_warps<HALF>(), halves = kGroupSlots / W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CtaWork w;
  __shared__ int r_s;
  __shared__ __align__(16) double rmax_s[W * kStride];
  __shared__ __align__(16) float amax_s[W * kTmaxSub];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* smem = reinterpret_cast<double*>(smem_raw + 128);
  const int per_sb = gblock * ntiles * halves;
  const int sb = static_cast<int>(blockIdx.x) / per_sb, rr = static_cast<int>(blockIdx.x) % per_sb;
  const int g0 = sb * gblock, gg = min(gblock, ngroups - g0);
  const int half = rr % halves, tile = (rr / halves) / gg, group = g0 + (rr / halves) % gg;
  if (group >= b.wl_group0[kFastRank + 1]) return;  // higher ranks: k_sweep_hi
  if (threadIdx.x == 0) {
    int r = 0;
    while (r < kFastRank && group >= b.wl_group0[r + 1]) ++r;
    r_s = r;
    cta_setup<HALF>(b, group, half, r, w, bars);
  }
  __syncthreads();
  if (w.ncand == 0) return;  // a group's second half can be empty
  switch (r_s) {
    case 0: sweep_cta<0, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 1: sweep_cta<1, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 2: sweep_cta<2, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 3: sweep_cta<3, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 4: sweep_cta<4, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 5: sweep_cta<5, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    case 6: sweep_cta<6, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    default: sweep_cta<7, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
  }
}

// Ranks kFastRank+1 .. kSweepRank (n_a = n_d = 4 genomes with grounded dead
// nodes; rare): a persistent kernel over their (tile, group) items, so its
// register allocation stays out of the common kernel and an empty bucket
// costs one short launch.
template <bool FULL, int TM, bool HALF>
__global__ void __launch_bounds__(32 * cta_warps<HALF>(), HALF ? 2 : 1) k_sweep_hi(DevGrid g, Batch b, int ntiles) {
  constexpr int W = cta_warps<HALF>(), halves = kGroupSlots / W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ CtaWork w;
  __shared__ int r_s;
  __shared__ __align__(16) double rmax_s[W * kStride];
  __shared__ __align__(16) float amax_s[W * kTmaxSub];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* smem = reinterpret_cast<double*>(smem_raw + 128);
  const int gbeg = b.wl_group0[kFastRank + 1], gend = b.wl_group0[kSweepRank + 1];
  const long items = static_cast<long>(gend - gbeg) * ntiles * halves;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    const int half = static_cast<int>(it % halves);
    const long gi = it / halves;
    const int group = gbeg + static_cast<int>(gi / ntiles), tile = static_cast<int>(gi % ntiles);
    __syncthreads();  // the previous item is done with the barriers and shared state
    if (threadIdx.x == 0) {
      int r = kFastRank + 1;
      while (r < kSweepRank && group >= b.wl_group0[r + 1]) ++r;
      r_s = r;
      cta_setup<HALF>(b, group, half, r, w, bars);
    }
    __syncthreads();
    if (w.ncand == 0) continue;
    switch (r_s) {
      case 8: sweep_cta<8, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
      case 9: sweep_cta<9, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
      case 10: sweep_cta<10, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
      default: sweep_cta<11, FULL, TM, HALF>(g, b, w, tile, smem, bars, rmax_s, amax_s); break;
    }
  }
}
static_assert(kSweepRank == 11 && kFastRank == 7, "k_sweep / k_sweep_hi rank switches");

// Masked sweep of one injection profile (multi-timestep screening,
// Batch::t_mode 2): each warp visits only the rows its candidate's all-profile
// mask marks for this tile (a few percent). The CTA's 16 masks are OR-ed into
// one union row list (rows hot for one candidate tend to be hot for many:
// ~8x fewer rows than the sum at cfg3); the T_base rows of the union are
// staged once per CTA by TMA bulk copies (1 KB per row) into a ring of
// 32-row batches, and each warp gathers only its own marked candidate rows.
// Per-profile data is compact (k_prep_mt): f_c and alpha of this profile, the
// L rows (profile 0) and the unscaled contingency factors rk are shared.
constexpr int kMaskBatch = 32;                               // union rows per ring stage
constexpr size_t kMaskStageBytes = kMaskBatch * kTileK * 8;  // T_base rows of one stage
constexpr int kMaskMaxStages = 4;
constexpr int kMaskWarps = kWarps / 2;       // half a candidate group per CTA, two CTAs per SM
constexpr int kMaskThreads = 32 * kMaskWarps;
constexpr size_t kMaskBudget = 110 * 1024;  // dynamic shared memory per CTA (two per SM)

// shared-memory plan of k_sweep_masked for E rows at row stride S
struct MaskedPlan {
  size_t su, ul, scr, ring;  // byte offsets: union words, union rows, per-warp row scratch, ring
  int stages;
};
__host__ __device__ inline MaskedPlan masked_plan(int E, int S) {
  MaskedPlan p;
  const int nch = (E + kChunk - 1) / kChunk;
  p.su = 0;
  p.ul = (static_cast<size_t>(nch) * 4 + 15) & ~size_t{15};
  p.scr = (p.ul + static_cast<size_t>(E) * 4 + 15) & ~size_t{15};
  p.ring = (p.scr + static_cast<size_t>(kMaskWarps) * 32 * S * 8 + 127) & ~size_t{127};
  const size_t left = kMaskBudget > p.ring ? kMaskBudget - p.ring : 0;
  const size_t st = left / kMaskStageBytes;
  p.stages = static_cast<int>(st < kMaskMaxStages ? st : kMaskMaxStages);
  return p;
}

template <int R>
__device__ __forceinline__ void masked_cta(const DevGrid& g, const Batch& b, const CtaWork& w, int tile,
                                           uint8_t* smem, uint64_t* full_bar, uint64_t* empty_bar, int nunion,
                                           double* rmax_s, float* amax_s, const MtMask& mm) {
  constexpr int S = row_stride(R);
  const MaskedPlan plan = masked_plan(g.E, S);
  const int NST = plan.stages;
  const int* ul = reinterpret_cast<const int*>(smem + plan.ul);
  const double* ring = reinterpret_cast<const double*>(smem + plan.ring);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* scr = reinterpret_cast<double*>(smem + plan.scr) + static_cast<size_t>(warp) * 32 * S;
  const int kb = tile * kTileK + lane * kKpl;
  double alpha[kKpl], rr[kKpl][R > 0 ? R : 1], energy[kKpl];
  bool kval[kKpl];
  int kbr[kKpl], rem[kMaxRemovedSweep];
  int cid = warp < w.ncand ? w.cand[warp] : -1;
  if (cid >= 0 && b.status[cid] != 0) cid = -1;
  const int c = cid >= 0 ? cid : w.cand[0];
  {
    const uint8_t* kf = b.kflag + static_cast<size_t>(c) * g.Kpad + kb;
#pragma unroll
    for (int i = 0; i < kKpl; ++i) {
      kbr[i] = kb + i < g.Ks ? g.ks_branch[kb + i] : -1;
      kval[i] = cid >= 0 && kf[i] == 0;
    }
#pragma unroll
    for (int q = 0; q < kMaxRemovedSweep; ++q) rem[q] = b.removed[static_cast<size_t>(c) * kMaxRemovedSweep + q];
  }
  const int ntiles = g.Kpad / kTileK;
  const uint32_t* mw = b.mask + (static_cast<size_t>(cid >= 0 ? cid : 0) * ntiles + tile) * b.nchunks;
  const size_t slot = static_cast<size_t>(w.group) * kGroupSlots + w.half * kMaskWarps + warp;
  unsigned long long* fmx = b.fmax;
  const double* tk_tile = g.TK + static_cast<size_t>(tile) * g.E * kTileK;
  const int nb = (nunion + kMaskBatch - 1) / kMaskBatch, nJ = nb * mm.np;  // batches over all profiles
  auto issue = [&](int J) {
    const int s = J % NST, r0 = (J % nb) * kMaskBatch, nr = min(kMaskBatch, nunion - r0);
    uint64_t* bar = full_bar + s;
    mbar_expect_tx(bar, static_cast<uint32_t>(nr * kTileK * 8));
    double* dst = const_cast<double*>(ring) + static_cast<size_t>(s) * kMaskBatch * kTileK;
    for (int r = 0; r < nr; ++r)
      bulk_g2s(dst + r * kTileK, tk_tile + static_cast<size_t>(ul[r0 + r]) * kTileK, kTileK * 8, bar);
  };
  if (threadIdx.x == 0)
    for (int J = 0; J < NST && J < nJ; ++J) issue(J);
  float* asub = amax_s + warp * kTmaxSub;
  double* rms = rmax_s + warp * kStride;
  const double* fc_p = b.fc_t;
  const float* rec_tile = nullptr;
  // per profile: alpha and R' = rk * alpha (k_prep's rounding), the stage-1
  // bound operands (sweep_cta: max |alpha - alpha0| per sub-tile as a float
  // rounded up, max |R'_q| over the tile, per warp)
  auto profile_setup = [&](int p) {
    const int t = mm.t0 + p;
    const double* kr = b.rk_mt + static_cast<size_t>(c) * g.Kpad * kStride + static_cast<size_t>(kb) * S;
    const double* al = b.al_t + p * mm.al_stride + static_cast<size_t>(c) * g.Kpad + kb;
#pragma unroll
    for (int i = 0; i < kKpl; ++i) {
      alpha[i] = al[i];
#pragma unroll
      for (int q = 0; q < R; ++q) rr[i][q] = kr[i * S + 1 + q] * alpha[i];
      energy[i] = 0.0;
    }
    fc_p = b.fc_t + p * mm.fc_stride;
    rec_tile = mm.tmax[t] + static_cast<size_t>(tile) * (g.E + kChunk) * kRec;
    fmx = b.fmax + p * mm.fmax_stride + static_cast<size_t>(cid >= 0 ? cid : 0) * g.E;
    const double* a0 = mm.alpha0[t];
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) a = fmax(a, fabs(alpha[k] - a0[kb + k]));
#pragma unroll
    for (int o = kSubLanes / 2; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane % kSubLanes == 0) asub[lane / kSubLanes] = __double2float_ru(a * (1.0 + 1e-12));
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double r = 0.0;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) r = fmax(r, fabs(rr[k][q]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (lane == 0) rms[q] = r * (1.0 + 1e-12);
    }
    __syncwarp();
  };
  // this lane's union row of batch j: own mask bit, candidate row, limit and
  // skip record, gathered one batch ahead (registers) while the current batch
  // computes; the row is kept only if this profile's own stage-1 bound (the
  // all-profile mask is the union over the day) cannot prove it safe
  int e_n = -1;
  bool marked_n = false;
  double lim_n = 0.0;
  double2 fr_n[S / 2];
  float4 rec_n[kRec / 4];
  auto gather = [&](int j) {
    const int idx = j * kMaskBatch + lane;
    e_n = j < nb && lane < kMaskBatch && idx < nunion ? ul[idx] : -1;
    marked_n = e_n >= 0 && cid >= 0 && ((mw[e_n >> 5] >> (e_n & 31)) & 1u);
    if (marked_n) {
      // L from profile 0's row, f_c of this profile
      const double2* fr = reinterpret_cast<const double2*>(b.feat + feat_index(static_cast<int>(slot), b.nchunks, e_n, R));
#pragma unroll
      for (int q = 0; q < S / 2; ++q) fr_n[q] = fr[q];
      fr_n[0].x = fc_p[static_cast<size_t>(cid) * g.E + e_n];
      lim_n = g.br_lim[e_n];
      const float4* rc = reinterpret_cast<const float4*>(rec_tile + static_cast<size_t>(e_n) * kRec);
#pragma unroll
      for (int q = 0; q < kRec / 4; ++q) rec_n[q] = rc[q];
    }
  };
  // stage 1 of sweep_cta on the gathered row (same rigorous bound)
  auto profile_hot = [&]() {
    const double lim = lim_n * (1.0 - 1e-12);
    const double* fl = reinterpret_cast<const double*>(fr_n);
    double l0 = 0.0, l1 = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (q & 1)
        l1 = fma(fabs(fl[1 + q]), rms[q], l1);
      else
        l0 = fma(fabs(fl[1 + q]), rms[q], l0);
    }
    const double lrb = l0 + l1, fc = fl[0];
    const float4* ar = reinterpret_cast<const float4*>(asub);
    float taf = 0.0f;
#pragma unroll
    for (int q = 0; q < kTmaxSub / 4; ++q) {
      const float4 t4 = rec_n[q], a4 = ar[q];
      taf = fmaxf(taf, fmaxf(fmaxf(__fmul_ru(t4.x, a4.x), __fmul_ru(t4.y, a4.y)),
                             fmaxf(__fmul_ru(t4.z, a4.z), __fmul_ru(t4.w, a4.w))));
    }
    const double2 d0 = reinterpret_cast<const double2*>(rec_n)[kTmaxSub / 4];
    const double gap = lim - fmax(fc + d0.x, -(fc + d0.y));
    const double s0 = 1e-12 * (fabs(fc) + fabs(d0.x) + fabs(d0.y));
    const double wd = static_cast<double>(taf) + lrb;
    return fma(wd, 1.0 + 1e-12, s0) >= gap;
  };
  for (int p = 0; p < mm.np; ++p) {
  profile_setup(p);
  gather(0);
  for (int j = 0; j < nb; ++j) {
    const int J = p * nb + j, s = J % NST;
    const int e_l = e_n;
    const bool marked = marked_n && profile_hot();
    const double lim_l = lim_n;
    if (marked) {
      double2* dst = reinterpret_cast<double2*>(scr + lane * S);
#pragma unroll
      for (int q = 0; q < S / 2; ++q) dst[q] = fr_n[q];
    }
    __syncwarp();
    gather(j + 1);
    unsigned need = __ballot_sync(0xffffffffu, marked);
    mbar_wait(full_bar + s, (J / NST) & 1);
    const double* st = ring + static_cast<size_t>(s) * kMaskBatch * kTileK + lane * kKpl;
    while (need) {
      const int u = __ffs(need) - 1;
      need &= need - 1;
      const int e = __shfl_sync(0xffffffffu, e_l, u);
      const double lim = __shfl_sync(0xffffffffu, lim_l, u);
      const double2 t01 = *reinterpret_cast<const double2*>(st + u * kTileK);
      const double2 t23 = *reinterpret_cast<const double2*>(st + u * kTileK + 2);
      const double tv[kKpl] = {t01.x, t01.y, t23.x, t23.y};
      const double* frow = scr + u * S;
      double fl[S];
#pragma unroll
      for (int q = 0; q < S / 2; ++q) {
        const double2 v = reinterpret_cast<const double2*>(frow)[q];
        fl[2 * q] = v.x;
        fl[2 * q + 1] = v.y;
      }
      double f1[kKpl];
      uint32_t mx = 0u;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) {
        double acc = fma(tv[k], alpha[k], fl[0]);
#pragma unroll
        for (int q = 0; q < R; ++q) acc = fma(fl[1 + q], rr[k][q], acc);
        f1[k] = acc;
        mx = max(mx, hi_abs(acc));
      }
      if (!__any_sync(0xffffffffu, mx >= hi_abs(lim))) continue;
      bool skip_row = false;
#pragma unroll
      for (int q = 0; q < kMaxRemovedSweep; ++q) skip_row |= e == rem[q];
      unsigned long long m = 0ull;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) {
        if (!kval[k] || skip_row || e == kbr[k]) continue;
        const double a = fabs(f1[k]);
        if (a > lim) {  // only a max above the limit is folded
          energy[k] += a - lim;
          m = max(m, static_cast<unsigned long long>(__double_as_longlong(a)));
        }
      }
      if (m > static_cast<unsigned long long>(__double_as_longlong(lim))) atomicMax(fmx + e, m);
    }
    // release the stage; thread 0 refills it once every warp has left it
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar + s);
    if (threadIdx.x == 0 && J + NST < nJ) {
      mbar_wait(empty_bar + s, (J / NST) & 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(J + NST);
    }
    __syncwarp();
  }
  if (cid >= 0) {
    double* en = b.energy + p * mm.energy_stride + static_cast<size_t>(cid) * g.Kall;
#pragma unroll
    for (int k = 0; k < kKpl; ++k)
      if (kval[k] && kb + k < g.Ks) en[g.ks_cont[kb + k]] = energy[k];
  }
  }  // profiles
}

template <int R>
__device__ __noinline__ void masked_cta_call(const DevGrid& g, const Batch& b, const CtaWork& w, int tile,
                                             uint8_t* smem, uint64_t* full_bar, uint64_t* empty_bar, int nunion,
                                             double* rmax_s, float* amax_s, const MtMask& mm) {
  masked_cta<R>(g, b, w, tile, smem, full_bar, empty_bar, nunion, rmax_s, amax_s, mm);
}

__global__ void __launch_bounds__(kMaskThreads, 2) k_sweep_masked(DevGrid g, Batch b, int ntiles, int ngroups,
                                                                  int gblock, MtMask mm) {
  extern __shared__ __align__(128) uint8_t msm[];
  __shared__ CtaWork w;
  __shared__ int r_s, nunion_s;
  __shared__ int wsum[kMaskWarps];
  __shared__ __align__(8) uint64_t bars[2 * kMaskMaxStages];
  __shared__ __align__(16) double rmax_s[kMaskWarps * kStride];
  __shared__ __align__(16) float amax_s[kMaskWarps * kTmaxSub];
  const int per_sb = gblock * ntiles * 2;
  const int sb = static_cast<int>(blockIdx.x) / per_sb, rr = static_cast<int>(blockIdx.x) % per_sb;
  const int g0 = sb * gblock, gg = min(gblock, ngroups - g0);
  const int half = rr & 1, tile = (rr >> 1) / gg, group = g0 + (rr >> 1) % gg;
  if (group >= b.wl_group0[kSweepRank + 1]) return;
  if (threadIdx.x == 0) {
    int r = 0;
    while (r < kSweepRank && group >= b.wl_group0[r + 1]) ++r;
    r_s = r;
    const int per = cand_per_cta(r);
    const int first = (group - b.wl_group0[r]) * per + half * kMaskWarps;
    int n = 0;
    for (int j = 0; j < kMaskWarps; ++j)
      if (first + j < b.wl_count[r]) w.cand[n++] = b.wl_list[b.wl_start[r] + first + j];
    w.ncand = n;
    w.group = group;
    w.half = half;
    for (int s = 0; s < kMaskMaxStages; ++s) {
      mbar_init(bars + s, 1);
      mbar_init(bars + kMaskMaxStages + s, kMaskWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (w.ncand == 0) return;  // the group's second half can be empty
  // union of the CTA's masks for this tile, then the union row list
  const int nch = b.nchunks;
  uint32_t* su = reinterpret_cast<uint32_t*>(msm);
  for (int c = threadIdx.x; c < nch; c += blockDim.x) su[c] = 0u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    int cid = warp < w.ncand ? w.cand[warp] : -1;
    if (cid >= 0 && b.status[cid] != 0) cid = -1;
    if (cid >= 0) {
      const uint32_t* mw = b.mask + (static_cast<size_t>(cid) * ntiles + tile) * nch;
      for (int c = lane; c < nch; c += 32) {
        const uint32_t v = mw[c];
        if (v) atomicOr(su + c, v);
      }
    }
  }
  __syncthreads();
  // block-wide exclusive scan of the per-thread row counts (contiguous word ranges)
  const int per_t = (nch + blockDim.x - 1) / blockDim.x;
  const int c_lo = min(nch, static_cast<int>(threadIdx.x) * per_t), c_hi = min(nch, c_lo + per_t);
  int cnt = 0;
  for (int c = c_lo; c < c_hi; ++c) cnt += __popc(su[c]);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < warp; ++i) base += wsum[i];
  if (threadIdx.x == blockDim.x - 1) nunion_s = base + incl;
  const int S = row_stride(r_s);
  int* ul = reinterpret_cast<int*>(msm + masked_plan(g.E, S).ul);
  int pos = base + incl - cnt;
  for (int c = c_lo; c < c_hi; ++c) {
    uint32_t v = su[c];
    while (v) {
      ul[pos++] = c * kChunk + __ffs(v) - 1;
      v &= v - 1;
    }
  }
  __syncthreads();
  uint8_t* sm = msm;
  uint64_t* fb = bars;
  uint64_t* eb = bars + kMaskMaxStages;
  const int nu = nunion_s;
  switch (r_s) {
    case 0: masked_cta<0>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 1: masked_cta<1>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 2: masked_cta<2>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 3: masked_cta<3>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 4: masked_cta<4>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 5: masked_cta<5>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    // higher ranks in their own call frames (register pressure of the common ones)
    case 6: masked_cta_call<6>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 7: masked_cta_call<7>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 8: masked_cta_call<8>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 9: masked_cta_call<9>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    case 10: masked_cta_call<10>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
    default: masked_cta_call<11>(g, b, w, tile, sm, fb, eb, nu, rmax_s, amax_s, mm); break;
  }
}

// ---------------------------------------------------------------- chunked sweep
// Scores-only sweep for ranks <= kChunkedMaxRank on one injection profile
// (the MapElites path). Persistent: every warp takes (candidate, tile) work
// items from a global counter (candidate-major, so concurrently running warps
// share the candidate's rows in L2) and runs them on its own, with no CTA-wide
// synchronization:
//   1. the candidate's alpha / R' of the tile in registers (4 contingencies per
//      lane), the bound operands max |alpha - alpha0| per sub-tile and max |R'_q|
//      per tile as in sweep_cta;
//   2. chunk test, one lane per 32-row chunk: every element of the chunk and
//      tile satisfies |f1| <= (base N-1 flow) + |f_c - f0| + |T_base||delta| +
//      sum_q |L_q||R'_q|, so the chunk is safe when
//        max|f_c - f0| + max_s Tmc_s delta_s + sum_q Lmax_q Rmax_q < Hc
//      (Crec: Tmc, Hc per (tile, chunk); csum: max|f_c - f0|, Lmax per
//      (candidate, chunk); FP32 with upward rounding and a 1e-6 relative
//      margin against a headroom already lowered for FP64 rounding). With the
//      rows in locality order (capi.cu sweep_row_order) most chunks of a tile
//      are far from the candidate's changes and pass;
//   3. the hot chunks' rows (candidate rows, limits, row skip records) are
//      staged by TMA bulk copies into a per-warp ring (lane 0 refills a stage
//      once the warp has left it) and run the row-level stages 1-3 of
//      sweep_cta unchanged (same arithmetic, so the result equals the dense
//      sweep bit for bit).
constexpr int kCkWarps = 8;                   // warps per CTA (independent), 2 CTAs per SM
constexpr int kCkThreads = 32 * kCkWarps;
constexpr int kCkMaxChunks = 512;             // E <= 16384 rows (16-bit hot-chunk list)
constexpr size_t kCkWarpBytes = 13 * 1024 + 512;  // shared memory per warp
constexpr size_t kCkHead = 64 + 128 + 32 + 2 * kCkMaxChunks;  // barriers, rms, asub, hot list
constexpr int kCkMaxStages = 4;

template <int R>
struct CkRing {
  static constexpr int S = row_stride(R);
  static constexpr size_t F = static_cast<size_t>(kChunk) * S * 8;  // candidate rows of one chunk
  static constexpr size_t L = kChunk * 8;                            // limits
  static constexpr size_t M = static_cast<size_t>(kChunk) * kRec * 4;  // row skip records
  static constexpr size_t stage = F + L + M;
  static constexpr size_t fit = (kCkWarpBytes - kCkHead) / stage;
  static constexpr int stages = fit < static_cast<size_t>(kCkMaxStages) ? static_cast<int>(fit) : kCkMaxStages;
  static_assert(stages >= 2, "chunked ring too small");
  static_assert(F % 16 == 0 && M % 16 == 0 && kCkHead % 16 == 0, "bulk copies move 16-byte multiples");
};
constexpr size_t kCkSmemBytes = kCkWarps * kCkWarpBytes;

// acc += d when d > 0 (a predicated add: the conditional add of the exact
// path without a select)
__device__ __forceinline__ void add_if_positive(double& acc, double d) {
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\t@p add.rn.f64 %0, %0, %1;\n\t}"
      : "+d"(acc)
      : "d"(d));
}

template <int R>
__device__ __forceinline__ void ck_item(const DevGrid& g, const Batch& b, int cid, int tile, uint8_t* ws,
                                        uint32_t& phase, unsigned (&stats)[6]) {
  using Rg = CkRing<R>;
  constexpr int S = Rg::S, NST = Rg::stages;
  const int lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ws);
  double* rms = reinterpret_cast<double*>(ws + 64);
  float* asub = reinterpret_cast<float*>(ws + 64 + 128);
  uint16_t* list = reinterpret_cast<uint16_t*>(ws + 64 + 128 + 32);
  uint8_t* ring = ws + kCkHead;
  const int kb = tile * kTileK + lane * kKpl;
  const int nch = b.nchunks;
  // the candidate's row block (chunk 0; chunk j at + j * kGroupSlots * kChunkRows * S),
  // its slot loaded at the item's start so the ring fills do not wait on it
  const double* fbase = b.feat + feat_index(b.slot[cid], nch, 0, R);
  double alpha[kKpl], rr[kKpl][R > 0 ? R : 1], energy[kKpl];
  bool kval[kKpl];
  int kbr[kKpl], rem[kMaxRemovedSweep];
  {
    const double* kd = b.kdat + static_cast<size_t>(cid) * g.Kpad * kStride + static_cast<size_t>(kb) * S;
    const uint8_t* kf = b.kflag + static_cast<size_t>(cid) * g.Kpad + kb;
#pragma unroll
    for (int i = 0; i < kKpl; ++i) {
      kbr[i] = kb + i < g.Ks ? g.ks_branch[kb + i] : -1;
      alpha[i] = __ldcs(kd + i * S);  // read once per launch: streaming
#pragma unroll
      for (int q = 0; q < R; ++q) rr[i][q] = __ldcs(kd + i * S + 1 + q);
      energy[i] = 0.0;
      kval[i] = kf[i] == 0;
    }
#pragma unroll
    for (int q = 0; q < kMaxRemovedSweep; ++q) rem[q] = b.removed[static_cast<size_t>(cid) * kMaxRemovedSweep + q];
  }
  // bound operands (sweep_cta): asub per sub-tile, rms per tile
  if (lane < kStride) rms[lane] = 0.0;
  __syncwarp();
  {
    // maxima as floats rounded up (looser by at most one float ulp: the bounds
    // stay rigorous), reduced with one REDUX each (non-negative float bits
    // order like the values)
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) a = fmax(a, fabs(alpha[k] - g.alpha0[kb + k]));
    const unsigned gmask = ((1u << kSubLanes) - 1u) << (lane & ~(kSubLanes - 1));
    const unsigned am = __reduce_max_sync(gmask, __float_as_uint(__double2float_ru(a * (1.0 + 1e-12))));
    if (lane % kSubLanes == 0) asub[lane / kSubLanes] = __uint_as_float(am);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      double r = 0.0;
#pragma unroll
      for (int k = 0; k < kKpl; ++k) r = fmax(r, fabs(rr[k][q]));
      const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(__double2float_ru(r * (1.0 + 1e-12))));
      if (lane == 0) rms[1 + q] = static_cast<double>(__uint_as_float(m));
    }
  }
  __syncwarp();
  constexpr bool kRegW = R <= 3;
  float areg[kRegW ? kTmaxSub : 1];
  double wreg[kRegW ? S : 1];
  if (kRegW) {
#pragma unroll
    for (int q = 0; q < kTmaxSub; ++q) areg[q] = asub[q];
#pragma unroll
    for (int q = 0; q < S; ++q) wreg[q] = rms[q];
  }
  // chunk tests -> hot-chunk list
  int nlist = 0;
  {
    float af[kTmaxSub], rf[R > 0 ? R : 1];
#pragma unroll
    for (int q = 0; q < kTmaxSub; ++q) af[q] = asub[q];
#pragma unroll
    for (int q = 0; q < R; ++q) rf[q] = __double2float_ru(rms[1 + q]);
    const float* crec = g.Crec + static_cast<size_t>(tile) * nch * kRec;
    const float* cs = b.csum + static_cast<size_t>(cid) * nch * kCsum;
    for (int cb = 0; cb < nch; cb += 32) {
      const int ch = cb + lane;
      bool hot = false;
      if (ch < nch) {
        const float4* rc = reinterpret_cast<const float4*>(crec + static_cast<size_t>(ch) * kRec);
        const float4 t0 = __ldg(rc), t1 = __ldg(rc + 1);
        const double2 hd = __ldg(reinterpret_cast<const double2*>(rc + 2));  // (min headroom, max d_e)
        const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs + static_cast<size_t>(ch) * kCsum));
        const float4 c1 = __ldg(reinterpret_cast<const float4*>(cs + static_cast<size_t>(ch) * kCsum) + 1);
        const float cv[kCsum] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        float td = fmaxf(fmaxf(fmaxf(__fmul_ru(t0.x, af[0]), __fmul_ru(t0.y, af[1])),
                               fmaxf(__fmul_ru(t0.z, af[2]), __fmul_ru(t0.w, af[3]))),
                         fmaxf(fmaxf(__fmul_ru(t1.x, af[4]), __fmul_ru(t1.y, af[5])),
                               fmaxf(__fmul_ru(t1.z, af[6]), __fmul_ru(t1.w, af[7]))));
        float wb = td;  // bound of |T_base||delta| + sum_q |L_q||R'_q| over the chunk and tile
#pragma unroll
        for (int q = 0; q < R; ++q) wb = __fmaf_ru(cv[1 + q], rf[q], wb);
        const float bnd = __fadd_ru(cv[0], wb);
        hot = static_cast<double>(__fmul_ru(bnd, 1.000001f)) >= hd.x;
        // row-coupled test (setup.cu k_chunk_rec): safe when
        // max_e (|f_c - f0|_e - H0_e) + max_e d_e + w < 0
        if (R + 2 <= kCsum && hot)
          hot = static_cast<double>(cv[kCsum - 1]) + static_cast<double>(__fmul_ru(wb, 1.000001f)) + hd.y >= 0.0;
      }
      const unsigned m = __ballot_sync(0xffffffffu, hot);
      if (hot) list[nlist + __popc(m & ((1u << lane) - 1))] = static_cast<uint16_t>(ch);
      nlist += __popc(m);
    }
    stats[4] += static_cast<unsigned>(nch);
    stats[5] += static_cast<unsigned>(nlist);
    stats[1] += static_cast<unsigned>(g.E);  // rows offered (every row of the tile)
  }
  __syncwarp();
  // stage of list entry j: j % NST; each stage barrier completes one phase per
  // fill and the warp waits for every fill, so the per-stage parity bits in
  // `phase` stay valid across items of different ring geometry
  auto issue = [&](int j) {  // lane 0
    const int st = j % NST;
    const int e0 = list[j] * kChunk;
    uint8_t* dst = ring + static_cast<size_t>(st) * Rg::stage;
    uint64_t* bar = bars + st;
    mbar_expect_tx(bar, static_cast<uint32_t>(Rg::stage));
    bulk_g2s(dst, fbase + static_cast<size_t>(list[j]) * (kGroupSlots * kChunkRows * S), static_cast<uint32_t>(Rg::F),
             bar);
    bulk_g2s(dst + Rg::F, g.br_lim + e0, static_cast<uint32_t>(Rg::L), bar);
    bulk_g2s(dst + Rg::F + Rg::L, g.Tmax + (static_cast<size_t>(tile) * (g.E + kChunk) + e0) * kRec,
             static_cast<uint32_t>(Rg::M), bar);
  };
  if (lane == 0)
    for (int j = 0; j < NST && j < nlist; ++j) issue(j);

  // exact path of a hot row: the full f1 of the lane's contingencies (same
  // FMA order as sweep_cta's stages 2-3, so bit-identical values), energies
  // per contingency in registers, the row's max over overloaded elements as
  // one warp reduction and one atomicMax. Stage 1 passes rows that are
  // overloaded for ~93 % (cfg4), so the per-row first-FMA and all-FMA
  // prefilters of sweep_cta are not repeated here.
  auto exact_row = [&](int e, double lim, const double* fr, const double (&tv)[kKpl]) {
    double fl[R > 0 ? R : 1];
#pragma unroll
    for (int q = 0; q < R; ++q) fl[q] = fr[1 + q];
    const double fc = fr[0];
    double mx = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) {
      double acc = fma(tv[k], alpha[k], fc);
#pragma unroll
      for (int q = 0; q < R; ++q) acc = fma(fl[q], rr[k][q], acc);
      const double a = fabs(acc);
      if (a > lim && kval[k] && e != kbr[k]) {
        energy[k] += a - lim;
        mx = fmax(mx, a);
      }
    }
    // warp max of non-negative doubles on their bit patterns (hi word, then lo)
    const unsigned long long bits = dbits(mx);
    const unsigned hi = static_cast<unsigned>(bits >> 32);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    if (mhi == 0u) return false;  // no overloaded element (an overload is > lim > 0)
    const unsigned sel = __ballot_sync(0xffffffffu, hi == mhi);
    if (hi == mhi) {
      const unsigned mlo = __reduce_max_sync(sel, static_cast<unsigned>(bits));
      if (lane == __ffs(sel) - 1)
        atomicMax(b.fmax + static_cast<size_t>(cid) * g.E + e, (static_cast<unsigned long long>(mhi) << 32) | mlo);
    }
    return true;
  };

  // fast form of exact_row when every contingency of the warp is valid and
  // row e is not the outaged branch of any of them (no per-element validity
  // tests): energies by a predicated add of a - lim > 0 (the same additions),
  // the row maximum over all elements (it is the maximum over the overloaded
  // ones whenever one exists, and then the only one stored)
  auto exact_row_fast = [&](int e, double lim, const double* fr, const double (&tv)[kKpl]) {
    double fl[R > 0 ? R : 1];
#pragma unroll
    for (int q = 0; q < R; ++q) fl[q] = fr[1 + q];
    const double fc = fr[0];
    double ma = 0.0;
#pragma unroll
    for (int k = 0; k < kKpl; ++k) {
      double acc = fma(tv[k], alpha[k], fc);
#pragma unroll
      for (int q = 0; q < R; ++q) acc = fma(fl[q], rr[k][q], acc);
      const double a = fabs(acc);
      add_if_positive(energy[k], a - lim);
      ma = a > ma ? a : ma;
    }
    const unsigned long long bits = dbits(ma);
    const unsigned hi = static_cast<unsigned>(bits >> 32);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned sel = __ballot_sync(0xffffffffu, hi == mhi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? static_cast<unsigned>(bits) : 0u);
    const unsigned long long m = (static_cast<unsigned long long>(mhi) << 32) | mlo;
    if (m <= dbits(lim)) return false;  // no overloaded element
    if (lane == __ffs(sel) - 1) atomicMax(b.fmax + static_cast<size_t>(cid) * g.E + e, m);
    return true;
  };
  const bool all_valid = __all_sync(0xffffffffu, kval[0] && kval[1] && kval[2] && kval[3]);
  static_assert(kKpl == 4, "all_valid covers four contingencies per lane");
  const uint32_t* diag_tile = g.diag_bits + static_cast<size_t>(tile) * nch;

  for (int j = 0; j < nlist; ++j) {
    const int st = j % NST;
    const uint8_t* sb = ring + static_cast<size_t>(st) * Rg::stage;
    mbar_wait(bars + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    const int e0 = list[j] * kChunk;
    const int rows = min(kChunk, g.E - e0);
    const double* sF = reinterpret_cast<const double*>(sb);
    const double* sL = reinterpret_cast<const double*>(sb + Rg::F);
    const float* sM = reinterpret_cast<const float*>(sb + Rg::F + Rg::L);
    // stage 1 (sweep_cta, same arithmetic): one lane per row; rows removed by
    // the genome carry no flow and are never scored
    bool hot = false;
    if (lane < rows) {
      bool removed = false;
#pragma unroll
      for (int q = 0; q < kMaxRemovedSweep; ++q) removed |= e0 + lane == rem[q];
      const double lim = sL[lane] * (1.0 - 1e-12);
      const float4* rec = reinterpret_cast<const float4*>(sM) + lane * (kRec / 4);
      const double2* fr = reinterpret_cast<const double2*>(sF + lane * S);
      const double2* wr = reinterpret_cast<const double2*>(rms);
      double l0 = 0.0, l1 = 0.0, fc = 0.0;
#pragma unroll
      for (int q = 0; q < S / 2; ++q) {
        const double2 p2 = fr[q];
        const double2 w2 = kRegW ? make_double2(wreg[kRegW ? 2 * q : 0], wreg[kRegW ? 2 * q + 1 : 0]) : wr[q];
        l0 = fma(fabs(p2.x), w2.x, l0);
        l1 = fma(fabs(p2.y), w2.y, l1);
        if (q == 0) fc = p2.x;
      }
      const double flo = fc;
      const double lrb = l0 + l1;
      const float4* ar = reinterpret_cast<const float4*>(asub);
      float taf = 0.0f;
#pragma unroll
      for (int q = 0; q < kTmaxSub / 4; ++q) {
        const float4 t4 = rec[q];
        const float4 a4 = kRegW ? make_float4(areg[kRegW ? 4 * q : 0], areg[kRegW ? 4 * q + 1 : 0],
                                              areg[kRegW ? 4 * q + 2 : 0], areg[kRegW ? 4 * q + 3 : 0])
                                : ar[q];
        taf = fmaxf(taf, fmaxf(fmaxf(__fmul_ru(t4.x, a4.x), __fmul_ru(t4.y, a4.y)),
                               fmaxf(__fmul_ru(t4.z, a4.z), __fmul_ru(t4.w, a4.w))));
      }
      const double2 d0 = reinterpret_cast<const double2*>(rec)[kTmaxSub / 4];
      const double gap = lim - fmax(fc + d0.x, -(flo + d0.y));
      const double s0 = 1e-12 * (fmax(fabs(fc), fabs(flo)) + fabs(d0.x) + fabs(d0.y));
      const double wd = static_cast<double>(taf) + lrb;
      hot = !removed && fma(wd, 1.0 + 1e-12, s0) >= gap;
    }
    unsigned need = __ballot_sync(0xffffffffu, hot);
    stats[3] += __popc(need);
    stats[0] += __popc(need);
    // exact path, NB rows' T_base tile rows in flight
    const uint32_t dword = need ? __ldg(diag_tile + list[j]) : 0u;
    constexpr int NB = R >= 6 ? 2 : 4;
    const double* tk_rows = g.TK + (static_cast<size_t>(tile) * g.E + e0) * kTileK + lane * kKpl;
    while (need) {
      int els[NB];
      int nu = 0;
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        els[u] = need ? __ffs(need) - 1 : -1;
        if (need) need &= need - 1, ++nu;
      }
      double2 t[NB][2];
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        const int el = els[u] >= 0 ? els[u] : els[0];
        const double2* src = reinterpret_cast<const double2*>(tk_rows + static_cast<size_t>(el) * kTileK);
        t[u][0] = __ldg(src);
        t[u][1] = __ldg(src + 1);
      }
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        if (u >= nu) break;
        const int el = els[u];
        const double tv[kKpl] = {t[u][0].x, t[u][0].y, t[u][1].x, t[u][1].y};
        const bool ok = all_valid && !((dword >> el) & 1u);
        stats[2] += (ok ? exact_row_fast(e0 + el, sL[el], sF + el * S, tv)
                        : exact_row(e0 + el, sL[el], sF + el * S, tv)) ? 1u : 0u;
      }
    }
    __syncwarp();
    if (lane == 0 && j + NST < nlist) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(j + NST);
    }
    __syncwarp();
  }
  double* en = b.energy + static_cast<size_t>(cid) * g.Kall;
#pragma unroll
  for (int k = 0; k < kKpl; ++k)
    if (kval[k] && kb + k < g.Ks && energy[k] != 0.0) en[g.ks_cont[kb + k]] = energy[k];  // zeroed per evaluation
}

template <int RLO, int RHI>
__device__ __forceinline__ void ck_dispatch(const DevGrid& g, const Batch& b, int r, int cid, int tile, uint8_t* ws,
                                            uint32_t& phase, unsigned (&stats)[6]) {
  if constexpr (RLO <= RHI) {
    if (r == RLO || RLO == RHI) {
      ck_item<RLO>(g, b, cid, tile, ws, phase, stats);
    } else {
      ck_dispatch<RLO + 1, RHI>(g, b, r, cid, tile, ws, phase, stats);
    }
  }
}

// ranks RLO..RHI (one kernel per rank class: each gets its own register allocation)
template <int RLO, int RHI>
__global__ void __launch_bounds__(kCkThreads, 2) k_sweep_chunked(DevGrid g, Batch b, int ntiles, unsigned* ctr) {
  extern __shared__ __align__(128) uint8_t ck_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ws = ck_smem + static_cast<size_t>(warp) * kCkWarpBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ws);
  if (lane == 0) {
    for (int s = 0; s < kCkMaxStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int first = b.wl_start[RLO];
  const int ncand = b.wl_start[RHI] + b.wl_count[RHI] - first;
  const unsigned items = static_cast<unsigned>(ncand) * static_cast<unsigned>(ntiles);  // the item counter is 32-bit
  uint32_t phase = 0;
  unsigned stats[6] = {0, 0, 0, 0, 0, 0};
  for (;;) {
    unsigned it = 0;
    if (lane == 0) it = atomicAdd(ctr, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= items) break;
    const unsigned ci = it / static_cast<unsigned>(ntiles);  // 32-bit division
    const int cid = b.wl_list[first + static_cast<int>(ci)];
    const int tile = static_cast<int>(it - ci * static_cast<unsigned>(ntiles));
    if (b.status[cid] != 0) continue;
    ck_dispatch<RLO, RHI>(g, b, b.rank[cid], cid, tile, ws, phase, stats);
  }
  if (lane == 0) {
    for (int i = 0; i < 6; ++i)
      if (stats[i]) atomicAdd(b.rows_done + i, static_cast<unsigned long long>(stats[i]));
  }
}

// Stable per-rank lists of swept candidates; bucket r is cut into CTA groups
// of cand_per_cta(r), and every swept candidate gets its row slot
// (group * kGroupSlots + position) so k_prep writes straight into the layout
// the sweep streams.
__global__ void k_bucket(Batch b) {
  // two passes over the batch in 1024-candidate chunks: per-rank counts, then
  // stable positions (rank bucket, then candidate order); one ballot per rank
  // per warp and one barrier per chunk and pass
  constexpr int NR = kSweepRank + 1;
  __shared__ int warp_tot[NR][32];
  __shared__ int run_s[NR], base_s[NR], gbase_s[NR];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < NR) run_s[threadIdx.x] = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int c0 = 0; c0 < b.n; c0 += blockDim.x) {
      const int c = c0 + threadIdx.x;
      const int rk = c < b.n ? b.rank[c] : -1;
      unsigned mine_m = 0u;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const unsigned m = __ballot_sync(0xffffffffu, rk == r);
        if (rk == r) mine_m = m;
        if (lane == 0) warp_tot[r][wid] = __popc(m);
      }
      __syncthreads();
      if (pass == 1 && rk >= 0 && rk < NR) {
        int off = 0;
        for (int x = 0; x < wid; ++x) off += warp_tot[rk][x];
        const int pos = run_s[rk] + off + __popc(mine_m & ((1u << lane) - 1));
        b.wl_list[base_s[rk] + pos] = c;
        b.slot[c] = (gbase_s[rk] + pos / cand_per_cta(rk)) * kGroupSlots + pos % cand_per_cta(rk);
      } else if (c < b.n && (rk < 0 || rk >= NR)) {
        b.slot[c] = -1;
      }
      __syncthreads();
      if (threadIdx.x < NR) {
        int tot = 0;
        for (int x = 0; x < nw; ++x) tot += warp_tot[threadIdx.x][x];
        run_s[threadIdx.x] += tot;
      }
      __syncthreads();
    }
    if (pass == 0 && threadIdx.x == 0) {
      int base = 0, group_base = 0;
      for (int r = 0; r < NR; ++r) {
        base_s[r] = base;
        gbase_s[r] = group_base;
        b.wl_start[r] = base;
        b.wl_count[r] = run_s[r];
        b.wl_group0[r] = group_base;
        base += run_s[r];
        group_base += (run_s[r] + cand_per_cta(r) - 1) / cand_per_cta(r);
        run_s[r] = 0;
      }
      b.wl_group0[NR] = group_base;
    }
    __syncthreads();
  }
}

}  // namespace

int sweep_tile_k() { return kTileK; }
// the masked timestep sweep needs two ring stages next to its row lists
bool masked_sweep_fits(int E) { return masked_plan(E, kStride).stages >= 2; }
int sweep_chunk() { return kChunk; }

void launch_sweep(const DevGrid& g, Batch& b, bool full, cudaStream_t stream, cudaEvent_t ev0, cudaEvent_t ev1,
                  int* launched) {
  static std::atomic<unsigned long long> configured{0};
  if (first_use_on_device(configured)) {
    const int sm = static_cast<int>(kSmemBytes), hm = static_cast<int>(kHalfSmemBytes);
    cudaFuncSetAttribute(k_sweep<true, kTmSingle, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep<false, kTmSingle, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep<false, kTmSingle, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hm);
    cudaFuncSetAttribute(k_sweep<false, kTmMask, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep<false, kTmMask, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hm);
    cudaFuncSetAttribute(k_sweep_hi<true, kTmSingle, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep_hi<false, kTmSingle, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep_hi<false, kTmSingle, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hm);
    cudaFuncSetAttribute(k_sweep_hi<false, kTmMask, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_sweep_hi<false, kTmMask, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hm);
    cudaFuncSetAttribute(k_sweep_chunked<0, kChunkedMaxRank>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kCkSmemBytes));
  }
  // group slots: every bucket rounds up to whole groups of kWarps candidates
  static const int gblock_env = [] {
    const char* v = std::getenv("TGB_SWEEP_GROUP_BLOCK");
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  const int ntiles = g.Kpad / kTileK, ngroups = max_sweep_groups(b.n);
  const int gblock = std::min(ngroups, gblock_env ? gblock_env : kGroupBlock);
  const unsigned grid = static_cast<unsigned>(ntiles) * ngroups;
  if (ev0) cudaEventRecord(ev0, stream);
  constexpr int kHiCtas = 148;  // persistent: one CTA per SM (two half-group CTAs)
  constexpr int hw = 32 * cta_warps<true>(), hh = kGroupSlots / cta_warps<true>();
  const bool half = g.E <= kHalfMaxRows;
  static const bool v1 = std::getenv("TGB_SWEEP_V1") != nullptr;  // A/B: the tile-streaming sweep for every rank
  const bool chunked = !v1 && g.Crec && b.csum && g.E <= kCkMaxChunks * kChunk;
  if (full) {
    k_sweep<true, kTmSingle, false><<<grid, kThreads, kSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
    k_sweep_hi<true, kTmSingle, false><<<kHiCtas, kThreads, kSmemBytes, stream>>>(g, b, ntiles);
  } else if (b.t_mode == kTmMask) {
    if (half) {
      k_sweep<false, kTmMask, true><<<grid * hh, hw, kHalfSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
      k_sweep_hi<false, kTmMask, true><<<kHiCtas * hh, hw, kHalfSmemBytes, stream>>>(g, b, ntiles);
    } else {
      k_sweep<false, kTmMask, false><<<grid, kThreads, kSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
      k_sweep_hi<false, kTmMask, false><<<kHiCtas, kThreads, kSmemBytes, stream>>>(g, b, ntiles);
    }
  } else if (chunked) {
    // ranks 0..7 in one persistent kernel (one work list, no tail between
    // rank classes; every rank variant fits the same 128 registers)
    cudaMemsetAsync(b.item_ctr, 0, sizeof(unsigned int), stream);
    // persistent: 2 CTAs per SM, fewer when the batch has fewer (candidate, tile) items than warps
    const int ck_grid = static_cast<int>(std::max<long>(1, std::min<long>(148 * 2, (static_cast<long>(b.n) * ntiles + kCkWarps - 1) / kCkWarps)));
    k_sweep_chunked<0, kChunkedMaxRank><<<ck_grid, kCkThreads, kCkSmemBytes, stream>>>(g, b, ntiles, b.item_ctr);
    k_sweep_hi<false, kTmSingle, false><<<kHiCtas, kThreads, kSmemBytes, stream>>>(g, b, ntiles);
  } else if (half) {
    k_sweep<false, kTmSingle, true><<<grid * hh, hw, kHalfSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
    k_sweep_hi<false, kTmSingle, true><<<kHiCtas * hh, hw, kHalfSmemBytes, stream>>>(g, b, ntiles);
  } else {
    k_sweep<false, kTmSingle, false><<<grid, kThreads, kSmemBytes, stream>>>(g, b, ntiles, ngroups, gblock);
    k_sweep_hi<false, kTmSingle, false><<<kHiCtas, kThreads, kSmemBytes, stream>>>(g, b, ntiles);
  }
  if (ev1) cudaEventRecord(ev1, stream);
  *launched += 2;
}

void launch_sweep_masked(const DevGrid& g, Batch& b, const MtMask& mm, cudaStream_t stream, cudaEvent_t ev0,
                         cudaEvent_t ev1, int* launched) {
  static std::atomic<unsigned long long> configured{0};
  if (first_use_on_device(configured))
    cudaFuncSetAttribute(k_sweep_masked, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kMaskBudget));
  const int ntiles = g.Kpad / kTileK, ngroups = max_sweep_groups(b.n);
  const int gblock = std::min(ngroups, kGroupBlock);
  const unsigned grid = 2u * static_cast<unsigned>(ntiles) * ngroups;  // half-group CTAs
  if (ev0) cudaEventRecord(ev0, stream);
  k_sweep_masked<<<grid, kMaskThreads, kMaskBudget, stream>>>(g, b, ntiles, ngroups, gblock, mm);
  if (ev1) cudaEventRecord(ev1, stream);
  *launched += 1;
}

void launch_bucket(Batch& b, cudaStream_t stream, int* launched) {
  k_bucket<<<1, 1024, 0, stream>>>(b);
  *launched += 1;
}

}  // namespace tgb
