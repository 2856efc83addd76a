// Batch buffers and launchers of the DC N-1 engine.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include "common.cuh"

namespace tgb {

struct TopoCore;                     // topo.cuh
size_t topo_core_bytes();

constexpr int kMaxRemovedSweep = 4;  // genome disconnections skipped in the sweep (n_d <= 4)
constexpr int kGroupSlots = 16;      // candidates per sweep CTA group (8 warps x 2)
constexpr int kChunkRows = 32;       // branch rows per sweep pipeline stage
constexpr int kCsum = 8;             // floats per (candidate, chunk) summary: max |f_c - f0|, max |L_0..6|
constexpr int kChunkedMaxRank = 7;   // ranks handled by the chunked sweep (higher ranks: k_sweep_hi)

// Ordered-integer key of a double (any sign): keys compare like the values.
__device__ inline unsigned long long order_key(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ inline double order_value(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// Doubles per candidate row (branch row f_c, L[0..r-1] or contingency row
// alpha, R'[0..r-1]) for update rank r, rounded up to whole double2.
__host__ __device__ constexpr int row_stride(int r) { return (r + 2) & ~1; }

// Row e of candidate c (sweep slot `slot`, update rank r) in the group-major
// candidate row array: [group][chunk][kGroupSlots][kChunkRows][row_stride(r)],
// each group owning a block sized for the largest stride.
__host__ __device__ inline size_t feat_index(int slot, int nchunks, int e, int r) {
  const int group = slot / kGroupSlots, pos = slot % kGroupSlots;
  const int chunk = e / kChunkRows, row = e % kChunkRows;
  return static_cast<size_t>(group) * nchunks * kGroupSlots * kChunkRows * kStride +
         ((static_cast<size_t>(chunk) * kGroupSlots + pos) * kChunkRows + row) * row_stride(r);
}

// Per-candidate scores, SoA (dc_engine.hpp:25-39).
struct Scores {
  double* lambda_o;
  int* lambda_c;
  int* lambda_c0;
  double* lambda_b;
  int* lambda_d;
  int* lambda_s;
  int* lambda_r;
  double* fitness;
  uint8_t* islanded;
  int* error;       // nonzero: capacity exceeded (host raises)
  int* worst_idx;   // [n][worst_k]
  double* worst_val;
  int* worst_n;
  int* isl_out;     // islanded contingencies
  int* isl_bus;     // islanded busbar outages
};

// Compact small-solve factors of one candidate for the split prep
// (k_prep_solve -> k_prep_rows; ranks <= kSweepRank, branch-space columns).
struct alignas(16) PcFac {
  double Sinv[kMaxSplits * kMaxSplits];  // ns x ns (ld kMaxSplits)
  double Y[kMaxSplits * kSweepRank];     // S^-1 Phi, ns x nv (ld kSweepRank)
  double Cinv[kSweepRank * kSweepRank];  // nv x nv (ld kSweepRank)
  double Rp[kMaxSplits + kSweepRank];    // [S^-1 phi_p ; -C^-1 rho_p]
  const double* base[kSweepRank];        // branch-space column sources (topo.cuh column_sources)
  int ns, nv;
};

// Device buffers of one evaluation batch (capacity fixed at allocation).
struct Batch {
  int n;                      // candidates in this launch
  const int* genomes;         // [n][n_a+n_d]
  DcParams params;
  int* status;                // 0 ok, 1 islanded, 2/3 capacity error
  int* err_sticky;            // per-context capacity-error word: k_finish ORs 1 into it for every lane whose
                              // status is a capacity error; the host checks it after loop steps and clears it
  TopoCore* topo;             // [n] topology analysis of k_analyze, reloaded by k_prep
  uint32_t* tbits;            // [n][2 * words] moved / removed branch bitmaps of the analysis
  int* rank;                  // low-rank update size, -1 when not swept
  int* removed;               // [n][kMaxRemovedSweep] genome-removed branches
  // Candidate branch rows (f_c, L[0..r-1], 0 padding) stored in the sweep's
  // group-major layout so one pipeline stage of a sweep CTA is one contiguous
  // block: [group][chunk][kGroupSlots][kChunkRows][row_stride(r)] (feat_index).
  double* feat;
  int* slot;                  // [n] group * kGroupSlots + position, -1 when not swept
  int nchunks;                // ceil(E / kChunkRows)
  unsigned long long* rows_done;  // [8] sweep stats: blocks computed / offered / overloaded / first FMA only,
                                  // chunk tests / hot chunks (chunked sweep)
  float* csum;                // [n][nchunks][kCsum] per (candidate, 32-row chunk): max |f_c - f0| and max |L_q|
                              // (q < rank) over the chunk's live rows, floats rounded up (k_prep; ranks <= 7)
  unsigned int* item_ctr;     // [4] work counters of the persistent chunked sweep (zeroed per evaluation)
  double* kdat;               // [n][Kpad * kStride]: Kpad rows of row_stride(r) doubles alpha, R'
                              // (single-branch contingencies)
  uint8_t* kflag;             // [n][Kpad] 0 ok, 1 islanded, 2 padding
  unsigned long long* fmax;   // [n][E] max |f| over contingencies (bits of a non-negative double). The FULL
                              // (FlowResult) sweep folds every element; the scores-only and masked sweeps fold
                              // only elements above the branch limit (the only values a score reads), so there
                              // an entry at or below the limit means "not overloaded", not the maximum: only
                              // FULL-path fmax may be exported as FlowResult::max_contingency (launch_extract)
  unsigned long long* fbus;   // [n][E] max |f| over busbar outages
  double* energy;             // [n][Kall] outage energy per contingency
  int* nc0;                   // [n] lambda_c0 of the candidate flows (k_prep)
  PcFac* pc;                  // [n] split-prep factors (k_prep_solve)
  // Multi-timestep screening (capi.cu, n_t > 1 profiles): k_prep (profile 0)
  // and k_prep_mt (the others) fold every profile's candidate flows and flow
  // factors into bounds over all profiles; k_sweep in mask mode (t_mode 1) marks the rows
  // of each (candidate, tile) that can overload at some profile, k_sweep in
  // masked mode (t_mode 2) then visits only those rows per profile.
  int t_mode;                 // 0 single profile, 1 mask generation, 2 masked sweep
  int no_worst;               // k_finish: skip the worst list (per-profile pass of a timestep grid)
  double* feat_mt;            // rows [key(max_t f_c), key(min_t f_c), L...] at row_stride(r + 1), feat_index layout;
                              // keys are the ordered bit patterns of doubles (order_key)
  unsigned long long* amx_mt; // [n][ntiles][kTmaxSub] max_t max |alpha_t - alpha0_t| per sub-tile (bits)
  unsigned long long* rmx_mt; // [n][ntiles][kStride] max_t max_k |R'_t[q, k]| per tile (bits, slot 1 + q)
  uint32_t* mask;             // [n][ntiles][nchunks] rows that can overload at some profile
  double* topo_sol;           // [n][kTopoSol] S^-1, Y, C^-1 of the first profile's small solve
  const double* fc_t;         // masked sweep: this profile's f_c [n][E] (k_prep_mt), L from feat (profile 0)
  const double* al_t;         // masked sweep: this profile's alpha [n][Kpad]
  const double* rk_mt;        // masked sweep: rk rows (MtProfiles::rk); R'_t = rk * alpha_t
  int* isl_out;               // [n] islanded special contingencies
  int* isl_bus;               // [n]
  int* wl_list;               // [n] candidates bucketed by rank
  int* wl_start;              // [kSweepRank+1]
  int* wl_count;              // [kSweepRank+1]
  int* wl_group0;             // [kSweepRank+2]
  Scores out;
};

struct EvalScratch {
  double* zprep;       // [zslots][Nr][kStride]
  int zslots;
  double* zspecial;    // [zslots_special][Nr][kMaxCols]
  int zslots_special;
};

// sweep_begin / sweep_end (optional) bracket the fused sweep launch for live timing.
// A second stream with fork / join events: launch_evaluate runs the special
// outages there, beside the prep and the sweep.
struct SideStream {
  cudaStream_t stream;
  cudaEvent_t fork, join;
};
void launch_evaluate(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                     cudaStream_t stream, int* kernels, cudaEvent_t sweep_begin = nullptr,
                     cudaEvent_t sweep_end = nullptr, const SideStream* side = nullptr);
// The phases launch_evaluate runs (returning kernels launched).
int launch_eval_reset(const DevGrid& g, Batch& b, cudaStream_t stream);
int launch_analyze(const DevGrid& g, Batch& b, int n_a, int n_d, cudaStream_t stream);
int launch_prep(const DevGrid& g, Batch& b, int n_a, int n_d, const EvalScratch& s, cudaStream_t stream);
// Multi-timestep screening: the candidate rows of profiles 1..n_t-1 in one pass
// (after launch_prep of profile 0 with t_index 0): per-profile base tables and
// the element strides between the profiles' row / contingency / energy / nc0
// arrays (profile 0 at the Batch pointers).
struct MtProfiles {
  const double* const* f0;       // [n_t] base flows
  const double* const* theta0;   // [n_t] base angles (reduced)
  const double* const* inj_net;  // [n_t] injections
  const double* const* alpha0;   // [n_t] unchanged-topology flow factors
  const float* const* tmax;      // [n_t] skip records
  int n_t;
  double* fc;  // [n_t][n][E] candidate flows per profile (compact)
  double* al;  // [n_t][n][Kpad] alpha per profile
  double* rk;  // [n][Kpad][kStride] rows [0, rk_0..rk_{r-1}] at row_stride(r), profile-independent
  size_t fc_stride, al_stride, energy_stride, nc0_stride;
};
int launch_prep_mt(const DevGrid& g, Batch& b, const MtProfiles& p, cudaStream_t stream);
int launch_special_finish(const DevGrid& g, Batch& b, int n_a, int n_d, bool full, const EvalScratch& s,
                          cudaStream_t stream);
void launch_extract(const DevGrid& g, Batch& b, double* base_out, double* fmax_out, double* fbus_out,
                    cudaStream_t stream);
// Timestep aggregation (host loops launch_evaluate over t with the per-t
// scores in `bt`): accumulate timestep t into (agg, agg_energy), then the
// fitness and worst list of the sums into b.out (b.energy = the summed energies).
int launch_accumulate_timestep(const Batch& bt, Scores& agg, double* agg_energy, int Kall, bool first,
                               cudaStream_t stream);
int launch_finish_aggregate(Batch& b, int Kall, cudaStream_t stream);
int launch_sum_profiles(const double* e, int n_t, size_t stride, size_t n, double* out, cudaStream_t stream);
int sweep_tile_k();
int sweep_chunk();
bool masked_sweep_fits(int E);  // k_sweep_masked's shared-memory plan holds for E rows
void launch_sweep(const DevGrid& g, Batch& b, bool full, cudaStream_t stream, cudaEvent_t ev0, cudaEvent_t ev1,
                  int* launched);
// Masked timestep sweep (Batch::t_mode 2) of profiles [t0, t0 + np): b's fc_t,
// al_t, energy and fmax point at profile t0's arrays, profile t0 + p at
// + p * the strides; per-profile skip records and alpha0 through device arrays.
struct MtMask {
  int t0, np;
  size_t fc_stride, al_stride, energy_stride, fmax_stride;
  const float* const* tmax;
  const double* const* alpha0;
};
constexpr int kMaskProfiles = 8;  // profiles per masked launch
void launch_sweep_masked(const DevGrid& g, Batch& b, const MtMask& mm, cudaStream_t stream, cudaEvent_t ev0,
                         cudaEvent_t ev1, int* launched);
// Rank buckets -> sweep groups; assigns every swept candidate its row slot.
void launch_bucket(Batch& b, cudaStream_t stream, int* launched);
// Upper bound on sweep groups for n candidates (every rank bucket rounds up).
inline int max_sweep_groups(int n) { return (n + kGroupSlots - 1) / kGroupSlots + kSweepRank + 1; }

// Base factorization on the device (dc_engine.cpp:88-116, importer.cpp:358-401):
// X = B_red^-1 by in-place Gauss-Jordan (B_red is SPD; no pivoting needed).
// Returns false when a pivot is not positive (disconnected grid).
bool device_spd_inverse(double* a, int n, cudaStream_t stream);
// build_ptdf (importer.cpp:358-401) from X = B_red^-1: out [E][N], slack column 0.
void launch_ptdf(int N, int E, int Nr, const int* red, const int* from, const int* to, const double* b,
                 const uint8_t* on, const double* X, double* out, cudaStream_t stream);
// Skip records of n_t profiles (contiguous, rec_floats each) combined into
// bounds over all profiles (multi-timestep screening).
void launch_rec_combine(const float* recs, size_t rec_floats, int n_t, float* out, cudaStream_t stream);
// Base N-1 headroom per branch row (lim - max_k |f0 + T_base alpha0|) for the
// sweep row order; needs g.{E, Nr, Ks, red, br_*, X, ks_branch}.
void launch_row_headroom(const DevGrid& g, const double* p_red, double* theta0, double* f0, double* tdiag, double* h,
                         cudaStream_t stream);
// Branch-space columns PhiA [A][E], act_nmv [A], PsiD [D][E] (DevGrid) from X.
void launch_phi_columns(const DevGrid& g, double* phiA, int* act_nmv, double* psiD, cudaStream_t stream);
// Chunk records (DevGrid::Crec) from a profile's skip records, base flows and limits.
void launch_chunk_records(const DevGrid& g, float* crec, cudaStream_t stream);
// DevGrid::row_static from the profile's base flows
void launch_row_static(const DevGrid& g, const double* f0, double4* out, cudaStream_t stream);
void launch_base_tables(const DevGrid& g, const double* p_red, double* theta0, double* f0, double* tdiag, double* tk,
                        float* tmax, double* alpha0, cudaStream_t stream);

}  // namespace tgb

namespace tgb {

// RAII device scratch for one-off host-requested outputs.
struct DeviceScratchGuard {
  double* ptr = nullptr;
  explicit DeviceScratchGuard(size_t n) { cudaMalloc(&ptr, (n ? n : 1) * sizeof(double)); }
  ~DeviceScratchGuard() { cudaFree(ptr); }
  DeviceScratchGuard(const DeviceScratchGuard&) = delete;
  DeviceScratchGuard& operator=(const DeviceScratchGuard&) = delete;
};

}  // namespace tgb
