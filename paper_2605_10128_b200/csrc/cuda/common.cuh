// Device-side tables and helpers shared by every kernel of the DC N-1 engine.
#pragma once

#include <atomic>

#include <cstdint>
#include <cuda_runtime.h>

namespace tgb {

// Compile-time capacities. The reference's QdConfig defaults are n_a=3, n_d=2
// (qd_optimizer.hpp:16-17); these bound the per-candidate low-rank update.
constexpr int kMaxSlots = 8;       // n_a + n_d
constexpr int kMaxSplits = 4;      // n_a
constexpr int kSweepRank = 11;     // largest update rank r (n_a = n_d = 4 plus grounded dead nodes)
constexpr int kStride = 12;        // max doubles per branch row (f_c, L[0..10]) and per contingency row
constexpr int kMaxMoved = 128;     // moved branch ends per candidate
constexpr int kMaxRemoved = 24;    // removed branches (genome + outage case)
constexpr int kMaxGround = 8;      // dead base nodes grounded
constexpr int kMaxCols = kMaxSplits + kMaxRemoved + kMaxGround;  // Z columns for the outage rebuild
constexpr int kTopoSol = kMaxSplits * kMaxSplits + kMaxSplits * kMaxCols + kMaxCols * kMaxCols;  // S^-1, Y, C^-1
constexpr int kMaxTerms = 512;     // sparse coefficients over all Z columns
constexpr int kMaxPMod = 32;       // omitted injections (p modifications)
constexpr int kMaxInjMoved = 64;   // injections moved to new nodes
constexpr int kTmaxSub = 8;        // sub-tiles of a sweep tile carrying their own max |T_base| per row
constexpr int kRec = kTmaxSub + 4; // floats per (tile, row) skip record: kTmaxSub sub-tile maxima of |T_base| (float,
                                   // rounded up), then max / min of T_base*alpha0 as two doubles (48 B)

// Flat, read-only network tables on the device (built once per context by
// engine_setup.cu from the host Grid/ActionTable).
struct DevGrid {
  int N, Nr, E, I, slack;
  int Ks, Kpad;   // single-branch contingencies handled by the fused sweep
  int Kx;         // special contingencies (multi-branch and/or injections)
  int Kall;       // all listed contingencies
  int Kb;         // busbar outages
  int S, A, D;
  const int* red;          // [N]   reduced index, slack -> -1
  const int* br_from;      // [E]
  const int* br_to;        // [E]
  const double* br_b;      // [E]   susceptance 1/x
  const double* br_lim;    // [E]
  const uint8_t* br_on;    // [E]
  const double* X;         // [Nr*Nr] inverse reduced susceptance (symmetric)
  const double* theta0;    // [Nr]  base angles X * p_red
  const double* f0;        // [E]   base flows
  const double4* row_static;  // [E] (f0, b, limit, in service) packed: one load per row in k_prep_rows
  const double* Tdiag;     // [E]   b_e a_e^T X a_e
  const int* node_ptr;     // [N+1] in-service incident branches
  const int* node_br;
  const int* node_inj_ptr; // [N+1] injections at node
  const int* node_inj;
  const int* inj_node;     // [I]
  const double* inj_net;   // [I]
  const int* ks_cont;      // [Ks]  contingency index
  const int* ks_branch;    // [Ks]
  const double* TK;        // [Kpad/128][E][128] T_base[e, ks_branch[k]] tiles (0 rows for out-of-service e)
  const float* Tmax;       // [Kpad/128][E + 32][kRec] skip record per (tile, row): max over each sub-tile of
                           // |T_base[e, k]|, then max_k and min_k of T_base[e, k] * alpha0[k] over the tile
  const double* alpha0;    // [Kpad] alpha of the unchanged topology, f0[beta] / (1 - Tdiag[beta]) (0 padding)
  const float* Crec;       // [Kpad/128][ceil(E/32)][kRec] chunk record per (tile, 32-row chunk): the max over the
                           // chunk's rows of each sub-tile maximum of Tmax (floats), then the chunk's base N-1
                           // headroom min_e (lim_e - max(f0_e + D0max, -(f0_e + D0min))) minus a rounding slack
                           // (double); the chunk-level skip bound of the scores-only sweep (sweep.cu)
  const uint32_t* diag_bits;  // [Kpad/128][ceil(E/32)] bit e%32 of word e/32: row e is the outaged branch of a
                              // contingency of the tile (the only rows with a diagonal element to exclude)
  const int* kx_cont;      // [Kx]
  const int* kx_br_ptr;    // [Kx+1]
  const int* kx_br;
  const int* kx_inj_ptr;   // [Kx+1]
  const int* kx_inj;
  const int* bo_station;   // [Kb]
  const int* bo_busbar;    // [Kb]
  const int* bo_def_ptr;   // [Kb+1] default implied sets (grid_model.cpp:217-227)
  const int* bo_def;
  const int* st_node;      // [S]
  const int* st_range_lo;  // [S] action id range (-1 when the station has none)
  const int* st_range_hi;  // [S]
  const int* st_term_ptr;  // [S+1]
  const int* term_kind;    // 0 from-end, 1 to-end, 2 injection
  const int* term_elem;
  const int* act_station;  // [A]
  const int* act_lambda_r; // [A]
  const uint8_t* act_group;// [A][n_terms(station)] at act_group_ptr
  const int* act_group_ptr;// [A+1]
  const int* act_imp_ptr;  // [A*?] implied set per (action, busbar): act_bb_ptr[a] + busbar -> range
  const int* act_bb_ptr;   // [A+1]
  const int* act_imp;
  const int* disc;         // [D] branch index of each disconnectable
  // Branch-space columns of the low-rank update, precomputed once per context
  // (setup.cu k_phi_cols; null when they do not fit the memory budget):
  // PhiA[a][e] = (X u_a)[from_e] - (X u_a)[to_e] for the split column u_a of
  // action a (all its base-active moved branch ends), PsiD[d][e] the same for
  // the removal column a_d of disconnectable d (topo.cuh column_sources).
  const double* PhiA;      // [A][E]
  const int* act_nmv;      // [A] base-active moved branch ends of each action (-1: no column)
  const double* PsiD;      // [D][E]
  const int* disc_of_br;   // [E] disconnectable index of a branch, -1
};

struct DcParams {
  double penalty;
  double weight_c0, weight_c;
  double lambda_b_pre;
  int worst_k;
  int variant;
  int n_a, n_d;
};

// Function attributes (shared-memory limits, carveouts) are per device: true
// the first time the calling thread's current device asks for `flags`.
inline bool first_use_on_device(std::atomic<unsigned long long>& flags) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  return !(flags.fetch_or(bit) & bit);
}

__device__ __forceinline__ unsigned long long dbits(double x) { return static_cast<unsigned long long>(__double_as_longlong(x)); }

// max on non-negative doubles through their ordered bit patterns
__device__ __forceinline__ void atomic_max_pos(unsigned long long* addr, double v) {
  atomicMax(addr, dbits(v));
}

}  // namespace tgb
