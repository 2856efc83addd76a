// MapElites device state: archive, lane RNG replay, mutation / crossover,
// sequential-equivalent insert (qd_optimizer.cpp:12-417).
#pragma once

#include "engine.cuh"

namespace tgb {

constexpr int kMaxCellCap = 16;  // QdConfig::cell_capacity supported on the device
constexpr int kRngReplay = 0;    // per-lane std::mt19937_64 + libstdc++ distributions (reference stream)
constexpr int kRngPhilox = 1;    // counter-based Philox4x32-10, same distributions

// QdConfig (qd_optimizer.hpp:15-32) as passed to kernels.
struct QdParams {
  int n_a, n_d, batch, cap;
  int d_max, s_max, r_max, cells;
  double p_action[4];
  double p_disc[4];
  double p_c1;
  double poisson_thr;  // exp(-mutation_mean), computed by the host libm like libstdc++ does
  unsigned long long seed;
  int n_actions, n_disc;
  int rng;             // kRngReplay (mt19937_64, bit-exact with the reference) or kRngPhilox
};

// Device archive of cells x cell_capacity entries, cell-major (Repertoire,
// qd_optimizer.hpp:60-81). Entries of a cell are kept sorted by fitness desc,
// ties in arrival order, exactly like the reference's upper_bound insert.
struct Archive {
  int* count;            // [cells]
  int* flat_start;       // [cells+1] exclusive prefix of count (Repertoire::member order)
  int* genome;           // [cells][cap][n_slots] as inserted
  int* key;              // [cells][cap][n_slots] canonical key: sorted actions, sorted disconnections (-1 padded)
  double* fitness;       // [cells][cap]
  double* lambda_o;
  int* lambda_c;
  int* lambda_c0;
  double* lambda_b;
  int* lambda_d;
  int* lambda_s;
  int* lambda_r;
  int* worst_idx;        // [cells][cap][worst_k]
  double* worst_val;
  int* worst_n;
  long long* iter;       // [1] global iteration counter (qd_optimizer.cpp:373)
};

struct QdState {
  QdParams p{};
  Archive a{};
  int n_slots = 0;
  int worst_k = 0;
  uint8_t* inserted = nullptr;  // [batch] Repertoire::insert results of the last insert
  int* lane_cell = nullptr;     // [batch]
  cudaGraphExec_t graph = nullptr;
  int graph_batch = 0;
  int kernels_per_iter = 0;
  void* arena = nullptr;        // owned by the context (DeviceArena*)
};

// Island exchange blob: one island's whole archive (cells x cap slots) in a
// fixed byte layout, so an NCCL allgather of equal-sized blobs moves every
// island's archive. Empty slots carry fitness -inf and are rejected by the
// merge insert like any non-finite fitness (qd_optimizer.cpp:283).
// Layout (all sections 8-byte aligned): fitness, lambda_o, lambda_b (f64[S]),
// worst_val (f64[S*wk]), genome (i32[S*ns]), lambda_c, lambda_c0, lambda_d,
// lambda_s, lambda_r, worst_n (i32[S]), worst_idx (i32[S*wk]).
struct BlobLayout {
  size_t fit, lo, lb, wval, gen, lc, lc0, ld, ls, lr, wn, widx, total;
  __host__ __device__ static size_t al(size_t x) { return (x + 7) & ~size_t{7}; }
  __host__ __device__ BlobLayout(int slots, int ns, int wk) {
    const size_t S = static_cast<size_t>(slots);
    size_t o = 0;
    fit = o, o += al(S * 8);
    lo = o, o += al(S * 8);
    lb = o, o += al(S * 8);
    wval = o, o += al(S * wk * 8);
    gen = o, o += al(S * ns * 4);
    lc = o, o += al(S * 4);
    lc0 = o, o += al(S * 4);
    ld = o, o += al(S * 4);
    ls = o, o += al(S * 4);
    lr = o, o += al(S * 4);
    wn = o, o += al(S * 4);
    widx = o, o += al(S * wk * 4);
    total = o;
  }
};

// Merge-side buffers: the gathered islands unpacked as one insert batch.
struct MergeBuffers {
  int capacity = 0;  // lanes
  int* genomes = nullptr;
  Scores sc{};
  int* lane_cell = nullptr;
  uint8_t* inserted = nullptr;
};

// Kernels launched by the context (capi.cu).
void launch_archive_reset(const QdState& q, cudaStream_t s);
void launch_offspring(const DevGrid& g, const QdState& q, int* genomes, cudaStream_t s);
// Returns the number of kernels launched.
int launch_insert(const QdState& q, const int* genomes, const Scores& sc, int n, int worst_k, bool advance_iter,
                  cudaStream_t s);
// Island exchange: pack this archive into `blob`
// (BlobLayout bytes); merge = clear the cells and insert the n_islands blobs in
// (island, cell, position) order with the Repertoire::insert semantics, so
// every island that merges the same gathered blobs holds the same archive.
void launch_archive_pack(const QdState& q, void* blob, cudaStream_t s);
int launch_archive_merge(const QdState& q, const void* blobs, int n_islands, MergeBuffers& m, cudaStream_t s);
// Score slices of a batch (lanes [lo, lo + n)) <-> BlobLayout(n) blobs, for
// the batch-sharded generation (each rank evaluates a slice, slices are
// allgathered, every rank inserts the whole batch).
void launch_scores_pack(const QdState& q, const int* genomes, const Scores& sc, int lo, int n, void* blob,
                        cudaStream_t s);
void launch_scores_unpack(const QdState& q, const void* blob, int lo, int n, const Scores& sc, cudaStream_t s);
void launch_mutate_lanes(const DevGrid& g, const QdState& q, const int* parents, const unsigned long long* seeds, int n,
                         int* children, cudaStream_t s);
void launch_crossover_lanes(const DevGrid& g, const QdState& q, const int* p1, const int* p2,
                            const unsigned long long* seeds, int n, int* children, cudaStream_t s);

}  // namespace tgb
