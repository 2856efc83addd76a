// MapElites device state: archive, lane RNG replay, mutation / crossover,
// sequential-equivalent insert (qd_optimizer.cpp:12-417).
#pragma once

#include "engine.cuh"

namespace tgb {

constexpr int kMaxCellCap = 16;  // QdConfig::cell_capacity supported on the device

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

// Kernels launched by the context (capi.cu).
void launch_archive_reset(const QdState& q, cudaStream_t s);
void launch_offspring(const DevGrid& g, const QdState& q, int* genomes, cudaStream_t s);
// Returns the number of kernels launched.
int launch_insert(const QdState& q, const int* genomes, const Scores& sc, int n, int worst_k, bool advance_iter,
                  cudaStream_t s);
void launch_mutate_lanes(const DevGrid& g, const QdState& q, const int* parents, const unsigned long long* seeds, int n,
                         int* children, cudaStream_t s);
void launch_crossover_lanes(const DevGrid& g, const QdState& q, const int* p1, const int* p2,
                            const unsigned long long* seeds, int n, int* children, cudaStream_t s);

}  // namespace tgb
