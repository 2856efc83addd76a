// Batched AC Newton-Raphson validation on the device.
//
// Replaces the reference's per-case CPU solve, AcNetwork::run_case / solve
// (ac_validator.cpp:26-272), and the case loops of AcValidator's baseline,
// worst_k_check and full_validation (ac_validator.cpp:313-473): every
// (genome, contingency) case of a validation batch is one CTA that runs the
// reference's algorithm — slack reachability, bus numbering, Ybus, polar
// Newton-Raphson from a flat start with a dense Jacobian solved by LU with
// partial pivoting, branch loadings — with its working set in shared memory
// (small networks) or in a per-CTA global scratch slot (large networks).
// Tables are in the grid's own branch order (not the DC engine's internal
// sweep order).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tgb {

struct AcGrid {
  int N, E, I, K, slack;
  const int* br_from;        // [E]
  const int* br_to;          // [E]
  const uint8_t* br_on;      // [E] in service
  const double* br_lim;      // [E] MW (MVA in the AC check, ac_validator.cpp:277)
  const double* br_r;        // [E] p.u.
  const double* br_x;        // [E] p.u.
  const double* br_bc;       // [E] total line charging p.u.
  const double* br_tap;      // [E] off-nominal ratio, from side
  const double* node_shunt;  // [N] shunt susceptance p.u.
  const int* node_ptr;       // [N+1] CSR of every branch at each of its ends (grid order)
  const int* node_br;
  const int* inj_node;       // [I]
  const double* inj_p;       // [I] MW
  const double* inj_q;       // [I] Mvar
  const double* inj_vset;    // [I] voltage setpoint p.u.
  const uint8_t* inj_gen;    // [I] generator (else load)
  const uint8_t* inj_has_vset;  // [I]
  const int* cont_br_ptr;    // [K+1] CSR of contingency branches
  const int* cont_br;
  const int* cont_inj_ptr;   // [K+1] CSR of contingency injections
  const int* cont_inj;
  const int* st_node;        // [S] the station's node
  const int* st_term_ptr;    // [S+1] station terminals
  const int* term_kind;      // 0 branch from-end, 1 branch to-end, 2 injection
  const int* term_elem;
  const int* act_station;    // [A]
  const int* act_group_ptr;  // [A+1]
  const uint8_t* act_group;  // per terminal of the action's station: 1 = moves to the new node
  const int* disc;           // [D] branch of each disconnectable
};

// Applied topologies of a genome batch (apply_genome, genome.cpp:76-110).
struct AcTopo {
  int* from;         // [G][E]
  int* to;           // [G][E]
  uint8_t* removed;  // [G][E]
  int* inj_node;     // [G][I]
  int* n_new;        // [G]
  int* split_node;   // [G][split_stride] base node of each split section (slot order)
  int split_stride;
};

// One validation batch of cases (genome index, contingency index or -1 for
// the base case). Optional outputs may be null.
struct AcCases {
  const int* genome;
  const int* cont;
  int n;
  uint8_t* converged;        // [n]
  int* iterations;           // [n]
  double* energy;            // [n] overload_energy (ac_validator.cpp:274-279), 0 unless converged
  int* critical;             // [n] critical_count (ac_validator.cpp:281-286), 0 unless converged
  double* loading;           // [n][E] MVA
  double* vm;                // [n][vm_stride]
  double* va;                // [n][vm_stride]
  int vm_stride;
  const uint8_t* fold_case;  // [n] the case enters the per-genome fold below (contingency cases)
  unsigned long long* fold;  // [G][E] max loading over converged fold cases (bits of non-negative doubles)
  int* nonconverged;         // [G] fold cases that did not converge
};

struct AcSolver {
  double tol;
  int max_iter;
  int n_bus;        // N + max new nodes per genome
  int nu;           // max unknowns, 2 (n_bus - 1)
  int in_smem;      // workspace in dynamic shared memory (else scratch + blockIdx.x * ws_bytes)
  size_t ws_bytes;  // per-CTA workspace
  unsigned char* scratch;
  unsigned* next_case;  // scratch path: dynamic case counter (zeroed per launch)
};

size_t ac_workspace_bytes(int n_bus, int nu, int E);
int ac_threads(int nu);
void ac_launch_topo(const AcGrid& g, const int* genomes, int n_genomes, int n_a, int n_d, const AcTopo& t,
                    cudaStream_t s);
void ac_launch_cases(const AcGrid& g, const AcTopo& t, const AcCases& c, const AcSolver& sv, int ctas,
                     cudaStream_t s);
// lambda_o / critical count per genome from the folded maxima
// (ac_validator.cpp:451-463, in branch order)
void ac_launch_fold_finish(const AcGrid& g, const unsigned long long* fold, int n_genomes, double* lambda_o,
                           int* critical, cudaStream_t s);

}  // namespace tgb
