// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A C++20 restatement of the reference's DC N-1 MapElites path
// (/root/reference/proj, "topopt"), written without Eigen so it builds in this
// image. It is the checker for the B200 product and the CPU baseline timed by
// bench.py (cpu_baseline.kind = "port"). Nothing in paper_2605_10128_b200/
// links or calls it; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it.
//
// Parity pinning: the reference cannot be compiled here (Eigen3 and the vendored
// json/doctest headers are absent, proj/CMakeLists.txt:12-21), so the oracle is
// pinned by the reference's own known-answer tests and rebuild oracles, ported
// in oracle/kats/kats.cpp and run by tests/test_oracle_kats.py.
//
// File map (reference file:line each part restates):
//   grid.cpp      grid_model.cpp:1-512, graph_utils.cpp:1-118
//   importer.cpp  importer.cpp:1-481
//   genome.cpp    genome.cpp:1-112
//   dc.cpp        dc_engine.cpp:1-470  (numerics substituted: see linalg.hpp)
//   qd.cpp        qd_optimizer.cpp:1-419, rng.hpp:1-23
//   fixtures.cpp  tests/helpers.hpp:1-583 (the reference's test oracles)
#pragma once

#include <array>
#include <atomic>
#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "linalg.hpp"

namespace oracle {

// ---- errors.hpp:9-34 --------------------------------------------------------
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValidationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IslandedContingency : std::runtime_error { using std::runtime_error::runtime_error; };
struct SingularSystem : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---- rng.hpp:9-21 -----------------------------------------------------------
inline std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t a, std::uint64_t b = 0) {
  return mix64(mix64(master ^ mix64(a)) ^ mix64(b + 0x632be59bd9b4e019ull));
}
using Rng = std::mt19937_64;

// ---- graph_utils.hpp:11-27 --------------------------------------------------
struct GraphEdge {
  int from = -1;
  int to = -1;
  bool active = true;
};
bool graph_connected(int n_nodes, const std::vector<GraphEdge>& edges,
                     const std::vector<int>& must_reach = {});
bool graph_connected_without(int n_nodes, const std::vector<GraphEdge>& edges,
                             const std::vector<int>& removed,
                             const std::vector<int>& must_reach = {});
std::vector<int> graph_bridges(int n_nodes, const std::vector<GraphEdge>& edges);

// ---- grid_model.hpp:16-139 --------------------------------------------------
enum class InjectionKind { Generator, Load };
struct Node {
  std::string id;
  std::string substation;
  double shunt_b_pu = 0.0;
};
struct Branch {
  std::string id;
  int from = -1, to = -1;
  double reactance = 0.0, resistance = 0.0, charging_b = 0.0, tap = 1.0;
  double flow_limit = 0.0;
  bool in_service = true;
};
struct Injection {
  std::string id;
  int node = -1;
  double p_mw = 0.0, q_mvar = 0.0;
  InjectionKind kind = InjectionKind::Load;
  std::optional<double> v_setpoint_pu;
  double net_mw() const { return kind == InjectionKind::Generator ? p_mw : -p_mw; }
};
struct ContingencyCase {
  std::string id;
  std::vector<int> branches;
  std::vector<int> injections;
};
struct BusbarOutage {
  std::string id;
  int substation = -1;
  std::string busbar;
};
enum class TerminalKind { BranchFrom, BranchTo, InjectionTerminal };
struct Terminal {
  std::string element;
  TerminalKind kind = TerminalKind::InjectionTerminal;
  int element_index = -1;
  std::vector<std::string> reachable;
  std::string default_busbar;
};
struct SubstationDetail {
  int node = -1;
  std::vector<std::string> busbars;
  std::vector<std::pair<std::string, std::string>> couplers;
  std::vector<Terminal> terminals;
  int busbar_index(const std::string& b) const;
};

class GridModel {
 public:
  std::vector<Node> nodes;
  std::vector<Branch> branches;
  std::vector<Injection> injections;
  std::vector<ContingencyCase> contingencies;
  std::vector<BusbarOutage> busbar_outages;
  std::vector<SubstationDetail> substations;
  int slack = -1;

  int node_index(const std::string& id) const;
  int branch_index(const std::string& id) const;
  int injection_index(const std::string& id) const;
  const std::vector<int>& branches_at(int node) const { return incident_[node]; }
  int substation_at(int node) const { return station_of_node_[node]; }
  std::vector<int> busbar_group(const SubstationDetail& detail, int busbar,
                                const std::vector<int>& open_couplers) const;
  std::vector<int> implied_branches(const BusbarOutage& outage) const;
  std::vector<int> implied_branches(const BusbarOutage& outage,
                                    const std::vector<int>& terminal_busbars,
                                    const std::vector<int>& open_couplers) const;
  void rebuild_indices();
  void validate() const;

 private:
  std::unordered_map<std::string, int> node_lookup_, branch_lookup_, injection_lookup_;
  std::vector<std::vector<int>> incident_;
  std::vector<int> station_of_node_;
};

GridModel grid_from_json_text(const std::string& text);
GridModel load_grid(const std::string& path);
std::string grid_to_json_text(const GridModel& grid);
std::uint64_t grid_content_hash(const GridModel& grid);
Vec base_power_vector(const GridModel& grid);

// ---- importer.hpp:19-95 -----------------------------------------------------
struct Action {
  int id = -1;
  int substation = -1;
  std::vector<char> group;
  std::vector<int> busbar_assignment;
  std::vector<int> open_couplers;
  int reassignment_distance = 0;
};
struct ActionSet {
  std::vector<Action> actions;
  std::vector<int> disconnectables;
  std::map<int, std::pair<int, int>> station_ranges;
  int substation_of(int action_id) const { return actions[action_id].substation; }
};
struct DcGraph {
  int n_nodes = 0;
  int slack = -1;
  struct Edge {
    int from, to;
    double susceptance;
    bool in_service;
  };
  std::vector<Edge> edges;
};
struct PTDFMatrix {
  Mat sensitivities;  // E x N, slack column zero
  int slack = -1;
};
struct EnumerationConfig {
  std::int64_t cap = std::int64_t{1} << 23;
  std::uint64_t seed = 0;
};
DcGraph dc_graph_from_grid(const GridModel& grid);
std::vector<int> find_bridges(const DcGraph& graph);
std::vector<int> enumerate_disconnectables(const GridModel& grid);
std::vector<Action> enumerate_station_actions(const GridModel& grid, int substation,
                                              const EnumerationConfig& cfg = {});
bool validate_action_islanding(const GridModel& grid, const Action& action);
ActionSet build_action_set(const GridModel& grid, const EnumerationConfig& cfg = {});
PTDFMatrix build_ptdf(const DcGraph& graph);
PTDFMatrix build_ptdf(const GridModel& grid);
std::string action_set_to_json_text(const ActionSet& actions, const GridModel& grid);
std::optional<ActionSet> action_set_from_json_text(const GridModel& grid, const std::string& text);

// ---- genome.hpp:13-58 -------------------------------------------------------
struct Genome {
  std::vector<int> action_slots;
  std::vector<int> disconnection_slots;
  static Genome empty(int n_a, int n_d) {
    return Genome{std::vector<int>(n_a, -1), std::vector<int>(n_d, -1)};
  }
  bool is_empty() const;
  int split_count() const;
  int disconnection_count() const;
  std::vector<int> action_ids() const;
  std::vector<int> disconnection_ids() const;
  std::string canonical_key() const;
};
bool genome_valid(const Genome& g, const ActionSet& actions);
int genome_distance(const Genome& a, const Genome& b);
struct AppliedTopology {
  std::vector<std::pair<int, int>> endpoints;
  std::vector<char> removed;
  std::vector<int> injection_node;
  std::vector<int> action_of_station;
  int n_new_nodes = 0;
};
AppliedTopology apply_genome(const GridModel& grid, const ActionSet& actions, const Genome& genome);

// ---- dc_engine.hpp:16-150 ---------------------------------------------------
struct DcConfig {
  double islanding_penalty_mw = 10000.0;
  int worst_k = 20;
  double weight_c0 = 200.0;
  double weight_c = 50.0;
  int fitness_variant = 1;
  int threads = 0;
};
struct ScoreVector {
  double lambda_o = 0.0;
  int lambda_c = 0;
  int lambda_c0 = 0;
  double lambda_b = 0.0;
  int lambda_d = 0, lambda_s = 0, lambda_r = 0;
  double fitness = 0.0;
  bool islanded = false;
  std::vector<std::pair<int, double>> worst_contingencies;
  static constexpr double kIslandedFitness = -std::numeric_limits<double>::infinity();
};
struct FlowResult {
  Vec base, max_contingency, max_busbar;
  std::vector<double> outage_energy;
  int islanded_outages = 0;
  int islanded_busbar_outages = 0;
};

class DcContext;

class FlowOperator {
 public:
  bool islanded() const { return islanded_; }
  int extra_nodes() const { return n_new_; }
  Vec flows(const Vec& p_full) const;
  const Vec& base_flows() const { return base_flows_; }
  int rank() const { return m_; }

 private:
  friend class DcContext;
  const DcContext* ctx_ = nullptr;
  bool islanded_ = false;
  int n_new_ = 0;
  std::vector<std::pair<int, int>> endpoints_;
  std::vector<char> removed_;
  std::vector<int> injection_node_;
  std::vector<int> action_of_station_;
  int m_ = 0;
  std::vector<std::pair<int, int>> pairs_;  // reduced endpoint indices, -1 = ground/slack
  Mat gain_;                                // X_aug * U  (dim x m)
  FullPivLU cap_;                           // capacitance, threshold 1e-10
  Vec base_theta_, base_flows_;

  int reduced(int full_node) const;
  Vec solve_sparse(const std::vector<std::pair<int, double>>& rhs) const;
  Vec apply_correction(Vec y) const;
  Vec flows_from_theta(const Vec& theta) const;
};

class DcContext {
 public:
  DcContext(const GridModel& grid, const ActionSet& actions, DcConfig config = {});
  const GridModel& grid() const { return *grid_; }
  const ActionSet& actions() const { return *actions_; }
  const DcConfig& config() const { return config_; }
  FlowOperator apply_topology(const Genome& genome) const;
  FlowResult screen_contingencies(const FlowOperator& op) const;
  ScoreVector compute_scores(const FlowResult& flows, const Genome& genome) const;
  ScoreVector evaluate(const Genome& genome) const;
  // evaluate + the FlowResult it was scored from (empty FlowResult when islanded)
  ScoreVector evaluate_with_flows(const Genome& genome, FlowResult* flows) const;
  std::vector<ScoreVector> evaluate_batch(const std::vector<Genome>& genomes, int batch_size) const;
  const ScoreVector& pre_optimization_score() const { return pre_score_; }
  double lambda_b_pre() const { return lambda_b_pre_; }

 private:
  friend class FlowOperator;
  FlowOperator build_operator(std::vector<std::pair<int, int>> endpoints, std::vector<char> removed,
                              std::vector<int> injection_node, std::vector<int> action_of_station,
                              int n_new, const std::vector<char>& omit_injection) const;
  struct ActionTopology {
    int station_node = -1;
    std::vector<std::vector<int>> implied_by_busbar;
  };
  const GridModel* grid_;
  const ActionSet* actions_;
  DcConfig config_;
  int n_nodes_ = 0, n_red_ = 0;
  std::vector<int> reduced_;
  Mat x_inv_;
  Vec p_base_, y_base_, limits_;
  std::vector<double> susceptance_;
  std::vector<char> in_service_;
  std::vector<ActionTopology> action_topo_;
  std::vector<std::vector<int>> default_implied_;
  double lambda_b_pre_ = 0.0;
  ScoreVector pre_score_;
};

// ---- qd_optimizer.hpp:15-118 ------------------------------------------------
struct QdConfig {
  int n_a = 3;
  int n_d = 2;
  int batch_size = 64;
  int iters_per_epoch = 500;
  int cell_capacity = 4;
  double mutation_mean = 2.0;
  std::array<double, 4> p_action{0.2, 0.2, 0.5, 0.1};
  std::array<double, 4> p_disc{0.25, 0.25, 0.5, 0.0};
  double p_crossover_parent1 = 0.75;
  int d_max = 2, s_max = 3, r_max = 45;
  std::uint64_t seed = 1;
  std::int64_t max_evaluations = -1;
  double max_seconds = -1.0;
};
inline int cell_count(const QdConfig& c) { return (c.d_max + 1) * (c.s_max + 1) * (c.r_max + 1); }
int descriptor_to_cell(int lambda_d, int lambda_s, int lambda_r, const QdConfig& cfg);
enum class MutationOp { Add, Remove, Change, Identity };
struct MutationTrace {
  std::vector<MutationOp> action_ops, disconnection_ops;
};
Genome mutate(const Genome& g, const ActionSet& actions, const QdConfig& cfg, Rng& rng,
              MutationTrace* trace = nullptr);
Genome crossover(const Genome& g1, const Genome& g2, const ActionSet& actions, const QdConfig& cfg,
                 Rng& rng);
struct RepertoireEntry {
  Genome genome;
  ScoreVector score;
  std::string key;
};
class Repertoire {
 public:
  explicit Repertoire(const QdConfig& cfg);
  bool insert(const Genome& genome, const ScoreVector& score);
  int total_size() const { return total_; }
  const RepertoireEntry& member(int flat_index) const;
  const std::vector<RepertoireEntry>& cell(int i) const { return cells_[i]; }
  int n_cells() const { return static_cast<int>(cells_.size()); }
  double best_fitness() const;
  std::vector<double> per_cell_best() const;

 private:
  QdConfig cfg_;
  std::vector<std::vector<RepertoireEntry>> cells_;
  int total_ = 0;
  mutable std::vector<std::pair<int, int>> flat_;
  mutable bool flat_dirty_ = true;
};
struct SnapshotEntry {
  int cell = 0;
  Genome genome;
  ScoreVector score;
};
struct RepertoireSnapshot {
  int epoch = 0;
  std::int64_t evaluations = 0;
  double best_fitness = 0.0;
  bool final = false;
  std::vector<SnapshotEntry> entries;
};
RepertoireSnapshot make_snapshot(const Repertoire& rep, int epoch, std::int64_t evaluations, bool final);
using SnapshotSink = std::function<void(RepertoireSnapshot)>;
struct OptimizerStats {
  std::int64_t evaluations = 0;
  int epochs = 0;
  std::vector<std::pair<std::int64_t, double>> fitness_trace;
};
struct OptimizerResult {
  Repertoire repertoire;
  OptimizerStats stats;
};
// Test hook (not in the reference): called after each iteration's evaluation
// with the iteration index, offspring and their scores.
using IterationTrace = std::function<void(std::int64_t, const std::vector<Genome>&, const std::vector<ScoreVector>&)>;
OptimizerResult run_optimizer(const DcContext& ctx, const QdConfig& cfg, const SnapshotSink& sink,
                              const std::atomic<bool>* stop = nullptr, const IterationTrace* trace = nullptr);

}  // namespace oracle

// ---- ac_validator.hpp:18-140 (restated in ac.cpp) ----------------------------
namespace oracle {

struct AcConfig {
  double tolerance_pu = 1e-6;
  int max_iterations = 30;
  int worst_k_nonconverged = 2;
  double nonconverged_fraction = 0.05;
  int similarity_distance = 1;
  double dominance_fitness_frac = 0.01;
  double improvement_threshold_frac = 0.05;
};

struct AcCaseResult {
  bool converged = false;
  int iterations = 0;
  Vec loading_mva;  // per branch, MVA (max of both ends); zero unless converged
  Vec vm_pu, va_rad;  // per bus (base nodes, then split sections)
};

class AcNetwork {
 public:
  AcNetwork(const GridModel& grid, const AppliedTopology& topology, AcConfig config = {});
  AcCaseResult run_case(int contingency) const;  // -1 = base case
  double overload_energy(const AcCaseResult& r) const;
  int critical_count(const AcCaseResult& r) const;

 private:
  const GridModel* grid_;
  AppliedTopology topo_;
  AcConfig cfg_;
  int n_buses_ = 0;
  AcCaseResult solve(const std::vector<char>& branch_out, const std::vector<char>& injection_out) const;
};

AcCaseResult ac_power_flow(const GridModel& grid, const AppliedTopology& topology, AcConfig config = {});

enum class RejectionReason {
  None, Nonconvergence, OverloadNotImproved, CriticalCountIncreased,
  EliminatedSimilar, EliminatedDominated, EliminatedBelowThreshold,
};
std::string to_string(RejectionReason reason);
enum class ValidationStage { None, WorstK, FullN1 };

struct ValidationRecord {
  Genome genome;
  ScoreVector dc_score;
  ValidationStage stage = ValidationStage::None;
  bool accepted = false;
  RejectionReason reason = RejectionReason::None;
  double ac_lambda_o = 0.0;
};
struct Candidate {
  Genome genome;
  ScoreVector dc_score;
};
struct EliminationOutcome {
  std::vector<int> queue;
  std::vector<std::pair<int, RejectionReason>> pruned;
};

class AcValidator {
 public:
  AcValidator(const GridModel& grid, const ActionSet& actions, const DcContext& dc, AcConfig config = {});
  const AcConfig& config() const { return cfg_; }
  double baseline_lambda_o() const { return base_lambda_o_; }
  int baseline_critical_count() const { return base_critical_; }
  bool baseline_base_converged() const { return base_converged_; }
  double baseline_base_energy() const { return base_energy_; }
  const std::vector<char>& baseline_case_converged() const { return case_converged_; }
  const std::vector<double>& baseline_case_energy() const { return case_energy_; }
  EliminationOutcome eliminate(const std::vector<Candidate>& candidates) const;
  RejectionReason worst_k_check(const Genome& genome, const ScoreVector& dc_score) const;
  ValidationRecord full_validation(const Genome& genome, const ScoreVector& dc_score) const;
  ValidationRecord validate(const Candidate& candidate);
  void record_elimination(const Candidate& candidate, RejectionReason reason);
  const std::vector<ValidationRecord>& records() const { return records_; }

 private:
  const GridModel* grid_;
  const ActionSet* actions_;
  AcConfig cfg_;
  double pre_fitness_ = 0.0;
  double base_lambda_o_ = 0.0;
  int base_critical_ = 0;
  bool base_converged_ = false;
  double base_energy_ = 0.0;
  std::vector<char> case_converged_;
  std::vector<double> case_energy_;
  struct Validated {
    Genome genome;
    int swd = 0;
    double fitness = 0.0;
  };
  std::vector<Validated> validated_;
  std::vector<ValidationRecord> records_;
};

std::string record_to_json(const ValidationRecord& record, const GridModel& grid, const ActionSet& actions);

}  // namespace oracle
