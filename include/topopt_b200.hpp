/*
 * topopt_b200.hpp — C++ host API of the B200 DC N-1 MapElites engine.
 *
 * Header-only C++20 layer over the C ABI (topopt_b200.h) that keeps the
 * reference's C++ surface for the hot path, names and semantics included, so
 * a C++ caller of arxiv/paper_2605_10128's `topopt` library switches by
 * changing the namespace (`topopt::` -> `topopt::b200::`):
 *
 *   errors.hpp:9-34          ParseError ... IoError (+ CudaError, CapacityError)
 *   grid_model.hpp:130-139   load_grid, grid_from_json_text, grid_to_json_text, grid_content_hash
 *   importer.hpp:68-94       EnumerationConfig, build_action_set, save/load_action_set
 *   genome.hpp:13-46         Genome (canonical_key, counts), genome_valid, genome_distance
 *   dc_engine.hpp:16-150     DcConfig, ScoreVector, FlowResult, DcContext::{evaluate,
 *                            evaluate_batch, evaluate_flows, pre_optimization_score, lambda_b_pre}
 *   ac_validator.hpp:18-140  AcConfig, AcCaseResult, RejectionReason, ValidationRecord, Candidate,
 *                            EliminationOutcome, AcValidator (GPU batches), record_to_json
 *   qd_optimizer.hpp:15-118  QdConfig, cell_count, descriptor_to_cell, RepertoireEntry,
 *                            Repertoire (read side), SnapshotEntry, RepertoireSnapshot,
 *                            SnapshotSink, OptimizerStats, OptimizerResult, run_optimizer
 *
 * Types are Eigen-free (FlowResult vectors are std::vector<double>). The
 * engine has no CPU path: every evaluation runs on the GPU behind the C ABI;
 * a missing device surfaces as CudaError. integration/dc_engine_b200.hpp
 * adapts the reference's own types (GridModel, ActionSet, ...) to the same
 * C ABI for callers that keep the reference's import step.
 */
#ifndef TOPOPT_B200_HPP
#define TOPOPT_B200_HPP

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "topopt_b200.h"

namespace topopt::b200 {

// ---- errors.hpp:9-34 --------------------------------------------------------
struct ParseError : std::runtime_error {
  explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
struct IslandedContingency : std::runtime_error {
  explicit IslandedContingency(const std::string& m) : std::runtime_error(m) {}
};
struct SingularSystem : std::runtime_error {
  explicit SingularSystem(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
// No reference counterpart: a CUDA failure (no device, launch error) and a
// candidate beyond a compile-time capacity of the engine (never a silent
// truncation).
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct CapacityError : std::runtime_error {
  explicit CapacityError(const std::string& m) : std::runtime_error(m) {}
};

// Every tg_status maps to its own exception type.
[[noreturn]] inline void throw_status(tg_status s) {
  const std::string msg = tg_last_error();
  switch (s) {
    case TG_PARSE_ERROR: throw ParseError(msg);
    case TG_VALIDATION_ERROR: throw ValidationError(msg);
    case TG_ISLANDED_CONTINGENCY: throw IslandedContingency(msg);
    case TG_SINGULAR_SYSTEM: throw SingularSystem(msg);
    case TG_CONFIG_ERROR: throw ConfigError(msg);
    case TG_IO_ERROR: throw IoError(msg);
    case TG_CUDA_ERROR: throw CudaError(msg);
    case TG_CAPACITY_ERROR: throw CapacityError(msg);
    default: throw std::runtime_error("topopt_b200: unknown status " + std::to_string(int(s)) + ": " + msg);
  }
}
inline void check(tg_status s) {
  if (s != TG_OK) throw_status(s);
}

namespace detail {
inline std::string take_string(char* p) {
  std::string s(p ? p : "");
  tg_free(p);
  return s;
}
}  // namespace detail

// ---- grid_model.hpp:80-139 ---------------------------------------------------
class GridModel {
 public:
  explicit GridModel(tg_grid* h) : h_(h, &tg_grid_destroy) { check(tg_grid_describe(h, &desc_)); }
  const tg_grid_desc& desc() const { return desc_; }
  tg_grid* handle() const { return h_.get(); }
  int n_nodes() const { return desc_.n_nodes; }
  int n_branches() const { return desc_.n_branches; }
  int n_injections() const { return desc_.n_injections; }
  int n_contingencies() const { return desc_.n_contingencies; }
  int n_busbar_outages() const { return desc_.n_busbar_outages; }
  int n_substations() const { return desc_.n_substations; }
  int slack() const { return desc_.slack; }

 private:
  std::shared_ptr<tg_grid> h_;
  tg_grid_desc desc_{};
};

inline GridModel grid_from_json_text(const std::string& text) {
  tg_grid* h = nullptr;
  check(tg_grid_from_json(text.data(), text.size(), &h));
  return GridModel(h);
}
inline GridModel load_grid(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open grid file '" + path.string() + "'");
  std::stringstream buf;
  buf << in.rdbuf();
  return grid_from_json_text(buf.str());
}
inline std::string grid_to_json_text(const GridModel& g) {
  char* p = nullptr;
  check(tg_grid_to_json(g.handle(), &p));
  return detail::take_string(p);
}
inline std::uint64_t grid_content_hash(const GridModel& g) {
  std::uint64_t h = 0;
  check(tg_grid_content_hash(g.handle(), &h));
  return h;
}

// ---- importer.hpp:19-94 ------------------------------------------------------
struct EnumerationConfig {
  std::int64_t cap = std::int64_t{1} << 23;
  std::uint64_t seed = 0;
  int device = -1;  // >= 0: islanding validation of the candidate splits on that GPU (same ids)
};

class ActionSet {
 public:
  ActionSet(tg_actionset* h, const GridModel& g) : h_(h, &tg_actionset_destroy), grid_(g) {
    check(tg_actionset_describe(h, g.handle(), &desc_));
  }
  const tg_actionset_desc& desc() const { return desc_; }
  tg_actionset* handle() const { return h_.get(); }
  int n_actions() const { return desc_.n_actions; }
  int n_disconnectables() const { return desc_.n_disconnectables; }
  int substation_of(int action_id) const { return desc_.action_substation[action_id]; }
  int disconnectable(int d) const { return desc_.disconnectables[d]; }
  int reassignment_distance(int action_id) const { return desc_.action_lambda_r[action_id]; }

 private:
  std::shared_ptr<tg_actionset> h_;
  GridModel grid_;  // keeps the grid alive (the description points into it)
  tg_actionset_desc desc_{};
};

inline ActionSet build_action_set(const GridModel& g, const EnumerationConfig& cfg = {}) {
  tg_actionset* h = nullptr;
  if (cfg.device >= 0)
    check(tg_actionset_build_device(g.handle(), cfg.seed, cfg.cap, cfg.device, &h));
  else
    check(tg_actionset_build(g.handle(), cfg.seed, cfg.cap, &h));
  return ActionSet(h, g);
}
inline void save_action_set(const ActionSet& a, const GridModel& g, const std::filesystem::path& path) {
  char* p = nullptr;
  check(tg_actionset_to_json(a.handle(), g.handle(), &p));
  const std::string text = detail::take_string(p);
  std::ofstream out(path);
  if (!out) throw IoError("cannot write action cache '" + path.string() + "'");
  out << text << "\n";
}
// Nothing on a missing file or a key (grid_content_hash) / id mismatch,
// importer.cpp:432-479.
inline std::optional<ActionSet> load_action_set(const GridModel& g, const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) return std::nullopt;
  std::stringstream buf;
  buf << in.rdbuf();
  const std::string text = buf.str();
  tg_actionset* h = nullptr;
  if (tg_actionset_from_json(g.handle(), text.data(), text.size(), &h) != TG_OK) return std::nullopt;
  return ActionSet(h, g);
}

// ---- genome.hpp:13-46 / genome.cpp:10-74 ------------------------------------
struct Genome {
  std::vector<int> action_slots;
  std::vector<int> disconnection_slots;

  static Genome empty(int n_a, int n_d) { return Genome{std::vector<int>(n_a, -1), std::vector<int>(n_d, -1)}; }
  int split_count() const {
    return static_cast<int>(std::count_if(action_slots.begin(), action_slots.end(), [](int a) { return a >= 0; }));
  }
  int disconnection_count() const {
    return static_cast<int>(
        std::count_if(disconnection_slots.begin(), disconnection_slots.end(), [](int d) { return d >= 0; }));
  }
  bool is_empty() const { return split_count() == 0 && disconnection_count() == 0; }
  std::vector<int> action_ids() const { return sorted_ids(action_slots); }
  std::vector<int> disconnection_ids() const { return sorted_ids(disconnection_slots); }
  std::string canonical_key() const {
    std::string key = "a:";
    for (int a : action_ids()) key += std::to_string(a) + ",";
    key += "d:";
    for (int d : disconnection_ids()) key += std::to_string(d) + ",";
    return key;
  }
  bool operator==(const Genome& o) const { return canonical_key() == o.canonical_key(); }

 private:
  static std::vector<int> sorted_ids(const std::vector<int>& v) {
    std::vector<int> ids;
    for (int x : v)
      if (x >= 0) ids.push_back(x);
    std::sort(ids.begin(), ids.end());
    return ids;
  }
};

inline bool genome_valid(const Genome& g, const ActionSet& a) {
  std::vector<int> subs, brs;
  for (int x : g.action_slots) {
    if (x < 0) continue;
    if (x >= a.n_actions()) return false;
    if (std::find(subs.begin(), subs.end(), a.substation_of(x)) != subs.end()) return false;
    subs.push_back(a.substation_of(x));
  }
  for (int d : g.disconnection_slots) {
    if (d < 0) continue;
    if (d >= a.n_disconnectables()) return false;
    if (std::find(brs.begin(), brs.end(), a.disconnectable(d)) != brs.end()) return false;
    brs.push_back(a.disconnectable(d));
  }
  return true;
}

inline int genome_distance(const Genome& a, const Genome& b) {
  auto sym = [](const std::vector<int>& x, const std::vector<int>& y) {
    std::vector<int> out;
    std::set_symmetric_difference(x.begin(), x.end(), y.begin(), y.end(), std::back_inserter(out));
    return static_cast<int>(out.size());
  };
  return sym(a.action_ids(), b.action_ids()) + sym(a.disconnection_ids(), b.disconnection_ids());
}

// ---- dc_engine.hpp:16-48 -----------------------------------------------------
struct DcConfig {
  double islanding_penalty_mw = 10000.0;
  int worst_k = 20;
  double weight_c0 = 200.0;
  double weight_c = 50.0;
  int fitness_variant = 1;
  int threads = 0;  // accepted and ignored: the batch runs on the GPU
};

struct ScoreVector {
  double lambda_o = 0.0;
  int lambda_c = 0;
  int lambda_c0 = 0;
  double lambda_b = 0.0;
  int lambda_d = 0;
  int lambda_s = 0;
  int lambda_r = 0;
  double fitness = 0.0;
  bool islanded = false;
  std::vector<std::pair<int, double>> worst_contingencies;
  static constexpr double kIslandedFitness = -std::numeric_limits<double>::infinity();
};

struct FlowResult {
  std::vector<double> base;             // signed N-0 flows, MW
  std::vector<double> max_contingency;  // elementwise max |flow| over outage cases
  std::vector<double> max_busbar;       // elementwise max |flow| over busbar outages
  std::vector<double> outage_energy;    // per contingency, islanding -> penalty
  int islanded_outages = 0;
  int islanded_busbar_outages = 0;
};

namespace detail {
// SoA output buffers of one tg_evaluate_batch call
struct ScoreBuffers {
  std::vector<double> lo, lb, fit, wv;
  std::vector<int32_t> lc, lc0, ld, ls, lr, wi, wn, io, ib;
  std::vector<uint8_t> isl;
  int k;
  ScoreBuffers(int n, int worst_k)
      : lo(n), lb(n), fit(n), wv(static_cast<size_t>(n) * worst_k), lc(n), lc0(n), ld(n), ls(n), lr(n),
        wi(static_cast<size_t>(n) * worst_k), wn(n), io(n), ib(n), isl(n), k(worst_k) {}
  tg_scores view() {
    return tg_scores{lo.data(), lc.data(), lc0.data(), lb.data(), ld.data(), ls.data(), lr.data(),
                     fit.data(), isl.data(), wi.data(), wv.data(), wn.data(), io.data(), ib.data()};
  }
  ScoreVector at(int i) const {
    ScoreVector s{lo[i], lc[i], lc0[i], lb[i], ld[i], ls[i], lr[i], fit[i], isl[i] != 0, {}};
    for (int j = 0; j < wn[i]; ++j)
      s.worst_contingencies.emplace_back(wi[static_cast<size_t>(i) * k + j], wv[static_cast<size_t>(i) * k + j]);
    return s;
  }
};
}  // namespace detail

// dc_engine.hpp:95-150: the device-resident context. Construction builds the
// base factorization and every device table on `device`; it is not copyable
// (one CUDA stream and one set of device buffers per context) and, like the
// reference's immutable context, evaluation does not change it.
class DcContext {
 public:
  DcContext(const GridModel& grid, const ActionSet& actions, DcConfig config = {}, int device = 0)
      : grid_(grid), actions_(actions), config_(config) {
    const tg_dc_config c{config.islanding_penalty_mw, config.worst_k, config.weight_c0, config.weight_c,
                         config.fitness_variant, config.threads};
    tg_context* h = nullptr;
    check(tg_context_create(&grid.desc(), &actions.desc(), &c, device, &h));
    h_ = h;
    detail::ScoreBuffers b(1, config.worst_k);
    tg_scores v = b.view();
    check(tg_pre_score(h_, &v, &lambda_b_pre_));
    pre_score_ = b.at(0);
  }
  ~DcContext() {
    if (h_) tg_context_destroy(h_);
  }
  DcContext(const DcContext&) = delete;
  DcContext& operator=(const DcContext&) = delete;

  const GridModel& grid() const { return grid_; }
  const ActionSet& actions() const { return actions_; }
  const DcConfig& config() const { return config_; }
  tg_context* handle() const { return h_; }

  ScoreVector evaluate(const Genome& g) const { return evaluate_batch({g}, 1).front(); }

  // dc_engine.cpp:439-468. Genomes may mix slot counts like the reference's
  // vector<Genome>: every genome is padded with empty slots (-1) to the
  // batch's widest action / disconnection slot count, which changes neither
  // its topology nor its score (genome.cpp:10-47).
  std::vector<ScoreVector> evaluate_batch(const std::vector<Genome>& gs, int batch_size) const {
    std::vector<ScoreVector> out;
    if (gs.empty()) return out;
    int na = 0, nd = 0;
    const std::vector<int32_t> flat = flatten(gs, na, nd);
    const int n = static_cast<int>(gs.size());
    detail::ScoreBuffers b(n, config_.worst_k);
    tg_scores v = b.view();
    check(tg_evaluate_batch(h_, flat.data(), n, na, nd, std::max(batch_size, n), &v, nullptr, nullptr, nullptr,
                            nullptr));
    out.reserve(n);
    for (int i = 0; i < n; ++i) out.push_back(b.at(i));
    return out;
  }

  // apply_topology + screen_contingencies of one genome (dc_engine.cpp:147-388):
  // the FlowResult, with its score.
  std::pair<FlowResult, ScoreVector> evaluate_flows(const Genome& g) const {
    int na = 0, nd = 0;
    const std::vector<int32_t> flat = flatten({g}, na, nd);
    const int E = grid_.n_branches(), K = grid_.n_contingencies();
    FlowResult f;
    f.base.resize(E);
    f.max_contingency.resize(E);
    f.max_busbar.resize(E);
    f.outage_energy.resize(K);
    detail::ScoreBuffers b(1, config_.worst_k);
    tg_scores v = b.view();
    check(tg_evaluate_batch(h_, flat.data(), 1, na, nd, 1, &v, f.base.data(), f.max_contingency.data(),
                            f.max_busbar.data(), K ? f.outage_energy.data() : nullptr));
    f.islanded_outages = b.io[0];
    f.islanded_busbar_outages = b.ib[0];
    return {std::move(f), b.at(0)};
  }

  const ScoreVector& pre_optimization_score() const { return pre_score_; }
  double lambda_b_pre() const { return lambda_b_pre_; }

 private:
  static std::vector<int32_t> flatten(const std::vector<Genome>& gs, int& na, int& nd) {
    na = nd = 0;
    for (const Genome& g : gs) {
      na = std::max(na, static_cast<int>(g.action_slots.size()));
      nd = std::max(nd, static_cast<int>(g.disconnection_slots.size()));
    }
    std::vector<int32_t> flat;
    flat.reserve(gs.size() * static_cast<size_t>(na + nd));
    for (const Genome& g : gs) {
      flat.insert(flat.end(), g.action_slots.begin(), g.action_slots.end());
      flat.insert(flat.end(), na - g.action_slots.size(), -1);
      flat.insert(flat.end(), g.disconnection_slots.begin(), g.disconnection_slots.end());
      flat.insert(flat.end(), nd - g.disconnection_slots.size(), -1);
    }
    return flat;
  }

  GridModel grid_;
  ActionSet actions_;
  DcConfig config_;
  tg_context* h_ = nullptr;
  ScoreVector pre_score_;
  double lambda_b_pre_ = 0.0;
};


// ---- ac_validator.hpp:18-140 ---------------------------------------------------
// The AC validation stage on the GPU (tg_ac_*): every power flow of a call is
// solved in one batch, one CTA per (genome, contingency) case. eliminate() and
// the validation history are host logic, as in the reference.
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
  std::vector<double> loading_mva;  // per branch, MVA
  std::vector<double> vm_pu, va_rad;  // per bus (base nodes, then split sections)
};

enum class RejectionReason {
  None, Nonconvergence, OverloadNotImproved, CriticalCountIncreased,
  EliminatedSimilar, EliminatedDominated, EliminatedBelowThreshold,
};
inline std::string to_string(RejectionReason r) {
  static const char* names[] = {"none", "nonconvergence", "overload_not_improved", "critical_count_increased",
                                "eliminated_similar", "eliminated_dominated", "eliminated_below_threshold"};
  return names[static_cast<int>(r)];
}
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
  AcValidator(const GridModel& grid, const ActionSet& actions, const DcContext& dc, AcConfig config = {},
              int device = 0)
      : grid_(grid), actions_(actions), config_(config) {
    const tg_ac_config c{config.tolerance_pu, config.max_iterations, config.worst_k_nonconverged,
                         config.nonconverged_fraction, config.similarity_distance, config.dominance_fitness_frac,
                         config.improvement_threshold_frac};
    check(tg_ac_context_create(grid.handle(), actions.handle(), dc.handle(), &c, device, &h_));
    tg_ac_baseline b{};
    check(tg_ac_baseline_get(h_, &b, nullptr, nullptr));
    baseline_lambda_o_ = b.lambda_o;
    baseline_critical_ = b.critical_count;
    pre_fitness_ = dc.pre_optimization_score().fitness;
  }
  ~AcValidator() {
    if (h_) tg_ac_context_destroy(h_);
  }
  AcValidator(const AcValidator&) = delete;
  AcValidator& operator=(const AcValidator&) = delete;

  const AcConfig& config() const { return config_; }
  double baseline_lambda_o() const { return baseline_lambda_o_; }
  int baseline_critical_count() const { return baseline_critical_; }
  tg_ac_context* handle() const { return h_; }

  // AcNetwork(grid, apply_genome(genome)).run_case(k) for every k (-1 = base case)
  std::vector<AcCaseResult> run_cases(const Genome& g, const std::vector<int>& contingencies) const {
    int na = static_cast<int>(g.action_slots.size()), nd = static_cast<int>(g.disconnection_slots.size());
    std::vector<int32_t> flat(g.action_slots.begin(), g.action_slots.end());
    flat.insert(flat.end(), g.disconnection_slots.begin(), g.disconnection_slots.end());
    const int n = static_cast<int>(contingencies.size()), E = grid_.n_branches(), V = grid_.n_nodes() + na;
    std::vector<int32_t> cg(n, 0), ck(contingencies.begin(), contingencies.end());
    std::vector<uint8_t> conv(n);
    std::vector<int32_t> it(n);
    std::vector<double> load(static_cast<size_t>(n) * E), vm(static_cast<size_t>(n) * V), va(vm.size());
    tg_ac_case_out o{conv.data(), it.data(), nullptr, nullptr, load.data(), vm.data(), va.data()};
    if (n) check(tg_ac_run_cases(h_, flat.data(), 1, na, nd, cg.data(), ck.data(), n, &o));
    std::vector<AcCaseResult> out(n);
    for (int i = 0; i < n; ++i) {
      out[i].converged = conv[i] != 0;
      out[i].iterations = it[i];
      out[i].loading_mva.assign(load.begin() + static_cast<size_t>(i) * E, load.begin() + static_cast<size_t>(i + 1) * E);
      out[i].vm_pu.assign(vm.begin() + static_cast<size_t>(i) * V, vm.begin() + static_cast<size_t>(i + 1) * V);
      out[i].va_rad.assign(va.begin() + static_cast<size_t>(i) * V, va.begin() + static_cast<size_t>(i + 1) * V);
    }
    return out;
  }
  AcCaseResult run_case(const Genome& g, int contingency) const { return run_cases(g, {contingency}).front(); }

  // ac_validator.cpp:345-397
  EliminationOutcome eliminate(const std::vector<Candidate>& cands) const {
    const double eps = config_.dominance_fitness_frac * std::abs(pre_fitness_);
    const double theta = config_.improvement_threshold_frac * std::abs(pre_fitness_);
    auto swd = [](const ScoreVector& s) { return s.lambda_d + s.lambda_s + s.lambda_r; };
    EliminationOutcome out;
    for (int i = 0; i < static_cast<int>(cands.size()); ++i) {
      const Candidate& c = cands[i];
      auto dominated_by = [&](int osw, double ofit) { return osw < swd(c.dc_score) && ofit >= c.dc_score.fitness - eps; };
      RejectionReason why = RejectionReason::None;
      for (const auto& v : validated_)
        if (genome_distance(c.genome, v.genome) <= config_.similarity_distance) {
          why = RejectionReason::EliminatedSimilar;
          break;
        }
      if (why == RejectionReason::None)
        for (const Candidate& o : cands)
          if (dominated_by(swd(o.dc_score), o.dc_score.fitness)) {
            why = RejectionReason::EliminatedDominated;
            break;
          }
      if (why == RejectionReason::None)
        for (const auto& v : validated_)
          if (dominated_by(v.swd, v.fitness)) {
            why = RejectionReason::EliminatedDominated;
            break;
          }
      if (why == RejectionReason::None &&
          (!std::isfinite(c.dc_score.fitness) || c.dc_score.fitness - pre_fitness_ < theta))
        why = RejectionReason::EliminatedBelowThreshold;
      if (why == RejectionReason::None)
        out.queue.push_back(i);
      else
        out.pruned.emplace_back(i, why);
    }
    std::sort(out.queue.begin(), out.queue.end(), [&](int a, int b) {
      if (cands[a].dc_score.fitness != cands[b].dc_score.fitness) return cands[a].dc_score.fitness > cands[b].dc_score.fitness;
      return cands[a].genome.canonical_key() < cands[b].genome.canonical_key();
    });
    return out;
  }

  // ac_validator.cpp:399-425, for a batch of genomes (one device batch)
  std::vector<RejectionReason> worst_k_check(const std::vector<Candidate>& cs) const {
    if (cs.empty()) return {};
    int na = 0, nd = 0, wk = 1;
    for (const Candidate& c : cs) {
      na = std::max(na, static_cast<int>(c.genome.action_slots.size()));
      nd = std::max(nd, static_cast<int>(c.genome.disconnection_slots.size()));
      wk = std::max(wk, static_cast<int>(c.dc_score.worst_contingencies.size()));
    }
    const int n = static_cast<int>(cs.size());
    std::vector<int32_t> flat = pad(cs, na, nd), wi(static_cast<size_t>(n) * wk, -1), wn(n), reason(n);
    for (int i = 0; i < n; ++i) {
      wn[i] = static_cast<int32_t>(cs[i].dc_score.worst_contingencies.size());
      for (int j = 0; j < wn[i]; ++j) wi[static_cast<size_t>(i) * wk + j] = cs[i].dc_score.worst_contingencies[j].first;
    }
    check(tg_ac_worst_k_check(h_, flat.data(), n, na, nd, wi.data(), wn.data(), wk, reason.data()));
    std::vector<RejectionReason> out(n);
    for (int i = 0; i < n; ++i) out[i] = static_cast<RejectionReason>(reason[i]);
    return out;
  }
  RejectionReason worst_k_check(const Genome& g, const ScoreVector& s) const { return worst_k_check({{g, s}}).front(); }

  // ac_validator.cpp:427-473, for a batch of genomes (one device batch)
  std::vector<ValidationRecord> full_validation(const std::vector<Candidate>& cs) const {
    if (cs.empty()) return {};
    int na = 0, nd = 0;
    for (const Candidate& c : cs) {
      na = std::max(na, static_cast<int>(c.genome.action_slots.size()));
      nd = std::max(nd, static_cast<int>(c.genome.disconnection_slots.size()));
    }
    const int n = static_cast<int>(cs.size());
    std::vector<int32_t> flat = pad(cs, na, nd), reason(n);
    std::vector<uint8_t> acc(n);
    std::vector<double> lo(n);
    check(tg_ac_full_validation(h_, flat.data(), n, na, nd, reason.data(), acc.data(), lo.data()));
    std::vector<ValidationRecord> out(n);
    for (int i = 0; i < n; ++i)
      out[i] = {cs[i].genome, cs[i].dc_score, ValidationStage::FullN1, acc[i] != 0,
                static_cast<RejectionReason>(reason[i]), lo[i]};
    return out;
  }
  ValidationRecord full_validation(const Genome& g, const ScoreVector& s) const { return full_validation({{g, s}}).front(); }

  // validate() for each candidate in order (ac_validator.cpp:475-495): the
  // worst-k stage of all of them as one device batch, the full N-1 stage of
  // the survivors as a second; the records equal a loop of validate calls.
  std::vector<ValidationRecord> validate_queue(const std::vector<Candidate>& cs) {
    for (const Candidate& c : cs)
      validated_.push_back({c.genome, c.dc_score.lambda_d + c.dc_score.lambda_s + c.dc_score.lambda_r, c.dc_score.fitness});
    const std::vector<RejectionReason> early = worst_k_check(cs);
    std::vector<Candidate> go;
    for (size_t i = 0; i < cs.size(); ++i)
      if (early[i] == RejectionReason::None) go.push_back(cs[i]);
    const std::vector<ValidationRecord> full = full_validation(go);
    std::vector<ValidationRecord> out;
    size_t j = 0;
    for (size_t i = 0; i < cs.size(); ++i) {
      if (early[i] == RejectionReason::None)
        out.push_back(full[j++]);
      else
        out.push_back({cs[i].genome, cs[i].dc_score, ValidationStage::WorstK, false, early[i], 0.0});
      records_.push_back(out.back());
    }
    return out;
  }
  ValidationRecord validate(const Candidate& c) { return validate_queue({c}).front(); }
  void record_elimination(const Candidate& c, RejectionReason reason) {
    records_.push_back({c.genome, c.dc_score, ValidationStage::None, false, reason, 0.0});
  }
  const std::vector<ValidationRecord>& records() const { return records_; }
  const GridModel& grid() const { return grid_; }
  const ActionSet& actions() const { return actions_; }

 private:
  static std::vector<int32_t> pad(const std::vector<Candidate>& cs, int na, int nd) {
    std::vector<int32_t> flat;
    for (const Candidate& c : cs) {
      flat.insert(flat.end(), c.genome.action_slots.begin(), c.genome.action_slots.end());
      flat.insert(flat.end(), na - c.genome.action_slots.size(), -1);
      flat.insert(flat.end(), c.genome.disconnection_slots.begin(), c.genome.disconnection_slots.end());
      flat.insert(flat.end(), nd - c.genome.disconnection_slots.size(), -1);
    }
    return flat;
  }
  struct Validated {
    Genome genome;
    int swd = 0;
    double fitness = 0.0;
  };
  GridModel grid_;
  ActionSet actions_;
  AcConfig config_;
  tg_ac_context* h_ = nullptr;
  double baseline_lambda_o_ = 0.0, pre_fitness_ = 0.0;
  int baseline_critical_ = 0;
  std::vector<Validated> validated_;
  std::vector<ValidationRecord> records_;
};

// ac_validator.cpp:497-534 (nlohmann ordered_json dump: compact, key order kept)
inline std::string record_to_json(const ValidationRecord& r, const GridModel& grid, const ActionSet& actions) {
  std::ostringstream o;
  o.precision(17);
  auto ids = [](std::vector<int> v) {
    std::sort(v.begin(), v.end());
    return v;
  };
  std::vector<int> acts, discs;
  for (int a : r.genome.action_slots)
    if (a >= 0) acts.push_back(a);
  for (int d : r.genome.disconnection_slots)
    if (d >= 0) discs.push_back(d);
  o << "{\"actions\":[";
  bool first = true;
  for (int a : ids(acts)) o << (first ? "" : ",") << a, first = false;
  o << "],\"disconnections\":[";
  first = true;
  for (int d : ids(discs)) {
    const char* id = tg_grid_branch_id(grid.handle(), actions.disconnectable(d));
    o << (first ? "" : ",") << '"' << (id ? id : "") << '"';
    first = false;
  }
  const double fit = std::isfinite(r.dc_score.fitness) ? r.dc_score.fitness : -1e30;
  const char* stage = r.stage == ValidationStage::None ? "eliminated" : r.stage == ValidationStage::WorstK ? "worst_k" : "full_n1";
  o << "],\"lambda_d\":" << r.dc_score.lambda_d << ",\"lambda_s\":" << r.dc_score.lambda_s
    << ",\"lambda_r\":" << r.dc_score.lambda_r << ",\"dc_fitness\":" << fit << ",\"dc_lambda_o\":" << r.dc_score.lambda_o
    << ",\"stage\":\"" << stage << "\",\"verdict\":\"" << (r.accepted ? "accepted" : "rejected")
    << "\",\"reason\":\"" << (r.accepted ? "" : to_string(r.reason)) << "\",\"ac_lambda_o\":" << r.ac_lambda_o << "}";
  return o.str();
}

// ---- qd_optimizer.hpp:15-118 -------------------------------------------------
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
  int d_max = 2;
  int s_max = 3;
  int r_max = 45;
  std::uint64_t seed = 1;
  std::int64_t max_evaluations = -1;
  double max_seconds = -1.0;
  // extension: 0 = the reference's per-lane mt19937_64 stream (bit for bit),
  // 1 = counter-based Philox (tg_qd_config::rng)
  int rng = 0;
};

inline int cell_count(const QdConfig& c) { return (c.d_max + 1) * (c.s_max + 1) * (c.r_max + 1); }

namespace detail {
inline tg_qd_config to_c(const QdConfig& q) {
  tg_qd_config c{};
  c.n_a = q.n_a;
  c.n_d = q.n_d;
  c.batch_size = q.batch_size;
  c.iters_per_epoch = q.iters_per_epoch;
  c.cell_capacity = q.cell_capacity;
  c.mutation_mean = q.mutation_mean;
  for (int i = 0; i < 4; ++i) c.p_action[i] = q.p_action[i], c.p_disc[i] = q.p_disc[i];
  c.p_crossover_parent1 = q.p_crossover_parent1;
  c.d_max = q.d_max;
  c.s_max = q.s_max;
  c.r_max = q.r_max;
  c.seed = q.seed;
  c.max_evaluations = q.max_evaluations;
  c.max_seconds = q.max_seconds;
  c.rng = q.rng;
  return c;
}
}  // namespace detail

inline int descriptor_to_cell(int lambda_d, int lambda_s, int lambda_r, const QdConfig& cfg) {
  const tg_qd_config c = detail::to_c(cfg);
  return tg_descriptor_to_cell(lambda_d, lambda_s, lambda_r, &c);
}

struct RepertoireEntry {
  Genome genome;
  ScoreVector score;
  std::string key;
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

using SnapshotSink = std::function<void(RepertoireSnapshot)>;

struct OptimizerStats {
  std::int64_t evaluations = 0;
  int epochs = 0;
  std::vector<std::pair<std::int64_t, double>> fitness_trace;
};

// Read side of the reference's Repertoire (qd_optimizer.hpp:62-81): the
// archive the device loop ended with, cells in cell order, entries ranked as
// Repertoire::insert keeps them. Insertion happens on the device.
class Repertoire {
 public:
  explicit Repertoire(const QdConfig& cfg) : cells_(cell_count(cfg)) {}
  int total_size() const { return total_; }
  int n_cells() const { return static_cast<int>(cells_.size()); }
  const std::vector<RepertoireEntry>& cell(int i) const { return cells_[i]; }
  const RepertoireEntry& member(int flat) const {
    for (const auto& c : cells_) {
      if (flat < static_cast<int>(c.size())) return c[flat];
      flat -= static_cast<int>(c.size());
    }
    throw std::out_of_range("repertoire member index");
  }
  double best_fitness() const {
    double b = -std::numeric_limits<double>::infinity();
    for (const auto& c : cells_)
      for (const auto& e : c) b = std::max(b, e.score.fitness);
    return b;
  }
  std::vector<double> per_cell_best() const {
    std::vector<double> out(cells_.size(), -std::numeric_limits<double>::infinity());
    for (size_t i = 0; i < cells_.size(); ++i)
      for (const auto& e : cells_[i]) out[i] = std::max(out[i], e.score.fitness);
    return out;
  }
  void add(int cell, Genome g, ScoreVector s) {
    std::string key = g.canonical_key();
    cells_[cell].push_back({std::move(g), std::move(s), std::move(key)});
    ++total_;
  }

 private:
  std::vector<std::vector<RepertoireEntry>> cells_;
  int total_ = 0;
};

struct OptimizerResult {
  Repertoire repertoire;
  OptimizerStats stats;
};

namespace detail {
inline RepertoireSnapshot from_view(const tg_snapshot_view& v, int n_a) {
  RepertoireSnapshot s{v.epoch, v.evaluations, v.best_fitness, v.final_snapshot != 0, {}};
  s.entries.reserve(v.n_entries);
  for (int i = 0; i < v.n_entries; ++i) {
    const int32_t* g = v.genome + static_cast<size_t>(i) * v.n_slots;
    Genome gen{{g, g + n_a}, {g + n_a, g + v.n_slots}};
    ScoreVector sc{v.lambda_o[i], v.lambda_c[i], v.lambda_c0[i], v.lambda_b[i], v.lambda_d[i],
                   v.lambda_s[i], v.lambda_r[i], v.fitness[i], false, {}};
    for (int j = 0; j < v.worst_n[i]; ++j)
      sc.worst_contingencies.emplace_back(v.worst_idx[static_cast<size_t>(i) * v.worst_k + j],
                                          v.worst_energy[static_cast<size_t>(i) * v.worst_k + j]);
    s.entries.push_back({v.cell[i], std::move(gen), std::move(sc)});
  }
  return s;
}
}  // namespace detail

// run_optimizer, qd_optimizer.cpp:344-417: the loop runs on the GPU (one CUDA
// graph per generation, no host round trip); `sink` receives one snapshot per
// epoch on the calling thread while the next epoch computes; `stop` is
// honoured before every generation. ConfigError exactly where the reference
// raises it.
inline OptimizerResult run_optimizer(const DcContext& ctx, const QdConfig& q, const SnapshotSink& sink,
                                     const std::atomic<bool>* stop = nullptr) {
  const tg_qd_config c = detail::to_c(q);
  struct User {
    const SnapshotSink* sink;
    int n_a;
    std::exception_ptr err;
  } user{&sink, q.n_a, nullptr};
  auto cb = [](const tg_snapshot_view* v, void* u) {
    auto* x = static_cast<User*>(u);
    if (!*x->sink || x->err) return;
    try {
      (*x->sink)(detail::from_view(*v, x->n_a));
    } catch (...) {
      x->err = std::current_exception();  // rethrown after the loop (no exception crosses the C ABI)
    }
  };
  // the engine polls a volatile int32 flag; a small thread mirrors the
  // reference's std::atomic<bool> into it
  volatile int32_t flag = 0;
  std::atomic<bool> done{false};
  std::thread mirror;
  if (stop)
    mirror = std::thread([&] {
      while (!done.load(std::memory_order_relaxed)) {
        if (stop->load(std::memory_order_relaxed)) flag = 1;
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    });
  constexpr int32_t kTraceCap = 1 << 16;
  std::vector<int64_t> tev(kTraceCap);
  std::vector<double> tbest(kTraceCap);
  tg_opt_stats st{};
  const tg_status rc =
      tg_optimizer_run(ctx.handle(), &c, cb, &user, stop ? &flag : nullptr, &st, tev.data(), tbest.data(), kTraceCap);
  done = true;
  if (mirror.joinable()) mirror.join();
  check(rc);
  if (user.err) std::rethrow_exception(user.err);
  OptimizerResult res{Repertoire(q), {st.evaluations, st.epochs, {}}};
  for (int i = 0; i < st.n_trace; ++i) res.stats.fitness_trace.emplace_back(tev[i], tbest[i]);
  tg_snapshot_view v{};
  check(tg_archive_export(ctx.handle(), &v));
  RepertoireSnapshot s = detail::from_view(v, q.n_a);
  for (SnapshotEntry& e : s.entries) res.repertoire.add(e.cell, std::move(e.genome), std::move(e.score));
  return res;
}

}  // namespace topopt::b200

#endif  // TOPOPT_B200_HPP
