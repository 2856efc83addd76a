// dc_engine_b200.hpp — reference-side shim: routes the reference's DC loop
// (topopt::DcContext::evaluate_batch, topopt::run_optimizer) to the B200
// engine through the C ABI (include/topopt_b200.h), taking the reference's
// own GridModel / ActionSet / Genome / QdConfig types.
//
// A maintainer adds this header to the reference build (proj/src) and links
// libtopopt_b200.so; the import step, the AC validator
// and the pipeline keep their reference code. tests/test_integration_shim.py
// compiles it against the reference headers (with integration/eigen_stub for
// the Eigen types the headers name) so it cannot drift from them.
//
// Reference interfaces used: grid_model.hpp:16-139, importer.hpp:19-35,
// genome.hpp:13-35, dc_engine.hpp:16-48 and 95-150, qd_optimizer.hpp:15-118,
// ac_validator.hpp:18-140, errors.hpp:9-34.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdint>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <topopt_b200.h>

#include "topopt/ac_validator.hpp"
#include "topopt/dc_engine.hpp"
#include "topopt/errors.hpp"
#include "topopt/qd_optimizer.hpp"

namespace topopt::b200 {

// Every tg_status raises the reference's exception of the same kind; the two
// engine-only kinds (device failure, capacity) raise std::runtime_error
// subclasses of their own, never ValidationError.
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct CapacityError : std::runtime_error {
  explicit CapacityError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(tg_status s) {
  if (s == TG_OK) return;
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
    default: throw std::runtime_error("topopt_b200 status " + std::to_string(int(s)) + ": " + msg);
  }
}

// Flattened copy of a GridModel (grid_model.hpp:80-127); the arrays live as
// long as the struct, tg_context_create reads them once.
struct GridArrays {
  std::vector<int32_t> from, to, inj_node, cbp{0}, cb, cip{0}, ci, sub_node, stp{0}, tkind, telem, bo_sub, bo_bb,
      bip{0}, bi;
  std::vector<double> x, lim, net;
  std::vector<uint8_t> on;
  tg_grid_desc desc{};

  explicit GridArrays(const GridModel& g) {
    for (const Branch& b : g.branches) {
      from.push_back(b.from);
      to.push_back(b.to);
      x.push_back(b.reactance);
      lim.push_back(b.flow_limit);
      on.push_back(b.in_service ? 1 : 0);
    }
    for (const Injection& i : g.injections) {
      inj_node.push_back(i.node);
      net.push_back(i.net_mw());
    }
    for (const ContingencyCase& c : g.contingencies) {
      cb.insert(cb.end(), c.branches.begin(), c.branches.end());
      cbp.push_back(static_cast<int32_t>(cb.size()));
      ci.insert(ci.end(), c.injections.begin(), c.injections.end());
      cip.push_back(static_cast<int32_t>(ci.size()));
    }
    for (const SubstationDetail& s : g.substations) {
      sub_node.push_back(s.node);
      for (const Terminal& t : s.terminals) {
        tkind.push_back(t.kind == TerminalKind::BranchFrom ? 0 : t.kind == TerminalKind::BranchTo ? 1 : 2);
        telem.push_back(t.element_index);
      }
      stp.push_back(static_cast<int32_t>(tkind.size()));
    }
    for (const BusbarOutage& bo : g.busbar_outages) {
      bo_sub.push_back(bo.substation);
      bo_bb.push_back(g.substations[bo.substation].busbar_index(bo.busbar));
      for (int e : g.implied_branches(bo)) bi.push_back(e);  // grid_model.cpp:217-227
      bip.push_back(static_cast<int32_t>(bi.size()));
    }
    desc.n_nodes = static_cast<int32_t>(g.nodes.size());
    desc.n_branches = static_cast<int32_t>(g.branches.size());
    desc.n_injections = static_cast<int32_t>(g.injections.size());
    desc.slack = g.slack;
    desc.branch_from = from.data();
    desc.branch_to = to.data();
    desc.branch_x = x.data();
    desc.branch_limit = lim.data();
    desc.branch_in_service = on.data();
    desc.injection_node = inj_node.data();
    desc.injection_net_mw = net.data();
    desc.n_contingencies = static_cast<int32_t>(g.contingencies.size());
    desc.cont_branch_ptr = cbp.data();
    desc.cont_branch = cb.data();
    desc.cont_inj_ptr = cip.data();
    desc.cont_inj = ci.data();
    desc.n_substations = static_cast<int32_t>(g.substations.size());
    desc.sub_node = sub_node.data();
    desc.sub_term_ptr = stp.data();
    desc.term_kind = tkind.data();
    desc.term_element = telem.data();
    desc.n_busbar_outages = static_cast<int32_t>(g.busbar_outages.size());
    desc.bo_substation = bo_sub.data();
    desc.bo_busbar = bo_bb.data();
    desc.bo_implied_ptr = bip.data();
    desc.bo_implied = bi.data();
    desc.n_timesteps = 1;  // the reference's single injection vector
    desc.injection_net_mw_t = nullptr;
  }
};

// Flattened ActionSet (importer.hpp:28-35) with the per-(action, busbar)
// implied branch lists the reference's DcContext precomputes
// (dc_engine.cpp:118-131).
struct ActionArrays {
  std::vector<int32_t> sub, lr, gp{0}, bbp{0}, ip{0}, imp, disc;
  std::vector<uint8_t> grp;
  tg_actionset_desc desc{};

  ActionArrays(const GridModel& g, const ActionSet& a) {
    for (const Action& act : a.actions) {
      sub.push_back(act.substation);
      lr.push_back(act.reassignment_distance);
      grp.insert(grp.end(), act.group.begin(), act.group.end());
      gp.push_back(static_cast<int32_t>(grp.size()));
      const SubstationDetail& st = g.substations[act.substation];
      for (const std::string& bb : st.busbars) {
        const BusbarOutage probe{"", act.substation, bb};
        for (int e : g.implied_branches(probe, act.busbar_assignment, act.open_couplers)) imp.push_back(e);
        ip.push_back(static_cast<int32_t>(imp.size()));
      }
      bbp.push_back(static_cast<int32_t>(ip.size()) - 1);
    }
    disc.assign(a.disconnectables.begin(), a.disconnectables.end());
    desc.n_actions = static_cast<int32_t>(a.actions.size());
    desc.action_substation = sub.data();
    desc.action_lambda_r = lr.data();
    desc.action_group_ptr = gp.data();
    desc.action_group = grp.data();
    desc.action_busbar_ptr = bbp.data();
    desc.action_implied_ptr = ip.data();
    desc.action_implied = imp.data();
    desc.n_disconnectables = static_cast<int32_t>(disc.size());
    desc.disconnectables = disc.data();
  }
};

// Drop-in for DcContext::evaluate_batch / evaluate (dc_engine.cpp:424-468).
class GpuDcContext {
 public:
  GpuDcContext(const GridModel& g, const ActionSet& a, DcConfig cfg = {}, int device = 0)
      : ga_(g), aa_(g, a), cfg_(cfg) {
    const tg_dc_config c{cfg.islanding_penalty_mw, cfg.worst_k, cfg.weight_c0, cfg.weight_c, cfg.fitness_variant,
                         cfg.threads};
    check(tg_context_create(&ga_.desc, &aa_.desc, &c, device, &ctx_));
  }
  ~GpuDcContext() { tg_context_destroy(ctx_); }
  GpuDcContext(const GpuDcContext&) = delete;
  GpuDcContext& operator=(const GpuDcContext&) = delete;

  ScoreVector evaluate(const Genome& g) const { return evaluate_batch({g}, 1).front(); }

  // Genomes may mix slot counts (vector<Genome>): each is padded with empty
  // slots to the widest one, which changes neither topology nor score.
  std::vector<ScoreVector> evaluate_batch(const std::vector<Genome>& gs, int batch_size) const {
    std::vector<ScoreVector> out;
    if (gs.empty()) return out;
    int na = 0, nd = 0;
    for (const Genome& g : gs) {
      na = std::max<int>(na, static_cast<int>(g.action_slots.size()));
      nd = std::max<int>(nd, static_cast<int>(g.disconnection_slots.size()));
    }
    const int n = static_cast<int>(gs.size()), k = cfg_.worst_k;
    std::vector<int32_t> flat;
    for (const Genome& g : gs) {
      flat.insert(flat.end(), g.action_slots.begin(), g.action_slots.end());
      flat.insert(flat.end(), na - g.action_slots.size(), -1);
      flat.insert(flat.end(), g.disconnection_slots.begin(), g.disconnection_slots.end());
      flat.insert(flat.end(), nd - g.disconnection_slots.size(), -1);
    }
    std::vector<double> lo(n), lb(n), fit(n), wv(static_cast<size_t>(n) * k);
    std::vector<int32_t> lc(n), lc0(n), ld(n), ls(n), lr(n), wi(static_cast<size_t>(n) * k), wn(n), io(n), ib(n);
    std::vector<uint8_t> isl(n);
    tg_scores s{lo.data(), lc.data(), lc0.data(), lb.data(), ld.data(), ls.data(), lr.data(),
                fit.data(), isl.data(), wi.data(), wv.data(), wn.data(), io.data(), ib.data()};
    check(tg_evaluate_batch(ctx_, flat.data(), n, na, nd, std::max(batch_size, n), &s, nullptr, nullptr, nullptr,
                            nullptr));
    out.resize(n);
    for (int i = 0; i < n; ++i) {
      ScoreVector& v = out[i];
      v.lambda_o = lo[i];
      v.lambda_c = lc[i];
      v.lambda_c0 = lc0[i];
      v.lambda_b = lb[i];
      v.lambda_d = ld[i];
      v.lambda_s = ls[i];
      v.lambda_r = lr[i];
      v.fitness = fit[i];
      v.islanded = isl[i] != 0;
      for (int j = 0; j < wn[i]; ++j)
        v.worst_contingencies.emplace_back(wi[static_cast<size_t>(i) * k + j], wv[static_cast<size_t>(i) * k + j]);
    }
    return out;
  }
  tg_context* handle() const { return ctx_; }

 private:
  GridArrays ga_;
  ActionArrays aa_;
  DcConfig cfg_;
  tg_context* ctx_ = nullptr;
};

// Drop-in for run_optimizer (qd_optimizer.cpp:344-417): the loop runs on the
// GPU; the sink receives one RepertoireSnapshot per epoch on the calling
// thread. Returns the stats (the archive is in the last snapshot).
inline OptimizerStats run_optimizer_gpu(const GpuDcContext& ctx, const QdConfig& q, const SnapshotSink& sink,
                                        const std::atomic<bool>* stop = nullptr) {
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
  c.rng = 0;  // the reference's mt19937_64 lane streams
  struct User {
    const SnapshotSink* sink;
    int na;
    std::exception_ptr err;
  } user{&sink, q.n_a, nullptr};
  auto cb = [](const tg_snapshot_view* v, void* u) {
    auto* x = static_cast<User*>(u);
    if (!*x->sink || x->err) return;
    try {
      RepertoireSnapshot s;
      s.epoch = v->epoch;
      s.evaluations = v->evaluations;
      s.best_fitness = v->best_fitness;
      s.final = v->final_snapshot != 0;
      for (int i = 0; i < v->n_entries; ++i) {
        const int32_t* g = v->genome + static_cast<size_t>(i) * v->n_slots;
        SnapshotEntry e;
        e.cell = v->cell[i];
        e.genome = Genome{{g, g + x->na}, {g + x->na, g + v->n_slots}};
        e.score.lambda_o = v->lambda_o[i];
        e.score.lambda_c = v->lambda_c[i];
        e.score.lambda_c0 = v->lambda_c0[i];
        e.score.lambda_b = v->lambda_b[i];
        e.score.lambda_d = v->lambda_d[i];
        e.score.lambda_s = v->lambda_s[i];
        e.score.lambda_r = v->lambda_r[i];
        e.score.fitness = v->fitness[i];
        for (int j = 0; j < v->worst_n[i]; ++j)
          e.score.worst_contingencies.emplace_back(v->worst_idx[static_cast<size_t>(i) * v->worst_k + j],
                                                   v->worst_energy[static_cast<size_t>(i) * v->worst_k + j]);
        s.entries.push_back(std::move(e));
      }
      (*x->sink)(std::move(s));
    } catch (...) {
      x->err = std::current_exception();
    }
  };
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
  constexpr int32_t kCap = 1 << 16;
  std::vector<int64_t> tev(kCap);
  std::vector<double> tbest(kCap);
  tg_opt_stats st{};
  const tg_status rc =
      tg_optimizer_run(ctx.handle(), &c, cb, &user, stop ? &flag : nullptr, &st, tev.data(), tbest.data(), kCap);
  done = true;
  if (mirror.joinable()) mirror.join();
  check(rc);
  if (user.err) std::rethrow_exception(user.err);
  OptimizerStats out;
  out.evaluations = st.evaluations;
  out.epochs = st.epochs;
  for (int i = 0; i < st.n_trace; ++i) out.fitness_trace.emplace_back(tev[i], tbest[i]);
  return out;
}


// Drop-in for AcValidator (ac_validator.hpp:93-140): the same members on the
// reference's own types; every power flow runs on the GPU (tg_ac_*, one CTA per
// (genome, contingency) case). The engine reads the grid through the
// reference's canonical dump (grid_to_json_text) and rebuilds the action set
// with the same ids. eliminate() and the history are the reference's host
// logic; validate_queue() validates a whole elimination queue with two device
// batches and records what a loop of validate() calls records.
class GpuAcValidator {
 public:
  GpuAcValidator(const GridModel& grid, const ActionSet& actions, const DcContext& dc, AcConfig config = {},
                 const GpuDcContext* gpu_dc = nullptr, int device = 0)
      : grid_(&grid), actions_(&actions), config_(config) {
    const std::string text = grid_to_json_text(grid);
    check(tg_grid_from_json(text.data(), text.size(), &tg_grid_));
    check(tg_actionset_build(tg_grid_, 0, 0, &tg_actions_));
    const tg_ac_config c{config.tolerance_pu, config.max_iterations, config.worst_k_nonconverged,
                         config.nonconverged_fraction, config.similarity_distance, config.dominance_fitness_frac,
                         config.improvement_threshold_frac};
    check(tg_ac_context_create(tg_grid_, tg_actions_, gpu_dc ? gpu_dc->handle() : nullptr, &c, device, &h_));
    tg_ac_baseline b{};
    check(tg_ac_baseline_get(h_, &b, nullptr, nullptr));
    baseline_lambda_o_ = b.lambda_o;
    baseline_critical_ = b.critical_count;
    pre_fitness_ = dc.pre_optimization_score().fitness;
  }
  ~GpuAcValidator() {
    if (h_) tg_ac_context_destroy(h_);
    if (tg_actions_) tg_actionset_destroy(tg_actions_);
    if (tg_grid_) tg_grid_destroy(tg_grid_);
  }
  GpuAcValidator(const GpuAcValidator&) = delete;
  GpuAcValidator& operator=(const GpuAcValidator&) = delete;

  const AcConfig& config() const { return config_; }
  double baseline_lambda_o() const { return baseline_lambda_o_; }
  int baseline_critical_count() const { return baseline_critical_; }

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
      for (const Validated& v : validated_)
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
        for (const Validated& v : validated_)
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

  // ac_validator.cpp:399-425 for a batch
  std::vector<RejectionReason> worst_k_check(const std::vector<Candidate>& cs) const {
    if (cs.empty()) return {};
    int na = 0, nd = 0, wk = 1;
    for (const Candidate& c : cs) {
      na = std::max<int>(na, static_cast<int>(c.genome.action_slots.size()));
      nd = std::max<int>(nd, static_cast<int>(c.genome.disconnection_slots.size()));
      wk = std::max<int>(wk, static_cast<int>(c.dc_score.worst_contingencies.size()));
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
  RejectionReason worst_k_check(const Genome& g, const ScoreVector& s) const { return worst_k_check({Candidate{g, s}}).front(); }

  // ac_validator.cpp:427-473 for a batch
  std::vector<ValidationRecord> full_validation(const std::vector<Candidate>& cs) const {
    std::vector<ValidationRecord> out;
    if (cs.empty()) return out;
    int na = 0, nd = 0;
    for (const Candidate& c : cs) {
      na = std::max<int>(na, static_cast<int>(c.genome.action_slots.size()));
      nd = std::max<int>(nd, static_cast<int>(c.genome.disconnection_slots.size()));
    }
    const int n = static_cast<int>(cs.size());
    std::vector<int32_t> flat = pad(cs, na, nd), reason(n);
    std::vector<uint8_t> acc(n);
    std::vector<double> lo(n);
    check(tg_ac_full_validation(h_, flat.data(), n, na, nd, reason.data(), acc.data(), lo.data()));
    out.resize(n);
    for (int i = 0; i < n; ++i) {
      out[i].genome = cs[i].genome;
      out[i].dc_score = cs[i].dc_score;
      out[i].stage = ValidationStage::FullN1;
      out[i].accepted = acc[i] != 0;
      out[i].reason = static_cast<RejectionReason>(reason[i]);
      out[i].ac_lambda_o = lo[i];
    }
    return out;
  }
  ValidationRecord full_validation(const Genome& g, const ScoreVector& s) const {
    return full_validation(std::vector<Candidate>{Candidate{g, s}}).front();
  }

  // ac_validator.cpp:475-495 for a whole queue
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
      if (early[i] == RejectionReason::None) {
        out.push_back(full[j++]);
      } else {
        ValidationRecord r;
        r.genome = cs[i].genome;
        r.dc_score = cs[i].dc_score;
        r.stage = ValidationStage::WorstK;
        r.reason = early[i];
        out.push_back(r);
      }
      records_.push_back(out.back());
    }
    return out;
  }
  ValidationRecord validate(const Candidate& c) { return validate_queue({c}).front(); }
  void record_elimination(const Candidate& c, RejectionReason reason) {
    ValidationRecord r;
    r.genome = c.genome;
    r.dc_score = c.dc_score;
    r.reason = reason;
    records_.push_back(r);
  }
  const std::vector<ValidationRecord>& records() const { return records_; }

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
  const GridModel* grid_;
  const ActionSet* actions_;
  AcConfig config_;
  tg_grid* tg_grid_ = nullptr;
  tg_actionset* tg_actions_ = nullptr;
  tg_ac_context* h_ = nullptr;
  double baseline_lambda_o_ = 0.0, pre_fitness_ = 0.0;
  int baseline_critical_ = 0;
  std::vector<Validated> validated_;
  std::vector<ValidationRecord> records_;
};

}  // namespace topopt::b200
