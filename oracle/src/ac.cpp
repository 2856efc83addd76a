// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
//
// Restatement of the reference's AC validation stage, ac_validator.cpp:1-536:
//   AcNetwork::solve        ac_validator.cpp:37-272  polar Newton-Raphson from a
//                           flat start on the live (slack-reachable) buses,
//                           dense Jacobian, LU with partial pivoting
//                           (Eigen partialPivLu, restated below)
//   overload_energy /
//   critical_count          ac_validator.cpp:274-288
//   AcValidator             ac_validator.cpp:311-495 baseline, eliminate,
//                           worst_k_check, full_validation, validate
//   record_to_json          ac_validator.cpp:497-534
// Checked by the reference's own tests (test_ac_validator.cpp), ported in
// oracle/kats/kats.cpp (ac_* KATs).
#include <algorithm>
#include <cmath>
#include <complex>

#include <nlohmann/json.hpp>

#include "oracle.hpp"

namespace oracle {

namespace {

constexpr double kMvaBase = 100.0;  // ac_validator.cpp:14
using cplx = std::complex<double>;

double positive_part(double x) { return x > 0.0 ? x : 0.0; }

// x = A^-1 b by LU with row partial pivoting (Eigen::PartialPivLU: the pivot
// of column k is the first largest |a_ik|, i >= k). A is row-major n x n and is
// overwritten. A zero pivot yields non-finite entries, which the caller tests
// (ac_validator.cpp:240-241), like Eigen.
Vec lu_solve(std::vector<double>& a, Vec b, int n) {
  auto at = [&](int i, int j) -> double& { return a[static_cast<std::size_t>(i) * n + j]; };
  for (int k = 0; k < n; ++k) {
    int p = k;
    double big = std::abs(at(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(at(i, k)) > big) big = std::abs(at(i, k)), p = i;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(at(k, j), at(p, j));
      std::swap(b[k], b[p]);
    }
    const double piv = at(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double l = at(i, k) / piv;
      at(i, k) = l;
      if (l == 0.0) continue;
      for (int j = k + 1; j < n; ++j) at(i, j) -= l * at(k, j);
      b[i] -= l * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= at(i, j) * b[j];
    b[i] = s / at(i, i);
  }
  return b;
}

}  // namespace

AcNetwork::AcNetwork(const GridModel& grid, const AppliedTopology& topology, AcConfig config)
    : grid_(&grid), topo_(topology), cfg_(config) {
  n_buses_ = static_cast<int>(grid.nodes.size()) + topo_.n_new_nodes;
}

// ac_validator.cpp:26-35
AcCaseResult AcNetwork::run_case(int contingency) const {
  std::vector<char> br_out(grid_->branches.size(), 0), inj_out(grid_->injections.size(), 0);
  if (contingency >= 0) {
    const ContingencyCase& c = grid_->contingencies[contingency];
    for (int e : c.branches) br_out[e] = 1;
    for (int i : c.injections) inj_out[i] = 1;
  }
  return solve(br_out, inj_out);
}

// ac_validator.cpp:37-272
AcCaseResult AcNetwork::solve(const std::vector<char>& br_out, const std::vector<char>& inj_out) const {
  const GridModel& g = *grid_;
  const int E = static_cast<int>(g.branches.size());
  const int I = static_cast<int>(g.injections.size());
  AcCaseResult res;
  res.loading_mva.assign(E, 0.0);
  res.vm_pu.assign(n_buses_, 0.0);
  res.va_rad.assign(n_buses_, 0.0);

  std::vector<char> live(E);
  for (int e = 0; e < E; ++e) live[e] = g.branches[e].in_service && !topo_.removed[e] && !br_out[e];

  // buses reachable from the slack over live branches (ac_validator.cpp:52-73)
  std::vector<std::vector<int>> nbr(n_buses_);
  for (int e = 0; e < E; ++e) {
    if (!live[e]) continue;
    nbr[topo_.endpoints[e].first].push_back(topo_.endpoints[e].second);
    nbr[topo_.endpoints[e].second].push_back(topo_.endpoints[e].first);
  }
  std::vector<char> seen(n_buses_, 0);
  std::vector<int> todo{g.slack};
  seen[g.slack] = 1;
  while (!todo.empty()) {
    const int v = todo.back();
    todo.pop_back();
    for (int w : nbr[v])
      if (!seen[w]) seen[w] = 1, todo.push_back(w);
  }
  // a floating live component or a stranded nonzero injection: not converged,
  // zero iterations (ac_validator.cpp:74-82)
  for (int e = 0; e < E; ++e)
    if (live[e] && !seen[topo_.endpoints[e].first]) return res;
  for (int i = 0; i < I; ++i) {
    if (inj_out[i]) continue;
    const Injection& q = g.injections[i];
    if ((q.p_mw != 0.0 || q.q_mvar != 0.0) && !seen[topo_.injection_node[i]]) return res;
  }

  std::vector<int> bus(n_buses_, -1), node_of;
  for (int v = 0; v < n_buses_; ++v)
    if (seen[v]) bus[v] = static_cast<int>(node_of.size()), node_of.push_back(v);
  const int n = static_cast<int>(node_of.size());
  const int sl = bus[g.slack];

  // specified injections, PV buses and their setpoints (ac_validator.cpp:94-115):
  // the first generator with a setpoint fixes a bus's magnitude
  Vec psp(n, 0.0), qsp(n, 0.0), vset(n, 1.0);
  std::vector<char> pv(n, 0);
  for (int i = 0; i < I; ++i) {
    if (inj_out[i]) continue;
    const Injection& q = g.injections[i];
    const int b = bus[topo_.injection_node[i]];
    if (b < 0) continue;
    if (q.kind == InjectionKind::Generator) {
      psp[b] += q.p_mw / kMvaBase;
      if (q.v_setpoint_pu) {
        if (!pv[b]) vset[b] = *q.v_setpoint_pu;
        pv[b] = 1;
      } else {
        qsp[b] += q.q_mvar / kMvaBase;
      }
    } else {
      psp[b] -= q.p_mw / kMvaBase;
      qsp[b] -= q.q_mvar / kMvaBase;
    }
  }

  // bus admittance matrix, pi model with off-nominal tap on the from side
  // (ac_validator.cpp:117-141)
  std::vector<cplx> Y(static_cast<std::size_t>(n) * n, cplx(0.0, 0.0));
  auto y_at = [&](int i, int j) -> cplx& { return Y[static_cast<std::size_t>(i) * n + j]; };
  std::vector<std::array<cplx, 4>> ybr(E);
  for (int e = 0; e < E; ++e) {
    if (!live[e]) continue;
    const Branch& br = g.branches[e];
    const cplx ys = 1.0 / cplx(br.resistance, br.reactance);
    const cplx ysh(0.0, br.charging_b / 2.0);
    const double t = br.tap;
    ybr[e] = {(ys + ysh) / (t * t), -ys / t, -ys / t, ys + ysh};
    const int f = bus[topo_.endpoints[e].first], to = bus[topo_.endpoints[e].second];
    y_at(f, f) += ybr[e][0];
    y_at(f, to) += ybr[e][1];
    y_at(to, f) += ybr[e][2];
    y_at(to, to) += ybr[e][3];
  }
  for (int v = 0; v < static_cast<int>(g.nodes.size()); ++v)
    if (bus[v] >= 0 && g.nodes[v].shunt_b_pu != 0.0) y_at(bus[v], bus[v]) += cplx(0.0, g.nodes[v].shunt_b_pu);
  auto G = [&](int i, int j) { return y_at(i, j).real(); };
  auto B = [&](int i, int j) { return y_at(i, j).imag(); };

  // flat start (ac_validator.cpp:143-147) and unknown ordering: angles of every
  // non-slack bus, then magnitudes of the PQ buses (148-156)
  Vec vm(n, 1.0), va(n, 0.0);
  for (int b = 0; b < n; ++b)
    if (pv[b] || b == sl) vm[b] = vset[b];
  std::vector<int> ang, mag;
  for (int b = 0; b < n; ++b) {
    if (b == sl) continue;
    ang.push_back(b);
    if (!pv[b]) mag.push_back(b);
  }
  const int na = static_cast<int>(ang.size()), nm = static_cast<int>(mag.size()), nu = na + nm;

  Vec P(n), Q(n);
  auto injections = [&] {  // ac_validator.cpp:159-173
    for (int i = 0; i < n; ++i) {
      double p = 0.0, q = 0.0;
      for (int k = 0; k < n; ++k) {
        if (G(i, k) == 0.0 && B(i, k) == 0.0) continue;
        const double th = va[i] - va[k], c = std::cos(th), s = std::sin(th);
        p += vm[i] * vm[k] * (G(i, k) * c + B(i, k) * s);
        q += vm[i] * vm[k] * (G(i, k) * s - B(i, k) * c);
      }
      P[i] = p;
      Q[i] = q;
    }
  };

  bool ok = false;
  int iters = 0;
  for (int it = 1; it <= cfg_.max_iterations; ++it) {  // ac_validator.cpp:175-244
    injections();
    iters = it;
    Vec dx(nu);
    double worst = 0.0;
    for (int r = 0; r < na; ++r) dx[r] = psp[ang[r]] - P[ang[r]], worst = std::max(worst, std::abs(dx[r]));
    for (int r = 0; r < nm; ++r)
      dx[na + r] = qsp[mag[r]] - Q[mag[r]], worst = std::max(worst, std::abs(dx[na + r]));
    if (!std::isfinite(worst) || worst > 1e8) break;  // diverged
    if (worst < cfg_.tolerance_pu) {
      ok = true;
      break;
    }
    if (it == cfg_.max_iterations) break;

    // Jacobian blocks dP/dtheta, dP/dV, dQ/dtheta, dQ/dV (ac_validator.cpp:186-236)
    std::vector<double> J(static_cast<std::size_t>(nu) * nu, 0.0);
    auto j_at = [&](int r, int c) -> double& { return J[static_cast<std::size_t>(r) * nu + c]; };
    for (int r = 0; r < na; ++r) {
      const int i = ang[r];
      for (int c = 0; c < na; ++c) {
        const int k = ang[c];
        if (i == k) {
          j_at(r, c) = -Q[i] - B(i, i) * vm[i] * vm[i];
        } else {
          const double th = va[i] - va[k];
          j_at(r, c) = vm[i] * vm[k] * (G(i, k) * std::sin(th) - B(i, k) * std::cos(th));
        }
      }
      for (int c = 0; c < nm; ++c) {
        const int k = mag[c];
        if (i == k) {
          j_at(r, na + c) = P[i] / vm[i] + G(i, i) * vm[i];
        } else {
          const double th = va[i] - va[k];
          j_at(r, na + c) = vm[i] * (G(i, k) * std::cos(th) + B(i, k) * std::sin(th));
        }
      }
    }
    for (int r = 0; r < nm; ++r) {
      const int i = mag[r];
      for (int c = 0; c < na; ++c) {
        const int k = ang[c];
        if (i == k) {
          j_at(na + r, c) = P[i] - G(i, i) * vm[i] * vm[i];
        } else {
          const double th = va[i] - va[k];
          j_at(na + r, c) = -vm[i] * vm[k] * (G(i, k) * std::cos(th) + B(i, k) * std::sin(th));
        }
      }
      for (int c = 0; c < nm; ++c) {
        const int k = mag[c];
        if (i == k) {
          j_at(na + r, na + c) = Q[i] / vm[i] - B(i, i) * vm[i];
        } else {
          const double th = va[i] - va[k];
          j_at(na + r, na + c) = vm[i] * (G(i, k) * std::sin(th) - B(i, k) * std::cos(th));
        }
      }
    }
    const Vec step = lu_solve(J, dx, nu);
    bool finite = true;
    for (double s : step) finite = finite && std::isfinite(s);
    if (!finite) break;
    for (int r = 0; r < na; ++r) va[ang[r]] += step[r];
    for (int r = 0; r < nm; ++r) vm[mag[r]] += step[na + r];
  }

  res.iterations = iters;
  if (!ok) return res;
  res.converged = true;
  for (int b = 0; b < n; ++b) res.vm_pu[node_of[b]] = vm[b], res.va_rad[node_of[b]] = va[b];
  // branch loading: larger apparent power of the two ends (ac_validator.cpp:254-270)
  for (int e = 0; e < E; ++e) {
    if (!live[e]) continue;
    const int f = bus[topo_.endpoints[e].first], to = bus[topo_.endpoints[e].second];
    const cplx vf = std::polar(vm[f], va[f]), vt = std::polar(vm[to], va[to]);
    const cplx sf = vf * std::conj(ybr[e][0] * vf + ybr[e][1] * vt);
    const cplx st = vt * std::conj(ybr[e][2] * vf + ybr[e][3] * vt);
    res.loading_mva[e] = std::max(std::abs(sf), std::abs(st)) * kMvaBase;
  }
  return res;
}

double AcNetwork::overload_energy(const AcCaseResult& r) const {  // ac_validator.cpp:274-279
  double s = 0.0;
  for (std::size_t e = 0; e < grid_->branches.size(); ++e)
    s += positive_part(r.loading_mva[e] - grid_->branches[e].flow_limit);
  return s;
}

int AcNetwork::critical_count(const AcCaseResult& r) const {  // ac_validator.cpp:281-286
  int c = 0;
  for (std::size_t e = 0; e < grid_->branches.size(); ++e) c += r.loading_mva[e] > grid_->branches[e].flow_limit;
  return c;
}

AcCaseResult ac_power_flow(const GridModel& grid, const AppliedTopology& topology, AcConfig config) {
  return AcNetwork(grid, topology, config).run_case(-1);
}

std::string to_string(RejectionReason r) {  // ac_validator.cpp:295-311
  switch (r) {
    case RejectionReason::None: return "none";
    case RejectionReason::Nonconvergence: return "nonconvergence";
    case RejectionReason::OverloadNotImproved: return "overload_not_improved";
    case RejectionReason::CriticalCountIncreased: return "critical_count_increased";
    case RejectionReason::EliminatedSimilar: return "eliminated_similar";
    case RejectionReason::EliminatedDominated: return "eliminated_dominated";
    case RejectionReason::EliminatedBelowThreshold: return "eliminated_below_threshold";
  }
  return "none";
}

// Baseline AC metrics of the unchanged grid (ac_validator.cpp:313-343): the
// base case, then every contingency; lambda_o and the critical count come from
// the per-branch maximum loading over the converged contingencies.
AcValidator::AcValidator(const GridModel& grid, const ActionSet& actions, const DcContext& dc, AcConfig config)
    : grid_(&grid), actions_(&actions), cfg_(config) {
  pre_fitness_ = dc.pre_optimization_score().fitness;
  const AcNetwork net(grid, apply_genome(grid, actions, Genome::empty(0, 0)), cfg_);
  const AcCaseResult base = net.run_case(-1);
  base_converged_ = base.converged;
  base_energy_ = base.converged ? net.overload_energy(base) : 0.0;
  const int E = static_cast<int>(grid.branches.size());
  const int K = static_cast<int>(grid.contingencies.size());
  Vec peak(E, 0.0);
  case_converged_.assign(K, 0);
  case_energy_.assign(K, 0.0);
  for (int k = 0; k < K; ++k) {
    const AcCaseResult r = net.run_case(k);
    case_converged_[k] = r.converged;
    if (!r.converged) continue;
    case_energy_[k] = net.overload_energy(r);
    for (int e = 0; e < E; ++e) peak[e] = std::max(peak[e], r.loading_mva[e]);
  }
  for (int e = 0; e < E; ++e) {
    base_lambda_o_ += positive_part(peak[e] - grid.branches[e].flow_limit);
    base_critical_ += peak[e] > grid.branches[e].flow_limit;
  }
}

// ac_validator.cpp:345-397
EliminationOutcome AcValidator::eliminate(const std::vector<Candidate>& cands) const {
  const double eps = cfg_.dominance_fitness_frac * std::abs(pre_fitness_);
  const double theta = cfg_.improvement_threshold_frac * std::abs(pre_fitness_);
  auto swd = [](const ScoreVector& s) { return s.lambda_d + s.lambda_s + s.lambda_r; };
  EliminationOutcome out;
  for (int i = 0; i < static_cast<int>(cands.size()); ++i) {
    const Candidate& c = cands[i];
    const int my_swd = swd(c.dc_score);
    auto dominated_by = [&](int other_swd, double other_fit) {
      return other_swd < my_swd && other_fit >= c.dc_score.fitness - eps;
    };
    RejectionReason why = RejectionReason::None;
    for (const Validated& v : validated_)
      if (genome_distance(c.genome, v.genome) <= cfg_.similarity_distance) {
        why = RejectionReason::EliminatedSimilar;
        break;
      }
    if (why == RejectionReason::None) {
      for (const Candidate& o : cands)
        if (dominated_by(swd(o.dc_score), o.dc_score.fitness)) {
          why = RejectionReason::EliminatedDominated;
          break;
        }
    }
    if (why == RejectionReason::None) {
      for (const Validated& v : validated_)
        if (dominated_by(v.swd, v.fitness)) {
          why = RejectionReason::EliminatedDominated;
          break;
        }
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

// ac_validator.cpp:399-425
RejectionReason AcValidator::worst_k_check(const Genome& genome, const ScoreVector& dc) const {
  const AcNetwork net(*grid_, apply_genome(*grid_, *actions_, genome), cfg_);
  const AcCaseResult base = net.run_case(-1);
  if (!base.converged) return RejectionReason::Nonconvergence;
  if (dc.worst_contingencies.empty()) return RejectionReason::None;
  double mine = net.overload_energy(base), ref = base_energy_;
  int failed = 0;
  for (const auto& wc : dc.worst_contingencies) {
    const int k = wc.first;
    const AcCaseResult r = net.run_case(k);
    if (!r.converged) {
      if (++failed > cfg_.worst_k_nonconverged) return RejectionReason::Nonconvergence;
      continue;
    }
    if (!case_converged_[k]) continue;
    mine += net.overload_energy(r);
    ref += case_energy_[k];
  }
  if (base_converged_ && mine >= ref) return RejectionReason::OverloadNotImproved;
  return RejectionReason::None;
}

// ac_validator.cpp:427-473
ValidationRecord AcValidator::full_validation(const Genome& genome, const ScoreVector& dc) const {
  ValidationRecord rec;
  rec.genome = genome;
  rec.dc_score = dc;
  rec.stage = ValidationStage::FullN1;
  const AcNetwork net(*grid_, apply_genome(*grid_, *actions_, genome), cfg_);
  const AcCaseResult base = net.run_case(-1);
  const int K = static_cast<int>(grid_->contingencies.size());
  const int E = static_cast<int>(grid_->branches.size());
  int failed = 0;
  Vec peak(E, 0.0);
  for (int k = 0; k < K; ++k) {
    const AcCaseResult r = net.run_case(k);
    if (!r.converged) {
      ++failed;
      continue;
    }
    for (int e = 0; e < E; ++e) peak[e] = std::max(peak[e], r.loading_mva[e]);
  }
  if (!base.converged || failed > cfg_.nonconverged_fraction * K) {
    rec.reason = RejectionReason::Nonconvergence;
    return rec;
  }
  double lo = 0.0;
  int crit = 0;
  for (int e = 0; e < E; ++e) {
    lo += positive_part(peak[e] - grid_->branches[e].flow_limit);
    crit += peak[e] > grid_->branches[e].flow_limit;
  }
  rec.ac_lambda_o = lo;
  if (!(lo < base_lambda_o_)) {
    rec.reason = RejectionReason::OverloadNotImproved;
    return rec;
  }
  if (crit > base_critical_) {
    rec.reason = RejectionReason::CriticalCountIncreased;
    return rec;
  }
  rec.accepted = true;
  return rec;
}

// ac_validator.cpp:475-495
ValidationRecord AcValidator::validate(const Candidate& c) {
  validated_.push_back({c.genome, c.dc_score.lambda_d + c.dc_score.lambda_s + c.dc_score.lambda_r, c.dc_score.fitness});
  const RejectionReason early = worst_k_check(c.genome, c.dc_score);
  ValidationRecord rec;
  if (early != RejectionReason::None) {
    rec.genome = c.genome;
    rec.dc_score = c.dc_score;
    rec.stage = ValidationStage::WorstK;
    rec.reason = early;
  } else {
    rec = full_validation(c.genome, c.dc_score);
  }
  records_.push_back(rec);
  return rec;
}

void AcValidator::record_elimination(const Candidate& c, RejectionReason reason) {
  ValidationRecord rec;
  rec.genome = c.genome;
  rec.dc_score = c.dc_score;
  rec.reason = reason;
  records_.push_back(rec);
}

// ac_validator.cpp:497-534
std::string record_to_json(const ValidationRecord& r, const GridModel& grid, const ActionSet& actions) {
  nlohmann::ordered_json j;
  j["actions"] = nlohmann::ordered_json::array();
  for (int a : r.genome.action_ids()) j["actions"].push_back(a);
  j["disconnections"] = nlohmann::ordered_json::array();
  for (int d : r.genome.disconnection_ids()) j["disconnections"].push_back(grid.branches[actions.disconnectables[d]].id);
  j["lambda_d"] = r.dc_score.lambda_d;
  j["lambda_s"] = r.dc_score.lambda_s;
  j["lambda_r"] = r.dc_score.lambda_r;
  j["dc_fitness"] = std::isfinite(r.dc_score.fitness) ? r.dc_score.fitness : -1e30;
  j["dc_lambda_o"] = r.dc_score.lambda_o;
  j["stage"] = r.stage == ValidationStage::None ? "eliminated" : r.stage == ValidationStage::WorstK ? "worst_k" : "full_n1";
  j["verdict"] = r.accepted ? "accepted" : "rejected";
  j["reason"] = r.accepted ? "" : to_string(r.reason);
  j["ac_lambda_o"] = r.ac_lambda_o;
  return j.dump();
}

}  // namespace oracle
