// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// extern "C" surface so pytest / bench.py (cpu_baseline) can drive the oracle
// through ctypes. Structured results are returned as JSON text (oc_free them).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>

#include "fixtures.hpp"

using namespace oracle;
using json = nlohmann::json;

namespace {
thread_local std::string g_err;
char* dup_str(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 1;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const IslandedContingency& e) {
    g_err = e.what();
    return 3;
  } catch (const SingularSystem& e) {
    g_err = e.what();
    return 4;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}
struct Ctx {
  GridModel grid;
  ActionSet actions;
  std::unique_ptr<DcContext> dc;
};
Genome genome_at(const int32_t* g, int na, int nd, int i) {
  Genome out = Genome::empty(na, nd);
  for (int k = 0; k < na; ++k) out.action_slots[k] = g[i * (na + nd) + k];
  for (int k = 0; k < nd; ++k) out.disconnection_slots[k] = g[i * (na + nd) + na + k];
  return out;
}
}  // namespace

extern "C" {

struct oc_qd_config {
  int32_t n_a, n_d, batch_size, iters_per_epoch, cell_capacity;
  double mutation_mean;
  double p_action[4];
  double p_disc[4];
  double p_crossover_parent1;
  int32_t d_max, s_max, r_max;
  uint64_t seed;
  int64_t max_evaluations;
  double max_seconds;
};

static QdConfig to_qd(const oc_qd_config* c) {
  QdConfig q;
  q.n_a = c->n_a;
  q.n_d = c->n_d;
  q.batch_size = c->batch_size;
  q.iters_per_epoch = c->iters_per_epoch;
  q.cell_capacity = c->cell_capacity;
  q.mutation_mean = c->mutation_mean;
  for (int i = 0; i < 4; ++i) q.p_action[i] = c->p_action[i], q.p_disc[i] = c->p_disc[i];
  q.p_crossover_parent1 = c->p_crossover_parent1;
  q.d_max = c->d_max;
  q.s_max = c->s_max;
  q.r_max = c->r_max;
  q.seed = c->seed;
  q.max_evaluations = c->max_evaluations;
  q.max_seconds = c->max_seconds;
  return q;
}

const char* oc_last_error() { return g_err.c_str(); }
void oc_free(void* p) { std::free(p); }

// Grid + action set + DC context in one handle (the oracle's DcContext keeps
// non-owning pointers, dc_engine.hpp:130-131, so the handle owns both).
int oc_context_create(const char* grid_json, uint64_t enum_seed, int64_t enum_cap, double penalty, int worst_k,
                      double w_c0, double w_c, int variant, int threads, void** out) {
  return guarded([&] {
    auto c = std::make_unique<Ctx>();
    c->grid = grid_from_json_text(grid_json);
    EnumerationConfig ec;
    ec.seed = enum_seed;
    if (enum_cap > 0) ec.cap = enum_cap;
    c->actions = build_action_set(c->grid, ec);
    DcConfig dc;
    dc.islanding_penalty_mw = penalty;
    dc.worst_k = worst_k;
    dc.weight_c0 = w_c0;
    dc.weight_c = w_c;
    dc.fitness_variant = variant;
    dc.threads = threads;
    c->dc = std::make_unique<DcContext>(c->grid, c->actions, dc);
    *out = c.release();
  });
}

void oc_context_destroy(void* h) { delete static_cast<Ctx*>(h); }

// grid_to_json_text / grid_content_hash (grid_model.cpp:423-503) and the
// action cache text (importer.cpp:407-430) of the context's grid / action set
char* oc_grid_json(void* h) { return dup_str(grid_to_json_text(static_cast<Ctx*>(h)->grid)); }
uint64_t oc_grid_hash(void* h) { return grid_content_hash(static_cast<Ctx*>(h)->grid); }
// build_ptdf (importer.cpp:358-401) of the context's grid: out [E][N] row-major
int oc_build_ptdf(void* h, double* out) {
  return guarded([&] {
    const PTDFMatrix p = build_ptdf(static_cast<Ctx*>(h)->grid);
    const int E = p.sensitivities.rows, N = p.sensitivities.cols;
    for (int e = 0; e < E; ++e)
      for (int v = 0; v < N; ++v) out[static_cast<size_t>(e) * N + v] = p.sensitivities(e, v);
  });
}
char* oc_action_cache(void* h) {
  auto* c = static_cast<Ctx*>(h);
  return dup_str(action_set_to_json_text(c->actions, c->grid));
}
// load_action_set (importer.cpp:432-479) of `text` against the context's grid:
// number of actions, -1 when the cache is rejected (hash or ids)
int64_t oc_action_cache_load(void* h, const char* text) {
  auto* c = static_cast<Ctx*>(h);
  auto s = action_set_from_json_text(c->grid, text);
  return s ? static_cast<int64_t>(s->actions.size()) : -1;
}

// JSON: {"n_nodes","n_branches","n_contingencies","n_busbar_outages","n_actions",
//        "disconnectables":[...],"actions":[{substation,group,busbars,open_couplers,lambda_r}],
//        "station_ranges":{sub:[b,e]}, "pre_score":{...}, "lambda_b_pre"}
char* oc_context_info(void* h) {
  auto* c = static_cast<Ctx*>(h);
  json j;
  j["n_nodes"] = c->grid.nodes.size();
  j["n_branches"] = c->grid.branches.size();
  j["n_injections"] = c->grid.injections.size();
  j["n_contingencies"] = c->grid.contingencies.size();
  j["n_busbar_outages"] = c->grid.busbar_outages.size();
  j["n_actions"] = c->actions.actions.size();
  j["disconnectables"] = c->actions.disconnectables;
  j["actions"] = json::array();
  for (const Action& a : c->actions.actions) {
    std::vector<int> grp(a.group.begin(), a.group.end());
    j["actions"].push_back({{"substation", a.substation},
                            {"group", grp},
                            {"busbars", a.busbar_assignment},
                            {"open_couplers", a.open_couplers},
                            {"lambda_r", a.reassignment_distance}});
  }
  j["station_ranges"] = json::object();
  for (const auto& [s, r] : c->actions.station_ranges) j["station_ranges"][std::to_string(s)] = {r.first, r.second};
  const ScoreVector& p = c->dc->pre_optimization_score();
  j["pre_score"] = {{"lambda_o", p.lambda_o}, {"lambda_c", p.lambda_c}, {"lambda_c0", p.lambda_c0},
                    {"lambda_b", p.lambda_b}, {"fitness", p.fitness}};
  j["lambda_b_pre"] = c->dc->lambda_b_pre();
  return dup_str(j.dump());
}

// Scores n genomes (row-major [n][na+nd], -1 empty). Scalar outputs are arrays
// of length n; worst lists are [n][worst_k] (index -1 padded). Flow outputs are
// optional (NULL to skip): base/fmax/fbus [n][E], energy [n][K].
int oc_evaluate(void* h, const int32_t* genomes, int na, int nd, int n, double* lambda_o, int32_t* lambda_c,
                int32_t* lambda_c0, double* lambda_b, int32_t* lambda_d, int32_t* lambda_s, int32_t* lambda_r,
                double* fitness, uint8_t* islanded, int32_t* worst_idx, double* worst_val, int32_t* worst_n,
                double* base, double* fmax, double* fbus, double* energy, int32_t* islanded_outages,
                int32_t* islanded_busbar) {
  return guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    const int ne = static_cast<int>(c->grid.branches.size());
    const int nk = static_cast<int>(c->grid.contingencies.size());
    const int wk = c->dc->config().worst_k;
    int workers = c->dc->config().threads > 0 ? c->dc->config().threads : static_cast<int>(std::thread::hardware_concurrency());
    workers = std::max(1, std::min(workers, n));
    std::atomic<int> next{0};
    auto work = [&] {
      for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
        FlowResult fr;
        ScoreVector s = c->dc->evaluate_with_flows(genome_at(genomes, na, nd, i), &fr);
        lambda_o[i] = s.lambda_o;
        lambda_c[i] = s.lambda_c;
        lambda_c0[i] = s.lambda_c0;
        lambda_b[i] = s.lambda_b;
        lambda_d[i] = s.lambda_d;
        lambda_s[i] = s.lambda_s;
        lambda_r[i] = s.lambda_r;
        fitness[i] = s.fitness;
        islanded[i] = s.islanded;
        worst_n[i] = static_cast<int32_t>(s.worst_contingencies.size());
        for (int k = 0; k < wk; ++k) {
          const bool on = k < static_cast<int>(s.worst_contingencies.size());
          worst_idx[i * wk + k] = on ? s.worst_contingencies[k].first : -1;
          worst_val[i * wk + k] = on ? s.worst_contingencies[k].second : 0.0;
        }
        const bool have = !s.islanded;
        for (int e = 0; e < ne; ++e) {
          if (base) base[static_cast<std::size_t>(i) * ne + e] = have ? fr.base[e] : 0.0;
          if (fmax) fmax[static_cast<std::size_t>(i) * ne + e] = have ? fr.max_contingency[e] : 0.0;
          if (fbus) fbus[static_cast<std::size_t>(i) * ne + e] = have ? fr.max_busbar[e] : 0.0;
        }
        if (energy)
          for (int k = 0; k < nk; ++k) energy[static_cast<std::size_t>(i) * nk + k] = have ? fr.outage_energy[k] : 0.0;
        if (islanded_outages) islanded_outages[i] = have ? fr.islanded_outages : 0;
        if (islanded_busbar) islanded_busbar[i] = have ? fr.islanded_busbar_outages : 0;
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < workers; ++w) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
  });
}

// Wall time of DcContext::evaluate_batch over `reps` passes (the reference's
// own threaded fan-out, dc_engine.cpp:439-468): the CPU baseline leg.
double oc_time_evaluate_batch(void* h, const int32_t* genomes, int na, int nd, int n, int reps) {
  auto* c = static_cast<Ctx*>(h);
  std::vector<Genome> batch;
  for (int i = 0; i < n; ++i) batch.push_back(genome_at(genomes, na, nd, i));
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) c->dc->evaluate_batch(batch, n);
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Reference-RNG replay of one lane's operator (qd_optimizer.cpp:380-395): for
// mutation lanes parents[0] is used, crossover uses both. seed is the lane
// seed (derive_seed(seed, iter, lane+1)); the parent index draws are NOT made
// here (the caller passes parents directly), matching mutate()/crossover().
int oc_mutate(void* h, const oc_qd_config* cfg, const int32_t* parent, uint64_t seed, int32_t* child, int32_t* ops,
              int32_t* n_ops) {
  return guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    QdConfig q = to_qd(cfg);
    Rng rng(seed);
    MutationTrace tr;
    Genome k = mutate(genome_at(parent, q.n_a, q.n_d, 0), c->actions, q, rng, &tr);
    for (int i = 0; i < q.n_a; ++i) child[i] = k.action_slots[i];
    for (int i = 0; i < q.n_d; ++i) child[q.n_a + i] = k.disconnection_slots[i];
    int m = 0;
    for (auto op : tr.action_ops) ops[m++] = static_cast<int>(op);
    for (auto op : tr.disconnection_ops) ops[m++] = 10 + static_cast<int>(op);
    *n_ops = m;
  });
}

int oc_crossover(void* h, const oc_qd_config* cfg, const int32_t* p1, const int32_t* p2, uint64_t seed, int32_t* child) {
  return guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    QdConfig q = to_qd(cfg);
    Rng rng(seed);
    Genome k = crossover(genome_at(p1, q.n_a, q.n_d, 0), genome_at(p2, q.n_a, q.n_d, 0), c->actions, q, rng);
    for (int i = 0; i < q.n_a; ++i) child[i] = k.action_slots[i];
    for (int i = 0; i < q.n_d; ++i) child[q.n_a + i] = k.disconnection_slots[i];
  });
}

// Full run_optimizer; returns JSON {"stats":{evaluations,epochs,fitness_trace},
// "snapshots":[{epoch,evaluations,best_fitness,final,entries:[[cell,[genome],fitness,ld,ls,lr,lo,lc,lc0,lb]]}]}
// (only the last snapshot's entries unless all_snapshots != 0).
char* oc_run_optimizer(void* h, const oc_qd_config* cfg, int all_snapshots) {
  char* out = nullptr;
  int rc = guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    QdConfig q = to_qd(cfg);
    json snaps = json::array();
    auto entries = [](const RepertoireSnapshot& s) {
      json e = json::array();
      for (const auto& x : s.entries) {
        std::vector<int> g = x.genome.action_slots;
        g.insert(g.end(), x.genome.disconnection_slots.begin(), x.genome.disconnection_slots.end());
        e.push_back({x.cell, g, x.score.fitness, x.score.lambda_d, x.score.lambda_s, x.score.lambda_r, x.score.lambda_o,
                     x.score.lambda_c, x.score.lambda_c0, x.score.lambda_b});
      }
      return e;
    };
    std::vector<RepertoireSnapshot> all;
    auto r = run_optimizer(*c->dc, q, [&](RepertoireSnapshot s) { all.push_back(std::move(s)); });
    for (std::size_t i = 0; i < all.size(); ++i) {
      const auto& s = all[i];
      json js = {{"epoch", s.epoch}, {"evaluations", s.evaluations}, {"best_fitness", s.best_fitness}, {"final", s.final}};
      if (all_snapshots || i + 1 == all.size()) js["entries"] = entries(s);
      snaps.push_back(js);
    }
    json j;
    j["stats"] = {{"evaluations", r.stats.evaluations}, {"epochs", r.stats.epochs}, {"fitness_trace", r.stats.fitness_trace}};
    j["snapshots"] = snaps;
    out = dup_str(j.dump());
  });
  return rc == 0 ? out : nullptr;
}

// run_optimizer with a per-iteration trace: JSON {"iters":[{"it":i,"genomes":[[..]..],
// "scores":[[fitness,ld,ls,lr,lo,lc,lc0,lb,worst_n,[idx..],[val..]]..]}], "stats":{...},
// "final":[[cell,[genome],fitness]...]}
char* oc_run_optimizer_trace(void* h, const oc_qd_config* cfg) {
  char* out = nullptr;
  int rc = guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    QdConfig q = to_qd(cfg);
    json iters = json::array();
    IterationTrace tr = [&](std::int64_t it, const std::vector<Genome>& kids, const std::vector<ScoreVector>& sc) {
      json gs = json::array(), ss = json::array();
      for (std::size_t i = 0; i < kids.size(); ++i) {
        std::vector<int> g = kids[i].action_slots;
        g.insert(g.end(), kids[i].disconnection_slots.begin(), kids[i].disconnection_slots.end());
        gs.push_back(g);
        std::vector<int> wi;
        std::vector<double> wv;
        for (const auto& [k, v] : sc[i].worst_contingencies) wi.push_back(k), wv.push_back(v);
        const double fit = std::isfinite(sc[i].fitness) ? sc[i].fitness : -1e300;
        ss.push_back({fit, sc[i].lambda_d, sc[i].lambda_s, sc[i].lambda_r, sc[i].lambda_o, sc[i].lambda_c,
                      sc[i].lambda_c0, sc[i].lambda_b, static_cast<int>(wi.size()), wi, wv});
      }
      iters.push_back({{"it", it}, {"genomes", gs}, {"scores", ss}});
    };
    auto r = run_optimizer(*c->dc, q, nullptr, nullptr, &tr);
    json fin = json::array();
    for (int cell = 0; cell < r.repertoire.n_cells(); ++cell)
      for (const auto& e : r.repertoire.cell(cell)) {
        std::vector<int> g = e.genome.action_slots;
        g.insert(g.end(), e.genome.disconnection_slots.begin(), e.genome.disconnection_slots.end());
        fin.push_back({cell, g, e.score.fitness});
      }
    json j;
    j["iters"] = iters;
    j["final"] = fin;
    j["stats"] = {{"evaluations", r.stats.evaluations}, {"epochs", r.stats.epochs}};
    out = dup_str(j.dump());
  });
  return rc == 0 ? out : nullptr;
}

// run_optimizer with a wall-clock stamp (seconds since the call) after each
// iteration's inserts: the reference arm of bench.py times the reference's own
// MapElites loop per generation. Returns the number of stamps written.
int oc_run_optimizer_timed(void* h, const oc_qd_config* cfg, double* stamps, int cap, int64_t* evaluations) {
  int n = 0;
  int rc = guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    QdConfig q = to_qd(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    IterationTrace tr = [&](std::int64_t, const std::vector<Genome>&, const std::vector<ScoreVector>&) {
      if (n < cap) stamps[n++] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    auto r = run_optimizer(*c->dc, q, nullptr, nullptr, &tr);
    *evaluations = r.stats.evaluations;
  });
  return rc == 0 ? n : -1;
}

// Seeded fixtures (tests/helpers.hpp:435-581).
char* oc_random_grid_json(uint64_t seed, int n_nodes, int extra_edges, int n_outages, int n_stations, int multi,
                          int injection_outages, int busbar_outages) {
  fx::RandomGridOptions o;
  o.n_nodes = n_nodes;
  o.extra_edges = extra_edges;
  o.n_outages = n_outages;
  o.n_stations = n_stations;
  o.multi_branch_outages = multi;
  o.injection_outages = injection_outages;
  o.busbar_outages = busbar_outages;
  char* out = nullptr;
  int rc = guarded([&] { out = dup_str(fx::random_grid_json(seed, o).dump()); });
  return rc == 0 ? out : nullptr;
}

int oc_random_genomes(void* h, int na, int nd, uint64_t seed, int n, int32_t* out) {
  return guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    std::mt19937_64 rng(seed);
    for (int i = 0; i < n; ++i) {
      Genome g = fx::random_genome(c->actions, na, nd, rng);
      for (int k = 0; k < na; ++k) out[i * (na + nd) + k] = g.action_slots[k];
      for (int k = 0; k < nd; ++k) out[i * (na + nd) + na + k] = g.disconnection_slots[k];
    }
  });
}

// Rebuild-from-scratch flows of a genome topology (helpers.hpp:228-281); the
// test oracle that pins both the restated engine and the GPU path.
int oc_rebuild_flows(void* h, const int32_t* genome, int na, int nd, double* flows, int32_t* singular) {
  return guarded([&] {
    auto* c = static_cast<Ctx*>(h);
    auto m = fx::materialize(c->grid, c->actions, genome_at(genome, na, nd, 0));
    try {
      Vec f = fx::rebuild_flows(m);
      for (std::size_t e = 0; e < f.size(); ++e) flows[e] = f[e];
      *singular = 0;
    } catch (const SingularSystem&) {
      *singular = 1;
    }
  });
}


// ---- AC validation (ac_validator.cpp) --------------------------------------
// Cases (genome index, contingency or -1) of a genome batch on `threads` host
// threads; any output pointer may be null (loading [n][E], vm / va [n][N + na]).
int oc_ac_cases(void* h, double tol, int max_iter, const int32_t* genomes, int na, int nd, const int32_t* case_g,
                const int32_t* case_k, int n, int threads, uint8_t* conv, int32_t* iters, double* energy,
                int32_t* crit, double* loading, double* vm, double* va) {
  return guarded([&] {
    Ctx* c = static_cast<Ctx*>(h);
    AcConfig cfg;
    cfg.tolerance_pu = tol;
    cfg.max_iterations = max_iter;
    const int E = static_cast<int>(c->grid.branches.size());
    const int V = static_cast<int>(c->grid.nodes.size()) + na;
    std::atomic<int> next{0};
    auto work = [&] {
      for (int i; (i = next.fetch_add(1)) < n;) {
        const AcNetwork net(c->grid, apply_genome(c->grid, c->actions, genome_at(genomes, na, nd, case_g[i])), cfg);
        const AcCaseResult r = net.run_case(case_k[i]);
        if (conv) conv[i] = r.converged;
        if (iters) iters[i] = r.iterations;
        if (energy) energy[i] = r.converged ? net.overload_energy(r) : 0.0;
        if (crit) crit[i] = r.converged ? net.critical_count(r) : 0;
        if (loading) std::copy(r.loading_mva.begin(), r.loading_mva.end(), loading + static_cast<size_t>(i) * E);
        if (vm)
          for (int v = 0; v < V; ++v) {
            vm[static_cast<size_t>(i) * V + v] = v < static_cast<int>(r.vm_pu.size()) ? r.vm_pu[v] : 0.0;
            va[static_cast<size_t>(i) * V + v] = v < static_cast<int>(r.va_rad.size()) ? r.va_rad[v] : 0.0;
          }
      }
    };
    const int T = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
  });
}

struct OcAc {
  Ctx* ctx;
  std::unique_ptr<AcValidator> val;
};

int oc_ac_validator_create(void* h, double tol, int max_iter, int q, double frac, int sim, double dom, double thr,
                           void** out) {
  return guarded([&] {
    Ctx* c = static_cast<Ctx*>(h);
    AcConfig cfg;
    cfg.tolerance_pu = tol;
    cfg.max_iterations = max_iter;
    cfg.worst_k_nonconverged = q;
    cfg.nonconverged_fraction = frac;
    cfg.similarity_distance = sim;
    cfg.dominance_fitness_frac = dom;
    cfg.improvement_threshold_frac = thr;
    auto v = std::make_unique<OcAc>();
    v->ctx = c;
    v->val = std::make_unique<AcValidator>(c->grid, c->actions, *c->dc, cfg);
    *out = v.release();
  });
}

void oc_ac_validator_destroy(void* v) { delete static_cast<OcAc*>(v); }

// lambda_o, critical, base_converged, base_energy; per contingency converged / energy
int oc_ac_baseline(void* v, double* lambda_o, int32_t* crit, uint8_t* base_conv, double* base_energy,
                   uint8_t* case_conv, double* case_energy) {
  return guarded([&] {
    const AcValidator& a = *static_cast<OcAc*>(v)->val;
    *lambda_o = a.baseline_lambda_o();
    *crit = a.baseline_critical_count();
    *base_conv = a.baseline_base_converged();
    *base_energy = a.baseline_base_energy();
    for (std::size_t k = 0; k < a.baseline_case_converged().size(); ++k) {
      case_conv[k] = a.baseline_case_converged()[k];
      case_energy[k] = a.baseline_case_energy()[k];
    }
  });
}

// worst_k_check per genome; worst lists [n][stride] with lengths worst_n
int oc_ac_worst_k(void* v, const int32_t* genomes, int na, int nd, int n, const int32_t* worst_idx,
                  const int32_t* worst_n, int stride, int32_t* reason) {
  return guarded([&] {
    const AcValidator& a = *static_cast<OcAc*>(v)->val;
    for (int i = 0; i < n; ++i) {
      ScoreVector s;
      for (int j = 0; j < worst_n[i]; ++j) s.worst_contingencies.emplace_back(worst_idx[i * stride + j], 1.0);
      reason[i] = static_cast<int32_t>(a.worst_k_check(genome_at(genomes, na, nd, i), s));
    }
  });
}

// full_validation per genome
int oc_ac_full(void* v, const int32_t* genomes, int na, int nd, int n, int32_t* reason, uint8_t* accepted,
               double* lambda_o) {
  return guarded([&] {
    const AcValidator& a = *static_cast<OcAc*>(v)->val;
    for (int i = 0; i < n; ++i) {
      const ValidationRecord r = a.full_validation(genome_at(genomes, na, nd, i), ScoreVector{});
      reason[i] = static_cast<int32_t>(r.reason);
      accepted[i] = r.accepted;
      lambda_o[i] = r.ac_lambda_o;
    }
  });
}

// tests/helpers.hpp:83-103 mini_congestion_grid, serialized (grid_to_json_text)
char* oc_mini_congestion_json() { return dup_str(grid_to_json_text(oracle::fx::mini_congestion_grid())); }
}  // extern "C"
