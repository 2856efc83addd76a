// C++ drop-in test: drives the engine through include/topopt_b200.hpp, the
// C++ surface that mirrors the reference's (dc_engine.hpp:95-150,
// qd_optimizer.hpp:116-118, grid_model.hpp:130-139, importer.hpp:80-94), the
// way a reference caller would after switching namespaces.
//
//   dropin_test host  GOLDEN_JSON          # no GPU: model, import, cache, errors
//   dropin_test gpu   GOLDEN_JSON OUT_JSON # evaluate vs the golden vectors,
//                                          # evaluate_flows, mixed slot counts,
//                                          # run_optimizer (sink, stop) -> OUT_JSON
//
// The golden vectors (tests/golden/grid14_congested_golden.json) are pinned
// to the oracle by tests/test_golden.py; tests/test_cpp_dropin.py runs this
// binary and compares OUT_JSON's optimizer run with the oracle's run_optimizer.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <nlohmann/json.hpp>
#include <sstream>
#include <string>
#include <vector>

#include "topopt_b200.hpp"

namespace tb = topopt::b200;
using json = nlohmann::json;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_fail;                                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
    }                                                                                 \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::string slurp(const std::filesystem::path& p) {
  std::ifstream in(p);
  std::stringstream b;
  b << in.rdbuf();
  return b.str();
}

// the golden file is written by Python's json (islanded fitness = -Infinity,
// not JSON): read non-finite numbers as null
static json parse_golden(const std::filesystem::path& p) {
  std::string t = slurp(p);
  for (const std::string tok : {"-Infinity", "Infinity", "NaN"})
    for (size_t at = t.find(tok); at != std::string::npos; at = t.find(tok, at)) t.replace(at, tok.size(), "null");
  return json::parse(t);
}

static bool close(double a, double b, double tol = 1e-9) {
  return std::abs(a - b) <= tol * std::max(1.0, std::abs(b));
}

static void host_checks(const std::filesystem::path& golden) {
  const json gold = parse_golden(golden);
  const auto grid_path = golden.parent_path() / gold["grid"].get<std::string>();
  const tb::GridModel g = tb::load_grid(grid_path);
  CHECK(g.n_nodes() == 14 && g.n_branches() == 20);
  CHECK(g.n_contingencies() == 10 && g.n_busbar_outages() == 1);
  const tb::ActionSet a = tb::build_action_set(g);
  CHECK(a.n_actions() > 0 && a.n_disconnectables() > 0);
  // canonical dump / hash are deterministic and the cache round-trips (importer.cpp:407-479)
  CHECK(tb::grid_content_hash(g) == tb::grid_content_hash(tb::grid_from_json_text(tb::grid_to_json_text(g))));
  const auto cache = std::filesystem::temp_directory_path() / "topopt_b200_dropin_actions.json";
  tb::save_action_set(a, g, cache);
  auto back = tb::load_action_set(g, cache);
  CHECK(back.has_value() && back->n_actions() == a.n_actions());
  for (int i = 0; back && i < a.n_actions(); ++i) CHECK(back->substation_of(i) == a.substation_of(i));
  const tb::GridModel other = tb::load_grid(golden.parent_path() / "data" / "grid14.json");
  CHECK(!tb::load_action_set(other, cache).has_value());  // key mismatch -> nothing
  CHECK(!tb::load_action_set(g, "/nonexistent/cache.json").has_value());
  std::filesystem::remove(cache);
  // genome helpers (genome.cpp:10-74)
  tb::Genome x{{3, -1, 1}, {-1, 0}}, y{{1, 3, -1}, {0, -1}};
  CHECK(x == y && x.canonical_key() == "a:1,3,d:0," && x.split_count() == 2 && x.disconnection_count() == 1);
  CHECK(tb::genome_distance(x, tb::Genome{{1, -1, -1}, {-1, -1}}) == 2);
  CHECK(tb::genome_valid(tb::Genome::empty(3, 2), a));
  CHECK(!tb::genome_valid(tb::Genome{{a.n_actions(), -1, -1}, {-1, -1}}, a));
  // descriptor_to_cell (qd_optimizer.cpp:12-17) KATs
  tb::QdConfig q;
  CHECK(tb::cell_count(q) == 552);
  CHECK(tb::descriptor_to_cell(0, 0, 0, q) == 0 && tb::descriptor_to_cell(1, 2, 3, q) == 1 + 3 * (2 + 4 * 3));
  CHECK(tb::descriptor_to_cell(9, 9, 99, q) == 551);
  // error kinds (errors.hpp:9-34), each status its own exception type
  CHECK(throws<tb::ParseError>([] { tb::grid_from_json_text("{not json"); }));
  CHECK(throws<tb::ParseError>([] { tb::grid_from_json_text(R"({"nodes": []})"); }));
  CHECK(throws<tb::IoError>([] { tb::load_grid("/nonexistent/grid.json"); }));
  json bad = json::parse(slurp(grid_path));
  bad["branches"][0]["to"] = "nowhere";
  CHECK(throws<tb::ValidationError>([&] { tb::grid_from_json_text(bad.dump()); }));
  json isl = json::parse(slurp(grid_path));
  // a contingency on the bridge b14 disconnects the base case (grid14.json: b14 is a bridge)
  std::string bridge;
  for (const auto& b : isl["branches"])
    if (b["id"] == "b14") bridge = "b14";
  if (!bridge.empty()) {
    isl["contingencies"].push_back({{"id", "c_bridge"}, {"branches", {bridge}}, {"injections", json::array()}});
    CHECK(throws<tb::IslandedContingency>([&] { tb::grid_from_json_text(isl.dump()); }));
  }
}

static void gpu_checks(const std::filesystem::path& golden, const std::filesystem::path& out_path) {
  const json gold = parse_golden(golden);
  const tb::GridModel g = tb::load_grid(golden.parent_path() / gold["grid"].get<std::string>());
  const tb::ActionSet a = tb::build_action_set(g);
  const tb::DcContext ctx(g, a);
  const int na = gold["n_a"];
  std::vector<tb::Genome> gs;
  for (const auto& row : gold["genomes"]) {
    std::vector<int> v = row.get<std::vector<int>>();
    gs.push_back({{v.begin(), v.begin() + na}, {v.begin() + na, v.end()}});
  }
  // DcContext::evaluate_batch vs the golden scores (dc_engine.cpp:424-468)
  const std::vector<tb::ScoreVector> sc = ctx.evaluate_batch(gs, 64);
  CHECK(sc.size() == gs.size());
  std::vector<double> lim;
  {
    const auto& d = g.desc();
    lim.assign(d.branch_limit, d.branch_limit + d.n_branches);
  }
  int knife_lanes = 0;
  for (size_t i = 0; i < gs.size(); ++i) {
    const json& s = gold["scores"][i];
    CHECK(sc[i].islanded == (s["islanded"].get<int>() != 0));
    CHECK(sc[i].lambda_d == s["lambda_d"] && sc[i].lambda_s == s["lambda_s"] && sc[i].lambda_r == s["lambda_r"]);
    if (sc[i].islanded) {
      CHECK(std::isinf(sc[i].fitness) && sc[i].fitness < 0);
      continue;
    }
    CHECK(close(sc[i].lambda_o, s["lambda_o"]));
    CHECK(close(sc[i].lambda_b, s["lambda_b"]));
    bool knife = false;
    const auto fm = s["fmax"].get<std::vector<double>>();
    for (size_t e = 0; e < fm.size(); ++e) knife |= std::abs(fm[e] - lim[e]) <= 1e-9 * std::max(1.0, lim[e]);
    if (sc[i].lambda_c == s["lambda_c"] && sc[i].lambda_c0 == s["lambda_c0"])
      CHECK(close(sc[i].fitness, s["fitness"]));
    else {
      CHECK(knife);
      ++knife_lanes;
    }
  }
  // evaluate == evaluate_batch; evaluate_flows gives the golden FlowResult
  for (size_t i = 0; i < gs.size(); i += 7) {
    const tb::ScoreVector one = ctx.evaluate(gs[i]);
    CHECK(one.fitness == sc[i].fitness || (std::isinf(one.fitness) && std::isinf(sc[i].fitness)));
    if (sc[i].islanded) continue;
    const auto [fr, s1] = ctx.evaluate_flows(gs[i]);
    const auto base = gold["scores"][i]["base"].get<std::vector<double>>();
    const auto fmax = gold["scores"][i]["fmax"].get<std::vector<double>>();
    for (size_t e = 0; e < base.size(); ++e) {
      CHECK(std::abs(fr.base[e] - base[e]) <= 1e-9 * (1.0 + std::abs(base[e])));
      CHECK(std::abs(fr.max_contingency[e] - fmax[e]) <= 1e-9 * (1.0 + std::abs(fmax[e])));
    }
    CHECK(close(s1.lambda_o, sc[i].lambda_o));
  }
  // mixed slot counts in one batch (vector<Genome> allows them): padded with
  // empty slots, same scores as the uniform genomes
  std::vector<tb::Genome> mixed;
  for (size_t i = 0; i < 12; ++i) {
    tb::Genome m = gs[i];
    while (!m.action_slots.empty() && m.action_slots.back() < 0) m.action_slots.pop_back();
    while (!m.disconnection_slots.empty() && m.disconnection_slots.back() < 0) m.disconnection_slots.pop_back();
    mixed.push_back(m);
  }
  const auto ms = ctx.evaluate_batch(mixed, 0);
  for (size_t i = 0; i < mixed.size(); ++i)
    CHECK(ms[i].fitness == sc[i].fitness || (std::isinf(ms[i].fitness) && std::isinf(sc[i].fitness)));
  // pre-optimization score (dc_engine.cpp:137-144): the empty genome's score
  CHECK(close(ctx.pre_optimization_score().fitness, sc[0].fitness) && ctx.lambda_b_pre() > 0.0);

  // run_optimizer (qd_optimizer.cpp:344-417) with a sink; the caller compares with the oracle
  tb::QdConfig q;
  q.seed = 1;
  q.batch_size = 64;
  q.iters_per_epoch = 7;
  q.max_evaluations = 3201;
  std::vector<tb::RepertoireSnapshot> snaps;
  const tb::OptimizerResult res = tb::run_optimizer(ctx, q, [&](tb::RepertoireSnapshot s) { snaps.push_back(std::move(s)); });
  CHECK(!snaps.empty() && snaps.back().final);
  CHECK(res.stats.evaluations == 3201 && res.stats.epochs == static_cast<int>(snaps.size()));
  CHECK(static_cast<int>(res.stats.fitness_trace.size()) == res.stats.epochs);
  CHECK(res.repertoire.total_size() == static_cast<int>(snaps.back().entries.size()));
  CHECK(res.repertoire.best_fitness() == snaps.back().best_fitness);
  for (const auto& e : snaps.back().entries)
    CHECK(e.cell == tb::descriptor_to_cell(e.score.lambda_d, e.score.lambda_s, e.score.lambda_r, q));
  json out;
  out["evaluations"] = res.stats.evaluations;
  out["epochs"] = res.stats.epochs;
  out["best_fitness"] = res.repertoire.best_fitness();
  out["n_snapshots"] = snaps.size();
  out["knife_lanes"] = knife_lanes;
  // stop flag (std::atomic<bool>*, qd_optimizer.hpp:116-118): set from the sink after the second epoch
  std::atomic<bool> stop{false};
  int seen = 0;
  tb::QdConfig q2 = q;
  q2.max_evaluations = -1;
  q2.iters_per_epoch = 2;
  const auto r2 = tb::run_optimizer(ctx, q2, [&](tb::RepertoireSnapshot) {
    if (++seen == 2) stop = true;
  }, &stop);
  // the flag is polled before every generation while the sink of an epoch
  // runs beside the next one (async snapshot copy): the run stops within a few
  // epochs of the request, never before it
  CHECK(r2.stats.epochs >= 2 && seen >= 2);
  out["stopped_epochs"] = r2.stats.epochs;
  // ConfigError where the reference raises it (qd_optimizer.cpp:347)
  tb::QdConfig bad = q;
  bad.batch_size = 0;
  CHECK(throws<tb::ConfigError>([&] { tb::run_optimizer(ctx, bad, {}); }));
  // a sink exception propagates to the caller (no exception crosses the C ABI)
  CHECK(throws<std::logic_error>([&] { tb::run_optimizer(ctx, q, [](tb::RepertoireSnapshot) { throw std::logic_error("x"); }); }));
  // AcValidator (ac_validator.hpp:93-140) on the GPU: baseline, worst-k and full
  // N-1 verdicts of the golden genomes (compared with the oracle by the caller),
  // the unchanged topology never improves on itself, validate_queue == stages
  {
    tb::AcValidator val(g, a, ctx);
    CHECK(val.baseline_lambda_o() > 0.0 && val.baseline_critical_count() >= 0);
    std::vector<tb::Candidate> cs;
    for (size_t i = 0; i < gs.size(); ++i) cs.push_back({gs[i], sc[i]});
    const auto wk = val.worst_k_check(cs);
    const auto full = val.full_validation(cs);
    CHECK(wk.size() == cs.size() && full.size() == cs.size());
    CHECK(val.worst_k_check(tb::Genome::empty(3, 2), sc[0]) == tb::RejectionReason::OverloadNotImproved);
    const tb::AcCaseResult base = val.run_case(tb::Genome::empty(3, 2), -1);
    CHECK(base.converged && base.iterations > 0 && static_cast<int>(base.loading_mva.size()) == g.n_branches());
    const auto recs = val.validate_queue(cs);
    for (size_t i = 0; i < cs.size(); ++i) {
      if (wk[i] == tb::RejectionReason::None)
        CHECK(recs[i].stage == tb::ValidationStage::FullN1 && recs[i].reason == full[i].reason);
      else
        CHECK(recs[i].stage == tb::ValidationStage::WorstK && recs[i].reason == wk[i]);
    }
    CHECK(val.records().size() == cs.size());
    const json rj = json::parse(tb::record_to_json(full[0], g, a));
    CHECK(rj["stage"] == "full_n1" && rj.contains("ac_lambda_o") && rj.contains("verdict"));
    json acj;
    acj["baseline_lambda_o"] = val.baseline_lambda_o();
    acj["baseline_critical"] = val.baseline_critical_count();
    for (size_t i = 0; i < cs.size(); ++i) {
      acj["worst_k"].push_back(static_cast<int>(wk[i]));
      acj["full_reason"].push_back(static_cast<int>(full[i].reason));
      acj["full_lambda_o"].push_back(full[i].ac_lambda_o);
    }
    out["ac"] = acj;
  }
  std::ofstream(out_path) << out.dump() << "\n";
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s host|gpu GOLDEN_JSON [OUT_JSON]\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1];
  try {
    host_checks(argv[2]);
    if (mode == "gpu") gpu_checks(argv[2], argc > 3 ? argv[3] : "dropin_out.json");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught exception: %s\n", e.what());
    return 1;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
