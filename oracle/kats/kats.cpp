// CPU ORACLE KNOWN-ANSWER TESTS — TEST INFRASTRUCTURE ONLY.
//
// Pins the oracle restatement to the reference's own test expectations. Each
// block cites the reference test it re-checks (proj/tests/*.cpp). Runs as a
// plain binary (no doctest in this image): prints one line per check group and
// exits non-zero on any failure. Driven by tests/test_oracle_kats.py.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../src/fixtures.hpp"

using namespace oracle;
using namespace oracle::fx;

namespace {

int g_fail = 0, g_pass = 0;
std::string g_case;

void expect(bool ok, const std::string& what) {
  if (ok) {
    ++g_pass;
  } else {
    ++g_fail;
    std::printf("  FAIL [%s] %s\n", g_case.c_str(), what.c_str());
  }
}
bool near(double a, double b, double tol = 1e-9) { return std::abs(a - b) <= tol * std::max(1.0, std::abs(b)); }
template <class F>
bool throws(F&& f) {
  try {
    f();
  } catch (...) {
    return true;
  }
  return false;
}
template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}
double rel_err(const Vec& got, const Vec& want) {
  double w = 0;
  for (std::size_t i = 0; i < got.size(); ++i)
    w = std::max(w, std::abs(got[i] - want[i]) / std::max(1.0, std::abs(want[i])));
  return w;
}
double abs_err(const Vec& a, const Vec& b) {
  double w = 0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]));
  return w;
}
Vec mat_vec(const Mat& m, const Vec& v) {
  Vec o(m.rows, 0.0);
  for (int j = 0; j < m.cols; ++j)
    for (int i = 0; i < m.rows; ++i) o[i] += m(i, j) * v[j];
  return o;
}
Vec cabs(Vec v) {
  for (double& x : v) x = std::abs(x);
  return v;
}
void fold_max(Vec& acc, const Vec& v) {
  for (std::size_t i = 0; i < v.size(); ++i) acc[i] = std::max(acc[i], std::abs(v[i]));
}

std::string g_data;
GridModel data_grid(const char* name) { return load_grid(g_data + "/" + name); }

std::map<std::string, std::function<void()>>& registry() {
  static std::map<std::string, std::function<void()>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry()[n] = std::move(f); }
};
#define KAT(name) \
  static void name(); \
  static Reg reg_##name(#name, name); \
  static void name()

// ------------------------------------------------------------ grid model
// test_grid_model.cpp:15-150
KAT(grid_model_loading) {
  GridModel g = two_node_grid();
  expect(g.nodes.size() == 2 && g.branches.size() == 1 && g.injections.size() == 2, "two-node counts");
  expect(g.slack == g.node_index("b"), "two-node slack");
  json zero = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}}},
               {"branches", {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.0}, {"limit_mw", 100.0}}}},
               {"slack", "a"}};
  expect(throws_as<ValidationError>([&] { grid_from_json(zero); }), "zero reactance rejected");
  expect(throws_as<ParseError>([] { grid_from_json_text("{not json"); }), "bad json");
  expect(throws_as<ParseError>([] { grid_from_json_text("{\"nodes\": []}"); }), "missing branches");
  json miss = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}}}, {"branches", {{{"id", "ab"}, {"from", "a"}, {"to", "b"}}}},
               {"slack", "a"}};
  expect(throws_as<ParseError>([&] { grid_from_json(miss); }), "missing field");
  json isl = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}}},
              {"branches",
               {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
              {"contingencies", {{{"id", "o1"}, {"branches", {"ab"}}}}},
              {"slack", "a"}};
  expect(throws_as<IslandedContingency>([&] { grid_from_json(isl); }), "islanding contingency rejected");
  GridModel g14 = data_grid("grid14.json");
  expect(g14.nodes.size() == 14 && g14.branches.size() == 20 && g14.contingencies.size() == 19, "14-bus counts");
  expect(g14.slack == g14.node_index("1"), "14-bus slack");
}

KAT(grid_model_power_vector) {
  GridModel g = two_node_grid();
  Vec p = base_power_vector(g);
  expect(near(p[g.node_index("a")], 100.0) && near(p[g.node_index("b")], -100.0), "two-node vector");
  GridModel g14 = data_grid("grid14.json");
  Vec p14 = base_power_vector(g14);
  double s = 0;
  for (double v : p14) s += v;
  expect(std::abs(s) < 1e-9, "14-bus balances");
  expect(near(p14[g14.node_index("3")], -94.2), "14-bus bus 3");
  for (std::uint64_t seed = 1; seed <= 10; ++seed) {
    Vec pr = base_power_vector(random_grid(seed));
    double t = 0;
    for (double v : pr) t += v;
    expect(std::abs(t) < 1e-9, "random grid balances");
  }
}

KAT(grid_model_roundtrip) {
  for (std::uint64_t seed : {3u, 7u, 11u}) {
    GridModel g = random_grid(seed);
    GridModel h = grid_from_json_text(grid_to_json_text(g));
    expect(grid_to_json_text(h) == grid_to_json_text(g), "text round trip");
    expect(grid_content_hash(h) == grid_content_hash(g), "hash round trip");
  }
}

KAT(grid_model_implied_branches) {
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}}},
            {"branches",
             {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ad"}, {"from", "a"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
            {"injections", {{{"id", "g"}, {"node", "a"}, {"p_mw", 50.0}, {"kind", "generator"}}}},
            {"substations", json::array({station_json("a", {"ab", "ac", "ad", "g"}, {"B1", "B1", "B2", "B2"})})},
            {"busbar_outages",
             {{{"id", "bo1"}, {"substation", "a"}, {"busbar", "B1"}}, {{"id", "bo2"}, {"substation", "a"}, {"busbar", "B2"}}}},
            {"slack", "c"}};
  GridModel g = grid_from_json(j);
  const int ab = g.branch_index("ab"), ac = g.branch_index("ac"), ad = g.branch_index("ad");
  expect(g.implied_branches(g.busbar_outages[0]) == std::vector<int>{ab, ac, ad}, "default implies all");
  std::vector<int> asg = {0, 0, 1, 1}, open = {0};
  expect(g.implied_branches(g.busbar_outages[0], asg, open) == std::vector<int>{ab, ac}, "B1 side");
  expect(g.implied_branches(g.busbar_outages[1], asg, open) == std::vector<int>{ad}, "B2 side");
}

// ------------------------------------------------------------ importer
// test_importer.cpp:15-353
KAT(importer_bridges) {
  expect(find_bridges(dc_graph_from_grid(triangle_grid())).empty(), "triangle no bridges");
  for (std::uint64_t seed = 1; seed <= 15; ++seed) {
    RandomGridOptions o;
    o.n_nodes = 30;
    o.extra_edges = static_cast<int>(seed % 4) * 6;
    GridModel g = random_grid(seed, o);
    auto got = find_bridges(dc_graph_from_grid(g));
    expect(std::set<int>(got.begin(), got.end()) == oracle_bridges(static_cast<int>(g.nodes.size()), oracle_edges(g)),
           "bridges vs brute force seed " + std::to_string(seed));
  }
}

KAT(importer_disconnectables) {
  expect(enumerate_disconnectables(triangle_grid(100, 100, 100, {"ab"})).empty(), "triangle with outage");
  expect(enumerate_disconnectables(triangle_grid()).size() == 3, "triangle without outages");
  for (std::uint64_t seed = 21; seed <= 40; ++seed) {
    RandomGridOptions o;
    o.n_nodes = 18;
    o.extra_edges = 14;
    o.n_outages = static_cast<int>(seed % 8);
    o.multi_branch_outages = true;
    GridModel g = random_grid(seed, o);
    auto got = enumerate_disconnectables(g);
    expect(std::set<int>(got.begin(), got.end()) == oracle_disconnectables(g), "disconnectables seed " + std::to_string(seed));
  }
  GridModel g14 = data_grid("grid14.json");
  auto got = enumerate_disconnectables(g14);
  expect(std::set<int>(got.begin(), got.end()) == oracle_disconnectables(g14), "14-bus disconnectables");
  // acceptance.cpp:110-129 (criterion 3)
  for (std::uint64_t seed = 3000; seed < 3020; ++seed) {
    RandomGridOptions o;
    o.n_nodes = 14 + static_cast<int>(seed % 12);
    o.extra_edges = 10 + static_cast<int>(seed % 9);
    o.n_outages = static_cast<int>(seed % 21);
    o.multi_branch_outages = true;
    GridModel g = random_grid(seed, o);
    auto d = enumerate_disconnectables(g);
    expect(std::set<int>(d.begin(), d.end()) == oracle_disconnectables(g), "criterion 3 seed " + std::to_string(seed));
  }
}

KAT(importer_enumeration) {
  json tri = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}}},
              {"branches",
               {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
              {"substations", json::array({station_json("a", {"ab", "ac"}, {"B1", "B2"})})},
              {"slack", "c"}};
  auto a1 = enumerate_station_actions(grid_from_json(tri), 0);
  expect(a1.size() == 1 && a1[0].group == std::vector<char>{0, 1} && a1[0].reassignment_distance == 0 &&
             a1[0].open_couplers == std::vector<int>{0},
         "two terminals, split defaults");
  tri["substations"] = json::array({station_json("a", {"ab", "ac"}, {"B1", "B1"})});
  auto a2 = enumerate_station_actions(grid_from_json(tri), 0);
  expect(a2.size() == 1 && a2[0].reassignment_distance == 1, "two terminals, moved one");
  json star = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}, {{"id", "e"}}}},
               {"branches",
                {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "ad"}, {"from", "a"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "ae"}, {"from", "a"}, {"to", "e"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
                 {{"id", "de"}, {"from", "d"}, {"to", "e"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
               {"substations", json::array({station_json("a", {"ab", "ac", "ad", "ae"})})},
               {"slack", "c"}};
  expect(enumerate_station_actions(grid_from_json(star), 0).size() == 7, "four free terminals -> 7");
  // acceptance.cpp:131-169 (criterion 4)
  json star2 = star;
  star2["substations"][0]["terminals"][3] = {{"element", "ae"}, {"reachable", {"B1"}}, {"default", "B1"}};
  expect(enumerate_station_actions(grid_from_json(star2), 0).size() == 3, "constrained station -> 3 (acceptance.cpp:156-161)");
  GridModel rg = random_grid(99, {.n_nodes = 25, .extra_edges = 20, .n_stations = 3});
  EnumerationConfig ec;
  ec.seed = 42;
  ec.cap = 4;
  auto s1 = enumerate_station_actions(rg, 0, ec), s2 = enumerate_station_actions(rg, 0, ec);
  bool same = s1.size() == s2.size();
  for (std::size_t i = 0; same && i < s1.size(); ++i) same = s1[i].group == s2[i].group;
  expect(same && s1.size() <= 4, "downsampled enumeration deterministic");
}

KAT(importer_islanding_filter) {
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}}},
            {"branches",
             {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
            {"injections", {{{"id", "l"}, {"node", "a"}, {"p_mw", 30.0}, {"kind", "load"}}}},
            {"substations", json::array({station_json("a", {"ab", "ac", "l"})})},
            {"slack", "c"}};
  GridModel g = grid_from_json(j);
  Action bad{-1, 0, {0, 0, 1}, {0, 0, 1}, {0}, 0}, fine{-1, 0, {0, 1, 1}, {0, 1, 1}, {0}, 0};
  expect(!validate_action_islanding(g, bad), "stranded load rejected");
  expect(validate_action_islanding(g, fine), "branch + load accepted");
  for (std::uint64_t seed = 50; seed <= 58; ++seed) {
    GridModel rg = random_grid(seed, {.n_nodes = 16, .extra_edges = 10, .n_outages = 4, .n_stations = 2});
    for (int s = 0; s < static_cast<int>(rg.substations.size()); ++s) {
      const SubstationDetail& st = rg.substations[s];
      for (const Action& a : enumerate_station_actions(rg, s)) {
        const int n = static_cast<int>(rg.nodes.size());
        auto edges = oracle_edges(rg);
        bool used = false;
        for (int t = 0; t < static_cast<int>(st.terminals.size()); ++t) {
          if (!a.group[t]) continue;
          const Terminal& term = st.terminals[t];
          used = true;
          if (term.kind == TerminalKind::InjectionTerminal) continue;
          (term.kind == TerminalKind::BranchFrom ? edges[term.element_index].from : edges[term.element_index].to) = n;
        }
        const int nt = used ? n + 1 : n;
        bool ok = oracle_connected(nt, edges);
        for (const auto& c : rg.contingencies) {
          if (!ok) break;
          auto cut = edges;
          for (int e : c.branches) cut[e].active = false;
          ok = oracle_connected(nt, cut);
        }
        expect(validate_action_islanding(rg, a) == ok, "islanding vs BFS oracle");
        int moved = 0;
        for (int t = 0; t < static_cast<int>(st.terminals.size()); ++t)
          if (st.busbars[a.busbar_assignment[t]] != st.terminals[t].default_busbar) ++moved;
        expect(moved == a.reassignment_distance && a.group[0] == 0, "action invariants");
      }
    }
  }
}

KAT(importer_ptdf) {
  GridModel g2 = two_node_grid();
  PTDFMatrix p = build_ptdf(g2);
  expect(near(p.sensitivities(0, g2.node_index("a")), 1.0) && near(p.sensitivities(0, g2.node_index("b")), 0.0),
         "two-node ptdf");
  expect(near(mat_vec(p.sensitivities, base_power_vector(g2))[0], 100.0), "two-node flow");
  GridModel tri = triangle_grid();
  Vec f = mat_vec(build_ptdf(tri).sensitivities, base_power_vector(tri));
  expect(near(f[tri.branch_index("ab")], 30.0) && near(f[tri.branch_index("ac")], 60.0) &&
             near(f[tri.branch_index("bc")], 30.0),
         "triangle 30/60/30");
  GridModel g14 = data_grid("grid14.json");
  Vec p14 = base_power_vector(g14);
  expect(abs_err(mat_vec(build_ptdf(g14).sensitivities, p14), angle_flows(dc_graph_from_grid(g14), p14)) < 1e-9,
         "14-bus ptdf == angle flows");
  for (std::uint64_t seed = 60; seed <= 66; ++seed) {
    GridModel g = random_grid(seed);
    Vec pp = base_power_vector(g), ff = mat_vec(build_ptdf(g).sensitivities, pp);
    Vec res(g.nodes.size(), 0.0);
    for (int e = 0; e < static_cast<int>(g.branches.size()); ++e)
      res[g.branches[e].from] += ff[e], res[g.branches[e].to] -= ff[e];
    double w = 0;
    for (int v = 0; v < static_cast<int>(g.nodes.size()); ++v)
      if (v != g.slack) w = std::max(w, std::abs(res[v] - pp[v]));
    expect(w < 1e-9, "nodal balance");
  }
  DcGraph dg;
  dg.n_nodes = 3;
  dg.slack = 0;
  dg.edges.push_back({0, 1, 10.0, true});
  dg.edges.push_back({1, 2, 10.0, false});
  expect(throws_as<SingularSystem>([&] { build_ptdf(dg); }), "disconnected ptdf raises");
}

KAT(importer_cache) {
  GridModel g = random_grid(70, {.n_nodes = 20, .extra_edges = 14, .n_outages = 3, .n_stations = 2});
  ActionSet s = build_action_set(g);
  expect(!s.actions.empty(), "actions exist");
  int covered = 0;
  for (const auto& [st, r] : s.station_ranges) {
    for (int a = r.first; a < r.second; ++a) expect(s.actions[a].substation == st, "range station");
    covered += r.second - r.first;
  }
  expect(covered == static_cast<int>(s.actions.size()), "ranges partition ids");
  auto back = action_set_from_json_text(g, action_set_to_json_text(s, g));
  expect(back && back->actions.size() == s.actions.size() && back->disconnectables == s.disconnectables, "cache reload");
  GridModel other = random_grid(71, {.n_nodes = 20, .extra_edges = 14});
  expect(!action_set_from_json_text(other, action_set_to_json_text(s, g)), "cache rejects other grid");
}

// ------------------------------------------------------------ DC engine
// test_dc_engine.cpp:26-526
KAT(dc_operator_vs_rebuild) {
  {
    GridModel g = triangle_grid();
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    Vec base = mat_vec(build_ptdf(g).sensitivities, base_power_vector(g));
    expect(rel_err(ctx.apply_topology(Genome::empty(3, 2)).base_flows(), base) < 1e-12, "empty genome == ptdf");
    expect(s.disconnectables.size() == 3, "triangle disconnectables");
    for (int d = 0; d < 3; ++d) {
      Genome gg = Genome::empty(3, 2);
      gg.disconnection_slots[0] = d;
      FlowOperator op = ctx.apply_topology(gg);
      expect(!op.islanded() && rel_err(op.base_flows(), rebuild_flows(materialize(g, s, gg))) < 1e-10,
             "single disconnection vs rebuild");
    }
  }
  {
    GridModel g14 = data_grid("grid14.json");
    json doc = json::parse(grid_to_json_text(g14));
    std::vector<std::string> el;
    for (const Branch& b : g14.branches)
      if (g14.nodes[b.from].id == "4" || g14.nodes[b.to].id == "4") el.push_back(b.id);
    el.push_back("load4");
    doc["substations"] = json::array({station_json("4", el)});
    GridModel g = grid_from_json(doc);
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    std::mt19937_64 rng(7);
    int checked = 0;
    for (int t = 0; t < 40; ++t) {
      Genome gg = random_genome(s, 3, 2, rng);
      FlowOperator op = ctx.apply_topology(gg);
      MaterializedTopology m = materialize(g, s, gg);
      if (op.islanded()) {
        expect(throws_as<SingularSystem>([&] { rebuild_flows(m); }), "islanded => rebuild singular");
        continue;
      }
      expect(rel_err(op.base_flows(), rebuild_flows(m)) < 1e-8, "14-bus split+disc vs rebuild");
      ++checked;
    }
    expect(checked > 10, "14-bus enough non-islanded");
  }
  std::mt19937_64 rng(123);
  for (std::uint64_t seed = 200; seed < 215; ++seed) {
    RandomGridOptions o;
    o.n_nodes = 12 + static_cast<int>(seed % 40);
    o.extra_edges = 8 + static_cast<int>(seed % 11);
    o.n_outages = 4;
    o.n_stations = 3;
    GridModel g = random_grid(seed, o);
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    for (int t = 0; t < 10; ++t) {
      Genome gg = random_genome(s, 3, 2, rng);
      FlowOperator op = ctx.apply_topology(gg);
      MaterializedTopology m = materialize(g, s, gg);
      if (op.islanded()) {
        expect(throws_as<SingularSystem>([&] { rebuild_flows(m); }), "random islanded");
        continue;
      }
      expect(rel_err(op.base_flows(), rebuild_flows(m)) < 1e-8, "random grid vs rebuild");
    }
  }
}

KAT(dc_linearity) {
  GridModel g = random_grid(300, {.n_nodes = 24, .extra_edges = 14, .n_stations = 2});
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  std::mt19937_64 rng(31);
  Genome gg = random_genome(s, 3, 2, rng);
  FlowOperator op = ctx.apply_topology(gg);
  expect(!op.islanded(), "linearity genome not islanded");
  const int dim = static_cast<int>(g.nodes.size()) + op.extra_nodes();
  std::uniform_real_distribution<double> u(-50.0, 50.0);
  for (int t = 0; t < 5; ++t) {
    Vec p1(dim), p2(dim), ps(dim);
    for (int i = 0; i < dim; ++i) p1[i] = u(rng), p2[i] = u(rng);
    for (int i = 0; i < dim; ++i) ps[i] = p1[i] + p2[i];
    Vec a = op.flows(ps), b1 = op.flows(p1), b2 = op.flows(p2);
    for (std::size_t i = 0; i < b1.size(); ++i) b1[i] += b2[i];
    expect(abs_err(a, b1) < 1e-9, "superposition");
  }
}

KAT(dc_screening_basics) {
  {
    GridModel g = triangle_grid(50, 50, 100);
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    ScoreVector sc = ctx.evaluate(Genome::empty(3, 2));
    expect(near(sc.lambda_o, 0.0) && sc.lambda_c == 0 && sc.lambda_c0 == 1 && near(sc.fitness, -200.0),
           "no outages: base metrics only");
  }
  {
    GridModel g = triangle_grid(100, 100, 100, {"ab"});
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    FlowResult fr = ctx.screen_contingencies(ctx.apply_topology(Genome::empty(3, 2)));
    expect(near(fr.max_contingency[g.branch_index("ac")], 90.0) && near(fr.max_contingency[g.branch_index("ab")], 0.0) &&
               near(fr.outage_energy[0], 0.0),
           "triangle outage ab -> ac carries 90");
  }
  {
    // acceptance.cpp:90-108 (criterion 2) and test_dc_engine.cpp:153-169
    GridModel g = data_grid("grid14.json");
    ActionSet s;
    DcContext ctx(g, s);
    FlowResult fr = ctx.screen_contingencies(ctx.apply_topology(Genome::empty(3, 2)));
    MaterializedTopology base = materialize(g, s, Genome::empty(3, 2));
    Vec want(g.branches.size(), 0.0);
    for (const auto& c : g.contingencies) {
      MaterializedTopology m = base;
      for (int e : c.branches) m.graph.edges[e].in_service = false;
      fold_max(want, rebuild_flows(m));
    }
    expect(abs_err(fr.max_contingency, want) < 1e-8, "14-bus screening vs rebuild");
  }
  {
    json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}}},
              {"branches",
               {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.2}, {"limit_mw", 100.0}},
                {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.2}, {"limit_mw", 100.0}},
                {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.2}, {"limit_mw", 100.0}}}},
              {"injections",
               {{{"id", "g"}, {"node", "a"}, {"p_mw", 90.0}, {"kind", "generator"}},
                {{"id", "lb"}, {"node", "b"}, {"p_mw", 60.0}, {"kind", "load"}},
                {{"id", "lc"}, {"node", "c"}, {"p_mw", 30.0}, {"kind", "load"}}}},
              {"contingencies", {{{"id", "load-b-out"}, {"injections", {"lb"}}}}},
              {"slack", "a"}};
    GridModel g = grid_from_json(j);
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    FlowResult fr = ctx.screen_contingencies(ctx.apply_topology(Genome::empty(3, 2)));
    Vec p(3, 0.0);
    p[g.node_index("c")] = -30.0;
    p[g.slack] = 30.0;
    expect(abs_err(fr.max_contingency, cabs(angle_flows(dc_graph_from_grid(g), p))) < 1e-9, "injection outage");
  }
}

KAT(dc_islanding_penalty) {
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}}},
            {"branches",
             {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bd"}, {"from", "b"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "da"}, {"from", "d"}, {"to", "a"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
            {"injections",
             {{{"id", "g"}, {"node", "b"}, {"p_mw", 50.0}, {"kind", "generator"}},
              {{"id", "l"}, {"node", "d"}, {"p_mw", 50.0}, {"kind", "load"}}}},
            {"contingencies", {{{"id", "ab-out"}, {"branches", {"ab"}}}}},
            {"slack", "a"}};
  GridModel g = grid_from_json(j);
  ActionSet s = build_action_set(g);
  DcConfig cfg;
  cfg.islanding_penalty_mw = 2500.0;
  DcContext ctx(g, s, cfg);
  auto find = [&](const std::string& id) {
    for (int d = 0; d < static_cast<int>(s.disconnectables.size()); ++d)
      if (g.branches[s.disconnectables[d]].id == id) return d;
    return -1;
  };
  Genome gg = Genome::empty(3, 2);
  gg.disconnection_slots[0] = find("bc");
  gg.disconnection_slots[1] = find("bd");
  ScoreVector sc = ctx.evaluate(gg);
  expect(!sc.islanded && near(sc.lambda_o, 2500.0) && sc.worst_contingencies.size() == 1 &&
             near(sc.worst_contingencies[0].second, 2500.0),
         "islanding contingency penalty 2500");
}

KAT(dc_scores) {
  GridModel g = triangle_grid();
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  FlowResult a;
  a.base.assign(3, 0.0);
  a.max_contingency = {110.0, 90.0, 0.0};
  a.max_busbar.assign(3, 0.0);
  a.outage_energy = {10.0};
  ScoreVector sa = ctx.compute_scores(a, Genome::empty(3, 2));
  expect(near(sa.lambda_o, 10.0) && sa.lambda_c == 1 && sa.lambda_c0 == 0 && near(sa.fitness, -60.0), "lambda_o=10 -> -60");
  FlowResult b;
  b.base = {101.0, 0.0, 0.0};
  b.max_contingency = {150.0, 150.0, 0.0};
  b.max_busbar.assign(3, 0.0);
  ScoreVector sb = ctx.compute_scores(b, Genome::empty(3, 2));
  expect(near(sb.lambda_o, 100.0) && sb.lambda_c0 == 1 && sb.lambda_c == 2 && near(sb.fitness, -400.0), "-400");
  expect(near(ctx.evaluate(Genome::empty(3, 2)).fitness, 0.0), "clean scores zero");
  std::mt19937_64 rng(17);
  std::uniform_real_distribution<double> u(0.0, 200.0);
  bool mono = true;
  for (int t = 0; t < 200; ++t) {
    FlowResult x;
    x.base.assign(3, 0.0);
    x.max_busbar.assign(3, 0.0);
    x.max_contingency.assign(3, 0.0);
    for (int e = 0; e < 3; ++e) x.max_contingency[e] = u(rng);
    FlowResult y = x;
    for (int e = 0; e < 3; ++e) y.max_contingency[e] += u(rng) * 0.2;
    ScoreVector p = ctx.compute_scores(x, Genome::empty(3, 2)), q = ctx.compute_scores(y, Genome::empty(3, 2));
    mono = mono && q.lambda_o >= p.lambda_o && q.lambda_c >= p.lambda_c;
  }
  expect(mono, "monotonicity");
}

KAT(dc_busbar_variant2) {
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}}},
            {"branches",
             {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ac"}, {"from", "a"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ad"}, {"from", "a"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
            {"injections",
             {{{"id", "g"}, {"node", "a"}, {"p_mw", 60.0}, {"kind", "generator"}},
              {{"id", "l"}, {"node", "c"}, {"p_mw", 60.0}, {"kind", "load"}}}},
            {"substations", json::array({station_json("a", {"ab", "ac", "ad", "g"})})},
            {"busbar_outages", {{{"id", "bo"}, {"substation", "a"}, {"busbar", "B1"}}}},
            {"slack", "c"}};
  GridModel g = grid_from_json(j);
  ActionSet s = build_action_set(g);
  DcConfig cfg;
  cfg.fitness_variant = 2;
  cfg.islanding_penalty_mw = 5000.0;
  DcContext ctx(g, s, cfg);
  expect(near(ctx.lambda_b_pre(), 5000.0) && near(ctx.pre_optimization_score().fitness, 0.0), "lambda_b_pre 5000");
  bool better = false, nonpos = true;
  for (int a = 0; a < static_cast<int>(s.actions.size()); ++a) {
    Genome gg = Genome::empty(3, 2);
    gg.action_slots[0] = a;
    ScoreVector sc = ctx.evaluate(gg);
    if (sc.islanded) continue;
    nonpos = nonpos && sc.fitness <= 0.0;
    better = better || sc.lambda_b < 5000.0;
  }
  expect(better && nonpos, "a split survives the busbar outage");
}

KAT(dc_batch_purity) {
  GridModel g = random_grid(400, {.n_nodes = 20, .extra_edges = 12, .n_outages = 5, .n_stations = 2});
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  std::mt19937_64 rng(9);
  std::vector<Genome> batch;
  for (int i = 0; i < 16; ++i) batch.push_back(random_genome(s, 3, 2, rng));
  batch.push_back(Genome::empty(3, 2));
  auto tog = ctx.evaluate_batch(batch, 64);
  bool ok = tog.size() == batch.size();
  for (std::size_t i = 0; ok && i < batch.size(); ++i) {
    ScoreVector one = ctx.evaluate(batch[i]);
    ok = tog[i].fitness == one.fitness && tog[i].lambda_o == one.lambda_o &&
         tog[i].worst_contingencies == one.worst_contingencies;
  }
  expect(ok, "batch == single");
  expect(tog.back().fitness == ctx.pre_optimization_score().fitness, "padded empty == pre score");
  std::vector<Genome> rev(batch.rbegin(), batch.rend());
  auto r = ctx.evaluate_batch(rev, 64);
  bool rok = true;
  for (std::size_t i = 0; i < batch.size(); ++i) rok = rok && r[batch.size() - 1 - i].fitness == tog[i].fitness;
  expect(rok, "reversal invariance");
  GridModel g2 = random_grid(500, {.n_nodes = 18, .extra_edges = 12, .n_outages = 6, .n_stations = 2});
  ActionSet s2 = build_action_set(g2);
  DcConfig c1, c3;
  c1.threads = 1;
  c3.threads = 3;
  DcContext serial(g2, s2, c1), par(g2, s2, c3);
  std::mt19937_64 r2(21);
  std::vector<Genome> b2;
  for (int i = 0; i < 40; ++i) b2.push_back(random_genome(s2, 3, 2, r2));
  auto x = serial.evaluate_batch(b2, 64), y = par.evaluate_batch(b2, 64);
  bool same = x.size() == y.size();
  for (std::size_t i = 0; same && i < x.size(); ++i)
    same = x[i].fitness == y[i].fitness && x[i].worst_contingencies == y[i].worst_contingencies;
  expect(same, "threads 1 == threads 3");
}

KAT(dc_scratch_cases) {
  std::mt19937_64 rng(808);
  int checked = 0, islanding = 0, busbar = 0;
  for (std::uint64_t seed = 600; seed < 612; ++seed) {
    RandomGridOptions o;
    o.n_nodes = 14 + static_cast<int>(seed % 20);
    o.extra_edges = 10 + static_cast<int>(seed % 7);
    o.n_outages = 6;
    o.n_stations = 2;
    o.multi_branch_outages = o.injection_outages = o.busbar_outages = true;
    GridModel g = random_grid(seed, o);
    ActionSet s = build_action_set(g);
    DcConfig cfg;
    cfg.islanding_penalty_mw = 7777.0;
    DcContext ctx(g, s, cfg);
    for (int t = 0; t < 6; ++t) {
      Genome gg = random_genome(s, 3, 2, rng);
      FlowOperator op = ctx.apply_topology(gg);
      if (op.islanded()) continue;
      FlowResult fr = ctx.screen_contingencies(op);
      Vec fold(g.branches.size(), 0.0);
      int isl = 0;
      for (int ci = 0; ci < static_cast<int>(g.contingencies.size()); ++ci) {
        const auto& c = g.contingencies[ci];
        auto f = scratch_outage_flows(g, s, gg, c.branches, c.injections);
        if (!f) {
          ++isl;
          ++islanding;
          expect(fr.outage_energy[ci] == cfg.islanding_penalty_mw, "islanded case energy = penalty");
          continue;
        }
        double en = 0;
        for (int e = 0; e < static_cast<int>(g.branches.size()); ++e)
          en += std::max(0.0, std::abs((*f)[e]) - g.branches[e].flow_limit);
        expect(std::abs(fr.outage_energy[ci] - en) < 1e-8, "case energy vs scratch");
        fold_max(fold, *f);
        ++checked;
      }
      expect(fr.islanded_outages == isl, "islanded count");
      expect(abs_err(fr.max_contingency, fold) < 1e-8, "contingency fold vs scratch");
      Vec bfold(g.branches.size(), 0.0);
      int bisl = 0;
      for (const auto& bo : g.busbar_outages) {
        auto f = scratch_outage_flows(g, s, gg, scratch_implied_branches(g, s, gg, bo), {});
        if (!f) {
          ++bisl;
          continue;
        }
        fold_max(bfold, *f);
        ++busbar;
      }
      expect(fr.islanded_busbar_outages == bisl, "busbar islanded count");
      expect(abs_err(fr.max_busbar, bfold) < 1e-8, "busbar fold vs scratch");
    }
  }
  expect(checked > 100 && islanding > 0 && busbar > 10, "coverage of scratch cases");
}

KAT(dc_slack_station_split) {
  json j = {{"nodes", {{{"id", "s"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}, {{"id", "e"}}}},
            {"branches",
             {{{"id", "sb"}, {"from", "s"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "sc"}, {"from", "s"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "sd"}, {"from", "s"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "se"}, {"from", "s"}, {"to", "e"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.2}, {"limit_mw", 100.0}},
              {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.2}, {"limit_mw", 100.0}},
              {{"id", "de"}, {"from", "d"}, {"to", "e"}, {"x_pu", 0.2}, {"limit_mw", 100.0}},
              {{"id", "eb"}, {"from", "e"}, {"to", "b"}, {"x_pu", 0.2}, {"limit_mw", 100.0}}}},
            {"injections",
             {{{"id", "g"}, {"node", "s"}, {"p_mw", 80.0}, {"kind", "generator"}},
              {{"id", "l"}, {"node", "d"}, {"p_mw", 80.0}, {"kind", "load"}}}},
            {"substations", json::array({station_json("s", {"sb", "sc", "sd", "se", "g"})})},
            {"slack", "s"}};
  GridModel g = grid_from_json(j);
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  int checked = 0;
  for (const Action& a : s.actions) {
    Genome gg = Genome::empty(3, 2);
    gg.action_slots[0] = a.id;
    FlowOperator op = ctx.apply_topology(gg);
    MaterializedTopology m = materialize(g, s, gg);
    if (op.islanded()) {
      expect(throws_as<SingularSystem>([&] { rebuild_flows(m); }), "slack split islanded");
      continue;
    }
    expect(abs_err(op.base_flows(), rebuild_flows(m)) < 1e-9, "slack split vs rebuild");
    ++checked;
  }
  expect(checked >= 3, "slack split coverage");
}

KAT(dc_genome_islanding) {
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "b"}}, {{"id", "c"}}, {{"id", "d"}}}},
            {"branches",
             {{{"id", "ab"}, {"from", "a"}, {"to", "b"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bc"}, {"from", "b"}, {"to", "c"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "ca"}, {"from", "c"}, {"to", "a"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "bd"}, {"from", "b"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}},
              {{"id", "cd"}, {"from", "c"}, {"to", "d"}, {"x_pu", 0.1}, {"limit_mw", 100.0}}}},
            {"injections",
             {{{"id", "g"}, {"node", "a"}, {"p_mw", 40.0}, {"kind", "generator"}},
              {{"id", "l"}, {"node", "d"}, {"p_mw", 40.0}, {"kind", "load"}}}},
            {"slack", "a"}};
  GridModel g = grid_from_json(j);
  ActionSet s = build_action_set(g);
  expect(s.disconnectables.size() == 5, "five disconnectables");
  DcContext ctx(g, s);
  auto find = [&](const std::string& id) {
    for (int d = 0; d < static_cast<int>(s.disconnectables.size()); ++d)
      if (g.branches[s.disconnectables[d]].id == id) return d;
    return -1;
  };
  Genome gg = Genome::empty(3, 2);
  gg.disconnection_slots[0] = find("bd");
  gg.disconnection_slots[1] = find("cd");
  ScoreVector sc = ctx.evaluate(gg);
  expect(sc.islanded && sc.fitness == ScoreVector::kIslandedFitness, "islanded sentinel");
}

// acceptance.cpp:51-88 (criterion 1)
KAT(acceptance_1_operator_vs_rebuild) {
  auto t0 = std::chrono::steady_clock::now();
  double worst = 0;
  int n = 0;
  std::mt19937_64 rng(4242);
  for (int trial = 0; trial < 50; ++trial) {
    RandomGridOptions o;
    o.n_nodes = 10 + (trial * 7) % 51;
    o.extra_edges = 6 + trial % 13;
    o.n_outages = 3 + trial % 5;
    o.n_stations = 2 + trial % 2;
    GridModel g = random_grid(1000 + trial, o);
    ActionSet s = build_action_set(g);
    DcContext ctx(g, s);
    for (int k = 0; k < 20; ++k) {
      Genome gg = random_genome(s, 3, 2, rng);
      FlowOperator op = ctx.apply_topology(gg);
      MaterializedTopology m = materialize(g, s, gg);
      if (op.islanded()) {
        expect(throws_as<SingularSystem>([&] { rebuild_flows(m); }), "criterion 1 islanded");
        continue;
      }
      worst = std::max(worst, rel_err(op.base_flows(), rebuild_flows(m)));
      ++n;
    }
  }
  double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("  criterion 1: %d genomes, max rel err %.2e, %.1f s\n", n, worst, sec);
  expect(worst < 1e-8 && sec < 60.0, "criterion 1");
}

// ------------------------------------------------------------ QD optimizer
// test_qd_optimizer.cpp:34-369, acceptance.cpp:171-295
KAT(qd_descriptor) {
  QdConfig c;
  expect(descriptor_to_cell(0, 0, 0, c) == 0 && descriptor_to_cell(1, 2, 0, c) == 7 &&
             descriptor_to_cell(2, 3, 45, c) == 551 && cell_count(c) == 552,
         "descriptor KATs");
  std::vector<int> hits(cell_count(c), 0);
  for (int d = 0; d <= c.d_max; ++d)
    for (int s = 0; s <= c.s_max; ++s)
      for (int r = 0; r <= c.r_max; ++r) ++hits[descriptor_to_cell(d, s, r, c)];
  bool bij = true;
  for (int h : hits) bij = bij && h == 1;
  expect(bij, "bijection");
  expect(descriptor_to_cell(0, 0, 99, c) == descriptor_to_cell(0, 0, 45, c), "clamp r");
}

double chi2(const std::map<MutationOp, int>& counts, const std::array<double, 4>& w, int n) {
  double st = 0;
  for (int op = 0; op < 4; ++op) {
    double e = w[op] * n;
    if (e == 0.0) continue;
    auto it = counts.find(static_cast<MutationOp>(op));
    double o = it == counts.end() ? 0.0 : it->second;
    st += (o - e) * (o - e) / e;
  }
  return st;
}

KAT(qd_mutation) {
  GridModel g = mini_congestion_grid();
  ActionSet s = build_action_set(g);
  QdConfig c;
  c.seed = 11;
  for (std::uint64_t seed = 0; seed < 50; ++seed) {
    Rng rng(seed);
    Genome k = mutate(Genome::empty(c.n_a, c.n_d), s, c, rng);
    expect((k.split_count() > 0 || k.disconnection_count() >= 1) && genome_valid(k, s), "forced add");
  }
  Rng rng(77);
  Genome cur = Genome::empty(c.n_a, c.n_d);
  bool ok = true;
  for (int step = 0; step < 10000; ++step) {
    cur = mutate(cur, s, c, rng);
    ok = ok && genome_valid(cur, s) && cur.split_count() <= c.n_a && cur.disconnection_count() <= c.n_d;
  }
  expect(ok, "10k chained mutations valid");
  expect(s.actions.size() >= 3, "mini grid actions");
  Genome parent = Genome::empty(c.n_a, c.n_d);
  parent.action_slots[0] = 0;
  parent.disconnection_slots[0] = 0;
  std::map<MutationOp, int> ac, dc;
  Rng r2(2024);
  for (int t = 0; t < 20000; ++t) {
    MutationTrace tr;
    mutate(parent, s, c, r2, &tr);
    ++ac[tr.action_ops[0]];
    ++dc[tr.disconnection_ops[0]];
  }
  expect(chi2(ac, c.p_action, 20000) < 11.345 && dc[MutationOp::Identity] == 0 && chi2(dc, c.p_disc, 20000) < 9.210,
         "operation frequencies");
}

KAT(qd_crossover) {
  GridModel g = mini_congestion_grid();
  ActionSet s = build_action_set(g);
  QdConfig c;
  c.seed = 11;
  auto r0 = s.station_ranges.begin(), r1 = std::next(r0);
  Genome p1 = Genome::empty(3, 2), p2 = Genome::empty(3, 2);
  p1.action_slots[0] = r0->second.first;
  p1.disconnection_slots[0] = 0;
  p2.action_slots[0] = r1->second.first;
  p2.disconnection_slots[0] = 1;
  QdConfig c1 = c;
  c1.p_crossover_parent1 = 1.0;
  Rng rng(5);
  bool same = true;
  for (int t = 0; t < 100; ++t) {
    Genome k = crossover(p1, p2, s, c1, rng);
    same = same && k.action_ids() == p1.action_ids() && k.disconnection_ids() == p1.disconnection_ids();
  }
  expect(same, "p_c1 = 1 reproduces parent 1");
  Rng r6(6);
  expect(crossover(Genome::empty(3, 2), Genome::empty(3, 2), s, c, r6).is_empty(), "empty x empty");
  Rng r7(7);
  std::mt19937_64 gr(8);
  bool valid = true;
  for (int t = 0; t < 10000; ++t) {
    Genome a = random_genome(s, 3, 2, gr), b = random_genome(s, 3, 2, gr);
    Genome k = crossover(a, b, s, c, r7);
    valid = valid && genome_valid(k, s);
    auto ia = a.action_ids(), ib = b.action_ids();
    for (int x : k.action_ids())
      valid = valid && (std::binary_search(ia.begin(), ia.end(), x) || std::binary_search(ib.begin(), ib.end(), x));
  }
  expect(valid, "crossover children valid and inherited");
}

KAT(qd_repertoire) {
  QdConfig c;
  c.cell_capacity = 2;
  Repertoire rep(c);
  ScoreVector s;
  s.lambda_d = 1;
  auto genome_d = [](int slot, int v) {
    Genome g = Genome::empty(3, 2);
    g.disconnection_slots[slot] = v;
    return g;
  };
  ScoreVector s1 = s, s2 = s, s3 = s, s5 = s;
  s1.fitness = -40;
  s2.fitness = -20;
  s3.fitness = -50;
  s5.fitness = -10;
  expect(rep.insert(genome_d(0, 0), s1) && rep.insert(genome_d(0, 1), s2), "fill cell");
  expect(!rep.insert(genome_d(0, 2), s3) && !rep.insert(genome_d(0, 2), s1), "full cell rejects <= min");
  expect(!rep.insert(genome_d(1, 0), s1) && rep.total_size() == 2, "duplicate key rejected");
  expect(rep.insert(genome_d(0, 3), s5) && rep.total_size() == 2 &&
             rep.cell(descriptor_to_cell(1, 0, 0, c))[0].score.fitness == -10.0,
         "better displaces worst");
  ScoreVector bad;
  bad.islanded = true;
  bad.fitness = ScoreVector::kIslandedFitness;
  expect(!rep.insert(genome_d(0, 4), bad), "islanded never enters");
}

std::string snap_text(const RepertoireSnapshot& s) {
  std::ostringstream o;
  o << s.epoch << "|" << s.evaluations << "|" << s.best_fitness << "|" << s.final;
  for (const auto& e : s.entries) o << ";" << e.cell << ":" << e.genome.canonical_key() << ":" << e.score.fitness;
  return o.str();
}

KAT(qd_optimizer_runs) {
  GridModel g = mini_congestion_grid();
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  QdConfig c;
  c.seed = 11;
  c.batch_size = 16;
  c.iters_per_epoch = 10;
  {
    QdConfig z = c;
    z.max_evaluations = 1;
    auto r = run_optimizer(ctx, z, nullptr);
    expect(r.repertoire.total_size() == 1 && r.stats.evaluations == 1 && r.repertoire.member(0).genome.is_empty(),
           "zero budget keeps the seed");
  }
  {
    QdConfig z = c;
    z.max_evaluations = 4000;
    auto r = run_optimizer(ctx, z, nullptr);
    expect(r.repertoire.best_fitness() > ctx.pre_optimization_score().fitness &&
               std::abs(r.repertoire.best_fitness()) < 1e-9,
           "finds the clearing disconnection");
  }
  {
    QdConfig z = c;
    z.max_evaluations = 3000;
    std::vector<RepertoireSnapshot> snaps;
    run_optimizer(ctx, z, [&](RepertoireSnapshot x) { snaps.push_back(std::move(x)); });
    bool elit = snaps.size() >= 2 && snaps.back().final;
    std::map<int, double> best;
    for (const auto& sn : snaps) {
      std::map<int, double> now;
      for (const auto& e : sn.entries) {
        elit = elit && genome_valid(e.genome, s) &&
               e.cell == descriptor_to_cell(e.score.lambda_d, e.score.lambda_s, e.score.lambda_r, z);
        auto it = now.find(e.cell);
        if (it == now.end() || e.score.fitness > it->second) now[e.cell] = e.score.fitness;
      }
      for (const auto& [cell, f] : best) elit = elit && now.count(cell) && now[cell] >= f - 1e-12;
      best = now;
    }
    expect(elit, "per-cell elitism and final flag");
  }
  {
    QdConfig z = c;
    z.max_evaluations = 2000;
    std::vector<std::string> a, b, d;
    run_optimizer(ctx, z, [&](RepertoireSnapshot x) { a.push_back(snap_text(x)); });
    run_optimizer(ctx, z, [&](RepertoireSnapshot x) { b.push_back(snap_text(x)); });
    z.seed = 12;
    run_optimizer(ctx, z, [&](RepertoireSnapshot x) { d.push_back(snap_text(x)); });
    expect(a == b && a != d, "determinism per seed");
  }
  {
    QdConfig z = c;
    z.max_evaluations = 10000;
    auto r = run_optimizer(ctx, z, nullptr);
    bool sp = false, di = false;
    for (int i = 0; i < r.repertoire.total_size(); ++i) {
      sp = sp || r.repertoire.member(i).score.lambda_s >= 1;
      di = di || r.repertoire.member(i).score.lambda_d >= 1;
    }
    expect(sp && di, "coverage");
  }
  {
    QdConfig z = c;
    z.batch_size = 0;
    expect(throws_as<ConfigError>([&] { run_optimizer(ctx, z, nullptr); }), "bad batch size");
  }
}

// acceptance.cpp:185-236 (criterion 6)
KAT(acceptance_6_operators) {
  GridModel g = data_grid("grid14_congested.json");
  ActionSet s = build_action_set(g);
  QdConfig c;
  int bad = 0;
  std::map<MutationOp, int> ac, dc;
  Rng rng(60601);
  std::mt19937_64 gr(60602);
  Genome stub = Genome::empty(c.n_a, c.n_d);
  stub.action_slots[0] = 0;
  stub.disconnection_slots[0] = 0;
  for (int t = 0; t < 50000; ++t) {
    MutationTrace tr;
    if (!genome_valid(mutate(stub, s, c, rng, &tr), s)) ++bad;
    ++ac[tr.action_ops[0]];
    ++dc[tr.disconnection_ops[0]];
  }
  for (int t = 0; t < 50000; ++t) {
    Genome a = random_genome(s, c.n_a, c.n_d, gr), b = random_genome(s, c.n_a, c.n_d, gr);
    if (!genome_valid(crossover(a, b, s, c, rng), s)) ++bad;
  }
  double x1 = chi2(ac, c.p_action, 50000), x2 = chi2(dc, c.p_disc, 50000);
  std::printf("  criterion 6: %d violations, chi2 %.2f / %.2f\n", bad, x1, x2);
  expect(bad == 0 && x1 < 11.345 && x2 < 9.210, "criterion 6");
}

// acceptance.cpp:238-295 (criterion 7)
KAT(acceptance_7_progress) {
  GridModel g = data_grid("grid14_congested.json");
  ActionSet s = build_action_set(g);
  DcContext ctx(g, s);
  const double pre_o = ctx.pre_optimization_score().lambda_o;
  expect(pre_o > 0.0, "fixture is congested");
  double opt = ctx.pre_optimization_score().fitness, drop = 0;
  for (int d = 0; d < static_cast<int>(s.disconnectables.size()); ++d) {
    Genome gg = Genome::empty(3, 2);
    gg.disconnection_slots[0] = d;
    ScoreVector sc = ctx.evaluate(gg);
    if (std::isfinite(sc.fitness)) opt = std::max(opt, sc.fitness);
    drop = std::max(drop, 1.0 - sc.lambda_o / pre_o);
  }
  for (int a = 0; a < static_cast<int>(s.actions.size()); ++a) {
    Genome gg = Genome::empty(3, 2);
    gg.action_slots[0] = a;
    ScoreVector sc = ctx.evaluate(gg);
    if (std::isfinite(sc.fitness)) opt = std::max(opt, sc.fitness);
  }
  expect(drop >= 0.8, "single disconnection removes >= 80% of lambda_o");
  QdConfig c;
  c.seed = 777;
  c.batch_size = 64;
  c.iters_per_epoch = 31;
  c.max_evaluations = 10000;
  auto r = run_optimizer(ctx, c, nullptr);
  const double best = r.repertoire.best_fitness();
  std::printf("  criterion 7: optimum %.3f reached %.3f, drop %.0f%%\n", opt, best, 100 * drop);
  expect(best >= opt - 0.05 * std::abs(opt), "criterion 7");
}


// ------------------------------------------------------------ AC validation
// test_ac_validator.cpp:15-395
namespace {
AppliedTopology no_split(const GridModel& g, const ActionSet& a) { return apply_genome(g, a, Genome::empty(0, 0)); }
json two_bus_json(double x, double r, double p, double q) {
  return {{"nodes", {{{"id", "s"}}, {{"id", "b"}}}},
          {"branches", {{{"id", "sb"}, {"from", "s"}, {"to", "b"}, {"x_pu", x}, {"r_pu", r}, {"limit_mw", 100.0}}}},
          {"injections", {{{"id", "l"}, {"node", "b"}, {"p_mw", p}, {"q_mvar", q}, {"kind", "load"}}}},
          {"slack", "s"}};
}
int slot_of_disconnectable(const GridModel& g, const ActionSet& a, const char* id) {
  for (int d = 0; d < static_cast<int>(a.disconnectables.size()); ++d)
    if (g.branches[a.disconnectables[d]].id == id) return d;
  return -1;
}
}  // namespace

KAT(ac_flat_and_two_bus) {
  {  // zero load: converges on the first mismatch test (test_ac_validator.cpp:31-47)
    GridModel g = grid_from_json(two_bus_json(0.1, 0.01, 0.0, 0.0));
    ActionSet a = build_action_set(g);
    AcCaseResult r = ac_power_flow(g, no_split(g, a));
    expect(r.converged && r.iterations == 1, "zero load converges in one iteration");
    expect(*std::max_element(r.loading_mva.begin(), r.loading_mva.end()) < 1e-9, "zero flows");
    expect(std::abs(r.vm_pu[g.node_index("b")] - 1.0) < 1e-12, "flat magnitude");
  }
  {  // two-bus load vs the Z-bus fixed point (49-75)
    GridModel g = grid_from_json(two_bus_json(0.1, 0.01, 50.0, 10.0));
    ActionSet a = build_action_set(g);
    AcCaseResult r = ac_power_flow(g, no_split(g, a));
    expect(r.converged, "two-bus converges");
    std::complex<double> v1(1.0, 0.0), z(0.01, 0.1), s(0.5, 0.1), v2 = v1;
    for (int i = 0; i < 500; ++i) v2 = v1 - z * std::conj(s / v2);
    const int b = g.node_index("b");
    expect(std::abs(std::polar(r.vm_pu[b], r.va_rad[b]) - v2) < 1e-6, "two-bus voltage = fixed point");
    const std::complex<double> sf = v1 * std::conj((v1 - v2) / z) * 100.0;
    expect(sf.real() > 50.0, "sending end covers losses");
    expect(std::abs(r.loading_mva[0] - std::abs(sf)) <= 1e-6 * std::abs(sf), "loading = |S_from|");
  }
  {  // beyond transfer capacity (170-184)
    GridModel g = grid_from_json(two_bus_json(0.5, 0.05, 400.0, 100.0));
    ActionSet a = build_action_set(g);
    expect(!ac_power_flow(g, no_split(g, a)).converged, "heavy load does not converge");
  }
}

KAT(ac_grid14_published) {  // test_ac_validator.cpp:77-134
  GridModel g = data_grid("grid14.json");
  ActionSet a;
  AcCaseResult r = ac_power_flow(g, no_split(g, a));
  expect(r.converged && r.iterations <= 10, "grid14 converges within 10 iterations");
  const std::vector<std::pair<const char*, double>> pub = {
      {"1", 1.060}, {"2", 1.045}, {"3", 1.010}, {"4", 1.018}, {"5", 1.020}, {"6", 1.070}, {"7", 1.062},
      {"8", 1.090}, {"9", 1.056}, {"10", 1.051}, {"11", 1.057}, {"12", 1.055}, {"13", 1.050}, {"14", 1.036}};
  for (auto& [bus, vm] : pub) expect(std::abs(r.vm_pu[g.node_index(bus)] - vm) < 1e-3, std::string("published vm ") + bus);
  // bus power balance against an independent Ybus (90-134)
  const int n = static_cast<int>(g.nodes.size());
  std::vector<std::complex<double>> V(n), S(n, 0.0);
  for (int v = 0; v < n; ++v) V[v] = std::polar(r.vm_pu[v], r.va_rad[v]);
  for (const Branch& br : g.branches) {
    const std::complex<double> y = 1.0 / std::complex<double>(br.resistance, br.reactance), ysh(0.0, br.charging_b / 2);
    const std::complex<double> i_f = (y + ysh) / (br.tap * br.tap) * V[br.from] - y / br.tap * V[br.to];
    const std::complex<double> i_t = -y / br.tap * V[br.from] + (y + ysh) * V[br.to];
    S[br.from] += V[br.from] * std::conj(i_f);
    S[br.to] += V[br.to] * std::conj(i_t);
  }
  for (int v = 0; v < n; ++v) S[v] += V[v] * std::conj(std::complex<double>(0.0, g.nodes[v].shunt_b_pu) * V[v]);
  for (int v = 0; v < n; ++v) {
    if (v == g.slack) continue;
    double p = 0, q = 0;
    bool pv = false;
    for (const Injection& inj : g.injections) {
      if (inj.node != v) continue;
      if (inj.kind == InjectionKind::Generator) {
        p += inj.p_mw / 100.0;
        pv = pv || inj.v_setpoint_pu.has_value();
      } else {
        p -= inj.p_mw / 100.0;
        q -= inj.q_mvar / 100.0;
      }
    }
    expect(std::abs(S[v].real() - p) < 1e-6, "P balance");
    if (!pv) expect(std::abs(S[v].imag() - q) < 1e-6, "Q balance");
  }
}

KAT(ac_islanding_contingency) {  // test_ac_validator.cpp:136-168
  GridModel g = mini_congestion_grid();
  ActionSet a = build_action_set(g);
  int pick = -1;
  for (const Action& act : a.actions) {
    const SubstationDetail& st = g.substations[act.substation];
    if (st.node != g.node_index("f")) continue;
    bool load_stays = false, mf_moves = true;
    for (int t = 0; t < static_cast<int>(st.terminals.size()); ++t) {
      if (st.terminals[t].element == "load" && !act.group[t]) load_stays = true;
      if ((st.terminals[t].element == "mf" || st.terminals[t].element == "mf2") && !act.group[t]) mf_moves = false;
    }
    if (load_stays && mf_moves) pick = act.id;
  }
  if (pick >= 0) {
    Genome gen = Genome::empty(3, 2);
    gen.action_slots[0] = pick;
    AcNetwork net(g, apply_genome(g, a, gen));
    expect(net.run_case(-1).converged, "split base converges");
    int af = -1;
    for (int k = 0; k < static_cast<int>(g.contingencies.size()); ++k)
      if (g.contingencies[k].id == "o-af") af = k;
    expect(af >= 0 && !net.run_case(af).converged, "stranding contingency does not converge");
  }
}

KAT(ac_validator_congestion) {  // test_ac_validator.cpp:186-233, 235-262
  GridModel g = mini_congestion_grid();
  ActionSet a = build_action_set(g);
  DcContext dc(g, a);
  AcValidator val(g, a, dc, {});
  expect(val.baseline_lambda_o() > 0.0, "baseline overload");
  const int mf = slot_of_disconnectable(g, a, "mf");
  expect(mf >= 0, "mf disconnectable");
  Genome clear = Genome::empty(3, 2);
  clear.disconnection_slots[0] = mf;
  const ScoreVector cs = dc.evaluate(clear);
  expect(std::abs(cs.fitness) < 1e-9, "clearing DC fitness 0");
  Genome none = Genome::empty(3, 2);
  expect(val.worst_k_check(none, dc.evaluate(none)) == RejectionReason::OverloadNotImproved, "unchanged never improves");
  expect(val.worst_k_check(clear, cs) == RejectionReason::None, "worst-k passes clearing");
  ValidationRecord rec = val.full_validation(clear, cs);
  expect(rec.accepted && rec.ac_lambda_o < val.baseline_lambda_o() && rec.stage == ValidationStage::FullN1,
         "full validation accepts clearing");
  AcValidator hist(g, a, dc, {});
  expect(hist.validate({clear, cs}).accepted, "validate accepts");
  EliminationOutcome out = hist.eliminate({{clear, cs}});
  expect(out.pruned.size() == 1 && out.pruned[0].second == RejectionReason::EliminatedSimilar && out.queue.empty(),
         "validated genome pruned as similar");
  for (double scale : {1.0, 0.9, 0.8}) {  // monotone in loading (235-262)
    json j = json::parse(grid_to_json_text(mini_congestion_grid()));
    for (json& inj : j["injections"]) {
      if (inj["kind"] != "load") continue;
      inj["p_mw"] = inj["p_mw"].get<double>() * scale;
      inj["q_mvar"] = inj["q_mvar"].get<double>() * scale;
    }
    GridModel gs = grid_from_json(j);
    ActionSet as = build_action_set(gs);
    DcContext dcs(gs, as);
    AcValidator vs(gs, as, dcs, {});
    if (vs.baseline_lambda_o() == 0.0) continue;
    Genome gg = Genome::empty(3, 2);
    gg.disconnection_slots[0] = slot_of_disconnectable(gs, as, "mf");
    ValidationRecord r = vs.full_validation(gg, dcs.evaluate(gg));
    expect(r.reason != RejectionReason::OverloadNotImproved && r.accepted, "accepted at smaller loads");
  }
  const std::string line = record_to_json(rec, g, a);  // 374-395
  json p = json::parse(line);
  expect(p.contains("verdict") && p.contains("reason") && p.contains("ac_lambda_o") && p["stage"] == "full_n1" &&
             p["lambda_d"] == 1,
         "record serializes");
}

KAT(ac_critical_count_rejection) {  // test_ac_validator.cpp:264-298
  json j = {{"nodes", {{{"id", "a"}}, {{"id", "m"}}, {{"id", "f"}}}},
            {"branches",
             {{{"id", "af"}, {"from", "a"}, {"to", "f"}, {"x_pu", 0.3}, {"limit_mw", 200.0}},
              {{"id", "am"}, {"from", "a"}, {"to", "m"}, {"x_pu", 0.05}, {"limit_mw", 107.0}},
              {{"id", "mf"}, {"from", "m"}, {"to", "f"}, {"x_pu", 0.05}, {"limit_mw", 45.0}},
              {{"id", "mf2"}, {"from", "m"}, {"to", "f"}, {"x_pu", 0.2}, {"limit_mw", 100.0}}}},
            {"injections",
             {{{"id", "g"}, {"node", "a"}, {"p_mw", 100.0}, {"kind", "generator"}, {"v_setpoint_pu", 1.02}},
              {{"id", "load"}, {"node", "f"}, {"p_mw", 100.0}, {"q_mvar", 20.0}, {"kind", "load"}}}},
            {"contingencies", {{{"id", "o-af"}, {"branches", {"af"}}}, {{"id", "o-am"}, {"branches", {"am"}}}}},
            {"slack", "a"}};
  GridModel g = grid_from_json(j);
  ActionSet a = build_action_set(g);
  DcContext dc(g, a);
  AcValidator val(g, a, dc, {});
  expect(val.baseline_critical_count() == 1, "one baseline critical branch");
  Genome gen = Genome::empty(3, 2);
  gen.disconnection_slots[0] = slot_of_disconnectable(g, a, "mf");
  ValidationRecord r = val.full_validation(gen, dc.evaluate(gen));
  expect(!r.accepted && r.reason == RejectionReason::CriticalCountIncreased && r.ac_lambda_o < val.baseline_lambda_o(),
         "criticals increased -> rejected");
}

KAT(ac_elimination) {  // test_ac_validator.cpp:300-372
  GridModel g = mini_congestion_grid();
  ActionSet a = build_action_set(g);
  DcContext dc(g, a);
  AcValidator val(g, a, dc, {});
  const double pre = dc.pre_optimization_score().fitness;
  expect(pre < 0.0, "congested pre fitness");
  auto make = [&](double fit, int d, int s, int r) {
    Candidate c;
    c.genome = Genome::empty(3, 2);
    c.genome.disconnection_slots[0] = d % 2;
    c.dc_score.fitness = fit;
    c.dc_score.lambda_d = d;
    c.dc_score.lambda_s = s;
    c.dc_score.lambda_r = r;
    return c;
  };
  {
    Candidate simple = make(-10.0, 1, 0, 0), twin = make(-10.0, 1, 1, 3);
    twin.genome.disconnection_slots[0] = 1;
    EliminationOutcome o = val.eliminate({simple, twin});
    expect(o.pruned.size() == 1 && o.pruned[0].first == 1 && o.pruned[0].second == RejectionReason::EliminatedDominated &&
               o.queue.size() == 1 && o.queue[0] == 0,
           "dominated pruned");
  }
  {
    EliminationOutcome o = val.eliminate({make(pre + 0.01 * std::abs(pre), 1, 0, 0)});
    expect(o.pruned.size() == 1 && o.pruned[0].second == RejectionReason::EliminatedBelowThreshold, "below threshold");
  }
  {
    Candidate good = make(-5.0, 1, 0, 0), better = make(-1.0, 1, 0, 0);
    better.genome.disconnection_slots[0] = 1;
    EliminationOutcome o = val.eliminate({good, better});
    expect(o.queue.size() == 2 && o.queue[0] == 1 && o.queue[1] == 0, "queue by DC fitness");
  }
  {
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<double> uf(pre, 0.0);
    std::uniform_int_distribution<int> ui(0, 3);
    std::vector<Candidate> pool;
    for (int i = 0; i < 60; ++i) {
      Candidate c;
      c.genome = random_genome(a, 3, 2, rng);
      c.dc_score.fitness = uf(rng);
      c.dc_score.lambda_d = c.genome.disconnection_count();
      c.dc_score.lambda_s = c.genome.split_count();
      c.dc_score.lambda_r = ui(rng);
      pool.push_back(c);
    }
    EliminationOutcome o = val.eliminate(pool);
    const double eps = val.config().dominance_fitness_frac * std::abs(pre);
    const double theta = val.config().improvement_threshold_frac * std::abs(pre);
    auto swd = [](const ScoreVector& s) { return s.lambda_d + s.lambda_s + s.lambda_r; };
    bool ok = o.queue.size() + o.pruned.size() == pool.size();
    for (int i : o.queue) {
      ok = ok && pool[i].dc_score.fitness - pre >= theta;
      for (const Candidate& other : pool)
        ok = ok && !(swd(other.dc_score) < swd(pool[i].dc_score) && other.dc_score.fitness >= pool[i].dc_score.fitness - eps);
    }
    expect(ok, "survivors fail every pruning predicate");
  }
}

}  // namespace

int main(int argc, char** argv) {
  g_data = argc > 1 ? argv[1] : "data";
  std::string only = argc > 2 ? argv[2] : "";
  for (auto& [name, fn] : registry()) {
    if (!only.empty() && name.find(only) == std::string::npos) continue;
    g_case = name;
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  FAIL [%s] exception: %s\n", name.c_str(), e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("oracle kats: %d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
