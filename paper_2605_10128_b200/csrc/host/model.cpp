// Host-side network model and import step (see model.hpp for the reference map).
#include <chrono>
#include <cstdlib>
#include "model.hpp"
#include "../cuda/islanding.cuh"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <random>
#include <set>
#include <thread>

#include "json_lite.hpp"

namespace tgb {

namespace {

using json::Value;

// splitmix-based seed derivation of rng.hpp:9-19
std::uint64_t mix(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
std::uint64_t derive(std::uint64_t master, std::uint64_t a, std::uint64_t b) {
  return mix(mix(master ^ mix(a)) ^ mix(b + 0x632be59bd9b4e019ull));
}

const Value& field(const Value& o, const char* key, const std::string& what) {
  const Value* v = o.find(key);
  if (!v) throw ParseError(what + ": missing field '" + key + "'");
  return *v;
}
std::string get_string(const Value& o, const char* key, const std::string& what) {
  const Value& v = field(o, key, what);
  if (!v.is_string()) throw ParseError(what + ": field '" + key + "' has the wrong type");
  return v.str;
}
double get_number(const Value& o, const char* key, const std::string& what) {
  const Value& v = field(o, key, what);
  if (!v.is_number()) throw ParseError(what + ": field '" + key + "' has the wrong type");
  if (!std::isfinite(v.num)) throw ParseError(what + ": non-finite number");
  return v.num;
}
double opt_number(const Value& o, const char* key, double dflt, const std::string& what) {
  const Value* v = o.find(key);
  if (!v) return dflt;
  if (!v->is_number()) throw ParseError(what + ": field '" + key + "' has the wrong type");
  if (!std::isfinite(v->num)) throw ParseError(what + ": non-finite number");
  return v->num;
}
std::vector<std::string> get_strings(const Value& o, const char* key, const std::string& what) {
  const Value& v = field(o, key, what);
  if (!v.is_array()) throw ParseError(what + ": field '" + key + "' has the wrong type");
  std::vector<std::string> out;
  for (const Value& x : v.arr) {
    if (!x.is_string()) throw ParseError(what + ": field '" + key + "' has the wrong type");
    out.push_back(x.str);
  }
  return out;
}
const std::vector<Value>& opt_array(const Value& o, const char* key) {
  static const std::vector<Value> none;
  const Value* v = o.find(key);
  if (!v || v->kind == Value::Null) return none;
  if (!v->is_array()) throw ParseError(std::string("field '") + key + "' must be an array");
  return v->arr;
}

// Active edges as CSR (offsets, (neighbour, edge) pairs): two flat arrays
// instead of one vector per node (the import runs these per candidate split).
struct Csr {
  std::vector<int> off;
  std::vector<std::pair<int, int>> nb;
  int degree(int v) const { return off[v + 1] - off[v]; }
};

Csr adjacency(int n, const std::vector<Edge>& edges, const std::vector<char>& cut) {
  Csr c;
  c.off.assign(n + 1, 0);
  auto live = [&](int e) { return edges[e].on && (cut.empty() || !cut[e]); };
  for (int e = 0; e < static_cast<int>(edges.size()); ++e)
    if (live(e)) ++c.off[edges[e].a + 1], ++c.off[edges[e].b + 1];
  for (int v = 0; v < n; ++v) c.off[v + 1] += c.off[v];
  c.nb.resize(c.off[n]);
  std::vector<int> fill(c.off.begin(), c.off.end() - 1);
  for (int e = 0; e < static_cast<int>(edges.size()); ++e)  // edge order per node, as push_back would give
    if (live(e)) c.nb[fill[edges[e].a]++] = {edges[e].b, e}, c.nb[fill[edges[e].b]++] = {edges[e].a, e};
  return c;
}

}  // namespace

// ---------------------------------------------------------------- graph
bool connected_with(int n, const std::vector<Edge>& edges, const std::vector<int>& must_reach,
                    const std::vector<int>& cut_list) {
  std::vector<char> cut;
  if (!cut_list.empty()) {
    cut.assign(edges.size(), 0);
    for (int e : cut_list) cut[e] = 1;
  }
  const Csr adj = adjacency(n, edges, cut);
  std::vector<char> need(n, 0);
  for (int v : must_reach) need[v] = 1;
  int root = must_reach.empty() ? -1 : must_reach.front();
  for (int v = 0; v < n; ++v)
    if (adj.degree(v) > 0) {
      need[v] = 1;
      if (root < 0) root = v;
    }
  if (root < 0) return true;
  std::vector<char> seen(n, 0);
  std::vector<int> q;
  q.reserve(n);
  q.push_back(root);
  seen[root] = 1;
  for (std::size_t h = 0; h < q.size(); ++h)
    for (int p = adj.off[q[h]]; p < adj.off[q[h] + 1]; ++p) {
      const int w = adj.nb[p].first;
      if (!seen[w]) seen[w] = 1, q.push_back(w);
    }
  for (int v = 0; v < n; ++v)
    if (need[v] && !seen[v]) return false;
  return true;
}

std::vector<int> bridges(int n, const std::vector<Edge>& edges) {
  const Csr adj = adjacency(n, edges, {});
  std::vector<int> tin(n, -1), low(n, 0), out;
  // explicit stack of (node, entering edge, next neighbour cursor)
  std::vector<std::array<int, 3>> st;
  int t = 0;
  for (int r = 0; r < n; ++r) {
    if (tin[r] >= 0 || adj.degree(r) == 0) continue;
    tin[r] = low[r] = t++;
    st.push_back({r, -1, adj.off[r]});
    while (!st.empty()) {
      auto& top = st.back();
      const int v = top[0];
      if (top[2] < adj.off[v + 1]) {
        auto [w, e] = adj.nb[top[2]++];
        if (e == top[1]) continue;
        if (tin[w] < 0) {
          tin[w] = low[w] = t++;
          st.push_back({w, e, adj.off[w]});
        } else {
          low[v] = std::min(low[v], tin[w]);
        }
      } else {
        const int via = top[1];
        st.pop_back();
        if (!st.empty()) {
          const int p = st.back()[0];
          low[p] = std::min(low[p], low[v]);
          if (low[v] > tin[p]) out.push_back(via);
        }
      }
    }
  }
  std::sort(out.begin(), out.end());
  return out;
}

// ---------------------------------------------------------------- grid
int Grid::station_at(int node) const { return station_of_node[node]; }
int Grid::branch_index(const std::string& id) const {
  auto it = branch_lookup.find(id);
  return it == branch_lookup.end() ? -1 : it->second;
}
int Grid::injection_index(const std::string& id) const {
  auto it = injection_lookup.find(id);
  return it == injection_lookup.end() ? -1 : it->second;
}

std::vector<int> Grid::implied_branches(int s, int busbar, const std::vector<int>& assign,
                                        const std::vector<int>& open) const {
  const Station& st = stations[s];
  const int nb = static_cast<int>(st.busbars.size());
  std::vector<char> in(nb, 0);
  std::vector<int> stack{busbar};
  in[busbar] = 1;
  while (!stack.empty()) {
    int v = stack.back();
    stack.pop_back();
    for (int c = 0; c < static_cast<int>(st.couplers.size()); ++c) {
      if (std::find(open.begin(), open.end(), c) != open.end()) continue;
      auto [a, b] = st.couplers[c];
      int w = a == v ? b : (b == v ? a : -1);
      if (w >= 0 && !in[w]) in[w] = 1, stack.push_back(w);
    }
  }
  std::vector<int> out;
  for (int t = 0; t < static_cast<int>(st.term_kind.size()); ++t) {
    if (st.term_kind[t] == kInjection) continue;
    const int e = st.term_index[t];
    if (!br_on[e]) continue;
    if (in[assign[t]]) out.push_back(e);
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

std::vector<int> Grid::default_implied(int bo) const {
  const Station& st = stations[bo_station[bo]];
  return implied_branches(bo_station[bo], bo_busbar[bo], st.term_default, {});
}

namespace {

void validate(const Grid& g) {
  const int n = g.n_nodes();
  for (int e = 0; e < g.n_branches(); ++e) {
    const std::string w = "branch '" + g.branch_id[e] + "'";
    if (g.br_from[e] == g.br_to[e]) throw ValidationError(w + " connects a node to itself");
    if (!(g.br_x[e] > 0.0)) throw ValidationError(w + " has non-positive reactance");
    if (!(g.br_limit[e] > 0.0)) throw ValidationError(w + " has non-positive flow limit");
  }
  if (g.slack < 0 || g.slack >= n) throw ValidationError("slack node is missing");
  std::vector<Edge> edges;
  for (int e = 0; e < g.n_branches(); ++e) edges.push_back({g.br_from[e], g.br_to[e], g.br_on[e] != 0});
  std::vector<int> all(n);
  std::iota(all.begin(), all.end(), 0);
  if (!connected_with(n, edges, all)) throw ValidationError("grid is disconnected in the base case");
  // grid_model.cpp:108-121 runs a BFS per contingency; a single-branch outage of
  // a connected grid disconnects it iff the branch is an in-service bridge, so
  // one bridge pass answers those (same verdicts, O(E) instead of O(K E)).
  std::vector<char> is_bridge(edges.size(), 0);
  for (int e : bridges(n, edges)) is_bridge[e] = 1;
  for (std::size_t c = 0; c < g.cont_id.size(); ++c) {
    if (g.cont_branches[c].empty() && g.cont_injections[c].empty())
      throw ValidationError("contingency '" + g.cont_id[c] + "' removes nothing");
    const auto& brs = g.cont_branches[c];
    const bool islands = brs.size() == 1 ? (edges[brs[0]].on && is_bridge[brs[0]])
                                         : !brs.empty() && !connected_with(n, edges, all, brs);
    if (islands) throw IslandedContingency("contingency '" + g.cont_id[c] + "' disconnects the base-case grid");
  }
  for (const Station& st : g.stations) {
    const std::string where = "substation at node '" + g.node_id[st.node] + "'";
    if (st.busbars.size() < 2) throw ValidationError(where + " needs at least 2 busbars");
    for (auto [a, b] : st.couplers)
      if (a < 0 || b < 0) throw ValidationError(where + " has a coupler on an unknown busbar");
    std::vector<Edge> ce;
    for (auto [a, b] : st.couplers) ce.push_back({a, b, true});
    std::vector<int> bb(st.busbars.size());
    std::iota(bb.begin(), bb.end(), 0);
    if (!connected_with(static_cast<int>(st.busbars.size()), ce, bb))
      throw ValidationError(where + " has a disconnected coupler graph");
    std::size_t expected = 0;
    for (int e = 0; e < g.n_branches(); ++e) expected += (g.br_from[e] == st.node) + (g.br_to[e] == st.node);
    for (int i = 0; i < g.n_injections(); ++i) expected += g.inj_node[i] == st.node;
    if (expected != st.term_kind.size())
      throw ValidationError(where + " lists " + std::to_string(st.term_kind.size()) + " terminals, expected " +
                            std::to_string(expected));
    for (std::size_t t = 0; t < st.term_kind.size(); ++t) {
      const std::string tw = "terminal '" + st.term_element[t] + "' at node '" + g.node_id[st.node] + "'";
      if (st.term_reach[t].empty()) throw ValidationError(tw + " reaches no busbar");
      for (int b : st.term_reach[t])
        if (b < 0) throw ValidationError(tw + " reaches an unknown busbar");
      if (st.term_default[t] < 0 ||
          std::find(st.term_reach[t].begin(), st.term_reach[t].end(), st.term_default[t]) == st.term_reach[t].end())
        throw ValidationError(tw + " defaults to an unreachable busbar");
    }
  }
}

}  // namespace

Grid load_grid_json(const std::string& text) {
  Value doc;
  try {
    doc = json::parse(text);
  } catch (const json::SyntaxError& e) {
    throw ParseError(std::string("invalid JSON: ") + e.what());
  }
  if (!doc.is_object() || !doc.has("nodes") || !doc.has("branches"))
    throw ParseError("grid file: missing 'nodes' or 'branches'");
  Grid g;
  for (const Value& jn : field(doc, "nodes", "grid").arr) {
    std::string id = get_string(jn, "id", "node");
    g.node_shunt.push_back(opt_number(jn, "shunt_b_pu", 0.0, "node '" + id + "'"));
    const Value* sub = jn.find("substation");
    g.node_sub.push_back(sub && sub->is_string() ? sub->str : std::string());
    if (!g.node_lookup.emplace(id, g.n_nodes()).second) throw ValidationError("duplicate node id '" + id + "'");
    g.node_id.push_back(std::move(id));
  }
  auto node_of = [&](const std::string& id, const std::string& what) {
    auto it = g.node_lookup.find(id);
    if (it == g.node_lookup.end()) throw ValidationError(what + " references unknown node '" + id + "'");
    return it->second;
  };
  for (const Value& jb : field(doc, "branches", "grid").arr) {
    std::string id = get_string(jb, "id", "branch");
    const std::string w = "branch '" + id + "'";
    g.br_from.push_back(node_of(get_string(jb, "from", w), w));
    g.br_to.push_back(node_of(get_string(jb, "to", w), w));
    g.br_x.push_back(get_number(jb, "x_pu", w));
    g.br_limit.push_back(get_number(jb, "limit_mw", w));
    g.br_r.push_back(opt_number(jb, "r_pu", 0.0, w));
    g.br_bc.push_back(opt_number(jb, "b_pu", 0.0, w));
    g.br_tap.push_back(opt_number(jb, "tap", 1.0, w));
    const Value* on = jb.find("in_service");
    g.br_on.push_back(on && on->is_bool() ? on->b : 1);
    if (!g.branch_lookup.emplace(id, g.n_branches() - 1).second) throw ValidationError("duplicate branch id '" + id + "'");
    g.branch_id.push_back(std::move(id));
  }
  for (const Value& ji : opt_array(doc, "injections")) {
    std::string id = get_string(ji, "id", "injection");
    const std::string w = "injection '" + id + "'";
    g.inj_node.push_back(node_of(get_string(ji, "node", w), w));
    g.inj_p.push_back(get_number(ji, "p_mw", w));
    g.inj_q.push_back(opt_number(ji, "q_mvar", 0.0, w));
    const std::string kind = get_string(ji, "kind", w);
    if (kind != "generator" && kind != "load") throw ParseError(w + ": kind must be 'generator' or 'load'");
    g.inj_gen.push_back(kind == "generator");
    const Value* vs = ji.find("v_setpoint_pu");
    g.inj_has_vset.push_back(vs != nullptr);
    g.inj_vset.push_back(vs ? vs->num : 0.0);
    if (const Value* v = vs) {
      if (kind == "load") throw ValidationError("load '" + id + "' carries a voltage setpoint");
      if (!(v->num > 0.0)) throw ValidationError("generator '" + id + "' has a non-positive voltage setpoint");
    }
    if (!g.injection_lookup.emplace(id, g.n_injections() - 1).second)
      throw ValidationError("duplicate injection id '" + id + "'");
    g.inj_id.push_back(std::move(id));
  }
  g.station_of_node.assign(g.n_nodes(), -1);
  for (const Value& js : opt_array(doc, "substations")) {
    Station st;
    const std::string nid = get_string(js, "node", "substation");
    const std::string w = "substation at node '" + nid + "'";
    st.node = node_of(nid, w);
    st.busbars = get_strings(js, "busbars", w);
    for (const Value& jc : opt_array(js, "couplers")) {
      if (!jc.is_array() || jc.arr.size() != 2 || !jc.arr[0].is_string() || !jc.arr[1].is_string())
        throw ParseError(w + ": coupler entries must be [busbar, busbar] pairs");
      st.couplers.emplace_back(st.busbar(jc.arr[0].str), st.busbar(jc.arr[1].str));
    }
    for (const Value& jt : opt_array(js, "terminals")) {
      const std::string el = get_string(jt, "element", w);
      std::vector<int> reach;
      for (const std::string& b : get_strings(jt, "reachable", w)) reach.push_back(st.busbar(b));
      const int def = st.busbar(get_string(jt, "default", w));
      int kind, idx = g.branch_index(el);
      if (idx >= 0) {
        if (g.br_from[idx] == st.node)
          kind = kFromEnd;
        else if (g.br_to[idx] == st.node)
          kind = kToEnd;
        else
          throw ValidationError(w + ": terminal '" + el + "' is a branch that does not end here");
      } else {
        idx = g.injection_index(el);
        if (idx < 0) throw ValidationError(w + ": terminal '" + el + "' matches no branch or injection");
        if (g.inj_node[idx] != st.node)
          throw ValidationError("terminal '" + el + "' at node '" + nid + "' does not match an injection at this node");
        kind = kInjection;
      }
      st.term_element.push_back(el);
      st.term_kind.push_back(kind);
      st.term_index.push_back(idx);
      st.term_reach.push_back(std::move(reach));
      st.term_default.push_back(def);
    }
    g.station_of_node[st.node] = static_cast<int>(g.stations.size());
    g.stations.push_back(std::move(st));
  }
  for (const Value& jc : opt_array(doc, "contingencies")) {
    std::string id = get_string(jc, "id", "contingency");
    const std::string w = "contingency '" + id + "'";
    std::vector<int> brs, injs;
    for (const Value& x : opt_array(jc, "branches")) {
      int e = x.is_string() ? g.branch_index(x.str) : -1;
      if (e < 0) throw ValidationError(w + " references an unknown branch");
      brs.push_back(e);
    }
    for (const Value& x : opt_array(jc, "injections")) {
      int i = x.is_string() ? g.injection_index(x.str) : -1;
      if (i < 0) throw ValidationError(w + " references an unknown injection");
      injs.push_back(i);
    }
    g.cont_id.push_back(std::move(id));
    g.cont_branches.push_back(std::move(brs));
    g.cont_injections.push_back(std::move(injs));
  }
  for (const Value& jb : opt_array(doc, "busbar_outages")) {
    std::string id = get_string(jb, "id", "busbar outage");
    const std::string w = "busbar outage '" + id + "'";
    const std::string nid = get_string(jb, "substation", w);
    const int s = g.station_of_node[node_of(nid, w)];
    if (s < 0) throw ValidationError(w + ": node '" + nid + "' has no substation detail");
    const int bb = g.stations[s].busbar(get_string(jb, "busbar", w));
    if (bb < 0) throw ValidationError(w + " references an unknown busbar");
    g.bo_id.push_back(std::move(id));
    g.bo_station.push_back(s);
    g.bo_busbar.push_back(bb);
  }
  const Value* sl = doc.find("slack");
  if (!sl) throw ParseError("grid file: missing 'slack'");
  if (!sl->is_string()) throw ParseError("grid file: 'slack' must be a node id");
  g.slack = node_of(sl->str, "slack");
  // timestep profiles (extension; see model.hpp)
  g.inj_p_t = g.inj_p;
  if (const Value* ts = doc.find("timesteps")) {
    if (!ts->is_object()) throw ParseError("'timesteps' must be an object");
    const Value* cnt = ts->find("count");
    if (!cnt || !cnt->is_number() || !cnt->integral || cnt->num < 1 || cnt->num > 8760)
      throw ParseError("'timesteps.count' must be an integer in [1, 8760]");
    g.n_t = static_cast<int>(cnt->num);
    const int I = g.n_injections();
    g.inj_p_t.assign(static_cast<size_t>(g.n_t) * I, 0.0);
    for (int t = 0; t < g.n_t; ++t)
      for (int i = 0; i < I; ++i) g.inj_p_t[static_cast<size_t>(t) * I + i] = g.inj_p[i];
    if (const Value* inj = ts->find("injections")) {
      if (!inj->is_object()) throw ParseError("'timesteps.injections' must be an object");
      for (const auto& kv : inj->obj) {
        const int i = g.injection_index(kv.first);
        if (i < 0) throw ValidationError("timestep profile for unknown injection '" + kv.first + "'");
        if (!kv.second.is_array() || static_cast<int>(kv.second.arr.size()) != g.n_t)
          throw ParseError("timestep profile of '" + kv.first + "' must be an array of 'count' numbers");
        for (int t = 0; t < g.n_t; ++t) {
          const Value& v = kv.second.arr[t];
          if (!v.is_number() || !std::isfinite(v.num)) throw ParseError("timestep profile of '" + kv.first + "': non-numeric value");
          g.inj_p_t[static_cast<size_t>(t) * I + i] = v.num;
        }
      }
    }
  }
  validate(g);
  return g;
}

std::vector<double> base_power_vector(const Grid& g) {
  std::vector<double> p(g.n_nodes(), 0.0);
  for (int i = 0; i < g.n_injections(); ++i) p[g.inj_node[i]] += g.inj_net(i);
  double total = 0.0;
  for (double v : p) total += v;
  p[g.slack] -= total;
  return p;
}

// ---------------------------------------------------------------- locality
std::vector<int> locality_rank(int n, const std::vector<std::pair<int, int>>& edges, int leaf) {
  std::vector<std::vector<int>> adj(n);
  for (auto [a, b] : edges) adj[a].push_back(b), adj[b].push_back(a);
  std::vector<int> rank(n, -1), part(n, 0), dist(n, -1);
  int next_rank = 0, next_part = 1;
  // BFS restricted to one part; returns visit order, fills dist
  auto bfs = [&](int src, int pid, std::vector<int>& order) {
    order.clear();
    order.push_back(src);
    dist[src] = 0;
    for (std::size_t h = 0; h < order.size(); ++h)
      for (int w : adj[order[h]])
        if (part[w] == pid && dist[w] < 0) dist[w] = dist[order[h]] + 1, order.push_back(w);
  };
  std::vector<std::pair<int, std::vector<int>>> stack;
  {
    std::vector<int> all(n);
    for (int v = 0; v < n; ++v) all[v] = v;
    stack.emplace_back(0, std::move(all));
  }
  std::vector<int> order, sub;
  while (!stack.empty()) {
    auto [pid, nodes] = std::move(stack.back());
    stack.pop_back();
    if (static_cast<int>(nodes.size()) <= leaf) {
      for (int v : nodes) rank[v] = next_rank++;
      continue;
    }
    // pseudo-peripheral start, then split the BFS order in halves (components
    // of a part are visited one after another)
    std::vector<int> seq;
    for (int v : nodes) dist[v] = -1;
    for (int root : nodes) {
      if (dist[root] >= 0) continue;
      bfs(root, pid, order);
      const int far = order.back();
      for (int v : order) dist[v] = -1;
      bfs(far, pid, order);
      seq.insert(seq.end(), order.begin(), order.end());
    }
    for (int v : nodes) dist[v] = -1;
    const std::size_t half = seq.size() / 2;
    std::vector<int> a(seq.begin(), seq.begin() + half), b(seq.begin() + half, seq.end());
    const int pa = next_part++, pb = next_part++;
    for (int v : a) part[v] = pa;
    for (int v : b) part[v] = pb;
    stack.emplace_back(pb, std::move(b));  // a is ranked first
    stack.emplace_back(pa, std::move(a));
  }
  return rank;
}

// ---------------------------------------------------------------- import
// Base branch graph, node CSR and contingency lists for the device graph kernels
// (cuda/islanding.cu).
SplitGraphDesc split_graph_desc(const Grid& g) {
  SplitGraphDesc gd;
  gd.n_nodes = g.n_nodes();
  gd.br_from.assign(g.br_from.begin(), g.br_from.end());
  gd.br_to.assign(g.br_to.begin(), g.br_to.end());
  gd.br_on.assign(g.br_on.begin(), g.br_on.end());
  std::vector<int> deg(g.n_nodes() + 1, 0);
  for (int e = 0; e < g.n_branches(); ++e) ++deg[g.br_from[e] + 1], ++deg[g.br_to[e] + 1];
  for (int v = 0; v < g.n_nodes(); ++v) deg[v + 1] += deg[v];
  gd.node_ptr = deg;
  gd.node_br.assign(deg.back(), 0);
  std::vector<int> fill(deg.begin(), deg.end() - 1);
  for (int e = 0; e < g.n_branches(); ++e) gd.node_br[fill[g.br_from[e]]++] = e, gd.node_br[fill[g.br_to[e]]++] = e;
  for (const auto& brs : g.cont_branches) {
    if (brs.size() == 1) gd.single_br.push_back(brs[0]);
    if (brs.size() > 1) {
      gd.multi_br.insert(gd.multi_br.end(), brs.begin(), brs.end());
      gd.multi_ptr.push_back(static_cast<int>(gd.multi_br.size()));
    }
    gd.cont_br.insert(gd.cont_br.end(), brs.begin(), brs.end());
    gd.cont_ptr.push_back(static_cast<int>(gd.cont_br.size()));
  }
  return gd;
}

// importer.cpp:42-70. device >= 0: the bridge passes (the base graph and the
// graph without each contingency's branches) run on that GPU, one CTA per pass
// (cuda/islanding.cu); a pass whose graph splits into components falls back to
// the host's general bridge search.
std::vector<int> enumerate_disconnectables(const Grid& g, int device) {
  const int ne = g.n_branches(), n = g.n_nodes();
  std::vector<Edge> edges;
  for (int e = 0; e < ne; ++e) edges.push_back({g.br_from[e], g.br_to[e], g.br_on[e] != 0});
  std::vector<char> out_of_play(ne, 0);
  for (int e = 0; e < ne; ++e) out_of_play[e] = !g.br_on[e];
  for (const auto& brs : g.cont_branches)
    for (int e : brs) out_of_play[e] = 1;
  auto host_pass = [&](int c) {  // c = contingency, or -1: the base graph
    auto cut = edges;
    if (c >= 0)
      for (int e : g.cont_branches[c]) cut[e].on = false;
    for (int e : bridges(n, cut)) out_of_play[e] = 1;
  };
  if (device >= 0) {
    std::vector<char> any;
    std::vector<int> fb;
    contingency_bridges_device(split_graph_desc(g), device, any, fb);
    for (int e = 0; e < ne; ++e)
      if (any[e]) out_of_play[e] = 1;
    const int K = static_cast<int>(g.cont_branches.size());
    for (int c : fb) host_pass(c < K ? c : -1);
  } else {
    host_pass(-1);
    for (int c = 0; c < static_cast<int>(g.cont_branches.size()); ++c)
      if (!g.cont_branches[c].empty()) host_pass(c);
  }
  std::vector<int> d;
  for (int e = 0; e < ne; ++e)
    if (!out_of_play[e]) d.push_back(e);
  return d;
}

namespace {

struct Realized {
  std::vector<int> assignment, open;
  int lambda_r = 0;
};

// BFS order over the coupler graph with neighbours sorted (importer.cpp:122-146)
std::vector<int> coupler_bfs(const std::vector<std::vector<int>>& nbr, int start) {
  std::vector<char> seen(nbr.size(), 0);
  std::vector<int> order{start};
  seen[start] = 1;
  for (std::size_t h = 0; h < order.size(); ++h)
    for (int w : nbr[order[h]])
      if (!seen[w]) seen[w] = 1, order.push_back(w);
  return order;
}

bool coupler_subset_connected(const std::vector<std::vector<int>>& nbr, const std::vector<char>& in) {
  int s = -1, cnt = 0;
  for (int v = 0; v < static_cast<int>(in.size()); ++v)
    if (in[v]) {
      if (s < 0) s = v;
      ++cnt;
    }
  if (cnt <= 1) return cnt == 1;
  std::vector<char> seen(in.size(), 0);
  std::vector<int> q{s};
  seen[s] = 1;
  for (std::size_t h = 0; h < q.size(); ++h)
    for (int w : nbr[q[h]])
      if (in[w] && !seen[w]) seen[w] = 1, q.push_back(w);
  return static_cast<int>(q.size()) == cnt;
}

// importer.cpp:171-235: grow group 0 as a BFS prefix from terminal 0's
// default busbar; smallest prefix serving both groups wins.
bool realize(const Station& st, const std::vector<char>& grp, Realized& r) {
  const int nb = static_cast<int>(st.busbars.size()), nt = static_cast<int>(st.term_kind.size());
  std::vector<std::vector<int>> nbr(nb);
  for (auto [a, b] : st.couplers) nbr[a].push_back(b), nbr[b].push_back(a);
  for (auto& v : nbr) std::sort(v.begin(), v.end());  // (neighbour, coupler) pairs sort by neighbour first
  std::vector<int> order = coupler_bfs(nbr, st.term_default[0]);
  if (static_cast<int>(order.size()) != nb) return false;
  std::vector<std::vector<int>> reach(nt);
  for (int t = 0; t < nt; ++t) {
    reach[t] = st.term_reach[t];
    std::sort(reach[t].begin(), reach[t].end());
  }
  for (int k = 0; k + 1 < nb; ++k) {
    std::vector<char> side0(nb, 0), side1(nb, 0);
    for (int i = 0; i <= k; ++i) side0[order[i]] = 1;
    for (int v = 0; v < nb; ++v) side1[v] = !side0[v];
    if (!coupler_subset_connected(nbr, side1)) continue;
    bool ok = true;
    for (int t = 0; t < nt && ok; ++t) {
      const auto& side = grp[t] ? side1 : side0;
      ok = std::any_of(reach[t].begin(), reach[t].end(), [&](int b) { return side[b] != 0; });
    }
    if (!ok) continue;
    r.assignment.assign(nt, -1);
    r.lambda_r = 0;
    for (int t = 0; t < nt; ++t) {
      const auto& side = grp[t] ? side1 : side0;
      const int def = st.term_default[t];
      if (side[def]) {
        r.assignment[t] = def;
        continue;
      }
      for (int b : order)
        if (side[b] && std::binary_search(reach[t].begin(), reach[t].end(), b)) {
          r.assignment[t] = b;
          break;
        }
      ++r.lambda_r;
    }
    r.open.clear();
    for (int c = 0; c < static_cast<int>(st.couplers.size()); ++c)
      if (side0[st.couplers[c].first] != side0[st.couplers[c].second]) r.open.push_back(c);
    return true;
  }
  return false;
}

// Split feasibility under the base case and every listed contingency
// (importer.cpp:288-339).
bool split_keeps_connected(const Grid& g, int s, const std::vector<char>& grp) {
  const int n = g.n_nodes();
  const Station& st = g.stations[s];
  std::vector<Edge> edges;
  for (int e = 0; e < g.n_branches(); ++e) edges.push_back({g.br_from[e], g.br_to[e], g.br_on[e] != 0});
  bool fresh_used = false;
  for (int t = 0; t < static_cast<int>(st.term_kind.size()); ++t) {
    if (!grp[t]) continue;
    if (st.term_kind[t] == kInjection) {
      fresh_used = true;
      continue;
    }
    Edge& e = edges[st.term_index[t]];
    (st.term_kind[t] == kFromEnd ? e.a : e.b) = n;
    fresh_used = fresh_used || e.on;
  }
  std::vector<int> must(n);
  std::iota(must.begin(), must.end(), 0);
  if (fresh_used) must.push_back(n);
  if (!connected_with(n + 1, edges, must)) return false;
  std::vector<char> is_bridge(edges.size(), 0);
  for (int e : bridges(n + 1, edges)) is_bridge[e] = 1;
  for (const auto& brs : g.cont_branches) {
    if (brs.empty()) continue;
    if (brs.size() == 1) {
      if (edges[brs[0]].on && is_bridge[brs[0]]) return false;
    } else if (!connected_with(n + 1, edges, must, brs)) {
      return false;
    }
  }
  return true;
}

}  // namespace

// importer.cpp:239-282 + 341-356. Ids: station order, then enumeration order.
ActionTable build_actions(const Grid& g, std::uint64_t seed, std::int64_t cap, int device) {
  ActionTable t;
  static const bool timing = std::getenv("TGB_IMPORT_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "import %s: %.3f s\n", what, std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  t.disconnectables = enumerate_disconnectables(g, device);
  lap("disconnectables");
  t.station_range.assign(g.stations.size(), {-1, -1});
  std::vector<std::pair<int, std::vector<char>>> pending;  // (station, group) in enumeration order
  for (int s = 0; s < static_cast<int>(g.stations.size()); ++s) {
    const Station& st = g.stations[s];
    const int nt = static_cast<int>(st.term_kind.size());
    if (st.busbars.size() < 2 || nt < 2) continue;
    std::mt19937_64 rng(derive(seed, 0x5741u, static_cast<std::uint64_t>(s)));
    std::vector<std::vector<char>> cands;
    std::set<std::string> seen;
    auto live = [&](int k) { return st.term_kind[k] == kInjection || g.br_on[st.term_index[k]]; };
    auto consider = [&](std::uint64_t mask) {
      std::vector<char> grp(nt, 0);
      for (int k = 1; k < nt; ++k) grp[k] = static_cast<char>((mask >> (k - 1)) & 1u);
      // electrical identity: unordered partition of live terminals (importer.cpp:87-103)
      std::vector<int> a, b;
      for (int k = 0; k < nt; ++k)
        if (live(k)) (grp[k] ? b : a).push_back(k);
      if (a.empty() || b.empty()) return;
      if (b.front() < a.front()) std::swap(a, b);
      std::string key;
      for (int k : a) key += std::to_string(k) + ",";
      key += "|";
      for (int k : b) key += std::to_string(k) + ",";
      if (!seen.insert(key).second) return;
      cands.push_back(std::move(grp));
    };
    const int free_bits = nt - 1;
    if (free_bits <= 30 && (std::int64_t{1} << free_bits) <= (cap << 1)) {
      for (std::uint64_t m = 1; m < (std::uint64_t{1} << free_bits); ++m) consider(m);
      if (static_cast<std::int64_t>(cands.size()) > cap) {
        std::vector<std::vector<char>> kept;
        std::sample(cands.begin(), cands.end(), std::back_inserter(kept), cap, rng);
        cands = std::move(kept);
      }
    } else {
      std::uniform_int_distribution<std::uint64_t> dist(1, (std::uint64_t{1} << free_bits) - 1);
      for (std::int64_t k = 0; k < cap * 2 && static_cast<std::int64_t>(cands.size()) < cap; ++k) consider(dist(rng));
    }
    for (auto& grp : cands) pending.push_back({s, std::move(grp)});
  }
  lap("enumeration");
  // realization + islanding validation of every candidate split are
  // independent (importer.cpp:288-356): fanned out over the host cores, ids
  // assigned afterwards in (station, enumeration) order as the reference does
  std::vector<Realized> real(pending.size());
  std::vector<char> keep(pending.size(), 0);
  if (device >= 0) {
    // realization on the host, islanding validation of every realized split
    // on the device (cuda/islanding.cu), one CTA per split
    std::vector<char> realized(pending.size(), 0);
    for (std::size_t i = 0; i < pending.size(); ++i)
      realized[i] = realize(g.stations[pending[i].first], pending[i].second, real[i]);
    const SplitGraphDesc gd = split_graph_desc(g);
    SplitCandidates cd;
    std::vector<std::size_t> idx;
    for (std::size_t i = 0; i < pending.size(); ++i) {
      if (!realized[i]) continue;
      const Station& st = g.stations[pending[i].first];
      const auto& grp = pending[i].second;
      bool fresh = false;
      for (int k = 0; k < static_cast<int>(st.term_kind.size()); ++k) {
        if (!grp[k]) continue;
        if (st.term_kind[k] == kInjection) {
          fresh = true;
          continue;
        }
        const int e = st.term_index[k];
        cd.moved.push_back(st.term_kind[k] == kFromEnd ? 1 + e : -(1 + e));
        fresh = fresh || g.br_on[e];
      }
      cd.moved_ptr.push_back(static_cast<int>(cd.moved.size()));
      cd.station_node.push_back(st.node);
      cd.fresh_used.push_back(fresh);
      idx.push_back(i);
    }
    std::vector<char> ok;
    validate_splits_device(gd, cd, device, ok);
    for (std::size_t j = 0; j < idx.size(); ++j) keep[idx[j]] = ok[j];
  } else {
    std::atomic<std::size_t> next{0};
    auto work = [&] {
      for (std::size_t i; (i = next.fetch_add(1)) < pending.size();) {
        const int s = pending[i].first;
        keep[i] = realize(g.stations[s], pending[i].second, real[i]) && split_keeps_connected(g, s, pending[i].second);
      }
    };
    const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                         static_cast<unsigned>(pending.size() / 8 + 1)));
    std::vector<std::thread> pool;
    for (unsigned k = 1; k < nth; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }
  for (std::size_t i = 0; i < pending.size(); ++i) {
    if (!keep[i]) continue;
    const int s = pending[i].first;
    if (t.station_range[s].first < 0) t.station_range[s].first = t.n_actions();
    t.station.push_back(s);
    t.group.push_back(std::move(pending[i].second));
    t.assignment.push_back(std::move(real[i].assignment));
    t.open_couplers.push_back(std::move(real[i].open));
    t.lambda_r.push_back(real[i].lambda_r);
    t.station_range[s].second = t.n_actions();
  }
  return t;
}

// Cache schema of importer.cpp:407-430 (grid_hash = grid_content_hash, grid_model.cpp:494-503).
std::string actions_to_json(const ActionTable& t, const Grid& g, std::uint64_t hash) {
  std::string o = "{\"grid_hash\":" + std::to_string(hash) + ",\"disconnectables\":[";
  for (std::size_t i = 0; i < t.disconnectables.size(); ++i)
    o += (i ? "," : "") + json::quote(g.branch_id[t.disconnectables[i]]);
  o += "],\"actions\":[";
  for (int a = 0; a < t.n_actions(); ++a) {
    const Station& st = g.stations[t.station[a]];
    o += a ? ",{" : "{";
    o += "\"node\":" + json::quote(g.node_id[st.node]) + ",\"group\":[";
    for (std::size_t k = 0; k < t.group[a].size(); ++k) o += (k ? "," : "") + std::to_string(int(t.group[a][k]));
    o += "],\"busbars\":[";
    for (std::size_t k = 0; k < t.assignment[a].size(); ++k)
      o += (k ? "," : "") + json::quote(st.busbars[t.assignment[a][k]]);
    o += "],\"open_couplers\":[";
    for (std::size_t k = 0; k < t.open_couplers[a].size(); ++k)
      o += (k ? "," : "") + std::to_string(t.open_couplers[a][k]);
    o += "],\"lambda_r\":" + std::to_string(t.lambda_r[a]) + "}";
  }
  return o + "]}";
}

bool actions_from_json(const std::string& text, const Grid& g, std::uint64_t hash, ActionTable& out) {
  Value doc;
  try {
    doc = json::parse(text);
  } catch (const json::SyntaxError&) {
    return false;
  }
  const Value* h = doc.find("grid_hash");
  if (!h || !h->is_number()) return false;
  if (!h->integral || h->u64 != hash) return false;
  ActionTable t;
  t.station_range.assign(g.stations.size(), {-1, -1});
  const Value* d = doc.find("disconnectables");
  const Value* acts = doc.find("actions");
  if (!d || !acts || !d->is_array() || !acts->is_array()) return false;
  for (const Value& x : d->arr) {
    const int e = x.is_string() ? g.branch_index(x.str) : -1;
    if (e < 0) return false;
    t.disconnectables.push_back(e);
  }
  for (const Value& ja : acts->arr) {
    const Value* node = ja.find("node");
    if (!node || !node->is_string()) return false;
    auto it = g.node_lookup.find(node->str);
    if (it == g.node_lookup.end()) return false;
    const int s = g.station_of_node[it->second];
    if (s < 0) return false;
    const Station& st = g.stations[s];
    std::vector<char> grp;
    std::vector<int> asg, open;
    for (const Value& x : field(ja, "group", "action").arr) grp.push_back(x.num != 0.0);
    for (const Value& x : field(ja, "busbars", "action").arr) {
      const int b = st.busbar(x.str);
      if (b < 0) return false;
      asg.push_back(b);
    }
    for (const Value& x : field(ja, "open_couplers", "action").arr) open.push_back(static_cast<int>(x.num));
    const int a = t.n_actions();
    t.station.push_back(s);
    t.group.push_back(std::move(grp));
    t.assignment.push_back(std::move(asg));
    t.open_couplers.push_back(std::move(open));
    t.lambda_r.push_back(static_cast<int>(field(ja, "lambda_r", "action").num));
    auto& r = t.station_range[s];
    if (r.first < 0)
      r = {a, a + 1};
    else
      r.second = a + 1;
  }
  out = std::move(t);
  return true;
}

}  // namespace tgb
