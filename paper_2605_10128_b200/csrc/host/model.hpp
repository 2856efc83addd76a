// Host-side network model and import step for the B200 engine.
//
// Mirrors the reference's data model and import semantics so that a grid file
// and the action ids derived from it are identical on both sides:
//   grid_model.hpp:16-139 / grid_model.cpp:79-413  -> Grid, load_grid_json, validate
//   graph_utils.cpp:31-116                          -> connected_with, bridges
//   importer.cpp:42-356                             -> build_actions (ids, order)
// Layout is flat (struct-of-arrays, index-based) because its only consumer is
// the device-table builder (engine_tables.cpp) and the C-ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace tgb {

// Error kinds of errors.hpp:9-34; the C-ABI maps each to a tg_status.
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValidationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IslandedContingency : std::runtime_error { using std::runtime_error::runtime_error; };
struct SingularSystem : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };

enum TermKind : int32_t { kFromEnd = 0, kToEnd = 1, kInjection = 2 };

struct Station {
  int node = -1;
  std::vector<std::string> busbars;
  std::vector<std::pair<int, int>> couplers;  // busbar index pairs
  // per terminal
  std::vector<std::string> term_element;
  std::vector<int> term_kind;
  std::vector<int> term_index;
  std::vector<std::vector<int>> term_reach;  // busbar indices, file order
  std::vector<int> term_default;
  int busbar(const std::string& name) const {
    for (int i = 0; i < static_cast<int>(busbars.size()); ++i)
      if (busbars[i] == name) return i;
    return -1;
  }
};

struct Grid {
  std::vector<std::string> node_id;
  std::vector<std::string> branch_id;
  std::vector<int> br_from, br_to;
  std::vector<double> br_x, br_limit;
  std::vector<char> br_on;
  std::vector<std::string> inj_id;
  std::vector<int> inj_node;
  std::vector<double> inj_p;
  std::vector<char> inj_gen;
  std::vector<std::string> cont_id;
  std::vector<std::vector<int>> cont_branches, cont_injections;
  std::vector<std::string> bo_id;
  std::vector<int> bo_station, bo_busbar;
  std::vector<Station> stations;
  int slack = -1;
  // fields that enter only the canonical dump (grid_to_json_text /
  // grid_content_hash, grid_model.cpp:423-503): node substation names and
  // shunts, branch r / charging / tap, injection q and voltage setpoints
  std::vector<std::string> node_sub;
  std::vector<double> node_shunt, br_r, br_bc, br_tap, inj_q, inj_vset;
  std::vector<char> inj_has_vset;
  // Timestep extension (not in the reference, whose GridModel carries one
  // injection vector, grid_model.hpp:36-46): top-level key
  //   "timesteps": {"count": T, "injections": {"<injection id>": [p_mw x T], ...}}
  // which the reference loader ignores. Injections without a profile keep p_mw.
  // n_t == 1 and inj_p_t == inj_p when the key is absent.
  int n_t = 1;
  std::vector<double> inj_p_t;  // [n_t][n_injections] p_mw
  double inj_net_t(int t, int i) const {
    const double p = inj_p_t[static_cast<size_t>(t) * inj_node.size() + i];
    return inj_gen[i] ? p : -p;
  }

  int n_nodes() const { return static_cast<int>(node_id.size()); }
  int n_branches() const { return static_cast<int>(br_from.size()); }
  int n_injections() const { return static_cast<int>(inj_node.size()); }
  double inj_net(int i) const { return inj_gen[i] ? inj_p[i] : -inj_p[i]; }
  int station_at(int node) const;
  int branch_index(const std::string& id) const;
  int injection_index(const std::string& id) const;

  // grid_model.cpp:187-242: in-service branches whose terminal busbar lies in
  // the failed busbar's coupler group (given assignment + open couplers).
  std::vector<int> implied_branches(int station, int busbar, const std::vector<int>& assignment,
                                    const std::vector<int>& open_couplers) const;
  std::vector<int> default_implied(int busbar_outage) const;

  std::unordered_map<std::string, int> node_lookup, branch_lookup, injection_lookup;
  std::vector<int> station_of_node;
};

// grid_model.cpp:263-413 + validate() 79-185. Throws the error kinds above.
Grid load_grid_json(const std::string& text);

// Net nodal injections, slack absorbing the residual (grid_model.cpp:505-510).
std::vector<double> base_power_vector(const Grid& g);

// ---- graph helpers (graph_utils.cpp) ---------------------------------------
struct Edge {
  int a, b;
  bool on;
};
bool connected_with(int n, const std::vector<Edge>& edges, const std::vector<int>& must_reach,
                    const std::vector<int>& cut = {});
std::vector<int> bridges(int n, const std::vector<Edge>& edges);

// ---- import (importer.hpp:19-95) ---------------------------------------------
struct ActionTable {
  // per action
  std::vector<int> station;
  std::vector<std::vector<char>> group;
  std::vector<std::vector<int>> assignment;
  std::vector<std::vector<int>> open_couplers;
  std::vector<int> lambda_r;
  std::vector<int> disconnectables;                  // branch indices, ascending
  std::vector<std::pair<int, int>> station_range;    // per station, (-1,-1) when none
  int n_actions() const { return static_cast<int>(station.size()); }
};

// Locality-preserving node ranking (recursive BFS bisection, leaves of at most
// `leaf` nodes): nodes close in the graph get close ranks. Used to order the
// contingency tiles of the sweep so each tile is electrically compact.
std::vector<int> locality_rank(int n, const std::vector<std::pair<int, int>>& edges, int leaf = 48);

// device >= 0: the bridge passes on that GPU (cuda/islanding.cu), same result
std::vector<int> enumerate_disconnectables(const Grid& g, int device = -1);
// device >= 0: the islanding validation of the candidate splits runs on that
// GPU (cuda/islanding.cu) instead of the host threads; same ids.
ActionTable build_actions(const Grid& g, std::uint64_t seed, std::int64_t cap, int device = -1);
std::string actions_to_json(const ActionTable& t, const Grid& g, std::uint64_t grid_hash);
bool actions_from_json(const std::string& text, const Grid& g, std::uint64_t grid_hash, ActionTable& out);
// grid_model.cpp:423-485: the reference's canonical serialization (nlohmann
// ordered_json, dump(2)); grid_model.cpp:494-503: FNV-1a over it, the key of
// the action cache (importer.cpp:407-479), so caches written by either side
// load on the other. host/grid_json.cpp.
std::string grid_to_json_text(const Grid& g);
std::uint64_t grid_content_hash(const Grid& g);

}  // namespace tgb
