// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// The reference's independent test oracles and seeded fixtures
// (tests/helpers.hpp:1-583), restated: tiny JSON grids, the seeded random grid
// and genome generators, rebuild-from-scratch flow oracles.
#pragma once

#include <optional>
#include <set>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "oracle.hpp"

namespace oracle::fx {

using json = nlohmann::json;

GridModel grid_from_json(const json& j);
GridModel two_node_grid();                                             // helpers.hpp:32-43
GridModel triangle_grid(double lab = 100, double lac = 100, double lbc = 100,
                        const std::vector<std::string>& outages = {});  // helpers.hpp:46-62
json station_json(const std::string& node, const std::vector<std::string>& elements,
                  const std::vector<std::string>& defaults = {});       // helpers.hpp:65-78
GridModel mini_congestion_grid();                                       // helpers.hpp:83-103

struct OracleEdge {
  int from, to;
  bool active;
};
bool oracle_connected(int n, const std::vector<OracleEdge>& edges);   // helpers.hpp:112-135
std::vector<OracleEdge> oracle_edges(const GridModel& g);
std::set<int> oracle_bridges(int n, const std::vector<OracleEdge>& edges);  // 144-153
std::set<int> oracle_disconnectables(const GridModel& g);                   // 156-181

struct ComposedTopology {
  std::vector<std::pair<int, int>> ends;
  std::vector<char> removed;
  std::vector<int> injection_node;
  int n_new = 0;
};
ComposedTopology compose_topology(const GridModel& g, const ActionSet& s, const Genome& genome);  // 193-219
struct MaterializedTopology {
  DcGraph graph;
  Vec injections;
  std::vector<char> removed;
  std::vector<int> injection_node;
};
MaterializedTopology materialize(const GridModel& g, const ActionSet& s, const Genome& genome);  // 228-275
Vec rebuild_flows(const MaterializedTopology& m);                                                 // 278-281
Vec angle_flows(const DcGraph& graph, const Vec& p);                                             // 284-313
std::optional<Vec> scratch_outage_flows(const GridModel& g, const ActionSet& s, const Genome& genome,
                                        const std::vector<int>& branches_out,
                                        const std::vector<int>& injections_out);  // 319-387
std::vector<int> scratch_implied_branches(const GridModel& g, const ActionSet& s, const Genome& genome,
                                          const BusbarOutage& outage);  // 392-431

struct RandomGridOptions {
  int n_nodes = 20;
  int extra_edges = 10;
  int n_outages = 5;
  int n_stations = 2;
  bool multi_branch_outages = false;
  bool injection_outages = false;
  bool busbar_outages = false;
};
json random_grid_json(std::uint64_t seed, const RandomGridOptions& opt = {});  // 435-553
GridModel random_grid(std::uint64_t seed, const RandomGridOptions& opt = {});
Genome random_genome(const ActionSet& s, int n_a, int n_d, std::mt19937_64& rng);  // 555-581

}  // namespace oracle::fx
