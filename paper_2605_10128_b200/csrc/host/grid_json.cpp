// Canonical grid serialization and content hash of the reference, so that the
// action cache (importer.cpp:407-479) is keyed identically on both sides.
//
//   grid_to_json_text   <- grid_model.cpp:423-485 (nlohmann::ordered_json, dump(2))
//   grid_content_hash   <- grid_model.cpp:494-503 (FNV-1a over that text)
//
// The reference builds the text with nlohmann/json (`using json =
// nlohmann::ordered_json`, grid_model.cpp:14); the hash depends on that
// library's number formatting (shortest round-trip digits, "1.0" for integral
// doubles) and indentation, so this file uses the same library (v3.11.3, the
// header the image ships) rather than a second formatter that could disagree
// on some double.
#include <nlohmann/json.hpp>

#include "model.hpp"

namespace tgb {

using ojson = nlohmann::ordered_json;

std::string grid_to_json_text(const Grid& g) {
  ojson doc;
  doc["nodes"] = ojson::array();
  for (int v = 0; v < g.n_nodes(); ++v) {
    ojson jn{{"id", g.node_id[v]}};
    if (!g.node_sub[v].empty()) jn["substation"] = g.node_sub[v];
    if (g.node_shunt[v] != 0.0) jn["shunt_b_pu"] = g.node_shunt[v];
    doc["nodes"].push_back(jn);
  }
  doc["branches"] = ojson::array();
  for (int e = 0; e < g.n_branches(); ++e) {
    ojson jb{{"id", g.branch_id[e]},
             {"from", g.node_id[g.br_from[e]]},
             {"to", g.node_id[g.br_to[e]]},
             {"x_pu", g.br_x[e]},
             {"limit_mw", g.br_limit[e]}};
    if (g.br_r[e] != 0.0) jb["r_pu"] = g.br_r[e];
    if (g.br_bc[e] != 0.0) jb["b_pu"] = g.br_bc[e];
    if (g.br_tap[e] != 1.0) jb["tap"] = g.br_tap[e];
    if (!g.br_on[e]) jb["in_service"] = false;
    doc["branches"].push_back(jb);
  }
  doc["injections"] = ojson::array();
  for (int i = 0; i < g.n_injections(); ++i) {
    ojson ji{{"id", g.inj_id[i]},
             {"node", g.node_id[g.inj_node[i]]},
             {"p_mw", g.inj_p[i]},
             {"q_mvar", g.inj_q[i]},
             {"kind", g.inj_gen[i] ? "generator" : "load"}};
    if (g.inj_has_vset[i]) ji["v_setpoint_pu"] = g.inj_vset[i];
    doc["injections"].push_back(ji);
  }
  doc["contingencies"] = ojson::array();
  for (size_t c = 0; c < g.cont_id.size(); ++c) {
    ojson jc{{"id", g.cont_id[c]}};
    jc["branches"] = ojson::array();
    for (int e : g.cont_branches[c]) jc["branches"].push_back(g.branch_id[e]);
    jc["injections"] = ojson::array();
    for (int i : g.cont_injections[c]) jc["injections"].push_back(g.inj_id[i]);
    doc["contingencies"].push_back(jc);
  }
  doc["busbar_outages"] = ojson::array();
  for (size_t b = 0; b < g.bo_id.size(); ++b) {
    const Station& st = g.stations[g.bo_station[b]];
    doc["busbar_outages"].push_back(
        ojson{{"id", g.bo_id[b]}, {"substation", g.node_id[st.node]}, {"busbar", st.busbars[g.bo_busbar[b]]}});
  }
  doc["substations"] = ojson::array();
  for (const Station& st : g.stations) {
    ojson js{{"node", g.node_id[st.node]}, {"busbars", st.busbars}};
    js["couplers"] = ojson::array();
    for (const auto& [a, b] : st.couplers) js["couplers"].push_back(ojson::array({st.busbars[a], st.busbars[b]}));
    js["terminals"] = ojson::array();
    for (size_t t = 0; t < st.term_kind.size(); ++t) {
      std::vector<std::string> reach;
      for (int r : st.term_reach[t]) reach.push_back(st.busbars[r]);
      js["terminals"].push_back(
          ojson{{"element", st.term_element[t]}, {"reachable", reach}, {"default", st.busbars[st.term_default[t]]}});
    }
    doc["substations"].push_back(js);
  }
  doc["slack"] = g.node_id[g.slack];
  return doc.dump(2);
}

std::uint64_t grid_content_hash(const Grid& g) {
  std::uint64_t h = 14695981039346656037ull;
  for (unsigned char c : grid_to_json_text(g)) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace tgb
