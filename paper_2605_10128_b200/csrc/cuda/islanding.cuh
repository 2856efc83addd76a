// Device islanding validation of candidate station splits (islanding.cu).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

namespace tgb {

// a candidate split beyond the kernel's shared-memory capacity (reported as
// TG_CAPACITY_ERROR by the C ABI, never truncated)
struct SplitCapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Base branch graph and the listed contingencies (grid order).
struct SplitGraphDesc {
  int n_nodes = 0;
  std::vector<int> br_from, br_to;
  std::vector<uint8_t> br_on;
  std::vector<int> node_ptr, node_br;    // CSR: every branch at both ends
  std::vector<int> single_br;            // branch of each single-branch contingency
  std::vector<int> multi_ptr{0}, multi_br;  // CSR of the multi-branch contingencies
  std::vector<int> cont_ptr{0}, cont_br;    // CSR of every contingency's branches (contingency_bridges_device)
};

// Candidate splits: split node, moved branch ends (+1 + e from end, -(1 + e)
// to end), whether the fresh node carries a terminal that counts
// (split_edges' new_node_used, importer.cpp:288-312).
struct SplitCandidates {
  std::vector<int> station_node;
  std::vector<int> moved_ptr{0}, moved;
  std::vector<uint8_t> fresh_used;
};

// keep[i] = validate_action_islanding (importer.cpp:314-339) of candidate i,
// computed on `device`.
void validate_splits_device(const SplitGraphDesc& g, const SplitCandidates& c, int device, std::vector<char>& keep);

// enumerate_disconnectables' bridge passes (importer.cpp:42-70) on `device`:
// is_bridge_any[e] = e is a bridge of the base graph or of the base graph
// without some contingency's branches. fallback_cases: cases (contingency index,
// or the number of contingencies for the base graph) whose graph has a second
// component; the caller runs the host pass for them.
void contingency_bridges_device(const SplitGraphDesc& g, int device, std::vector<char>& is_bridge_any,
                                std::vector<int>& fallback_cases);

}  // namespace tgb
