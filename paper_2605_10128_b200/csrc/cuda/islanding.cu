// Islanding validation of candidate station splits on the device (SURVEY
// §8(f) row 3; importer.cpp:284-339 validate_action_islanding).
//
// One CTA per candidate split. The split graph is the base branch graph with
// the moved branch ends attached to a fresh node n (split_edges,
// importer.cpp:288-312). The CTA
//   1. runs a level-synchronous BFS from node 0 over the live branches,
//      recording each reached node's tree edge and depth, and checks that
//      every base node (and the fresh node when it carries a terminal) is
//      reached (graph_connected with must_reach, graph_utils.cpp:31-64);
//   2. marks every tree edge covered by a non-tree edge (the tree paths from
//      both ends of the non-tree edge up to their lowest common ancestor): a
//      live branch is a bridge iff it is an uncovered tree edge — the same set
//      graph_bridges (graph_utils.cpp:66-116) returns;
//   3. rejects the split if a single-branch contingency's live branch is a
//      bridge, and runs one more BFS without the branches of each
//      multi-branch contingency (graph_connected_without).
// The result is an exact graph property (no floating point), so the action
// ids equal the reference's.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "islanding.cuh"

namespace tgb {

namespace {

constexpr int kIslThreads = 256;
constexpr int kIslMaxMoved = 256;  // moved branch ends per candidate kept in shared memory

struct IslGraph {
  int N, E;
  const int* br_from;
  const int* br_to;
  const uint8_t* br_on;
  const int* node_ptr;  // [N+1] CSR of every branch at each end (in-service or not)
  const int* node_br;
  int n_single;         // single-branch contingencies
  const int* single_br;
  int n_multi;          // multi-branch contingencies (CSR)
  const int* multi_ptr;
  const int* multi_br;
};

struct IslCands {
  int n;
  const int* station_node;  // [n] the split node s
  const int* moved_ptr;     // [n+1] CSR of moved branch ends: +1 + e = from end, -(1 + e) = to end
  const int* moved;
  const uint8_t* fresh_used;  // [n] the fresh node carries a live branch or an injection
  uint8_t* keep;              // [n] out
};

struct IslScratch {
  int* dist;      // [slots][N+1]
  int* par_edge;  // [slots][N+1]
  int* queue;     // [slots][2][N+1]
  uint8_t* cov;   // [slots][E] covered tree edge / 2 = tree edge
};

struct Split {
  int s, n, nm;
  int* mv;          // shared: moved ends (signed, see IslCands)
  uint32_t* mbits;  // shared: bit e of (from-moved | to-moved) branches
};

__device__ __forceinline__ bool moved_end(const Split& sp, int e, bool from_end) {
  if (!((sp.mbits[e >> 5] >> (e & 31)) & 1u)) return false;
  const int code = from_end ? 1 + e : -(1 + e);
  for (int i = 0; i < sp.nm; ++i)
    if (sp.mv[i] == code) return true;
  return false;
}

__device__ __forceinline__ void ends(const IslGraph& g, const Split& sp, int e, int& a, int& b) {
  a = g.br_from[e];
  b = g.br_to[e];
  if ((sp.mbits[e >> 5] >> (e & 31)) & 1u) {
    if (moved_end(sp, e, true)) a = sp.n;
    if (moved_end(sp, e, false)) b = sp.n;
  }
}

__device__ __forceinline__ bool excluded(const int* x0, const int* x1, int e) {
  for (const int* p = x0; p < x1; ++p)
    if (*p == e) return true;
  return false;
}

// BFS from node 0 over live, non-excluded branches; returns the number of
// reached nodes among the attached ones (every base node, plus the fresh node
// when `fresh_attached`) that were NOT reached (0 = connected).
__device__ int bfs(const IslGraph& g, const Split& sp, const int* x0, const int* x1, bool fresh_attached, int* dist,
                   int* par_edge, int* q0, int* q1, int* shv) {
  const int tid = threadIdx.x, nn = g.N + 1;
  for (int v = tid; v < nn; v += kIslThreads) dist[v] = -1, par_edge[v] = -1;
  __syncthreads();
  if (tid == 0) {
    dist[0] = 0;
    q0[0] = 0;
    shv[0] = 1;  // frontier size
  }
  __syncthreads();
  int level = 0;
  int* cur = q0;
  int* nxt = q1;
  for (;;) {
    const int fs = shv[0];
    if (fs == 0) break;
    if (tid == 0) shv[1] = 0;
    __syncthreads();
    for (int i = tid; i < fs; i += kIslThreads) {
      const int v = cur[i];
      auto visit = [&](int e) {
        if (!g.br_on[e] || (x0 && excluded(x0, x1, e))) return;
        int a, b;
        ends(g, sp, e, a, b);
        if (a != v && b != v) return;  // this end moved away from v
        const int w = a == v ? b : a;
        if (atomicCAS(dist + w, -1, level + 1) == -1) {
          par_edge[w] = e;
          nxt[atomicAdd(shv + 1, 1)] = w;
        }
      };
      if (v < g.N) {
        for (int k = g.node_ptr[v]; k < g.node_ptr[v + 1]; ++k) visit(g.node_br[k]);
      } else {
        for (int k = 0; k < sp.nm; ++k) visit(sp.mv[k] > 0 ? sp.mv[k] - 1 : -sp.mv[k] - 1);
      }
    }
    __syncthreads();
    if (tid == 0) shv[0] = shv[1];
    __syncthreads();
    int* t = cur;
    cur = nxt;
    nxt = t;
    ++level;
  }
  int missing = 0;
  for (int v = tid; v < nn; v += kIslThreads)
    if (dist[v] < 0 && (v < g.N || fresh_attached)) ++missing;
  return __syncthreads_count(missing > 0);
}

__global__ void __launch_bounds__(kIslThreads) k_split_valid(IslGraph g, IslCands c, IslScratch sc) {
  __shared__ int mv[kIslMaxMoved];
  __shared__ int shv[2];
  extern __shared__ uint32_t mbits[];
  const int tid = threadIdx.x, nn = g.N + 1, words = (g.E + 31) >> 5;
  int* dist = sc.dist + static_cast<size_t>(blockIdx.x) * nn;
  int* pe = sc.par_edge + static_cast<size_t>(blockIdx.x) * nn;
  int* q0 = sc.queue + static_cast<size_t>(blockIdx.x) * 2 * nn;
  int* q1 = q0 + nn;
  uint8_t* cov = sc.cov + static_cast<size_t>(blockIdx.x) * g.E;
  for (int ci = blockIdx.x; ci < c.n; ci += gridDim.x) {
    const int m0 = c.moved_ptr[ci], nm = c.moved_ptr[ci + 1] - m0;
    for (int w = tid; w < words; w += kIslThreads) mbits[w] = 0u;
    __syncthreads();
    for (int i = tid; i < nm; i += kIslThreads) {
      const int code = c.moved[m0 + i];
      mv[i] = code;
      const int e = code > 0 ? code - 1 : -code - 1;
      atomicOr(mbits + (e >> 5), 1u << (e & 31));
    }
    __syncthreads();
    Split sp{c.station_node[ci], g.N, nm, mv, mbits};
    const bool fresh = c.fresh_used[ci];
    bool ok = bfs(g, sp, nullptr, nullptr, fresh, dist, pe, q0, q1, shv) == 0;
    if (ok && g.n_single > 0) {
      // tree edges (2), then covered ones (1): walk both ends of every live
      // non-tree edge up to their lowest common ancestor
      for (int e = tid; e < g.E; e += kIslThreads) cov[e] = 0;
      __syncthreads();
      for (int v = tid; v < nn; v += kIslThreads)
        if (pe[v] >= 0) cov[pe[v]] = 2;
      __syncthreads();
      for (int e = tid; e < g.E; e += kIslThreads) {
        if (!g.br_on[e]) continue;
        int a, b;
        ends(g, sp, e, a, b);
        if (pe[a] == e || pe[b] == e) continue;  // tree edge
        if (dist[a] < 0) continue;  // outside the reached component (isolated fresh node)
        while (a != b) {
          if (dist[a] >= dist[b]) {
            const int pa = pe[a];
            cov[pa] = 3;
            int x, y;
            ends(g, sp, pa, x, y);
            a = x == a ? y : x;
          } else {
            const int pb = pe[b];
            cov[pb] = 3;
            int x, y;
            ends(g, sp, pb, x, y);
            b = x == b ? y : x;
          }
        }
      }
      __syncthreads();
      bool bridge_hit = false;
      for (int k = tid; k < g.n_single; k += kIslThreads) {
        const int e = g.single_br[k];
        if (g.br_on[e] && cov[e] == 2) bridge_hit = true;  // uncovered tree edge
      }
      ok = !__syncthreads_or(bridge_hit);
    }
    for (int k = 0; ok && k < g.n_multi; ++k)
      ok = bfs(g, sp, g.multi_br + g.multi_ptr[k], g.multi_br + g.multi_ptr[k + 1], fresh, dist, pe, q0, q1, shv) == 0;
    if (tid == 0) c.keep[ci] = ok;
    __syncthreads();
  }
}


// Bridges of the base graph without each contingency's branches
// (enumerate_disconnectables, importer.cpp:42-70): one CTA per case (case
// n_cases = the base graph itself), BFS from node 0 over the live,
// non-excluded branches, tree-path covering by the non-tree ones; every
// uncovered tree edge is a bridge of that graph and is OR-ed into `bridges`.
// A case whose graph leaves a live branch unreached from node 0 (a second
// component) is flagged for the host's general bridge pass.
__global__ void __launch_bounds__(kIslThreads) k_cont_bridges(IslGraph g, const int* cptr, const int* cbr, int n_cases,
                                                              IslScratch sc, uint32_t* bridges, int* fallback) {
  __shared__ int shv[2];
  __shared__ int mv_dummy[1];
  extern __shared__ uint32_t mb_zero[];  // no moved ends: an all-zero bitmap over the branches
  const int tid = threadIdx.x, nn = g.N + 1, words = (g.E + 31) >> 5;
  int* dist = sc.dist + static_cast<size_t>(blockIdx.x) * nn;
  int* pe = sc.par_edge + static_cast<size_t>(blockIdx.x) * nn;
  int* q0 = sc.queue + static_cast<size_t>(blockIdx.x) * 2 * nn;
  int* q1 = q0 + nn;
  uint8_t* cov = sc.cov + static_cast<size_t>(blockIdx.x) * g.E;
  for (int w = tid; w < words; w += kIslThreads) mb_zero[w] = 0u;
  __syncthreads();
  // no split: a graph with no moved ends (the fresh node n = N stays isolated)
  Split sp{-1, g.N, 0, mv_dummy, mb_zero};
  for (int ci = blockIdx.x; ci <= n_cases; ci += gridDim.x) {
    const int* x0 = ci < n_cases ? cbr + cptr[ci] : nullptr;
    const int* x1 = ci < n_cases ? cbr + cptr[ci + 1] : nullptr;
    if (ci < n_cases && x0 == x1) continue;  // empty contingency: nothing removed
    bfs(g, sp, x0, x1, false, dist, pe, q0, q1, shv);
    for (int e = tid; e < g.E; e += kIslThreads) cov[e] = 0;
    __syncthreads();
    bool stray = false;
    for (int e = tid; e < g.E; e += kIslThreads) {
      if (!g.br_on[e] || (x0 && excluded(x0, x1, e))) continue;
      int a = g.br_from[e], b = g.br_to[e];
      if (dist[a] < 0 || dist[b] < 0) {
        stray = true;
        continue;
      }
      if (pe[a] == e || pe[b] == e) continue;  // tree edge
      while (a != b) {
        if (dist[a] >= dist[b]) {
          const int pa = pe[a];
          cov[pa] = 1;
          a = g.br_from[pa] == a ? g.br_to[pa] : g.br_from[pa];
        } else {
          const int pb = pe[b];
          cov[pb] = 1;
          b = g.br_from[pb] == b ? g.br_to[pb] : g.br_from[pb];
        }
      }
    }
    if (__syncthreads_or(stray)) {
      if (tid == 0) fallback[ci] = 1;
      continue;
    }
    for (int v = tid; v < nn; v += kIslThreads) {
      const int e = pe[v];
      if (e >= 0 && !cov[e]) atomicOr(bridges + (e >> 5), 1u << (e & 31));
    }
    __syncthreads();
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* up(const std::vector<T>& v, std::vector<void*>& owned) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)), "cudaMalloc");
  owned.push_back(p);
  if (!v.empty()) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  return static_cast<T*>(p);
}

}  // namespace

void validate_splits_device(const SplitGraphDesc& gd, const SplitCandidates& cd, int device, std::vector<char>& keep) {
  const int n = static_cast<int>(cd.station_node.size());
  keep.assign(n, 0);
  if (n == 0) return;
  ck(cudaSetDevice(device), "cudaSetDevice");
  int max_moved = 0;
  for (int i = 0; i < n; ++i) max_moved = std::max(max_moved, cd.moved_ptr[i + 1] - cd.moved_ptr[i]);
  if (max_moved > kIslMaxMoved)
    throw SplitCapacityError("a station split moves " + std::to_string(max_moved) + " branch ends (device limit " +
                             std::to_string(kIslMaxMoved) + ")");
  std::vector<void*> owned;
  struct Free {
    std::vector<void*>& o;
    ~Free() {
      for (void* p : o) cudaFree(p);
    }
  } guard{owned};
  IslGraph g{};
  g.N = gd.n_nodes;
  g.E = static_cast<int>(gd.br_from.size());
  g.br_from = up(gd.br_from, owned);
  g.br_to = up(gd.br_to, owned);
  g.br_on = up(gd.br_on, owned);
  g.node_ptr = up(gd.node_ptr, owned);
  g.node_br = up(gd.node_br, owned);
  g.n_single = static_cast<int>(gd.single_br.size());
  g.single_br = up(gd.single_br, owned);
  g.n_multi = static_cast<int>(gd.multi_ptr.size()) - 1;
  g.multi_ptr = up(gd.multi_ptr, owned);
  g.multi_br = up(gd.multi_br, owned);
  IslCands c{};
  c.n = n;
  c.station_node = up(cd.station_node, owned);
  c.moved_ptr = up(cd.moved_ptr, owned);
  c.moved = up(cd.moved, owned);
  c.fresh_used = up(cd.fresh_used, owned);
  std::vector<uint8_t> zeros(n, 0);
  c.keep = up(zeros, owned);
  const int slots = std::min(n, 148 * 4);
  const size_t nn = static_cast<size_t>(g.N) + 1;
  IslScratch sc{};
  void* p = nullptr;
  ck(cudaMalloc(&p, slots * nn * sizeof(int) * 4 + static_cast<size_t>(slots) * std::max(g.E, 1)), "cudaMalloc");
  owned.push_back(p);
  sc.dist = static_cast<int*>(p);
  sc.par_edge = sc.dist + slots * nn;
  sc.queue = sc.par_edge + slots * nn;
  sc.cov = reinterpret_cast<uint8_t*>(sc.queue + 2 * slots * nn);
  const size_t smem = static_cast<size_t>((g.E + 31) / 32) * 4;
  if (smem > 48 * 1024) ck(cudaFuncSetAttribute(k_split_valid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(smem)), "smem attribute");
  k_split_valid<<<slots, kIslThreads, smem>>>(g, c, sc);
  ck(cudaGetLastError(), "k_split_valid launch");
  std::vector<uint8_t> out(n);
  ck(cudaMemcpy(out.data(), c.keep, n, cudaMemcpyDeviceToHost), "D2H keep");
  for (int i = 0; i < n; ++i) keep[i] = out[i];
}


void contingency_bridges_device(const SplitGraphDesc& gd, int device, std::vector<char>& is_bridge_any,
                                std::vector<int>& fallback_cases) {
  const int E = static_cast<int>(gd.br_from.size());
  const int n_cases = static_cast<int>(gd.cont_ptr.size()) - 1;
  is_bridge_any.assign(E, 0);
  fallback_cases.clear();
  ck(cudaSetDevice(device), "cudaSetDevice");
  std::vector<void*> owned;
  struct Free {
    std::vector<void*>& o;
    ~Free() {
      for (void* p : o) cudaFree(p);
    }
  } guard{owned};
  IslGraph g{};
  g.N = gd.n_nodes;
  g.E = E;
  g.br_from = up(gd.br_from, owned);
  g.br_to = up(gd.br_to, owned);
  g.br_on = up(gd.br_on, owned);
  g.node_ptr = up(gd.node_ptr, owned);
  g.node_br = up(gd.node_br, owned);
  const int* cptr = up(gd.cont_ptr, owned);
  const int* cbr = up(gd.cont_br, owned);
  const int slots = std::min(n_cases + 1, 148 * 4);
  const size_t nn = static_cast<size_t>(g.N) + 1;
  IslScratch sc{};
  void* p = nullptr;
  ck(cudaMalloc(&p, slots * nn * sizeof(int) * 4 + static_cast<size_t>(slots) * std::max(E, 1)), "cudaMalloc");
  owned.push_back(p);
  sc.dist = static_cast<int*>(p);
  sc.par_edge = sc.dist + slots * nn;
  sc.queue = sc.par_edge + slots * nn;
  sc.cov = reinterpret_cast<uint8_t*>(sc.queue + 2 * slots * nn);
  const int words = (E + 31) / 32;
  std::vector<uint32_t> zeros(std::max(words, 1), 0u);
  uint32_t* bits = up(zeros, owned);
  std::vector<int> fz(n_cases + 1, 0);
  int* fb = up(fz, owned);
  const size_t smem = static_cast<size_t>((E + 31) / 32) * 4;
  if (smem > 48 * 1024) ck(cudaFuncSetAttribute(k_cont_bridges, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                static_cast<int>(smem)), "smem attribute");
  k_cont_bridges<<<slots, kIslThreads, smem>>>(g, cptr, cbr, n_cases, sc, bits, fb);
  ck(cudaGetLastError(), "k_cont_bridges launch");
  std::vector<uint32_t> hb(std::max(words, 1));
  ck(cudaMemcpy(hb.data(), bits, hb.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H bridges");
  ck(cudaMemcpy(fz.data(), fb, fz.size() * sizeof(int), cudaMemcpyDeviceToHost), "D2H fallback");
  for (int e = 0; e < E; ++e) is_bridge_any[e] = (hb[e >> 5] >> (e & 31)) & 1u;
  for (int c = 0; c <= n_cases; ++c)
    if (fz[c]) fallback_cases.push_back(c);
}

}  // namespace tgb
