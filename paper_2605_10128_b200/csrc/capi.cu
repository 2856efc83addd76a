// C-ABI implementation: host model objects, device context, evaluation and
// optimizer entry points (declared in include/topopt_b200.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/topopt_b200.h"
#include "cuda/ac.cuh"
#include "cuda/engine.cuh"
#include "cuda/islanding.cuh"
#include "cuda/qd.cuh"
#include "host/model.hpp"
#include "host/snapshot.hpp"

namespace {

thread_local std::string g_error;

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

// host/islands.cpp reports through the same per-thread message as the C ABI
namespace tgb {
void set_last_error(const std::string& m) { g_error = m; }
}  // namespace tgb

namespace {

template <class F>
tg_status guarded(F&& f) {
  try {
    f();
    return TG_OK;
  } catch (const tgb::ParseError& e) {
    g_error = e.what();
    return TG_PARSE_ERROR;
  } catch (const tgb::ValidationError& e) {
    g_error = e.what();
    return TG_VALIDATION_ERROR;
  } catch (const tgb::IslandedContingency& e) {
    g_error = e.what();
    return TG_ISLANDED_CONTINGENCY;
  } catch (const tgb::SingularSystem& e) {
    g_error = e.what();
    return TG_SINGULAR_SYSTEM;
  } catch (const tgb::ConfigError& e) {
    g_error = e.what();
    return TG_CONFIG_ERROR;
  } catch (const tgb::IoError& e) {
    g_error = e.what();
    return TG_IO_ERROR;
  } catch (const CudaFailure& e) {
    g_error = e.what();
    return TG_CUDA_ERROR;
  } catch (const CapacityFailure& e) {
    g_error = e.what();
    return TG_CAPACITY_ERROR;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TG_VALIDATION_ERROR;
  }
}

// Device allocation owner.
class DeviceArena {
 public:
  ~DeviceArena() {
    for (void* p : ptrs_) cudaFree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    ptrs_.push_back(p);
    bytes_ += n * sizeof(T);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v, cudaStream_t s) {
    T* d = alloc<T>(v.size());
    if (!v.empty()) check(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
    return d;
  }
  size_t bytes() const { return bytes_; }

 private:
  std::vector<void*> ptrs_;
  size_t bytes_ = 0;
};

}  // namespace

// ---------------------------------------------------------------- host objects
struct tg_grid {
  tgb::Grid g;
  std::vector<int32_t> br_from, br_to, inj_node, cont_bptr, cont_b, cont_iptr, cont_i, sub_node, sub_tptr, tkind,
      telem, bo_sub, bo_bb, bo_iptr, bo_i;
  std::vector<double> br_x, br_lim, inj_net, inj_net_t;
  std::vector<uint8_t> br_on;
};

struct tg_actionset {
  tgb::ActionTable t;
  std::vector<int32_t> station, lambda_r, gptr, bbptr, iptr, imp, disc;
  std::vector<uint8_t> group;
};

namespace {

void flatten_grid(tg_grid& h) {
  const tgb::Grid& g = h.g;
  h.br_from.assign(g.br_from.begin(), g.br_from.end());
  h.br_to.assign(g.br_to.begin(), g.br_to.end());
  h.br_x = g.br_x;
  h.br_lim = g.br_limit;
  h.br_on.assign(g.br_on.begin(), g.br_on.end());
  h.inj_node.assign(g.inj_node.begin(), g.inj_node.end());
  h.inj_net.clear();
  for (int i = 0; i < g.n_injections(); ++i) h.inj_net.push_back(g.inj_net(i));
  h.inj_net_t.clear();
  for (int t = 0; t < g.n_t; ++t)
    for (int i = 0; i < g.n_injections(); ++i) h.inj_net_t.push_back(g.inj_net_t(t, i));
  h.cont_bptr = {0};
  h.cont_iptr = {0};
  h.cont_b.clear();
  h.cont_i.clear();
  for (size_t c = 0; c < g.cont_id.size(); ++c) {
    for (int e : g.cont_branches[c]) h.cont_b.push_back(e);
    for (int i : g.cont_injections[c]) h.cont_i.push_back(i);
    h.cont_bptr.push_back(static_cast<int32_t>(h.cont_b.size()));
    h.cont_iptr.push_back(static_cast<int32_t>(h.cont_i.size()));
  }
  h.sub_node.clear();
  h.sub_tptr = {0};
  h.tkind.clear();
  h.telem.clear();
  for (const auto& st : g.stations) {
    h.sub_node.push_back(st.node);
    for (size_t t = 0; t < st.term_kind.size(); ++t) {
      h.tkind.push_back(st.term_kind[t]);
      h.telem.push_back(st.term_index[t]);
    }
    h.sub_tptr.push_back(static_cast<int32_t>(h.tkind.size()));
  }
  h.bo_sub.assign(g.bo_station.begin(), g.bo_station.end());
  h.bo_bb.assign(g.bo_busbar.begin(), g.bo_busbar.end());
  h.bo_iptr = {0};
  h.bo_i.clear();
  for (size_t b = 0; b < g.bo_id.size(); ++b) {
    for (int e : g.default_implied(static_cast<int>(b))) h.bo_i.push_back(e);
    h.bo_iptr.push_back(static_cast<int32_t>(h.bo_i.size()));
  }
}

void flatten_actions(tg_actionset& a, const tgb::Grid& g) {
  const tgb::ActionTable& t = a.t;
  a.station.assign(t.station.begin(), t.station.end());
  a.lambda_r.assign(t.lambda_r.begin(), t.lambda_r.end());
  a.gptr = {0};
  a.group.clear();
  a.bbptr = {0};
  a.iptr = {0};
  a.imp.clear();
  for (int k = 0; k < t.n_actions(); ++k) {
    for (char x : t.group[k]) a.group.push_back(static_cast<uint8_t>(x));
    a.gptr.push_back(static_cast<int32_t>(a.group.size()));
    const auto& st = g.stations[t.station[k]];
    for (int bb = 0; bb < static_cast<int>(st.busbars.size()); ++bb) {
      for (int e : g.implied_branches(t.station[k], bb, t.assignment[k], t.open_couplers[k])) a.imp.push_back(e);
      a.iptr.push_back(static_cast<int32_t>(a.imp.size()));
    }
    a.bbptr.push_back(static_cast<int32_t>(a.iptr.size() - 1));
  }
  a.disc.assign(t.disconnectables.begin(), t.disconnectables.end());
}

}  // namespace

// ---------------------------------------------------------------- device context
struct tg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  DeviceArena arena;
  tgb::DevGrid g{};
  tgb::DcParams params{};
  int n_cont = 0;
  int worst_k = 20;
  int64_t launches = 0;
  tgb::SideStream side{nullptr, nullptr, nullptr};  // special outages beside the prep / sweep (launch_evaluate)
  // evaluation batch buffers
  int capacity = 0;
  std::unique_ptr<DeviceArena> batch_arena;
  tgb::Batch batch{};
  tgb::EvalScratch scratch{};
  int* d_genomes = nullptr;
  // pre-optimization score
  std::vector<double> pre;  // lambda_o, lambda_c, lambda_c0, lambda_b, fitness
  double lambda_b_pre = 0.0;
  // optimizer state
  std::unique_ptr<tgb::QdState> qd;
  // snapshots (make_snapshot): archive blob packed on the device, copied to
  // pinned host memory (ring of kSnapSlots for the asynchronous hand-off of
  // tg_optimizer_run), decoded on the host
  static constexpr int kSnapSlots = 2;
  tgb::HostSnapshot snap;
  size_t snap_bytes = 0;
  void* snap_dev[kSnapSlots] = {nullptr, nullptr};
  uint8_t* snap_host[kSnapSlots] = {nullptr, nullptr};
  cudaEvent_t snap_ev[kSnapSlots] = {nullptr, nullptr};
  void snap_buffers(size_t bytes);
  void free_snap_buffers();
  int n_a_cap = 4, n_d_cap = 4;
  // grid-dependent sizes checked against the engine's compile-time capacities
  // (common.cuh): outage removal sets (multi-branch contingencies, busbar
  // implied sets), outage injection sets, per-station injection / branch
  // terminals (moved by one split)
  int max_outage_removed = 0, max_outage_inj = 0, max_station_inj = 0, max_station_br = 0;
  std::vector<int> br_perm;   // internal branch index -> the grid's (empty: identity); see sweep_row_order
  int* err_sticky = nullptr;  // device word: a capacity error happened in some lane since the last check
  int* err_host = nullptr;    // pinned mirror of err_sticky, copied after every enqueued loop step
  cudaEvent_t err_ev = nullptr;
  bool err_pending = false;
  void check_capacity(int n_a, int n_d) const;
  void check_sticky();  // synchronizing check
  void poll_sticky();   // non-blocking: raises if an earlier step's mirror landed with an error
  void mirror_sticky(); // enqueue the mirror copy after the steps just enqueued
  // live timing of the fused sweep (bench.py roofline)
  bool time_sweep = false;
  cudaEvent_t sw0 = nullptr, sw1 = nullptr;
  double sweep_ms = 0.0;
  int64_t sweep_launches = 0;
  // timestep extension: per-timestep table views (gt[0] == g), per-timestep
  // scores / energies of the batch being aggregated
  int n_t = 1;
  std::vector<tgb::DevGrid> gt;
  tgb::Scores tscores{};
  double* tenergy = nullptr;
  // multi-timestep screening (one mask pass over all profiles, then a masked
  // sweep per profile): needs the same zero pattern of injections in every
  // profile (then the topology analysis is shared) and room for every
  // profile's candidate rows
  bool mt_ok = false;
  bool mt_pattern_ok = false;  // injection zero pattern identical across profiles
  tgb::MtProfiles mt_prof{};   // per-profile table pointers (device arrays)
  tgb::DevGrid g_mt{};          // t = 0 view with the all-profile skip records
  double* mt_fc = nullptr;      // [n_t][n][E] candidate flows per profile
  double* mt_al = nullptr;      // [n_t][n][Kpad] alpha per profile
  double* mt_rk = nullptr;      // [cap][Kpad][kStride] profile-independent contingency factors
  unsigned long long* mt_fmax = nullptr;  // [kMaskProfiles][cap][E] max |f| per profile of one masked launch
  double* mt_energy = nullptr;  // [n_t][cap][Kall]
  int* mt_nc0 = nullptr;        // [n_t][cap]
  // island merge buffers (allocated on the first merge)
  std::unique_ptr<DeviceArena> merge_arena;
  tgb::MergeBuffers merge{};
  // step-wise optimizer state
  int64_t qd_evaluations = 0;
  int qd_epoch = 0;

  void ensure_capacity(int n);
  void run_batch(int n, int n_a, int n_d, bool full);
  // Enqueues the evaluation of batch.n candidates (all timesteps); returns
  // kernels launched. timed: every sweep launch bracketed by sw0 / sw1 and
  // accumulated into sweep_ms (synchronizes).
  int enqueue_evaluate(int n_a, int n_d, bool full, bool timed = false) {
    return enqueue_evaluate(batch, n_a, n_d, full, timed);
  }
  int enqueue_evaluate(tgb::Batch& bv, int n_a, int n_d, bool full, bool timed);
  int enqueue_evaluate_mt(tgb::Batch& bv, int n_a, int n_d, bool timed);
  void time_sweep_done();
};

void tg_context::check_capacity(int n_a, int n_d) const {
  auto fail = [](const std::string& what) {
    throw CapacityFailure(what + " exceeds the engine's compile-time capacity (common.cuh)");
  };
  if (max_outage_removed + n_d > tgb::kMaxRemoved)
    fail("an outage removal set of " + std::to_string(max_outage_removed) + " branches plus " + std::to_string(n_d) +
         " genome disconnections (limit " + std::to_string(tgb::kMaxRemoved) + ")");
  if (n_a * max_station_inj > tgb::kMaxInjMoved)
    fail(std::to_string(n_a) + " splits of stations with " + std::to_string(max_station_inj) +
         " injection terminals (limit " + std::to_string(tgb::kMaxInjMoved) + " moved injections)");
  if (n_a * max_station_br > tgb::kMaxMoved)
    fail(std::to_string(n_a) + " splits of stations with " + std::to_string(max_station_br) +
         " branch terminals (limit " + std::to_string(tgb::kMaxMoved) + " moved branch ends)");
}

// Capacity errors of lanes evaluated inside the device loop (k_finish ORs
// them into err_sticky): raised by the next host-visible call, never dropped.
void tg_context::check_sticky() {
  int v = 0;
  check(cudaMemcpyAsync(&v, err_sticky, sizeof(int), cudaMemcpyDeviceToHost, stream), "error word D2H");
  check(cudaStreamSynchronize(stream), "error word");
  if (v) {
    check(cudaMemsetAsync(err_sticky, 0, sizeof(int), stream), "error word reset");
    throw CapacityFailure("a candidate exceeded the engine's compile-time capacity (rank/removed/moved limits) "
                          "during the optimizer loop");
  }
}

void tg_context::poll_sticky() {
  if (!err_pending) return;
  const cudaError_t r = cudaEventQuery(err_ev);
  if (r == cudaErrorNotReady) return;
  check(r, "error word");
  err_pending = false;
  if (*err_host) check_sticky();
}

void tg_context::mirror_sticky() {
  if (!err_host) {
    check(cudaMallocHost(reinterpret_cast<void**>(&err_host), sizeof(int)), "cudaMallocHost");
    *err_host = 0;
    check(cudaEventCreateWithFlags(&err_ev, cudaEventDisableTiming), "event");
  }
  check(cudaMemcpyAsync(err_host, err_sticky, sizeof(int), cudaMemcpyDeviceToHost, stream), "error word D2H");
  check(cudaEventRecord(err_ev, stream), "event record");
  err_pending = true;
}

void tg_context::snap_buffers(size_t bytes) {
  if (bytes <= snap_bytes) return;
  check(cudaStreamSynchronize(stream), "snapshot buffers");
  free_snap_buffers();
  for (int i = 0; i < kSnapSlots; ++i) {
    check(cudaMalloc(&snap_dev[i], bytes), "cudaMalloc");
    check(cudaMallocHost(reinterpret_cast<void**>(&snap_host[i]), bytes), "cudaMallocHost");
    check(cudaEventCreateWithFlags(&snap_ev[i], cudaEventDisableTiming), "event");
  }
  snap_bytes = bytes;
}

void tg_context::free_snap_buffers() {
  for (int i = 0; i < kSnapSlots; ++i) {
    if (snap_dev[i]) cudaFree(snap_dev[i]);
    if (snap_host[i]) cudaFreeHost(snap_host[i]);
    if (snap_ev[i]) cudaEventDestroy(snap_ev[i]);
    snap_dev[i] = nullptr;
    snap_host[i] = nullptr;
    snap_ev[i] = nullptr;
  }
  snap_bytes = 0;
}

void tg_context::ensure_capacity(int n) {
  if (n <= capacity) return;
  const int cap = std::max(n, 64);
  if (qd && qd->graph) {  // the captured iteration points at the old buffers
    cudaGraphExecDestroy(qd->graph);
    qd->graph = nullptr;
  }
  batch_arena = std::make_unique<DeviceArena>();
  DeviceArena& A = *batch_arena;
  tgb::Batch& b = batch;
  b = tgb::Batch{};  // every pointer below is reallocated or stays null
  b.err_sticky = err_sticky;
  mt_ok = false;
  const size_t E = g.E, Kp = g.Kpad, Ka = std::max(g.Kall, 1);
  d_genomes = A.alloc<int>(static_cast<size_t>(cap) * tgb::kMaxSlots);
  b.status = A.alloc<int>(cap);
  b.rank = A.alloc<int>(cap);
  b.topo = reinterpret_cast<tgb::TopoCore*>(A.alloc<uint8_t>(static_cast<size_t>(cap) * tgb::topo_core_bytes()));
  b.tbits = A.alloc<uint32_t>(static_cast<size_t>(cap) * 2 * ((E + 31) / 32));
  b.removed = A.alloc<int>(static_cast<size_t>(cap) * tgb::kMaxRemovedSweep);
  b.nchunks = static_cast<int>((E + tgb::kChunkRows - 1) / tgb::kChunkRows);
  b.feat = A.alloc<double>(static_cast<size_t>(tgb::max_sweep_groups(cap)) * b.nchunks * tgb::kGroupSlots *
                           tgb::kChunkRows * tgb::kStride);
  b.slot = A.alloc<int>(cap);
  b.rows_done = A.alloc<unsigned long long>(8);
  check(cudaMemset(b.rows_done, 0, 8 * sizeof(unsigned long long)), "memset");
  b.csum = A.alloc<float>(static_cast<size_t>(cap) * b.nchunks * tgb::kCsum);
  b.item_ctr = A.alloc<unsigned int>(4);
  b.kdat = A.alloc<double>(static_cast<size_t>(cap) * std::max<size_t>(Kp, 1) * tgb::kStride);
  b.kflag = A.alloc<uint8_t>(static_cast<size_t>(cap) * std::max<size_t>(Kp, 1));
  b.fmax = A.alloc<unsigned long long>(static_cast<size_t>(cap) * E);
  b.fbus = A.alloc<unsigned long long>(static_cast<size_t>(cap) * E);
  // zero once: grids without busbar outages never write it (no per-evaluation reset)
  check(cudaMemset(b.fbus, 0, static_cast<size_t>(cap) * E * sizeof(unsigned long long)), "memset");
  b.energy = A.alloc<double>(static_cast<size_t>(cap) * Ka);
  b.isl_out = A.alloc<int>(cap);
  b.isl_bus = A.alloc<int>(cap);
  b.nc0 = A.alloc<int>(cap);
  b.pc = A.alloc<tgb::PcFac>(cap);
  b.wl_list = A.alloc<int>(cap);
  b.wl_start = A.alloc<int>(tgb::kSweepRank + 1);
  b.wl_count = A.alloc<int>(tgb::kSweepRank + 1);
  b.wl_group0 = A.alloc<int>(tgb::kSweepRank + 2);
  tgb::Scores& o = b.out;
  o.lambda_o = A.alloc<double>(cap);
  o.lambda_c = A.alloc<int>(cap);
  o.lambda_c0 = A.alloc<int>(cap);
  o.lambda_b = A.alloc<double>(cap);
  o.lambda_d = A.alloc<int>(cap);
  o.lambda_s = A.alloc<int>(cap);
  o.lambda_r = A.alloc<int>(cap);
  o.fitness = A.alloc<double>(cap);
  o.islanded = A.alloc<uint8_t>(cap);
  o.error = A.alloc<int>(cap);
  o.worst_idx = A.alloc<int>(static_cast<size_t>(cap) * std::max(worst_k, 1));
  o.worst_val = A.alloc<double>(static_cast<size_t>(cap) * std::max(worst_k, 1));
  o.worst_n = A.alloc<int>(cap);
  o.isl_out = A.alloc<int>(cap);
  o.isl_bus = A.alloc<int>(cap);
  if (n_t > 1) {
    tgb::Scores& ts = tscores;
    ts = o;  // same shapes
    ts.lambda_o = A.alloc<double>(cap);
    ts.lambda_c = A.alloc<int>(cap);
    ts.lambda_c0 = A.alloc<int>(cap);
    ts.lambda_b = A.alloc<double>(cap);
    ts.lambda_d = A.alloc<int>(cap);
    ts.lambda_s = A.alloc<int>(cap);
    ts.lambda_r = A.alloc<int>(cap);
    ts.fitness = A.alloc<double>(cap);
    ts.islanded = A.alloc<uint8_t>(cap);
    ts.error = A.alloc<int>(cap);
    ts.worst_idx = A.alloc<int>(static_cast<size_t>(cap) * std::max(worst_k, 1));
    ts.worst_val = A.alloc<double>(static_cast<size_t>(cap) * std::max(worst_k, 1));
    ts.worst_n = A.alloc<int>(cap);
    ts.isl_out = A.alloc<int>(cap);
    ts.isl_bus = A.alloc<int>(cap);
    tenergy = A.alloc<double>(static_cast<size_t>(cap) * Ka);
    // multi-timestep screening buffers, when they fit in half of the free memory
    const size_t feat_sz = static_cast<size_t>(tgb::max_sweep_groups(cap)) * b.nchunks * tgb::kGroupSlots *
                           tgb::kChunkRows * tgb::kStride;
    const size_t kdat_sz = static_cast<size_t>(cap) * std::max<size_t>(Kp, 1) * tgb::kStride;
    const size_t ntiles = std::max<size_t>(Kp / tgb::sweep_tile_k(), 1);
    const size_t need = sizeof(double) * (static_cast<size_t>(n_t) * cap * (static_cast<size_t>(E) + Kp + Ka) +
                                          feat_sz + kdat_sz + static_cast<size_t>(tgb::kMaskProfiles) * cap * E) +
                        static_cast<size_t>(n_t) * cap * sizeof(int) +
                        static_cast<size_t>(cap) * ntiles * (tgb::kTmaxSub + tgb::kStride) * 8 +
                        static_cast<size_t>(cap) * ntiles * b.nchunks * 4;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    static const bool mt_disabled = std::getenv("TGB_NO_MT_SCREEN") != nullptr;  // A/B switch
    mt_ok = mt_pattern_ok && !mt_disabled && need < free_b / 2 && tgb::masked_sweep_fits(g.E);
    if (mt_ok) {
      mt_fc = A.alloc<double>(static_cast<size_t>(n_t) * cap * std::max<size_t>(E, 1));
      mt_al = A.alloc<double>(static_cast<size_t>(n_t) * cap * std::max<size_t>(Kp, 1));
      mt_rk = A.alloc<double>(kdat_sz);
      mt_fmax = A.alloc<unsigned long long>(static_cast<size_t>(tgb::kMaskProfiles) * cap * std::max<size_t>(E, 1));
      mt_energy = A.alloc<double>(static_cast<size_t>(n_t) * cap * Ka);
      mt_nc0 = A.alloc<int>(static_cast<size_t>(n_t) * cap);
      b.feat_mt = A.alloc<double>(feat_sz);
      b.amx_mt = A.alloc<unsigned long long>(static_cast<size_t>(cap) * ntiles * tgb::kTmaxSub);
      b.rmx_mt = A.alloc<unsigned long long>(static_cast<size_t>(cap) * ntiles * tgb::kStride);
      b.mask = A.alloc<uint32_t>(static_cast<size_t>(cap) * ntiles * b.nchunks);
      b.topo_sol = A.alloc<double>(static_cast<size_t>(cap) * tgb::kTopoSol);
    }
  }
  // Z scratch: bounded so huge grids stay within a fixed budget
  const size_t row_prep = static_cast<size_t>(std::max(g.Nr, 1)) * tgb::kStride * sizeof(double);
  const size_t budget = size_t{2} << 30;
  scratch.zslots = static_cast<int>(std::max<size_t>(1, std::min<size_t>(cap, budget / row_prep)));
  scratch.zprep = A.alloc<double>(static_cast<size_t>(scratch.zslots) * std::max(g.Nr, 1) * tgb::kStride);
  const size_t row_sp = static_cast<size_t>(std::max(g.Nr, 1)) * tgb::kMaxCols * sizeof(double);
  scratch.zslots_special = static_cast<int>(std::max<size_t>(1, std::min<size_t>(1024, (size_t{1} << 30) / row_sp)));
  scratch.zspecial = A.alloc<double>(static_cast<size_t>(scratch.zslots_special) * std::max(g.Nr, 1) * tgb::kMaxCols);
  capacity = cap;
}

void tg_context::time_sweep_done() {
  check(cudaEventSynchronize(sw1), "sweep timing");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, sw0, sw1), "sweep timing");
  sweep_ms += ms;
  ++sweep_launches;
}

int tg_context::enqueue_evaluate(tgb::Batch& bv, int n_a, int n_d, bool full, bool timed) {
  int kernels = 0;
  if (timed && !sw0) {
    check(cudaEventCreate(&sw0), "event");
    check(cudaEventCreate(&sw1), "event");
  }
  if (n_t == 1) {
    tgb::launch_evaluate(g, bv, n_a, n_d, full, scratch, stream, &kernels, timed ? sw0 : nullptr,
                         timed ? sw1 : nullptr, &side);
    if (timed) time_sweep_done();
    return kernels;
  }
  // timesteps: the pipeline once per injection profile into the per-t
  // buffers, accumulated into batch.out / batch.energy, then the fitness and
  // worst list of the sums (engine.cu, k_accum_t / k_finish_agg)
  if (full) throw tgb::ConfigError("FlowResult outputs are per timestep; request them on a single-timestep grid");
  if (mt_ok) return enqueue_evaluate_mt(bv, n_a, n_d, timed);
  tgb::Batch bt = bv;
  bt.out = tscores;
  bt.energy = tenergy;
  bt.no_worst = 1;
  for (int t = 0; t < n_t; ++t) {
    int k = 0;
    tgb::launch_evaluate(gt[t], bt, n_a, n_d, false, scratch, stream, &k, timed ? sw0 : nullptr,
                         timed ? sw1 : nullptr);
    if (timed) time_sweep_done();
    kernels += k + tgb::launch_accumulate_timestep(bt, bv.out, bv.energy, g.Kall, t == 0, stream);
  }
  kernels += tgb::launch_finish_aggregate(bv, g.Kall, stream);
  return kernels;
}

// Multi-timestep screening: analysis once (the topology does not depend on the
// profile), candidate rows of every profile (k_prep folds bounds over all
// profiles), one mask pass over all profiles (k_sweep mode 1), then per profile
// the masked sweep (mode 2), special outages, scores, accumulation.
int tg_context::enqueue_evaluate_mt(tgb::Batch& bv, int n_a, int n_d, bool timed) {
  const int n = bv.n, ntiles = std::max(g.Kpad / tgb::sweep_tile_k(), 1);
  const size_t Ka = std::max(g.Kall, 1);
  int kernels = 0;
  auto view = [&](int t) {
    tgb::Batch b = bv;  // feat / kdat: profile 0's rows (the batch's own arrays)
    b.fc_t = mt_fc + static_cast<size_t>(t) * n * g.E;
    b.al_t = mt_al + static_cast<size_t>(t) * n * g.Kpad;
    b.rk_mt = mt_rk;
    b.energy = mt_energy + static_cast<size_t>(t) * n * Ka;
    b.nc0 = mt_nc0 + static_cast<size_t>(t) * n;
    return b;
  };
  tgb::Batch b0 = view(0);
  b0.feat_mt = nullptr;  // the analysis does not touch the bounds
  kernels += tgb::launch_analyze(g, b0, n_a, n_d, stream);
  check(cudaMemsetAsync(bv.amx_mt, 0, static_cast<size_t>(n) * ntiles * tgb::kTmaxSub * 8, stream), "memset");
  check(cudaMemsetAsync(bv.rmx_mt, 0, static_cast<size_t>(n) * ntiles * tgb::kStride * 8, stream), "memset");
  check(cudaMemsetAsync(mt_energy, 0, static_cast<size_t>(n_t) * n * Ka * sizeof(double), stream), "memset");
  {
    // profile 0 (factors, L rows, bounds), then every later profile in one pass
    tgb::Batch b0p = view(0);
    kernels += tgb::launch_prep(gt[0], b0p, n_a, n_d, scratch, stream);
    tgb::MtProfiles P = mt_prof;
    P.fc = mt_fc;
    P.al = mt_al;
    P.rk = mt_rk;
    P.fc_stride = static_cast<size_t>(n) * g.E;
    P.al_stride = static_cast<size_t>(n) * g.Kpad;
    P.energy_stride = static_cast<size_t>(n) * Ka;
    P.nc0_stride = static_cast<size_t>(n);
    kernels += tgb::launch_prep_mt(g, b0p, P, stream);
  }
  tgb::Batch bm = view(0);
  bm.t_mode = 1;
  if (g.Ks > 0) tgb::launch_sweep(g_mt, bm, false, stream, timed ? sw0 : nullptr, timed ? sw1 : nullptr, &kernels);
  if (timed && g.Ks > 0) time_sweep_done();
  // masked sweeps of kMaskProfiles profiles per launch (per-profile fmax
  // buffers), then per profile special outages, scores, accumulation
  const size_t fmax_n = static_cast<size_t>(n) * g.E;
  for (int t0 = 0; t0 < n_t; t0 += tgb::kMaskProfiles) {
    const int np = std::min(tgb::kMaskProfiles, n_t - t0);
    tgb::Batch bs = view(t0);
    bs.t_mode = 2;
    bs.fmax = mt_fmax;
    check(cudaMemsetAsync(mt_fmax, 0, np * fmax_n * sizeof(unsigned long long), stream), "memset");
    if (g.Ks > 0) {
      tgb::MtMask mm{t0, np, static_cast<size_t>(n) * g.E, static_cast<size_t>(n) * g.Kpad,
                     static_cast<size_t>(n) * Ka, fmax_n, mt_prof.tmax, mt_prof.alpha0};
      tgb::launch_sweep_masked(gt[t0], bs, mm, stream, timed ? sw0 : nullptr, timed ? sw1 : nullptr, &kernels);
      if (timed) time_sweep_done();
    }
    for (int p = 0; p < np; ++p) {
      const int t = t0 + p;
      tgb::Batch bt = view(t);
      bt.out = tscores;
      bt.no_worst = 1;
      bt.feat_mt = nullptr;
      bt.amx_mt = nullptr;
      bt.rmx_mt = nullptr;
      bt.fmax = mt_fmax + p * fmax_n;
      check(cudaMemsetAsync(bt.fbus, 0, fmax_n * sizeof(unsigned long long), stream), "memset");
      check(cudaMemsetAsync(bt.isl_out, 0, n * sizeof(int), stream), "memset");
      check(cudaMemsetAsync(bt.isl_bus, 0, n * sizeof(int), stream), "memset");
      kernels += tgb::launch_special_finish(gt[t], bt, n_a, n_d, false, scratch, stream);
      kernels += tgb::launch_accumulate_timestep(bt, bv.out, nullptr, g.Kall, t == 0, stream);
    }
  }
  kernels += tgb::launch_sum_profiles(mt_energy, n_t, static_cast<size_t>(n) * Ka, static_cast<size_t>(n) * g.Kall,
                                      bv.energy, stream);
  kernels += tgb::launch_finish_aggregate(bv, g.Kall, stream);
  return kernels;
}

void tg_context::run_batch(int n, int n_a, int n_d, bool full) {
  batch.n = n;
  batch.genomes = d_genomes;
  batch.params = params;
  launches += enqueue_evaluate(n_a, n_d, full, time_sweep && g.Ks > 0);
  check(cudaGetLastError(), "evaluate launch");
}

namespace {

void copy_scores(tg_context* ctx, int n, tg_scores* out) {
  if (!out) return;
  const tgb::Scores& o = ctx->batch.out;
  cudaStream_t s = ctx->stream;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    if (dst) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "scores D2H");
  };
  cp(out->lambda_o, o.lambda_o, n * sizeof(double));
  cp(out->lambda_c, o.lambda_c, n * sizeof(int));
  cp(out->lambda_c0, o.lambda_c0, n * sizeof(int));
  cp(out->lambda_b, o.lambda_b, n * sizeof(double));
  cp(out->lambda_d, o.lambda_d, n * sizeof(int));
  cp(out->lambda_s, o.lambda_s, n * sizeof(int));
  cp(out->lambda_r, o.lambda_r, n * sizeof(int));
  cp(out->fitness, o.fitness, n * sizeof(double));
  cp(out->islanded, o.islanded, n * sizeof(uint8_t));
  cp(out->worst_n, o.worst_n, n * sizeof(int));
  cp(out->islanded_outages, o.isl_out, n * sizeof(int));
  cp(out->islanded_busbar_outages, o.isl_bus, n * sizeof(int));
  cp(out->worst_idx, o.worst_idx, static_cast<size_t>(n) * ctx->worst_k * sizeof(int));
  cp(out->worst_energy, o.worst_val, static_cast<size_t>(n) * ctx->worst_k * sizeof(double));
}

void check_errors(tg_context* ctx, int n) {
  std::vector<int> err(n);
  check(cudaMemcpyAsync(err.data(), ctx->batch.out.error, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream),
        "error D2H");
  check(cudaStreamSynchronize(ctx->stream), "evaluate");
  // this call reports its own lanes: the loop's sticky word starts clean
  check(cudaMemsetAsync(ctx->err_sticky, 0, sizeof(int), ctx->stream), "error word reset");
  for (int i = 0; i < n; ++i)
    if (err[i] != 0)
      throw CapacityFailure("candidate " + std::to_string(i) +
                            " exceeds the engine's compile-time capacity (rank/removed/moved limits)");
}

}  // namespace

extern "C" {

const char* tg_last_error(void) { return g_error.c_str(); }
const char* tg_version(void) { return "topopt_b200 0.1 (sm_100a)"; }
void tg_free(void* p) { std::free(p); }

tg_status tg_grid_from_json(const char* text, size_t len, tg_grid** out) {
  return guarded([&] {
    auto h = std::make_unique<tg_grid>();
    h->g = tgb::load_grid_json(std::string(text, len));
    flatten_grid(*h);
    *out = h.release();
  });
}

void tg_grid_destroy(tg_grid* grid) { delete grid; }

tg_status tg_grid_to_json(const tg_grid* grid, char** text_out) {
  return guarded([&] {
    const std::string s = tgb::grid_to_json_text(grid->g);
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    *text_out = p;
  });
}

tg_status tg_build_ptdf(const tg_grid* grid, int device, double* out) {
  return guarded([&] {
    const tgb::Grid& g = grid->g;
    const int N = g.n_nodes(), E = g.n_branches(), Nr = N - 1;
    check(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t s = nullptr;
    check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    DeviceArena A;
    std::vector<int> red(N, -1);
    for (int v = 0, r = 0; v < N; ++v)
      if (v != g.slack) red[v] = r++;
    std::vector<double> b(E), bred(static_cast<size_t>(Nr) * Nr, 0.0);
    for (int e = 0; e < E; ++e) {
      b[e] = 1.0 / g.br_x[e];
      if (!g.br_on[e]) continue;
      const int i = red[g.br_from[e]], j = red[g.br_to[e]];
      if (i >= 0) bred[static_cast<size_t>(i) * Nr + i] += b[e];
      if (j >= 0) bred[static_cast<size_t>(j) * Nr + j] += b[e];
      if (i >= 0 && j >= 0) bred[static_cast<size_t>(i) * Nr + j] -= b[e], bred[static_cast<size_t>(j) * Nr + i] -= b[e];
    }
    double* X = A.upload(bred, s);
    const bool ok = tgb::device_spd_inverse(X, Nr, s);
    if (!ok) {
      cudaStreamDestroy(s);
      throw tgb::SingularSystem("susceptance matrix is singular; the grid is disconnected");
    }
    std::vector<uint8_t> on(g.br_on.begin(), g.br_on.end());
    double* d_out = A.alloc<double>(static_cast<size_t>(E) * N);
    tgb::launch_ptdf(N, E, Nr, A.upload(red, s), A.upload(std::vector<int>(g.br_from.begin(), g.br_from.end()), s),
                     A.upload(std::vector<int>(g.br_to.begin(), g.br_to.end()), s), A.upload(b, s), A.upload(on, s), X,
                     d_out, s);
    check(cudaGetLastError(), "ptdf");
    check(cudaMemcpyAsync(out, d_out, static_cast<size_t>(E) * N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "ptdf");
    cudaStreamDestroy(s);
  });
}

tg_status tg_grid_content_hash(const tg_grid* grid, uint64_t* hash) {
  return guarded([&] { *hash = tgb::grid_content_hash(grid->g); });
}

const char* tg_grid_branch_id(const tg_grid* grid, int32_t e) {
  if (!grid || e < 0 || e >= grid->g.n_branches()) return nullptr;
  return grid->g.branch_id[e].c_str();
}

tg_status tg_grid_describe(const tg_grid* h, tg_grid_desc* d) {
  return guarded([&] {
    const tgb::Grid& g = h->g;
    d->n_nodes = g.n_nodes();
    d->n_branches = g.n_branches();
    d->n_injections = g.n_injections();
    d->slack = g.slack;
    d->branch_from = h->br_from.data();
    d->branch_to = h->br_to.data();
    d->branch_x = h->br_x.data();
    d->branch_limit = h->br_lim.data();
    d->branch_in_service = h->br_on.data();
    d->injection_node = h->inj_node.data();
    d->injection_net_mw = h->inj_net.data();
    d->n_contingencies = static_cast<int32_t>(g.cont_id.size());
    d->cont_branch_ptr = h->cont_bptr.data();
    d->cont_branch = h->cont_b.data();
    d->cont_inj_ptr = h->cont_iptr.data();
    d->cont_inj = h->cont_i.data();
    d->n_substations = static_cast<int32_t>(g.stations.size());
    d->sub_node = h->sub_node.data();
    d->sub_term_ptr = h->sub_tptr.data();
    d->term_kind = h->tkind.data();
    d->term_element = h->telem.data();
    d->n_busbar_outages = static_cast<int32_t>(g.bo_id.size());
    d->bo_substation = h->bo_sub.data();
    d->bo_busbar = h->bo_bb.data();
    d->bo_implied_ptr = h->bo_iptr.data();
    d->bo_implied = h->bo_i.data();
    d->n_timesteps = g.n_t;
    d->injection_net_mw_t = g.n_t > 1 ? h->inj_net_t.data() : nullptr;
  });
}

tg_status tg_actionset_build(const tg_grid* grid, uint64_t seed, int64_t cap, tg_actionset** out) {
  return guarded([&] {
    auto a = std::make_unique<tg_actionset>();
    a->t = tgb::build_actions(grid->g, seed, cap > 0 ? cap : (int64_t{1} << 23));
    flatten_actions(*a, grid->g);
    *out = a.release();
  });
}

tg_status tg_actionset_build_device(const tg_grid* grid, uint64_t seed, int64_t cap, int device, tg_actionset** out) {
  return guarded([&] {
    if (device < 0) throw tgb::ConfigError("device must be >= 0");
    auto a = std::make_unique<tg_actionset>();
    try {
      a->t = tgb::build_actions(grid->g, seed, cap > 0 ? cap : (int64_t{1} << 23), device);
    } catch (const tgb::SplitCapacityError& e) {
      throw CapacityFailure(e.what());
    } catch (const std::runtime_error& e) {
      if (dynamic_cast<const tgb::ParseError*>(&e) || dynamic_cast<const tgb::ValidationError*>(&e)) throw;
      throw CudaFailure(e.what());
    }
    flatten_actions(*a, grid->g);
    *out = a.release();
  });
}

tg_status tg_actionset_from_json(const tg_grid* grid, const char* text, size_t len, tg_actionset** out) {
  return guarded([&] {
    auto a = std::make_unique<tg_actionset>();
    if (!tgb::actions_from_json(std::string(text, len), grid->g, tgb::grid_content_hash(grid->g), a->t))
      throw tgb::IoError("action cache does not match this grid");
    flatten_actions(*a, grid->g);
    *out = a.release();
  });
}

tg_status tg_actionset_to_json(const tg_actionset* set, const tg_grid* grid, char** text_out) {
  return guarded([&] {
    std::string s = tgb::actions_to_json(set->t, grid->g, tgb::grid_content_hash(grid->g));
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    *text_out = p;
  });
}

void tg_actionset_destroy(tg_actionset* set) { delete set; }

tg_status tg_actionset_describe(const tg_actionset* a, const tg_grid*, tg_actionset_desc* d) {
  return guarded([&] {
    d->n_actions = a->t.n_actions();
    d->action_substation = a->station.data();
    d->action_lambda_r = a->lambda_r.data();
    d->action_group_ptr = a->gptr.data();
    d->action_group = a->group.data();
    d->action_busbar_ptr = a->bbptr.data();
    d->action_implied_ptr = a->iptr.data();
    d->action_implied = a->imp.data();
    d->n_disconnectables = static_cast<int32_t>(a->disc.size());
    d->disconnectables = a->disc.data();
  });
}

}  // extern "C"

namespace {

// B_red^-1 of the grid (dc_engine.cpp:88-116): assembled on the host in the
// grid's own branch order, inverted on the device. Node space only, so it is
// shared by every branch (row) order.
double* base_inverse(tg_context* ctx, const tg_grid_desc* gd) {
  const int N = gd->n_nodes, E = gd->n_branches, Nr = N - 1;
  std::vector<int> red(N, -1);
  for (int v = 0, r = 0; v < N; ++v)
    if (v != gd->slack) red[v] = r++;
  std::vector<double> bred(static_cast<size_t>(Nr) * Nr, 0.0);
  for (int e = 0; e < E; ++e) {
    if (!gd->branch_in_service[e]) continue;
    const double b = 1.0 / gd->branch_x[e];
    const int i = red[gd->branch_from[e]], j = red[gd->branch_to[e]];
    if (i >= 0) bred[static_cast<size_t>(i) * Nr + i] += b;
    if (j >= 0) bred[static_cast<size_t>(j) * Nr + j] += b;
    if (i >= 0 && j >= 0) bred[static_cast<size_t>(i) * Nr + j] -= b, bred[static_cast<size_t>(j) * Nr + i] -= b;
  }
  double* X = ctx->arena.upload(bred, ctx->stream);
  if (!tgb::device_spd_inverse(X, Nr, ctx->stream))
    throw tgb::SingularSystem("susceptance matrix is singular; the grid is disconnected");
  return X;
}

// Sweep row order: the engine numbers branches internally so that each
// 32-row chunk of the sweep holds electrically close branches (recursive
// bisection of the node graph, tgb::locality_rank), with the rows whose base
// N-1 headroom is under 5 % of their limit (near-overloaded in the unchanged
// topology) last. A chunk far from a candidate's changes is then proved safe
// by one chunk-level bound (sweep.cu). Returns internal -> original branch
// index; empty (identity) for grids below the sweep's scale.
std::vector<int> sweep_row_order(tg_context* ctx, const tg_grid_desc* gd, const double* X) {
  const int N = gd->n_nodes, E = gd->n_branches, I = gd->n_injections;
  if (E < 512 || getenv("TGB_NO_ROW_ORDER")) return {};
  cudaStream_t s = ctx->stream;
  DeviceArena tmp;
  std::vector<int> red(N, -1);
  for (int v = 0, r = 0; v < N; ++v)
    if (v != gd->slack) red[v] = r++;
  std::vector<int> ks;
  for (int c = 0; c < gd->n_contingencies; ++c)
    if (gd->cont_branch_ptr[c + 1] - gd->cont_branch_ptr[c] == 1 && gd->cont_inj_ptr[c + 1] == gd->cont_inj_ptr[c])
      ks.push_back(gd->cont_branch[gd->cont_branch_ptr[c]]);
  std::vector<double> b(E), p(N, 0.0);
  for (int e = 0; e < E; ++e) b[e] = 1.0 / gd->branch_x[e];
  for (int i = 0; i < I; ++i) p[gd->injection_node[i]] += gd->injection_net_mw[i];
  double tot = 0.0;
  for (double v : p) tot += v;
  p[gd->slack] -= tot;
  std::vector<double> pr(N - 1);
  for (int v = 0; v < N; ++v)
    if (red[v] >= 0) pr[red[v]] = p[v];
  tgb::DevGrid g{};
  g.N = N;
  g.Nr = N - 1;
  g.E = E;
  g.Ks = static_cast<int>(ks.size());
  g.red = tmp.upload(red, s);
  g.br_from = tmp.upload(std::vector<int>(gd->branch_from, gd->branch_from + E), s);
  g.br_to = tmp.upload(std::vector<int>(gd->branch_to, gd->branch_to + E), s);
  g.br_b = tmp.upload(b, s);
  g.br_lim = tmp.upload(std::vector<double>(gd->branch_limit, gd->branch_limit + E), s);
  g.br_on = tmp.upload(std::vector<uint8_t>(gd->branch_in_service, gd->branch_in_service + E), s);
  g.ks_branch = tmp.upload(ks.empty() ? std::vector<int>{0} : ks, s);
  g.X = X;
  double* h = tmp.alloc<double>(E);
  tgb::launch_row_headroom(g, tmp.upload(pr, s), tmp.alloc<double>(N), tmp.alloc<double>(E), tmp.alloc<double>(E), h,
                           s);
  check(cudaGetLastError(), "row headroom");
  std::vector<double> hh(E);
  check(cudaMemcpyAsync(hh.data(), h, E * sizeof(double), cudaMemcpyDeviceToHost, s), "headroom D2H");
  check(cudaStreamSynchronize(s), "row headroom");
  std::vector<std::pair<int, int>> edges;
  for (int e = 0; e < E; ++e)
    if (gd->branch_in_service[e]) edges.emplace_back(gd->branch_from[e], gd->branch_to[e]);
  const std::vector<int> rank = tgb::locality_rank(N, edges);
  std::vector<int> perm(E);
  for (int e = 0; e < E; ++e) perm[e] = e;
  auto key = [&](int e) {
    const int tight = hh[e] < 0.05 * gd->branch_limit[e] ? 1 : 0;
    const int a = rank[gd->branch_from[e]], c = rank[gd->branch_to[e]];
    return std::make_tuple(tight, std::min(a, c), std::max(a, c));
  };
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return key(x) < key(y); });
  return perm;
}

// Grid / action descriptors with branches renumbered (internal e = original
// perm[e]); every branch reference is mapped, everything else is shared.
struct PermutedDesc {
  tg_grid_desc gd;
  tg_actionset_desc ad{};
  std::vector<int32_t> from, to, cont_branch, term_element, bo_implied, act_implied, disc;
  std::vector<double> x, lim;
  std::vector<uint8_t> on;
  PermutedDesc(const tg_grid_desc& g, const tg_actionset_desc* a, const std::vector<int>& perm) : gd(g) {
    const int E = g.n_branches;
    std::vector<int> inv(E);
    for (int e = 0; e < E; ++e) inv[perm[e]] = e;
    for (int e = 0; e < E; ++e) {
      from.push_back(g.branch_from[perm[e]]);
      to.push_back(g.branch_to[perm[e]]);
      x.push_back(g.branch_x[perm[e]]);
      lim.push_back(g.branch_limit[perm[e]]);
      on.push_back(g.branch_in_service[perm[e]]);
    }
    for (int i = 0; i < g.cont_branch_ptr[g.n_contingencies]; ++i) cont_branch.push_back(inv[g.cont_branch[i]]);
    const int nterm = g.sub_term_ptr[g.n_substations];
    for (int q = 0; q < nterm; ++q)
      term_element.push_back(g.term_kind[q] == 2 ? g.term_element[q] : inv[g.term_element[q]]);
    for (int i = 0; i < g.bo_implied_ptr[g.n_busbar_outages]; ++i) bo_implied.push_back(inv[g.bo_implied[i]]);
    gd.branch_from = from.data();
    gd.branch_to = to.data();
    gd.branch_x = x.data();
    gd.branch_limit = lim.data();
    gd.branch_in_service = on.data();
    gd.cont_branch = cont_branch.data();
    gd.term_element = term_element.data();
    gd.bo_implied = bo_implied.data();
    if (a) {
      ad = *a;
      const int nslots = a->n_actions > 0 ? a->action_busbar_ptr[a->n_actions] : 0;
      const int nimp = a->n_actions > 0 ? a->action_implied_ptr[nslots] : 0;
      for (int i = 0; i < nimp; ++i) act_implied.push_back(inv[a->action_implied[i]]);
      for (int d = 0; d < a->n_disconnectables; ++d) disc.push_back(inv[a->disconnectables[d]]);
      ad.action_implied = act_implied.data();
      ad.disconnectables = disc.data();
    }
  }
};

void context_build(tg_context* ctx, const tg_grid_desc* gd, const tg_actionset_desc* ad, const tg_dc_config* cfg,
                   double* X_base) {
    cudaStream_t s = ctx->stream;
    DeviceArena& A = ctx->arena;
    tgb::DevGrid& g = ctx->g;
    const int N = gd->n_nodes, E = gd->n_branches, I = gd->n_injections;
    g.N = N;
    g.Nr = N - 1;
    g.E = E;
    g.I = I;
    g.slack = gd->slack;
    std::vector<int> red(N, -1);
    for (int v = 0, r = 0; v < N; ++v)
      if (v != gd->slack) red[v] = r++;
    std::vector<double> b(E);
    for (int e = 0; e < E; ++e) b[e] = 1.0 / gd->branch_x[e];
    // node incidence (in-service) and node injections
    std::vector<int> nptr(N + 1, 0), nbr, iptr(N + 1, 0), ninj;
    for (int e = 0; e < E; ++e)
      if (gd->branch_in_service[e]) ++nptr[gd->branch_from[e] + 1], ++nptr[gd->branch_to[e] + 1];
    for (int v = 0; v < N; ++v) nptr[v + 1] += nptr[v];
    nbr.resize(nptr[N]);
    {
      std::vector<int> fill(nptr.begin(), nptr.end() - 1);
      for (int e = 0; e < E; ++e)
        if (gd->branch_in_service[e]) nbr[fill[gd->branch_from[e]]++] = e, nbr[fill[gd->branch_to[e]]++] = e;
    }
    for (int i = 0; i < I; ++i) ++iptr[gd->injection_node[i] + 1];
    for (int v = 0; v < N; ++v) iptr[v + 1] += iptr[v];
    ninj.resize(iptr[N]);
    {
      std::vector<int> fill(iptr.begin(), iptr.end() - 1);
      for (int i = 0; i < I; ++i) ninj[fill[gd->injection_node[i]]++] = i;
    }
    // contingencies: single-branch (fused sweep) vs special (outage rebuild)
    std::vector<int> ks_cont, ks_br, kx_cont, kx_bptr{0}, kx_b, kx_iptr{0}, kx_i;
    for (int c = 0; c < gd->n_contingencies; ++c) {
      const int b0 = gd->cont_branch_ptr[c], b1 = gd->cont_branch_ptr[c + 1];
      const int i0 = gd->cont_inj_ptr[c], i1 = gd->cont_inj_ptr[c + 1];
      if (b1 - b0 == 1 && i1 == i0) {
        ks_cont.push_back(c);
        ks_br.push_back(gd->cont_branch[b0]);
      } else {
        kx_cont.push_back(c);
        for (int p = b0; p < b1; ++p) kx_b.push_back(gd->cont_branch[p]);
        for (int p = i0; p < i1; ++p) kx_i.push_back(gd->cont_inj[p]);
        kx_bptr.push_back(static_cast<int>(kx_b.size()));
        kx_iptr.push_back(static_cast<int>(kx_i.size()));
      }
    }
    // locality order of the sweep's contingency tiles: each 128-wide tile holds
    // electrically close branches, so most (branch row, tile) blocks of a
    // candidate are provably below their limits and skipped exactly
    {
      std::vector<std::pair<int, int>> edges;
      for (int e = 0; e < E; ++e)
        if (gd->branch_in_service[e]) edges.emplace_back(gd->branch_from[e], gd->branch_to[e]);
      const std::vector<int> rank = tgb::locality_rank(N, edges);
      std::vector<int> perm(ks_cont.size());
      for (size_t i = 0; i < perm.size(); ++i) perm[i] = static_cast<int>(i);
      auto key = [&](int i) {
        const int b = ks_br[i];
        return std::make_pair(std::min(rank[gd->branch_from[b]], rank[gd->branch_to[b]]),
                              std::max(rank[gd->branch_from[b]], rank[gd->branch_to[b]]));
      };
      std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return key(x) < key(y); });
      std::vector<int> c2, b2;
      for (int i : perm) c2.push_back(ks_cont[i]), b2.push_back(ks_br[i]);
      ks_cont.swap(c2);
      ks_br.swap(b2);
    }
    // capacities (common.cuh) against this grid: checked here and per call
    for (size_t c = 0; c + 1 < kx_bptr.size(); ++c) {
      ctx->max_outage_removed = std::max(ctx->max_outage_removed, kx_bptr[c + 1] - kx_bptr[c]);
      ctx->max_outage_inj = std::max(ctx->max_outage_inj, kx_iptr[c + 1] - kx_iptr[c]);
    }
    for (int bo = 0; bo < gd->n_busbar_outages; ++bo)
      ctx->max_outage_removed = std::max(ctx->max_outage_removed, gd->bo_implied_ptr[bo + 1] - gd->bo_implied_ptr[bo]);
    if (ad && ad->n_actions > 0 && gd->n_busbar_outages > 0) {
      const int nslots = ad->action_busbar_ptr[ad->n_actions];
      for (int i = 0; i < nslots; ++i)
        ctx->max_outage_removed =
            std::max(ctx->max_outage_removed, ad->action_implied_ptr[i + 1] - ad->action_implied_ptr[i]);
    }
    for (int st = 0; st < gd->n_substations; ++st) {
      int ni = 0, nb = 0;
      for (int q = gd->sub_term_ptr[st]; q < gd->sub_term_ptr[st + 1]; ++q) (gd->term_kind[q] == 2 ? ni : nb) += 1;
      ctx->max_station_inj = std::max(ctx->max_station_inj, ni);
      ctx->max_station_br = std::max(ctx->max_station_br, nb);
    }
    if (ctx->max_outage_removed > tgb::kMaxRemoved)
      throw CapacityFailure("an outage removes " + std::to_string(ctx->max_outage_removed) +
                            " branches; the engine's compile-time capacity is " + std::to_string(tgb::kMaxRemoved));
    if (ctx->max_outage_inj > tgb::kMaxPMod)
      throw CapacityFailure("a contingency drops " + std::to_string(ctx->max_outage_inj) +
                            " injections; the engine's compile-time capacity is " + std::to_string(tgb::kMaxPMod));
    if (ctx->max_station_inj > tgb::kMaxInjMoved || ctx->max_station_br > tgb::kMaxMoved)
      throw CapacityFailure("a substation has more terminals than the engine's compile-time capacity");
    ctx->err_sticky = A.alloc<int>(1);
    check(cudaMemsetAsync(ctx->err_sticky, 0, sizeof(int), s), "error word");
    const int tile = tgb::sweep_tile_k();
    g.Ks = static_cast<int>(ks_cont.size());
    g.Kpad = ((g.Ks + tile - 1) / tile) * tile;
    g.Kx = static_cast<int>(kx_cont.size());
    g.Kall = gd->n_contingencies;
    g.Kb = gd->n_busbar_outages;
    g.S = gd->n_substations;
    g.A = ad ? ad->n_actions : 0;
    g.D = ad ? ad->n_disconnectables : 0;
    // station action ranges (actions of one station are contiguous)
    std::vector<int> lo(g.S, -1), hi(g.S, -1);
    for (int a = 0; a < g.A; ++a) {
      const int st = ad->action_substation[a];
      if (lo[st] < 0) lo[st] = a;
      else if (hi[st] != a) throw tgb::ValidationError("actions of a substation must be contiguous");
      hi[st] = a + 1;
    }
    auto v32 = [](const int32_t* p, size_t n) { return std::vector<int>(p, p + n); };
    g.red = A.upload(red, s);
    g.br_from = A.upload(v32(gd->branch_from, E), s);
    g.br_to = A.upload(v32(gd->branch_to, E), s);
    g.br_b = A.upload(b, s);
    {
      // padded to whole sweep chunks: the sweep streams limits in 16-byte bulk copies
      std::vector<double> lim(gd->branch_limit, gd->branch_limit + E);
      lim.resize(E + tgb::sweep_chunk(), 0.0);
      g.br_lim = A.upload(lim, s);
    }
    g.br_on = A.upload(std::vector<uint8_t>(gd->branch_in_service, gd->branch_in_service + E), s);
    g.node_ptr = A.upload(nptr, s);
    g.node_br = A.upload(nbr, s);
    g.node_inj_ptr = A.upload(iptr, s);
    g.node_inj = A.upload(ninj, s);
    g.inj_node = A.upload(v32(gd->injection_node, I), s);
    g.inj_net = A.upload(std::vector<double>(gd->injection_net_mw, gd->injection_net_mw + I), s);
    g.ks_cont = A.upload(ks_cont, s);
    g.ks_branch = A.upload(ks_br, s);
    {
      // rows that are the outaged branch of some contingency of a sweep tile
      // (the chunked sweep's exact path checks its diagonal only there)
      const int tk = tgb::sweep_tile_k(), nt = std::max(g.Kpad / tk, 1), nw = (E + 31) / 32;
      std::vector<uint32_t> diag(static_cast<size_t>(nt) * nw, 0u);
      for (int k = 0; k < static_cast<int>(ks_br.size()); ++k)
        diag[static_cast<size_t>(k / tk) * nw + ks_br[k] / 32] |= 1u << (ks_br[k] % 32);
      g.diag_bits = A.upload(diag, s);
    }
    g.kx_cont = A.upload(kx_cont, s);
    g.kx_br_ptr = A.upload(kx_bptr, s);
    g.kx_br = A.upload(kx_b, s);
    g.kx_inj_ptr = A.upload(kx_iptr, s);
    g.kx_inj = A.upload(kx_i, s);
    g.bo_station = A.upload(v32(gd->bo_substation, g.Kb), s);
    g.bo_busbar = A.upload(v32(gd->bo_busbar, g.Kb), s);
    g.bo_def_ptr = A.upload(v32(gd->bo_implied_ptr, g.Kb + 1), s);
    g.bo_def = A.upload(v32(gd->bo_implied, gd->bo_implied_ptr[g.Kb]), s);
    g.st_node = A.upload(v32(gd->sub_node, g.S), s);
    g.st_range_lo = A.upload(lo, s);
    g.st_range_hi = A.upload(hi, s);
    g.st_term_ptr = A.upload(v32(gd->sub_term_ptr, g.S + 1), s);
    g.term_kind = A.upload(v32(gd->term_kind, gd->sub_term_ptr[g.S]), s);
    g.term_elem = A.upload(v32(gd->term_element, gd->sub_term_ptr[g.S]), s);
    if (g.A > 0) {
      g.act_station = A.upload(v32(ad->action_substation, g.A), s);
      g.act_lambda_r = A.upload(v32(ad->action_lambda_r, g.A), s);
      g.act_group_ptr = A.upload(v32(ad->action_group_ptr, g.A + 1), s);
      g.act_group = A.upload(std::vector<uint8_t>(ad->action_group, ad->action_group + ad->action_group_ptr[g.A]), s);
      g.act_bb_ptr = A.upload(v32(ad->action_busbar_ptr, g.A + 1), s);
      const int nslots = ad->action_busbar_ptr[g.A];
      g.act_imp_ptr = A.upload(v32(ad->action_implied_ptr, nslots + 1), s);
      g.act_imp = A.upload(v32(ad->action_implied, ad->action_implied_ptr[nslots]), s);
    } else {
      g.act_station = A.alloc<int>(1);
      g.act_lambda_r = A.alloc<int>(1);
      g.act_group_ptr = A.alloc<int>(1);
      g.act_group = A.alloc<uint8_t>(1);
      g.act_bb_ptr = A.alloc<int>(1);
      g.act_imp_ptr = A.alloc<int>(1);
      g.act_imp = A.alloc<int>(1);
    }
    g.disc = g.D > 0 ? A.upload(v32(ad->disconnectables, g.D), s) : A.alloc<int>(1);

    // base factorization (base_inverse, in the grid's own branch order)
    const int Nr = g.Nr;
    g.X = X_base;
    // branch-space columns of every action / disconnectable (topo.cuh
    // column_sources): k_prep reads a candidate's update columns instead of
    // building Z = X [U | V]; skipped when they would take more than 1/8 of
    // the free memory (k_prep then builds Z)
    g.PhiA = nullptr;
    g.PsiD = nullptr;
    {
      std::vector<int> dob(E, -1);
      for (int d = 0; d < g.D; ++d) dob[ad->disconnectables[d]] = d;
      g.disc_of_br = A.upload(dob, s);
      size_t free_b = 0, total_b = 0;
      check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      const size_t need = static_cast<size_t>(g.A + g.D) * E * sizeof(double);
      static const bool off = std::getenv("TGB_NO_PHI_COLUMNS") != nullptr;  // A/B switch
      if (!off && g.A + g.D > 0 && need <= free_b / 8) {
        double* phi = A.alloc<double>(static_cast<size_t>(g.A + g.D) * E);
        int* nmv = A.alloc<int>(std::max(g.A, 1));
        g.PhiA = phi;
        g.PsiD = phi + static_cast<size_t>(g.A) * E;
        g.act_nmv = nmv;
        tgb::launch_phi_columns(g, phi, nmv, phi + static_cast<size_t>(g.A) * E, s);
        check(cudaGetLastError(), "phi columns");
      } else {
        g.act_nmv = A.alloc<int>(1);
      }
    }
    // base tables per injection profile (timestep extension; T = 1 is the reference)
    const int T = std::max(1, gd->n_timesteps);
    if (T > 1 && !gd->injection_net_mw_t) throw tgb::ConfigError("n_timesteps > 1 needs injection_net_mw_t");
    double* tdiag = A.alloc<double>(E);
    double* tk = A.alloc<double>(static_cast<size_t>(E) * std::max(g.Kpad, 1));
    const int ntiles = g.Kpad / tgb::sweep_tile_k();
    const size_t tmax_n = static_cast<size_t>(std::max(ntiles, 1)) * (E + tgb::sweep_chunk()) * tgb::kRec;
    g.Tdiag = tdiag;
    g.TK = tk;
    ctx->n_t = T;
    ctx->gt.clear();
    float* tmax_all = A.alloc<float>(static_cast<size_t>(T) * tmax_n);
    check(cudaMemsetAsync(tmax_all, 0, static_cast<size_t>(T) * tmax_n * sizeof(float), s), "tmax");
    ctx->mt_pattern_ok = T > 1;
    for (int t = 1; t < T && ctx->mt_pattern_ok; ++t)
      for (int i = 0; i < I; ++i)
        if ((gd->injection_net_mw_t[static_cast<size_t>(t) * I + i] == 0.0) != (gd->injection_net_mw_t[i] == 0.0)) {
          ctx->mt_pattern_ok = false;
          break;
        }
    for (int t = 0; t < T; ++t) {
      const double* net = T > 1 ? gd->injection_net_mw_t + static_cast<size_t>(t) * I : gd->injection_net_mw;
      std::vector<double> p(N, 0.0);
      for (int i = 0; i < I; ++i) p[gd->injection_node[i]] += net[i];
      double tot = 0.0;
      for (double v : p) tot += v;
      p[gd->slack] -= tot;
      std::vector<double> pr(Nr);
      for (int v = 0; v < N; ++v)
        if (red[v] >= 0) pr[red[v]] = p[v];
      tgb::DevGrid gv = g;
      if (T > 1) gv.inj_net = A.upload(std::vector<double>(net, net + I), s);
      double* d_pr = A.upload(pr, s);
      double* theta0 = A.alloc<double>(Nr);
      double* f0 = A.alloc<double>(E);
      float* tmax = tmax_all + static_cast<size_t>(t) * tmax_n;
      double* alpha0 = A.alloc<double>(std::max(g.Kpad, 1));
      gv.theta0 = theta0;
      gv.f0 = f0;
      gv.Tmax = tmax;
      gv.alpha0 = alpha0;
      tgb::launch_base_tables(gv, d_pr, theta0, f0, tdiag, tk, tmax, alpha0, s);
      check(cudaGetLastError(), "base tables");
      double4* rstat = A.alloc<double4>(std::max(E, 1));
      tgb::launch_row_static(gv, f0, rstat, s);
      gv.row_static = rstat;
      if (g.Kpad > 0) {
        float* crec = A.alloc<float>(static_cast<size_t>(ntiles) * ((E + tgb::kChunkRows - 1) / tgb::kChunkRows) *
                                     tgb::kRec);
        tgb::launch_chunk_records(gv, crec, s);
        check(cudaGetLastError(), "chunk records");
        gv.Crec = crec;
      }
      ctx->gt.push_back(gv);
    }
    g = ctx->gt[0];
    ctx->g_mt = g;
    {
      // per-profile table pointers for k_prep_mt
      std::vector<const double*> f0p, thp, injp, a0p;
      std::vector<const float*> tmp;
      for (const auto& gv : ctx->gt) {
        f0p.push_back(gv.f0);
        thp.push_back(gv.theta0);
        injp.push_back(gv.inj_net);
        a0p.push_back(gv.alpha0);
        tmp.push_back(gv.Tmax);
      }
      ctx->mt_prof.tmax = A.upload(tmp, s);
      ctx->mt_prof.f0 = A.upload(f0p, s);
      ctx->mt_prof.theta0 = A.upload(thp, s);
      ctx->mt_prof.inj_net = A.upload(injp, s);
      ctx->mt_prof.alpha0 = A.upload(a0p, s);
      ctx->mt_prof.n_t = T;
    }
    if (T > 1) {
      float* rec_mt = A.alloc<float>(tmax_n);
      tgb::launch_rec_combine(tmax_all, tmax_n, T, rec_mt, s);
      ctx->g_mt.Tmax = rec_mt;
    }
    check(cudaStreamSynchronize(s), "context setup");

    ctx->n_cont = gd->n_contingencies;
    ctx->worst_k = cfg ? cfg->worst_k : 20;
    ctx->params.penalty = cfg ? cfg->islanding_penalty_mw : 10000.0;
    ctx->params.weight_c0 = cfg ? cfg->weight_c0 : 200.0;
    ctx->params.weight_c = cfg ? cfg->weight_c : 50.0;
    ctx->params.variant = cfg ? cfg->fitness_variant : 1;
    ctx->params.worst_k = ctx->worst_k;
    ctx->params.lambda_b_pre = 0.0;
    if (ctx->params.variant != 1 && ctx->params.variant != 2)
      throw tgb::ConfigError("fitness_variant must be 1 or 2");

    // pre-optimization score of the unchanged topology (dc_engine.cpp:137-144)
    ctx->ensure_capacity(1);
    std::vector<int> empty(1, -1);
    check(cudaMemcpyAsync(ctx->d_genomes, empty.data(), sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
    // lambda_b_pre is not known yet: score with variant 1, whose fitness equals the
    // variant-2 pre-score (clip(lambda_b - lambda_b_pre) = 0 for the unchanged topology)
    const int variant = ctx->params.variant;
    ctx->params.variant = 1;
    ctx->run_batch(1, 1, 0, false);
    ctx->params.variant = variant;
    check_errors(ctx, 1);
    double lo_ = 0, lb_ = 0, fit = 0;
    int lc = 0, lc0 = 0;
    const tgb::Scores& o = ctx->batch.out;
    check(cudaMemcpy(&lo_, o.lambda_o, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    check(cudaMemcpy(&lb_, o.lambda_b, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    check(cudaMemcpy(&fit, o.fitness, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    check(cudaMemcpy(&lc, o.lambda_c, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    check(cudaMemcpy(&lc0, o.lambda_c0, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    ctx->lambda_b_pre = lb_;
    ctx->params.lambda_b_pre = lb_;
    ctx->pre = {lo_, static_cast<double>(lc), static_cast<double>(lc0), lb_, fit};
}

}  // namespace

extern "C" {
tg_status tg_context_create(const tg_grid_desc* gd, const tg_actionset_desc* ad, const tg_dc_config* cfg, int device,
                            tg_context** out) {
  return guarded([&] {
    auto ctx = std::make_unique<tg_context>();
    ctx->device = device;
    check(cudaSetDevice(device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    // side stream of launch_evaluate (special outages beside the prep / sweep);
    // created here, not inside a graph capture
    check(cudaStreamCreateWithFlags(&ctx->side.stream, cudaStreamNonBlocking), "side stream");
    check(cudaEventCreateWithFlags(&ctx->side.fork, cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&ctx->side.join, cudaEventDisableTiming), "event");
    if (gd->n_nodes < 2) throw tgb::ValidationError("grid needs at least two nodes");
    double* X = base_inverse(ctx.get(), gd);
    std::vector<int> perm = sweep_row_order(ctx.get(), gd, X);
    if (perm.empty()) {
      context_build(ctx.get(), gd, ad, cfg, X);
    } else {
      PermutedDesc pd(*gd, ad, perm);
      context_build(ctx.get(), &pd.gd, ad ? &pd.ad : nullptr, cfg, X);
      ctx->br_perm = std::move(perm);
    }
    *out = ctx.release();
  });
}

void tg_context_destroy(tg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->qd) {
    if (ctx->qd->graph) cudaGraphExecDestroy(ctx->qd->graph);
    delete static_cast<DeviceArena*>(ctx->qd->arena);
    ctx->qd.reset();
  }
  ctx->batch_arena.reset();
  ctx->free_snap_buffers();
  cudaStream_t s = ctx->stream;
  if (ctx->sw0) cudaEventDestroy(ctx->sw0), cudaEventDestroy(ctx->sw1);
  if (ctx->side.stream) {
    cudaStreamSynchronize(ctx->side.stream);
    cudaStreamDestroy(ctx->side.stream);
    cudaEventDestroy(ctx->side.fork);
    cudaEventDestroy(ctx->side.join);
  }
  if (ctx->err_host) cudaFreeHost(ctx->err_host), cudaEventDestroy(ctx->err_ev);
  delete ctx;
  cudaStreamDestroy(s);
}

tg_status tg_evaluate_batch(tg_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                            int32_t batch_size, tg_scores* out, double* base_flows, double* max_contingency,
                            double* max_busbar, double* outage_energy) {
  return guarded([&] {
    if (n < 0 || n_a < 0 || n_d < 0 || n_a > tgb::kMaxSplits || n_d > tgb::kMaxRemovedSweep)
      throw tgb::ConfigError("genome slots exceed the engine capacity (n_a <= 4, n_d <= 4)");
    if (n == 0) return;
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    for (int64_t i = 0; i < static_cast<int64_t>(n) * (n_a + n_d); ++i) {
      const int v = genomes[i];
      const int slot = static_cast<int>(i % (n_a + n_d));
      if (v < -1 || (slot < n_a && v >= ctx->g.A) || (slot >= n_a && v >= ctx->g.D))
        throw tgb::ValidationError("genome slot value out of range");
    }
    ctx->check_capacity(n_a, n_d);
    (void)batch_size;  // padding lanes are empty genomes whose scores are dropped
    ctx->ensure_capacity(n);
    check(cudaMemcpyAsync(ctx->d_genomes, genomes, static_cast<size_t>(n) * (n_a + n_d) * sizeof(int),
                          cudaMemcpyHostToDevice, ctx->stream),
          "genomes H2D");
    const bool full = base_flows || max_contingency || max_busbar || outage_energy;
    ctx->run_batch(n, n_a, n_d, full);
    copy_scores(ctx, n, out);
    const size_t ne = static_cast<size_t>(n) * ctx->g.E;
    if (base_flows || max_contingency || max_busbar) {
      tgb::DeviceScratchGuard tmp(ne);
      std::vector<double> stage(ctx->br_perm.empty() ? 0 : ne);
      // per-branch outputs leave in the grid's branch order (internal rows: sweep_row_order)
      auto fetch = [&](double* dst) {
        double* land = ctx->br_perm.empty() ? dst : stage.data();
        check(cudaMemcpyAsync(land, tmp.ptr, ne * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        check(cudaStreamSynchronize(ctx->stream), "sync");
        if (!ctx->br_perm.empty()) {
          const int E = ctx->g.E;
          for (int i = 0; i < n; ++i)
            for (int e = 0; e < E; ++e)
              dst[static_cast<size_t>(i) * E + ctx->br_perm[e]] = stage[static_cast<size_t>(i) * E + e];
        }
      };
      if (base_flows) {
        tgb::launch_extract(ctx->g, ctx->batch, tmp.ptr, nullptr, nullptr, ctx->stream);
        fetch(base_flows);
      }
      if (max_contingency) {
        tgb::launch_extract(ctx->g, ctx->batch, nullptr, tmp.ptr, nullptr, ctx->stream);
        fetch(max_contingency);
      }
      if (max_busbar) {
        tgb::launch_extract(ctx->g, ctx->batch, nullptr, nullptr, tmp.ptr, ctx->stream);
        fetch(max_busbar);
      }
    }
    if (outage_energy && ctx->g.Kall > 0)
      check(cudaMemcpyAsync(outage_energy, ctx->batch.energy, static_cast<size_t>(n) * ctx->g.Kall * sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream),
            "energy D2H");
    check_errors(ctx, n);
    // islanded genomes report zero flows / energies (FlowResult is not built, dc_engine.cpp:426-435)
    if (outage_energy && ctx->g.Kall > 0) {
      std::vector<uint8_t> isl(n);
      check(cudaMemcpy(isl.data(), ctx->batch.out.islanded, n, cudaMemcpyDeviceToHost), "D2H");
      for (int i = 0; i < n; ++i)
        if (isl[i]) std::fill(outage_energy + static_cast<size_t>(i) * ctx->g.Kall,
                              outage_energy + static_cast<size_t>(i + 1) * ctx->g.Kall, 0.0);
    }
    check(cudaStreamSynchronize(ctx->stream), "evaluate");
  });
}

tg_status tg_evaluate_batch_device(tg_context* ctx, const int32_t* d_genomes, int32_t n, int32_t n_a, int32_t n_d,
                                   tg_scores* d_out) {
  return guarded([&] {
    if (n_a > tgb::kMaxSplits || n_d > tgb::kMaxRemovedSweep)
      throw tgb::ConfigError("genome slots exceed the engine capacity (n_a <= 4, n_d <= 4)");
    if (n <= 0) return;
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    ctx->check_capacity(n_a, n_d);
    ctx->ensure_capacity(n);
    check(cudaMemcpyAsync(ctx->d_genomes, d_genomes, static_cast<size_t>(n) * (n_a + n_d) * sizeof(int),
                          cudaMemcpyDeviceToDevice, ctx->stream),
          "genomes D2D");
    ctx->run_batch(n, n_a, n_d, false);
    if (d_out) {
      const tgb::Scores& o = ctx->batch.out;
      auto cp = [&](void* dst, const void* src, size_t bytes) {
        if (dst) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "scores D2D");
      };
      cp(d_out->fitness, o.fitness, n * sizeof(double));
      cp(d_out->lambda_o, o.lambda_o, n * sizeof(double));
      cp(d_out->lambda_c, o.lambda_c, n * sizeof(int));
      cp(d_out->lambda_c0, o.lambda_c0, n * sizeof(int));
      cp(d_out->islanded, o.islanded, n * sizeof(uint8_t));
    }
  });
}

tg_status tg_pre_score(tg_context* ctx, tg_scores* out, double* lambda_b_pre) {
  return guarded([&] {
    if (lambda_b_pre) *lambda_b_pre = ctx->lambda_b_pre;
    if (!out) return;
    if (out->lambda_o) out->lambda_o[0] = ctx->pre[0];
    if (out->lambda_c) out->lambda_c[0] = static_cast<int32_t>(ctx->pre[1]);
    if (out->lambda_c0) out->lambda_c0[0] = static_cast<int32_t>(ctx->pre[2]);
    if (out->lambda_b) out->lambda_b[0] = ctx->pre[3];
    if (out->fitness) out->fitness[0] = ctx->pre[4];
    if (out->lambda_d) out->lambda_d[0] = 0;
    if (out->lambda_s) out->lambda_s[0] = 0;
    if (out->lambda_r) out->lambda_r[0] = 0;
    if (out->islanded) out->islanded[0] = 0;
  });
}

int32_t tg_descriptor_to_cell(int32_t d, int32_t s, int32_t r, const tg_qd_config* c) {
  d = std::min(d, c->d_max);
  s = std::min(s, c->s_max);
  r = std::min(r, c->r_max);
  return d + (c->d_max + 1) * (s + (c->s_max + 1) * r);
}

tg_status tg_context_info(tg_context* ctx, int64_t* v, int32_t n) {
  return guarded([&] {
    const int64_t vals[] = {ctx->g.N, ctx->g.E, ctx->g.Kall, ctx->g.Ks, ctx->g.Kx, ctx->g.Kb,
                            ctx->g.A, ctx->g.D, ctx->g.Kpad, static_cast<int64_t>(ctx->arena.bytes())};
    for (int i = 0; i < n && i < static_cast<int>(sizeof(vals) / sizeof(vals[0])); ++i) v[i] = vals[i];
  });
}

int64_t tg_kernel_launches(tg_context* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

// ---------------------------------------------------------------- MapElites loop
namespace {

tgb::QdParams qd_params(tg_context* ctx, const tg_qd_config* c) {
  if (c->batch_size <= 0) throw tgb::ConfigError("batch size must be positive");
  if (c->n_a < 0 || c->n_d < 0 || c->n_a > tgb::kMaxSplits || c->n_d > tgb::kMaxRemovedSweep)
    throw tgb::ConfigError("n_a and n_d must lie in [0, 4] on the device");
  if (c->cell_capacity <= 0 || c->cell_capacity > tgb::kMaxCellCap)
    throw tgb::ConfigError("cell_capacity must lie in [1, 16] on the device");
  if (!(c->mutation_mean < 12.0))
    throw tgb::ConfigError("mutation_mean >= 12 (libstdc++ rejection sampler) is not replayed on the device");
  if (c->d_max < 0 || c->s_max < 0 || c->r_max < 0) throw tgb::ConfigError("descriptor bounds must be >= 0");
  ctx->check_capacity(c->n_a, c->n_d);
  tgb::QdParams p{};
  p.n_a = c->n_a;
  p.n_d = c->n_d;
  p.batch = c->batch_size;
  p.cap = c->cell_capacity;
  p.d_max = c->d_max;
  p.s_max = c->s_max;
  p.r_max = c->r_max;
  p.cells = (c->d_max + 1) * (c->s_max + 1) * (c->r_max + 1);
  for (int i = 0; i < 4; ++i) p.p_action[i] = c->p_action[i], p.p_disc[i] = c->p_disc[i];
  p.p_c1 = c->p_crossover_parent1;
  p.poisson_thr = std::exp(-c->mutation_mean);  // poisson_distribution::param_type::_M_initialize
  p.seed = c->seed;
  p.n_actions = ctx->g.A;
  p.n_disc = ctx->g.D;
  if (c->rng != tgb::kRngReplay && c->rng != tgb::kRngPhilox) throw tgb::ConfigError("rng must be 0 (replay) or 1 (philox)");
  p.rng = c->rng;
  return p;
}

void qd_setup(tg_context* ctx, const tgb::QdParams& p) {
  auto& q = ctx->qd;
  const bool same = q && q->p.cells == p.cells && q->p.cap == p.cap && q->p.n_a == p.n_a && q->p.n_d == p.n_d &&
                    q->p.batch >= p.batch;
  if (!same) {
    if (q && q->graph) cudaGraphExecDestroy(q->graph);
    delete static_cast<DeviceArena*>(q ? q->arena : nullptr);
    q = std::make_unique<tgb::QdState>();
    ctx->merge.capacity = 0;  // merge buffers are sized for the old slot layout
    auto* A = new DeviceArena();
    q->arena = A;
    const size_t slots = static_cast<size_t>(p.cells) * p.cap;
    const int ns = p.n_a + p.n_d, wk = std::max(ctx->worst_k, 1);
    tgb::Archive& a = q->a;
    a.count = A->alloc<int>(p.cells);
    a.flat_start = A->alloc<int>(p.cells + 1);
    a.genome = A->alloc<int>(slots * std::max(ns, 1));
    a.key = A->alloc<int>(slots * std::max(ns, 1));
    a.fitness = A->alloc<double>(slots);
    a.lambda_o = A->alloc<double>(slots);
    a.lambda_c = A->alloc<int>(slots);
    a.lambda_c0 = A->alloc<int>(slots);
    a.lambda_b = A->alloc<double>(slots);
    a.lambda_d = A->alloc<int>(slots);
    a.lambda_s = A->alloc<int>(slots);
    a.lambda_r = A->alloc<int>(slots);
    a.worst_idx = A->alloc<int>(slots * wk);
    a.worst_val = A->alloc<double>(slots * wk);
    a.worst_n = A->alloc<int>(slots);
    a.iter = A->alloc<long long>(1);
    q->inserted = A->alloc<uint8_t>(std::max(p.batch, 1));
    q->lane_cell = A->alloc<int>(std::max(p.batch, 1));
    q->graph_batch = 0;
  }
  if (q->graph && std::memcmp(&q->p, &p, sizeof(p)) != 0) {
    cudaGraphExecDestroy(q->graph);
    q->graph = nullptr;
  }
  q->p = p;
  q->n_slots = p.n_a + p.n_d;
  q->worst_k = ctx->worst_k;
}

// Snapshot of the device archive (make_snapshot, qd_optimizer.cpp:331-342):
// enqueue the blob pack + D2H into ring slot `slot`, completion recorded on
// snap_ev[slot]; decode_snapshot turns the pinned blob into ctx->snap.
void enqueue_snapshot(tg_context* ctx, int slot) {
  const tgb::QdState& q = *ctx->qd;
  ctx->snap_buffers(tgb::BlobLayout(q.p.cells * q.p.cap, q.n_slots, q.worst_k).total);
  tgb::launch_archive_pack(q, ctx->snap_dev[slot], ctx->stream);
  ctx->launches += 1;
  check(cudaMemcpyAsync(ctx->snap_host[slot], ctx->snap_dev[slot], ctx->snap_bytes, cudaMemcpyDeviceToHost,
                        ctx->stream), "snapshot D2H");
  check(cudaEventRecord(ctx->snap_ev[slot], ctx->stream), "snapshot event");
}

void decode_snapshot(tg_context* ctx, int slot, int epoch, int64_t evaluations, bool fin) {
  const tgb::QdState& q = *ctx->qd;
  ctx->snap.from_blob(ctx->snap_host[slot], q.p.cells, q.p.cap, q.n_slots, q.worst_k, epoch, evaluations, fin);
}

// Synchronous snapshot (tg_qd_fetch, tg_archive_replay, run end).
void fetch_archive(tg_context* ctx, int epoch, int64_t evaluations, bool fin) {
  enqueue_snapshot(ctx, 0);
  check(cudaEventSynchronize(ctx->snap_ev[0]), "snapshot");
  decode_snapshot(ctx, 0, epoch, evaluations, fin);
}

// One MapElites iteration: offspring -> DC N-1 evaluation -> archive insert.
int enqueue_iteration(tg_context* ctx) {
  tgb::QdState& q = *ctx->qd;
  const int B = q.p.batch;
  tgb::launch_offspring(ctx->g, q, ctx->d_genomes, ctx->stream);
  ctx->batch.n = B;
  ctx->batch.genomes = ctx->d_genomes;
  ctx->batch.params = ctx->params;
  const int kernels = ctx->enqueue_evaluate(q.p.n_a, q.p.n_d, false);
  const int ins = tgb::launch_insert(q, ctx->d_genomes, ctx->batch.out, B, ctx->worst_k, true, ctx->stream);
  return 1 + kernels + ins;
}

}  // namespace

extern "C" {

tg_status tg_qd_begin(tg_context* ctx, const tg_qd_config* cfg) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->g.A == 0 && ctx->g.D == 0)
      throw tgb::ConfigError("nothing to optimize: no actions and no disconnectable branches");
    const tgb::QdParams p = qd_params(ctx, cfg);
    qd_setup(ctx, p);
    tgb::QdState& q = *ctx->qd;
    ctx->ensure_capacity(p.batch);
    check(cudaMemsetAsync(ctx->err_sticky, 0, sizeof(int), ctx->stream), "error word reset");
    ctx->err_pending = false;
    cudaStream_t s = ctx->stream;
    // seed the archive with the unchanged topology (qd_optimizer.cpp:361-363)
    tgb::launch_archive_reset(q, s);
    check(cudaMemsetAsync(ctx->d_genomes, 0xff, static_cast<size_t>(q.n_slots) * sizeof(int), s), "seed genome");
    ctx->run_batch(1, p.n_a, p.n_d, false);
    ctx->launches += tgb::launch_insert(q, ctx->d_genomes, ctx->batch.out, 1, ctx->worst_k, false, s);
    ctx->qd_evaluations = 1;
    ctx->qd_epoch = 0;
    // the whole iteration as one CUDA graph (no host round trip per generation)
    if (!q.graph || q.graph_batch != p.batch) {
      if (q.graph) cudaGraphExecDestroy(q.graph);
      cudaGraph_t graph;
      check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
      q.kernels_per_iter = enqueue_iteration(ctx);
      check(cudaStreamEndCapture(s, &graph), "capture end");
      check(cudaGraphInstantiate(&q.graph, graph, 0), "graph instantiate");
      cudaGraphDestroy(graph);
      q.graph_batch = p.batch;
    }
  });
}

tg_status tg_qd_step(tg_context* ctx, int32_t n_iters) {
  return guarded([&] {
    if (!ctx->qd || !ctx->qd->graph) throw tgb::ConfigError("call tg_qd_begin first");
    ctx->poll_sticky();  // an earlier step's capacity error surfaces here (no synchronization)
    if (ctx->time_sweep) {
      // instrumented path: same kernels launched directly, sweep bracketed by events
      tgb::QdState& q = *ctx->qd;
      for (int i = 0; i < n_iters; ++i) {
        tgb::launch_offspring(ctx->g, q, ctx->d_genomes, ctx->stream);
        ctx->run_batch(q.p.batch, q.p.n_a, q.p.n_d, false);
        ctx->launches += 1 + tgb::launch_insert(q, ctx->d_genomes, ctx->batch.out, q.p.batch, ctx->worst_k, true,
                                                ctx->stream);
      }
      ctx->qd_evaluations += static_cast<int64_t>(n_iters) * q.p.batch;
      ctx->mirror_sticky();
      return;
    }
    for (int i = 0; i < n_iters; ++i) check(cudaGraphLaunch(ctx->qd->graph, ctx->stream), "graph launch");
    ctx->launches += static_cast<int64_t>(n_iters) * ctx->qd->kernels_per_iter;
    ctx->qd_evaluations += static_cast<int64_t>(n_iters) * ctx->qd->p.batch;
    ctx->mirror_sticky();
  });
}

// ---- batch-sharded generation (SURVEY.md 8(e) parity mode)
namespace {
tgb::Scores offset_scores(const tgb::Scores& o, int lo, int wk) {
  tgb::Scores v = o;
  v.lambda_o += lo, v.lambda_c += lo, v.lambda_c0 += lo, v.lambda_b += lo, v.lambda_d += lo, v.lambda_s += lo;
  v.lambda_r += lo, v.fitness += lo, v.islanded += lo, v.error += lo, v.worst_n += lo, v.isl_out += lo;
  v.isl_bus += lo;
  v.worst_idx += static_cast<size_t>(lo) * wk;
  v.worst_val += static_cast<size_t>(lo) * wk;
  return v;
}
void check_lane_range(tg_context* ctx, int lo, int hi) {
  if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
  if (lo < 0 || hi < lo || hi > ctx->qd->p.batch) throw tgb::ConfigError("lane range outside the batch");
}
}  // namespace

tg_status tg_qd_generation_begin(tg_context* ctx) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    tgb::launch_offspring(ctx->g, *ctx->qd, ctx->d_genomes, ctx->stream);
    ctx->launches += 1;
    check(cudaGetLastError(), "offspring");
  });
}

tg_status tg_qd_evaluate_lanes(tg_context* ctx, int32_t lo, int32_t hi) {
  return guarded([&] {
    check_lane_range(ctx, lo, hi);
    if (hi == lo) return;
    const tgb::QdState& q = *ctx->qd;
    tgb::Batch bv = ctx->batch;
    bv.n = hi - lo;
    bv.genomes = ctx->d_genomes + static_cast<size_t>(lo) * q.n_slots;
    bv.params = ctx->params;
    bv.out = offset_scores(ctx->batch.out, lo, std::max(ctx->worst_k, 1));
    ctx->launches += ctx->enqueue_evaluate(bv, q.p.n_a, q.p.n_d, false, false);
    check(cudaGetLastError(), "evaluate lanes");
  });
}

tg_status tg_qd_scores_blob_bytes(tg_context* ctx, int32_t n, int64_t* bytes) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    *bytes = static_cast<int64_t>(tgb::BlobLayout(n, ctx->qd->n_slots, ctx->qd->worst_k).total);
  });
}

tg_status tg_qd_scores_pack(tg_context* ctx, int32_t lo, int32_t hi, void* d_blob) {
  return guarded([&] {
    check_lane_range(ctx, lo, hi);
    tgb::launch_scores_pack(*ctx->qd, ctx->d_genomes, ctx->batch.out, lo, hi - lo, d_blob, ctx->stream);
    ctx->launches += 1;
    check(cudaGetLastError(), "scores pack");
  });
}

tg_status tg_qd_scores_unpack(tg_context* ctx, int32_t lo, int32_t hi, const void* d_blob) {
  return guarded([&] {
    check_lane_range(ctx, lo, hi);
    tgb::launch_scores_unpack(*ctx->qd, d_blob, lo, hi - lo, ctx->batch.out, ctx->stream);
    ctx->launches += 1;
    check(cudaGetLastError(), "scores unpack");
  });
}

tg_status tg_qd_generation_end(tg_context* ctx) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    tgb::QdState& q = *ctx->qd;
    ctx->launches += tgb::launch_insert(q, ctx->d_genomes, ctx->batch.out, q.p.batch, ctx->worst_k, true,
                                        ctx->stream);
    ctx->qd_evaluations += q.p.batch;
    check(cudaGetLastError(), "insert");
    ctx->poll_sticky();
    ctx->mirror_sticky();
  });
}

tg_status tg_qd_fetch(tg_context* ctx, int32_t final_snapshot, tg_snapshot_view* out) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    ctx->check_sticky();
    fetch_archive(ctx, ctx->qd_epoch, ctx->qd_evaluations, final_snapshot != 0);
    if (out) *out = ctx->snap.view;
  });
}

tg_status tg_qd_offspring(tg_context* ctx, int32_t* genomes_out) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    tgb::QdState& q = *ctx->qd;
    tgb::launch_offspring(ctx->g, q, ctx->d_genomes, ctx->stream);
    ctx->launches += 1;
    check(cudaMemcpyAsync(genomes_out, ctx->d_genomes, static_cast<size_t>(q.p.batch) * q.n_slots * sizeof(int),
                          cudaMemcpyDeviceToHost, ctx->stream),
          "offspring D2H");
    check(cudaStreamSynchronize(ctx->stream), "offspring");
  });
}

tg_status tg_qd_insert(tg_context* ctx, const int32_t* genomes, const tg_scores* sc) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    tgb::QdState& q = *ctx->qd;
    const int n = q.p.batch, wk = ctx->worst_k;
    const tgb::Scores& o = ctx->batch.out;
    cudaStream_t s = ctx->stream;
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
      if (!src) throw tgb::ConfigError("insert needs every score field");
      check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "insert H2D");
    };
    h2d(ctx->d_genomes, genomes, static_cast<size_t>(n) * q.n_slots * sizeof(int));
    h2d(o.fitness, sc->fitness, n * sizeof(double));
    h2d(o.lambda_o, sc->lambda_o, n * sizeof(double));
    h2d(o.lambda_c, sc->lambda_c, n * sizeof(int));
    h2d(o.lambda_c0, sc->lambda_c0, n * sizeof(int));
    h2d(o.lambda_b, sc->lambda_b, n * sizeof(double));
    h2d(o.lambda_d, sc->lambda_d, n * sizeof(int));
    h2d(o.lambda_s, sc->lambda_s, n * sizeof(int));
    h2d(o.lambda_r, sc->lambda_r, n * sizeof(int));
    h2d(o.worst_n, sc->worst_n, n * sizeof(int));
    h2d(o.worst_idx, sc->worst_idx, static_cast<size_t>(n) * wk * sizeof(int));
    h2d(o.worst_val, sc->worst_energy, static_cast<size_t>(n) * wk * sizeof(double));
    ctx->launches += tgb::launch_insert(q, ctx->d_genomes, o, n, wk, true, s);
    ctx->qd_evaluations += n;
    check(cudaStreamSynchronize(s), "insert");
  });
}

tg_status tg_archive_blob_bytes(tg_context* ctx, int64_t* bytes) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    const tgb::QdState& q = *ctx->qd;
    *bytes = static_cast<int64_t>(tgb::BlobLayout(q.p.cells * q.p.cap, q.n_slots, q.worst_k).total);
  });
}

tg_status tg_archive_pack(tg_context* ctx, void* d_blob) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    if (!d_blob) throw tgb::ConfigError("null blob");
    tgb::launch_archive_pack(*ctx->qd, d_blob, ctx->stream);
    ctx->launches += 1;
    check(cudaGetLastError(), "archive pack");
  });
}

tg_status tg_archive_merge(tg_context* ctx, const void* d_blobs, int32_t n_islands) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("call tg_qd_begin first");
    if (n_islands <= 0 || !d_blobs) throw tgb::ConfigError("merge needs at least one island blob");
    tgb::QdState& q = *ctx->qd;
    const int n = q.p.cells * q.p.cap * n_islands;
    tgb::MergeBuffers& m = ctx->merge;
    if (m.capacity < n) {
      ctx->merge_arena = std::make_unique<DeviceArena>();
      DeviceArena& A = *ctx->merge_arena;
      const size_t wk = std::max(ctx->worst_k, 1);
      m = tgb::MergeBuffers{};
      m.capacity = n;
      m.genomes = A.alloc<int>(static_cast<size_t>(n) * std::max(q.n_slots, 1));
      m.sc.fitness = A.alloc<double>(n);
      m.sc.lambda_o = A.alloc<double>(n);
      m.sc.lambda_b = A.alloc<double>(n);
      m.sc.lambda_c = A.alloc<int>(n);
      m.sc.lambda_c0 = A.alloc<int>(n);
      m.sc.lambda_d = A.alloc<int>(n);
      m.sc.lambda_s = A.alloc<int>(n);
      m.sc.lambda_r = A.alloc<int>(n);
      m.sc.worst_n = A.alloc<int>(n);
      m.sc.worst_idx = A.alloc<int>(static_cast<size_t>(n) * wk);
      m.sc.worst_val = A.alloc<double>(static_cast<size_t>(n) * wk);
      m.lane_cell = A.alloc<int>(n);
      m.inserted = A.alloc<uint8_t>(n);
    }
    ctx->launches += tgb::launch_archive_merge(q, d_blobs, n_islands, m, ctx->stream);
    check(cudaGetLastError(), "archive merge");
  });
}

struct tg_channel {
  explicit tg_channel(size_t capacity) : q(capacity) {}
  tgb::SnapshotChannel q;
  std::unique_ptr<tgb::HostSnapshot> popped;  // backs the view returned by the last pop
};

tg_channel* tg_channel_create(int64_t capacity) {
  try {
    return new tg_channel(static_cast<size_t>(capacity > 0 ? capacity : 0));
  } catch (...) {
    return nullptr;
  }
}
void tg_channel_destroy(tg_channel* ch) { delete ch; }
void tg_channel_push(tg_channel* ch, const tg_snapshot_view* v) {
  if (!ch || !v) return;
  auto s = std::make_unique<tgb::HostSnapshot>();
  s->from_view(*v);
  ch->q.push(std::move(s));
}
void tg_channel_sink(const tg_snapshot_view* v, void* channel) { tg_channel_push(static_cast<tg_channel*>(channel), v); }
void tg_channel_close(tg_channel* ch) {
  if (ch) ch->q.close();
}
int32_t tg_channel_pop(tg_channel* ch, int32_t blocking, tg_snapshot_view* out) {
  if (!ch) return 0;
  auto s = ch->q.pop(blocking != 0);
  if (!s) return 0;
  ch->popped = std::move(s);
  if (out) *out = ch->popped->view;
  return 1;
}
int64_t tg_channel_pending(tg_channel* ch) { return ch ? static_cast<int64_t>(ch->q.pending()) : 0; }
int64_t tg_channel_dropped(tg_channel* ch) { return ch ? static_cast<int64_t>(ch->q.dropped()) : 0; }

void* tg_context_stream(tg_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

tg_status tg_sweep_timing(tg_context* ctx, int32_t enable, double* total_ms, int64_t* launches) {
  return guarded([&] {
    if (total_ms) *total_ms = ctx->sweep_ms;
    if (launches) *launches = ctx->sweep_launches;
    ctx->time_sweep = enable != 0;
    ctx->sweep_ms = 0.0;
    ctx->sweep_launches = 0;
  });
}

tg_status tg_sweep_rows(tg_context* ctx, int64_t* computed, int64_t* offered, int64_t* overloaded, int64_t* partial) {
  return guarded([&] {
    unsigned long long v[4] = {0, 0, 0, 0};
    if (ctx->batch.rows_done) {
      check(cudaMemcpyAsync(v, ctx->batch.rows_done, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream), "rows D2H");
      check(cudaMemsetAsync(ctx->batch.rows_done, 0, sizeof(v), ctx->stream), "rows reset");
      check(cudaStreamSynchronize(ctx->stream), "rows");
    }
    if (computed) *computed = static_cast<int64_t>(v[0]);
    if (offered) *offered = static_cast<int64_t>(v[1]);
    if (overloaded) *overloaded = static_cast<int64_t>(v[2]);
    if (partial) *partial = static_cast<int64_t>(v[3]);
  });
}

tg_status tg_sweep_chunks(tg_context* ctx, int64_t* tested, int64_t* hot) {
  return guarded([&] {
    unsigned long long v[2] = {0, 0};
    if (ctx->batch.rows_done) {
      check(cudaMemcpyAsync(v, ctx->batch.rows_done + 4, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
      check(cudaMemsetAsync(ctx->batch.rows_done + 4, 0, sizeof(v), ctx->stream), "chunks reset");
      check(cudaStreamSynchronize(ctx->stream), "chunks");
    }
    if (tested) *tested = static_cast<int64_t>(v[0]);
    if (hot) *hot = static_cast<int64_t>(v[1]);
  });
}

tg_status tg_batch_ranks(tg_context* ctx, int32_t n, int32_t* ranks) {
  return guarded([&] {
    check(cudaMemcpyAsync(ranks, ctx->batch.rank, static_cast<size_t>(n) * sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream), "ranks D2H");
    check(cudaStreamSynchronize(ctx->stream), "ranks");
  });
}

tg_status tg_optimizer_run(tg_context* ctx, const tg_qd_config* cfg, tg_snapshot_cb cb, void* user,
                           const volatile int32_t* stop, tg_opt_stats* stats, int64_t* trace_ev, double* trace_best,
                           int32_t trace_cap) {
  const auto t0 = std::chrono::steady_clock::now();
  tg_status st = tg_qd_begin(ctx, cfg);
  if (st != TG_OK) return st;
  return guarded([&] {
    tgb::QdState& q = *ctx->qd;
    cudaStream_t s = ctx->stream;
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    auto exhausted = [&] {
      if (stop && *stop) return true;
      if (cfg->max_evaluations >= 0 && ctx->qd_evaluations >= cfg->max_evaluations) return true;
      if (cfg->max_seconds >= 0.0 && elapsed() >= cfg->max_seconds) return true;
      return false;
    };
    // at most kInFlight generations queued ahead of the device, so stop /
    // max_seconds act within a few generations (qd_optimizer.cpp:365-376)
    constexpr int kInFlight = 4;
    cudaEvent_t ev[kInFlight];
    for (auto& e : ev) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    int n_trace = 0;
    int64_t launched = 0;
    bool emitted_final = false;
    // Snapshot hand-off: each epoch's archive is packed
    // and copied to pinned memory asynchronously; the sink runs on this thread
    // once the copy has landed, while the device already works on the next
    // epoch (same content and order as make_snapshot after each epoch,
    // qd_optimizer.cpp:403-410).
    struct Pending {
      int slot, epoch;
      int64_t evaluations;
      bool fin;
    };
    std::deque<Pending> pending;
    int next_slot = 0;
    auto deliver = [&](bool wait_all) {
      while (!pending.empty()) {
        const Pending p = pending.front();
        if (!wait_all) {
          const cudaError_t r = cudaEventQuery(ctx->snap_ev[p.slot]);
          if (r == cudaErrorNotReady) return;
          check(r, "snapshot");
        } else {
          check(cudaEventSynchronize(ctx->snap_ev[p.slot]), "snapshot");
        }
        decode_snapshot(ctx, p.slot, p.epoch, p.evaluations, p.fin);
        pending.pop_front();
        if (trace_ev && trace_best && n_trace < trace_cap) {
          trace_ev[n_trace] = p.evaluations;
          trace_best[n_trace] = ctx->snap.view.best_fitness;
        }
        ++n_trace;
        if (cb) cb(&ctx->snap.view, user);
      }
    };
    auto snapshot = [&](bool fin) {
      if (static_cast<int>(pending.size()) == tg_context::kSnapSlots) {  // ring full: the oldest goes first
        check(cudaEventSynchronize(ctx->snap_ev[pending.front().slot]), "snapshot");
        deliver(false);
      }
      enqueue_snapshot(ctx, next_slot);
      pending.push_back({next_slot, ctx->qd_epoch, ctx->qd_evaluations, fin});
      next_slot = (next_slot + 1) % tg_context::kSnapSlots;
    };
    while (!exhausted()) {
      for (int it = 0; it < cfg->iters_per_epoch && !exhausted(); ++it) {
        if (launched >= kInFlight) check(cudaEventSynchronize(ev[launched % kInFlight]), "throttle");
        check(cudaGraphLaunch(q.graph, s), "graph launch");
        check(cudaEventRecord(ev[launched % kInFlight], s), "event record");
        ++launched;
        ctx->launches += q.kernels_per_iter;
        ctx->qd_evaluations += q.p.batch;
        deliver(false);
      }
      ++ctx->qd_epoch;
      const bool fin = exhausted();
      snapshot(fin);
      if (fin) {
        emitted_final = true;
        break;
      }
    }
    if (!emitted_final) snapshot(true);
    deliver(true);
    for (auto& e : ev) cudaEventDestroy(e);
    // capacity errors of any generation of the run surface here (sticky word)
    ctx->check_sticky();
    if (stats) {
      stats->evaluations = ctx->qd_evaluations;
      stats->epochs = ctx->qd_epoch;
      stats->n_trace = std::min(n_trace, trace_cap);
    }
  });
}

tg_status tg_archive_export(tg_context* ctx, tg_snapshot_view* out) {
  return guarded([&] {
    if (!ctx->qd) throw tgb::ConfigError("no archive: run the optimizer or a replay first");
    *out = ctx->snap.view;
  });
}

tg_status tg_archive_replay(tg_context* ctx, const tg_qd_config* cfg, const int32_t* genomes, int32_t n,
                            const tg_scores* sc, uint8_t* inserted) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tg_qd_config c2 = *cfg;
    c2.batch_size = std::max(n, 1);
    const tgb::QdParams p = qd_params(ctx, &c2);
    qd_setup(ctx, p);
    tgb::QdState& q = *ctx->qd;
    ctx->ensure_capacity(std::max(n, 1));
    cudaStream_t s = ctx->stream;
    tgb::launch_archive_reset(q, s);
    if (n > 0) {
      const tgb::Scores& o = ctx->batch.out;
      auto h2d = [&](void* dst, const void* src, size_t bytes) {
        if (!src) throw tgb::ConfigError("replay needs fitness, lambda_d/s/r and worst lists");
        check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "replay H2D");
      };
      const int wk = ctx->worst_k;
      h2d(ctx->d_genomes, genomes, static_cast<size_t>(n) * q.n_slots * sizeof(int));
      h2d(o.fitness, sc->fitness, n * sizeof(double));
      h2d(o.lambda_d, sc->lambda_d, n * sizeof(int));
      h2d(o.lambda_s, sc->lambda_s, n * sizeof(int));
      h2d(o.lambda_r, sc->lambda_r, n * sizeof(int));
      std::vector<double> zd(n, 0.0);
      std::vector<int> zi(static_cast<size_t>(n) * std::max(wk, 1), 0);
      std::vector<double> zw(static_cast<size_t>(n) * std::max(wk, 1), 0.0);
      h2d(o.lambda_o, sc->lambda_o ? sc->lambda_o : zd.data(), n * sizeof(double));
      h2d(o.lambda_b, sc->lambda_b ? sc->lambda_b : zd.data(), n * sizeof(double));
      h2d(o.lambda_c, sc->lambda_c ? sc->lambda_c : zi.data(), n * sizeof(int));
      h2d(o.lambda_c0, sc->lambda_c0 ? sc->lambda_c0 : zi.data(), n * sizeof(int));
      h2d(o.worst_n, sc->worst_n ? sc->worst_n : zi.data(), n * sizeof(int));
      h2d(o.worst_idx, sc->worst_idx ? sc->worst_idx : zi.data(), zi.size() * sizeof(int));
      h2d(o.worst_val, sc->worst_energy ? sc->worst_energy : zw.data(), zw.size() * sizeof(double));
      ctx->launches += tgb::launch_insert(q, ctx->d_genomes, o, n, wk, false, s);
      if (inserted) check(cudaMemcpyAsync(inserted, q.inserted, n, cudaMemcpyDeviceToHost, s), "inserted D2H");
    }
    fetch_archive(ctx, 0, n, true);
  });
}

tg_status tg_mutate_lanes(tg_context* ctx, const tg_qd_config* cfg, const int32_t* parents, const uint64_t* seeds,
                          int32_t n, int32_t* children) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tg_qd_config c2 = *cfg;
    c2.batch_size = std::max(n, 1);
    const tgb::QdParams p = qd_params(ctx, &c2);
    tgb::QdState tmp;
    tmp.p = p;
    const size_t ns = p.n_a + p.n_d;
    DeviceArena A;
    int* dp = A.alloc<int>(n * ns);
    int* dc = A.alloc<int>(n * ns);
    auto* ds = A.alloc<unsigned long long>(n);
    check(cudaMemcpyAsync(dp, parents, n * ns * sizeof(int), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    check(cudaMemcpyAsync(ds, seeds, n * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    tgb::launch_mutate_lanes(ctx->g, tmp, dp, ds, n, dc, ctx->stream);
    ctx->launches += 1;
    check(cudaMemcpyAsync(children, dc, n * ns * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check(cudaStreamSynchronize(ctx->stream), "mutate");
  });
}

tg_status tg_crossover_lanes(tg_context* ctx, const tg_qd_config* cfg, const int32_t* p1, const int32_t* p2,
                             const uint64_t* seeds, int32_t n, int32_t* children) {
  return guarded([&] {
    check(cudaSetDevice(ctx->device), "cudaSetDevice");
    tg_qd_config c2 = *cfg;
    c2.batch_size = std::max(n, 1);
    const tgb::QdParams p = qd_params(ctx, &c2);
    tgb::QdState tmp;
    tmp.p = p;
    const size_t ns = p.n_a + p.n_d;
    DeviceArena A;
    int* d1 = A.alloc<int>(n * ns);
    int* d2 = A.alloc<int>(n * ns);
    int* dc = A.alloc<int>(n * ns);
    auto* ds = A.alloc<unsigned long long>(n);
    check(cudaMemcpyAsync(d1, p1, n * ns * sizeof(int), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    check(cudaMemcpyAsync(d2, p2, n * ns * sizeof(int), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    check(cudaMemcpyAsync(ds, seeds, n * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    tgb::launch_crossover_lanes(ctx->g, tmp, d1, d2, ds, n, dc, ctx->stream);
    ctx->launches += 1;
    check(cudaMemcpyAsync(children, dc, n * ns * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    check(cudaStreamSynchronize(ctx->stream), "crossover");
  });
}

}  // extern "C"

namespace tgb {
double measure_fp64_peak(int device);
}

extern "C" tg_status tg_fp64_peak(int device, double* tflops) {
  return guarded([&] {
    *tflops = tgb::measure_fp64_peak(device);
    check(cudaGetLastError(), "fp64 peak");
  });
}

// ---------------------------------------------------------------- AC validation
// AcValidator (ac_validator.hpp:93-140) on the device: the baseline at
// creation, then worst-k and full N-1 stages for whole batches of genomes.
struct tg_ac_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  DeviceArena arena;
  tgb::AcGrid g{};
  tg_ac_config cfg{};
  int N = 0, E = 0, I = 0, K = 0, A = 0, D = 0;
  double pre_fitness = 0.0;
  // baseline of the unchanged grid (ac_validator.cpp:313-343)
  double base_lambda_o = 0.0;
  int base_critical = 0;
  bool base_converged = false;
  double base_energy = 0.0;
  std::vector<uint8_t> case_conv;
  std::vector<double> case_energy;
  int64_t launches = 0;
  // per-call buffers (grow only)
  std::unique_ptr<DeviceArena> work;
  size_t cap_genomes = 0, cap_cases = 0, cap_scratch = 0, cap_rows = 0;
  int cap_slots = 0;
  int *d_genomes = nullptr, *d_case_g = nullptr, *d_case_k = nullptr, *d_iters = nullptr, *d_crit = nullptr,
      *d_nonconv = nullptr, *d_fcrit = nullptr;
  int *t_from = nullptr, *t_to = nullptr, *t_inode = nullptr, *t_nnew = nullptr, *t_split = nullptr;
  uint8_t *t_rem = nullptr, *d_conv = nullptr, *d_foldcase = nullptr;
  double *d_energy = nullptr, *d_flo = nullptr, *d_loading = nullptr, *d_vm = nullptr, *d_va = nullptr;
  unsigned long long* d_fold = nullptr;
  unsigned char* d_scratch = nullptr;
  unsigned* d_next_case = nullptr;
  // pinned host staging of one call's inputs and per-case outputs (grow only)
  unsigned char* h_stage = nullptr;
  size_t h_stage_cap = 0;

  struct Result {
    std::vector<uint8_t> conv;
    std::vector<int32_t> iters, crit;
    std::vector<double> energy;
    std::vector<int32_t> nonconv, fold_crit;  // per genome (fold runs)
    std::vector<double> fold_lambda_o;
  };
  // Runs cases (genome index, contingency index) of a genome batch; with
  // `fold`, contingency cases (k >= 0) fold their loadings per genome.
  Result run(const int32_t* genomes, int n_genomes, int n_a, int n_d, const std::vector<int32_t>& cg,
             const std::vector<int32_t>& ck, bool fold, double* loading, double* vm, double* va);
};

namespace {
constexpr size_t kAcSmemMax = 200 * 1024;
constexpr size_t kAcScratchBudget = size_t(4) << 30;

tgb::AcSolver ac_solver(const tg_ac_context& ctx, int n_a) {
  tgb::AcSolver sv{};
  sv.tol = ctx.cfg.tolerance_pu;
  sv.max_iter = ctx.cfg.max_iterations;
  sv.n_bus = ctx.N + n_a;
  sv.nu = 2 * (sv.n_bus - 1);
  if (static_cast<double>(sv.nu) * sv.nu * 8.0 > double(size_t(1) << 30))
    throw CapacityFailure("dense AC Jacobian of " + std::to_string(sv.nu) +
                          " unknowns exceeds the 1 GiB per-case workspace of the batched solver");
  sv.ws_bytes = tgb::ac_workspace_bytes(sv.n_bus, sv.nu, ctx.E);
  sv.in_smem = sv.ws_bytes <= kAcSmemMax;
  return sv;
}
}  // namespace

tg_ac_context::Result tg_ac_context::run(const int32_t* genomes, int n_genomes, int n_a, int n_d,
                                         const std::vector<int32_t>& cg, const std::vector<int32_t>& ck, bool fold,
                                         double* loading, double* vm, double* va) {
  if (n_a < 0 || n_d < 0 || n_a > 64 || n_d > 64) throw tgb::ValidationError("bad genome slot counts");
  for (int i = 0; i < n_genomes; ++i) {
    for (int s = 0; s < n_a; ++s) {
      const int a = genomes[static_cast<size_t>(i) * (n_a + n_d) + s];
      if (a < -1 || a >= A) throw tgb::ValidationError("action id out of range in genome " + std::to_string(i));
    }
    for (int s = 0; s < n_d; ++s) {
      const int d = genomes[static_cast<size_t>(i) * (n_a + n_d) + n_a + s];
      if (d < -1 || d >= D) throw tgb::ValidationError("disconnection id out of range in genome " + std::to_string(i));
    }
  }
  const int nc = static_cast<int>(cg.size());
  for (int c = 0; c < nc; ++c)
    if (cg[c] < 0 || cg[c] >= n_genomes || ck[c] < -1 || ck[c] >= K)
      throw tgb::ValidationError("AC case " + std::to_string(c) + " out of range");
  const tgb::AcSolver sv0 = ac_solver(*this, n_a);
  // HBM-scratch path: one slot per resident CTA, four 256-thread CTAs per SM (64 registers)
  int slots = sv0.in_smem ? nc  // one CTA per case: the block scheduler balances the uneven Newton runs
                          : std::max(1, std::min<int>({nc, 148 * 4, static_cast<int>(kAcScratchBudget / sv0.ws_bytes)}));
  const size_t scratch = sv0.in_smem ? 0 : static_cast<size_t>(slots) * sv0.ws_bytes;
  const size_t rows = loading ? static_cast<size_t>(nc) * E : 0;
  const size_t vrows = vm ? static_cast<size_t>(nc) * (N + n_a) : 0;
  check(cudaSetDevice(device), "cudaSetDevice");
  if (!work || static_cast<size_t>(n_genomes) > cap_genomes || static_cast<size_t>(nc) > cap_cases ||
      scratch > cap_scratch || rows + 2 * vrows > cap_rows || n_a + n_d > cap_slots) {
    check(cudaStreamSynchronize(stream), "AC sync");
    work.reset(new DeviceArena);
    cap_genomes = std::max<size_t>(n_genomes, 2 * cap_genomes);
    cap_cases = std::max<size_t>(nc, 2 * cap_cases);
    cap_scratch = std::max(scratch, cap_scratch);
    cap_rows = std::max(rows + 2 * vrows, cap_rows);
    cap_slots = std::max(n_a + n_d, std::max(cap_slots, 8));
    d_genomes = work->alloc<int>(cap_genomes * cap_slots);
    t_from = work->alloc<int>(cap_genomes * E);
    t_to = work->alloc<int>(cap_genomes * E);
    t_rem = work->alloc<uint8_t>(cap_genomes * E);
    t_inode = work->alloc<int>(cap_genomes * std::max(I, 1));
    t_nnew = work->alloc<int>(cap_genomes);
    t_split = work->alloc<int>(cap_genomes * cap_slots);
    d_fold = work->alloc<unsigned long long>(cap_genomes * E);
    d_nonconv = work->alloc<int>(cap_genomes);
    d_flo = work->alloc<double>(cap_genomes);
    d_fcrit = work->alloc<int>(cap_genomes);
    d_case_g = work->alloc<int>(cap_cases);
    d_case_k = work->alloc<int>(cap_cases);
    d_foldcase = work->alloc<uint8_t>(cap_cases);
    d_conv = work->alloc<uint8_t>(cap_cases);
    d_iters = work->alloc<int>(cap_cases);
    d_crit = work->alloc<int>(cap_cases);
    d_energy = work->alloc<double>(cap_cases);
    d_loading = work->alloc<double>(std::max<size_t>(cap_rows, 1));
    d_scratch = cap_scratch ? work->alloc<unsigned char>(cap_scratch) : nullptr;
    d_next_case = work->alloc<unsigned>(1);
  }
  // inputs and per-case outputs through one pinned staging block (pageable
  // copies would each be staged by the driver synchronously)
  const size_t gbytes = sizeof(int32_t) * n_genomes * (n_a + n_d), cbytes = sizeof(int32_t) * nc;
  auto up16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  const size_t o_g = 0, o_cg = up16(gbytes), o_ck = o_cg + up16(cbytes), o_fc = o_ck + up16(cbytes);
  const size_t o_conv = o_fc + up16(nc), o_iters = o_conv + up16(nc), o_crit = o_iters + up16(cbytes);
  const size_t o_energy = o_crit + up16(cbytes), o_nonconv = o_energy + up16(sizeof(double) * nc);
  const size_t o_fcrit = o_nonconv + up16(sizeof(int) * n_genomes), o_flo = o_fcrit + up16(sizeof(int) * n_genomes);
  const size_t stage_bytes = o_flo + up16(sizeof(double) * n_genomes);
  if (stage_bytes > h_stage_cap) {
    check(cudaStreamSynchronize(stream), "AC sync");
    if (h_stage) cudaFreeHost(h_stage);
    h_stage = nullptr;
    h_stage_cap = std::max(stage_bytes, 2 * h_stage_cap);
    check(cudaMallocHost(reinterpret_cast<void**>(&h_stage), h_stage_cap), "cudaMallocHost");
  }
  if (n_genomes) std::memcpy(h_stage + o_g, genomes, gbytes);
  std::memcpy(h_stage + o_cg, cg.data(), cbytes);
  std::memcpy(h_stage + o_ck, ck.data(), cbytes);
  uint8_t* fc = h_stage + o_fc;
  for (int c = 0; c < nc; ++c) fc[c] = fold && ck[c] >= 0;
  if (n_genomes)
    check(cudaMemcpyAsync(d_genomes, h_stage + o_g, gbytes, cudaMemcpyHostToDevice, stream), "AC genomes H2D");
  check(cudaMemcpyAsync(d_case_g, h_stage + o_cg, cbytes, cudaMemcpyHostToDevice, stream), "AC cases");
  check(cudaMemcpyAsync(d_case_k, h_stage + o_ck, cbytes, cudaMemcpyHostToDevice, stream), "AC cases");
  check(cudaMemcpyAsync(d_foldcase, fc, nc, cudaMemcpyHostToDevice, stream), "AC cases");
  if (fold) {
    check(cudaMemsetAsync(d_fold, 0, sizeof(unsigned long long) * n_genomes * E, stream), "AC fold reset");
    check(cudaMemsetAsync(d_nonconv, 0, sizeof(int) * n_genomes, stream), "AC fold reset");
  }
  tgb::AcTopo tp{t_from, t_to, t_rem, t_inode, t_nnew, t_split, std::max(n_a, 1)};
  tgb::ac_launch_topo(g, d_genomes, n_genomes, n_a, n_d, tp, stream);
  tgb::AcCases io{};
  io.genome = d_case_g;
  io.cont = d_case_k;
  io.n = nc;
  io.converged = d_conv;
  io.iterations = d_iters;
  io.energy = d_energy;
  io.critical = d_crit;
  io.loading = loading ? d_loading : nullptr;
  io.vm_stride = N + n_a;
  io.vm = vm ? d_loading + rows : nullptr;
  io.va = vm ? d_loading + rows + vrows : nullptr;
  io.fold_case = d_foldcase;
  io.fold = fold ? d_fold : nullptr;
  io.nonconverged = fold ? d_nonconv : nullptr;
  tgb::AcSolver sv = sv0;
  sv.scratch = d_scratch;
  sv.next_case = sv.in_smem ? nullptr : d_next_case;
  if (!sv.in_smem) check(cudaMemsetAsync(d_next_case, 0, sizeof(unsigned), stream), "AC case counter");
  tgb::ac_launch_cases(g, tp, io, sv, slots, stream);
  launches += 2;
  if (fold) {
    tgb::ac_launch_fold_finish(g, d_fold, n_genomes, d_flo, d_fcrit, stream);
    ++launches;
  }
  check(cudaGetLastError(), "AC launch");
  Result r;
  check(cudaMemcpyAsync(h_stage + o_conv, d_conv, nc, cudaMemcpyDeviceToHost, stream), "AC D2H");
  check(cudaMemcpyAsync(h_stage + o_iters, d_iters, cbytes, cudaMemcpyDeviceToHost, stream), "AC D2H");
  check(cudaMemcpyAsync(h_stage + o_crit, d_crit, cbytes, cudaMemcpyDeviceToHost, stream), "AC D2H");
  check(cudaMemcpyAsync(h_stage + o_energy, d_energy, sizeof(double) * nc, cudaMemcpyDeviceToHost, stream), "AC D2H");
  if (loading)
    check(cudaMemcpyAsync(loading, d_loading, sizeof(double) * rows, cudaMemcpyDeviceToHost, stream), "AC D2H");
  if (vm) {
    check(cudaMemcpyAsync(vm, d_loading + rows, sizeof(double) * vrows, cudaMemcpyDeviceToHost, stream), "AC D2H");
    check(cudaMemcpyAsync(va, d_loading + rows + vrows, sizeof(double) * vrows, cudaMemcpyDeviceToHost, stream), "AC D2H");
  }
  if (fold) {
    check(cudaMemcpyAsync(h_stage + o_nonconv, d_nonconv, sizeof(int) * n_genomes, cudaMemcpyDeviceToHost, stream),
          "AC D2H");
    check(cudaMemcpyAsync(h_stage + o_fcrit, d_fcrit, sizeof(int) * n_genomes, cudaMemcpyDeviceToHost, stream), "AC D2H");
    check(cudaMemcpyAsync(h_stage + o_flo, d_flo, sizeof(double) * n_genomes, cudaMemcpyDeviceToHost, stream), "AC D2H");
  }
  check(cudaStreamSynchronize(stream), "AC cases");
  auto take = [&](auto& v, size_t off, size_t count) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    v.resize(count);
    std::memcpy(v.data(), h_stage + off, sizeof(T) * count);
  };
  take(r.conv, o_conv, nc);
  take(r.iters, o_iters, nc);
  take(r.crit, o_crit, nc);
  take(r.energy, o_energy, nc);
  if (fold) {
    take(r.nonconv, o_nonconv, n_genomes);
    take(r.fold_crit, o_fcrit, n_genomes);
    take(r.fold_lambda_o, o_flo, n_genomes);
  }
  return r;
}

extern "C" {

tg_status tg_ac_context_create(const tg_grid* grid, const tg_actionset* actions, tg_context* dc,
                               const tg_ac_config* cfg, int device, tg_ac_context** out) {
  return guarded([&] {
    if (!grid || !actions || !out) throw tgb::ConfigError("null argument");
    *out = nullptr;
    std::unique_ptr<tg_ac_context> ctx(new tg_ac_context);
    ctx->device = device;
    ctx->cfg = cfg ? *cfg : tg_ac_config{1e-6, 30, 2, 0.05, 1, 0.01, 0.05};
    if (ctx->cfg.max_iterations < 1 || !(ctx->cfg.tolerance_pu > 0.0)) throw tgb::ConfigError("bad AcConfig");
    check(cudaSetDevice(device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    const tgb::Grid& G = grid->g;
    ctx->N = G.n_nodes();
    ctx->E = G.n_branches();
    ctx->I = G.n_injections();
    ctx->K = static_cast<int>(G.cont_id.size());
    ctx->A = actions->t.n_actions();
    ctx->D = static_cast<int>(actions->t.disconnectables.size());
    cudaStream_t s = ctx->stream;
    DeviceArena& ar = ctx->arena;
    tgb::AcGrid& g = ctx->g;
    g.N = ctx->N, g.E = ctx->E, g.I = ctx->I, g.K = ctx->K, g.slack = G.slack;
    g.br_from = ar.upload(grid->br_from, s);
    g.br_to = ar.upload(grid->br_to, s);
    g.br_on = ar.upload(grid->br_on, s);
    g.br_lim = ar.upload(grid->br_lim, s);
    g.br_r = ar.upload(G.br_r, s);
    g.br_x = ar.upload(G.br_x, s);
    g.br_bc = ar.upload(G.br_bc, s);
    g.br_tap = ar.upload(G.br_tap, s);
    g.node_shunt = ar.upload(G.node_shunt, s);
    {
      // CSR of every branch at both of its ends, grid order (the sparse Ybus of k_ac_case)
      std::vector<int32_t> ptr(ctx->N + 1, 0), br;
      for (int e = 0; e < ctx->E; ++e) ++ptr[G.br_from[e] + 1], ++ptr[G.br_to[e] + 1];
      for (int v = 0; v < ctx->N; ++v) ptr[v + 1] += ptr[v];
      br.assign(ptr.back(), 0);
      std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
      for (int e = 0; e < ctx->E; ++e) br[fill[G.br_from[e]]++] = e, br[fill[G.br_to[e]]++] = e;
      g.node_ptr = ar.upload(ptr, s);
      g.node_br = ar.upload(br, s);
    }
    g.st_node = ar.upload(grid->sub_node, s);
    g.inj_node = ar.upload(grid->inj_node, s);
    g.inj_p = ar.upload(G.inj_p, s);
    g.inj_q = ar.upload(G.inj_q, s);
    g.inj_vset = ar.upload(G.inj_vset, s);
    std::vector<uint8_t> gen(G.inj_gen.begin(), G.inj_gen.end()), hv(G.inj_has_vset.begin(), G.inj_has_vset.end());
    g.inj_gen = ar.upload(gen, s);
    g.inj_has_vset = ar.upload(hv, s);
    g.cont_br_ptr = ar.upload(grid->cont_bptr, s);
    g.cont_br = ar.upload(grid->cont_b, s);
    g.cont_inj_ptr = ar.upload(grid->cont_iptr, s);
    g.cont_inj = ar.upload(grid->cont_i, s);
    g.st_term_ptr = ar.upload(grid->sub_tptr, s);
    g.term_kind = ar.upload(grid->tkind, s);
    g.term_elem = ar.upload(grid->telem, s);
    g.act_station = ar.upload(actions->station, s);
    g.act_group_ptr = ar.upload(actions->gptr, s);
    g.act_group = ar.upload(actions->group, s);
    g.disc = ar.upload(actions->disc, s);
    // pre-optimization DC fitness (ac_validator.cpp:315), from the DC context
    if (dc) {
      ctx->pre_fitness = dc->pre.size() > 4 ? dc->pre[4] : 0.0;
    }
    // baseline: the unchanged grid's base case and every contingency
    const int K = ctx->K;
    std::vector<int32_t> cg(K + 1, 0), ck(K + 1);
    for (int k = 0; k <= K; ++k) ck[k] = k - 1;
    const tg_ac_context::Result r = ctx->run(nullptr, 1, 0, 0, cg, ck, true, nullptr, nullptr, nullptr);
    ctx->base_converged = r.conv[0];
    ctx->base_energy = r.conv[0] ? r.energy[0] : 0.0;
    ctx->case_conv.assign(r.conv.begin() + 1, r.conv.end());
    ctx->case_energy.assign(K, 0.0);
    for (int k = 0; k < K; ++k)
      if (ctx->case_conv[k]) ctx->case_energy[k] = r.energy[k + 1];
    ctx->base_lambda_o = r.fold_lambda_o[0];
    ctx->base_critical = r.fold_crit[0];
    *out = ctx.release();
  });
}

void tg_ac_context_destroy(tg_ac_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->work.reset();
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

tg_status tg_ac_baseline_get(tg_ac_context* ctx, tg_ac_baseline* out, uint8_t* case_converged, double* case_energy) {
  return guarded([&] {
    if (!ctx || !out) throw tgb::ConfigError("null argument");
    out->lambda_o = ctx->base_lambda_o;
    out->critical_count = ctx->base_critical;
    out->base_converged = ctx->base_converged;
    out->base_energy = ctx->base_energy;
    out->pre_fitness = ctx->pre_fitness;
    if (case_converged) std::copy(ctx->case_conv.begin(), ctx->case_conv.end(), case_converged);
    if (case_energy) std::copy(ctx->case_energy.begin(), ctx->case_energy.end(), case_energy);
  });
}

tg_status tg_ac_run_cases(tg_ac_context* ctx, const int32_t* genomes, int32_t n_genomes, int32_t n_a, int32_t n_d,
                          const int32_t* case_genome, const int32_t* case_contingency, int32_t n_cases,
                          tg_ac_case_out* out) {
  return guarded([&] {
    if (!ctx || !out || n_cases < 0 || n_genomes < 0 || (n_genomes && !genomes) ||
        (n_cases && (!case_genome || !case_contingency)))
      throw tgb::ConfigError("bad argument");
    if (n_cases == 0) return;
    std::vector<int32_t> cg(case_genome, case_genome + n_cases), ck(case_contingency, case_contingency + n_cases);
    if ((out->vm_pu == nullptr) != (out->va_rad == nullptr)) throw tgb::ConfigError("vm_pu and va_rad go together");
    const tg_ac_context::Result r =
        ctx->run(genomes, n_genomes, n_a, n_d, cg, ck, false, out->loading_mva, out->vm_pu, out->va_rad);
    if (out->converged) std::copy(r.conv.begin(), r.conv.end(), out->converged);
    if (out->iterations) std::copy(r.iters.begin(), r.iters.end(), out->iterations);
    if (out->overload_energy) std::copy(r.energy.begin(), r.energy.end(), out->overload_energy);
    if (out->critical_count) std::copy(r.crit.begin(), r.crit.end(), out->critical_count);
  });
}

tg_status tg_ac_worst_k_check(tg_ac_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                              const int32_t* worst_idx, const int32_t* worst_n, int32_t worst_stride, int32_t* reason) {
  return guarded([&] {
    if (!ctx || n < 0 || (n && (!genomes || !worst_idx || !worst_n || !reason)) || worst_stride < 0)
      throw tgb::ConfigError("bad argument");
    if (n == 0) return;
    // cases: per genome the base case, then its worst contingencies in list order
    std::vector<int32_t> cg, ck, first(n);
    for (int i = 0; i < n; ++i) {
      if (worst_n[i] < 0 || worst_n[i] > worst_stride) throw tgb::ValidationError("bad worst list length");
      first[i] = static_cast<int32_t>(cg.size());
      cg.push_back(i), ck.push_back(-1);
      for (int j = 0; j < worst_n[i]; ++j) cg.push_back(i), ck.push_back(worst_idx[static_cast<size_t>(i) * worst_stride + j]);
    }
    const tg_ac_context::Result r = ctx->run(genomes, n, n_a, n_d, cg, ck, false, nullptr, nullptr, nullptr);
    // ac_validator.cpp:399-425, summed in list order
    for (int i = 0; i < n; ++i) {
      const int b = first[i];
      if (!r.conv[b]) {
        reason[i] = TG_AC_NONCONVERGENCE;
        continue;
      }
      if (worst_n[i] == 0) {
        reason[i] = TG_AC_NONE;
        continue;
      }
      double mine = r.energy[b], ref = ctx->base_energy;
      int failed = 0;
      int verdict = -1;
      for (int j = 0; j < worst_n[i]; ++j) {
        const int k = ck[b + 1 + j];
        if (!r.conv[b + 1 + j]) {
          if (++failed > ctx->cfg.worst_k_nonconverged) {
            verdict = TG_AC_NONCONVERGENCE;
            break;
          }
          continue;
        }
        if (!ctx->case_conv[k]) continue;
        mine += r.energy[b + 1 + j];
        ref += ctx->case_energy[k];
      }
      if (verdict < 0) verdict = (ctx->base_converged && mine >= ref) ? TG_AC_OVERLOAD_NOT_IMPROVED : TG_AC_NONE;
      reason[i] = verdict;
    }
  });
}

tg_status tg_ac_full_validation(tg_ac_context* ctx, const int32_t* genomes, int32_t n, int32_t n_a, int32_t n_d,
                                int32_t* reason, uint8_t* accepted, double* ac_lambda_o) {
  return guarded([&] {
    if (!ctx || n < 0 || (n && (!genomes || !reason))) throw tgb::ConfigError("bad argument");
    if (n == 0) return;
    const int K = ctx->K;
    std::vector<int32_t> cg, ck;
    cg.reserve(static_cast<size_t>(n) * (K + 1));
    ck.reserve(cg.capacity());
    for (int i = 0; i < n; ++i)
      for (int k = -1; k < K; ++k) cg.push_back(i), ck.push_back(k);
    const tg_ac_context::Result r = ctx->run(genomes, n, n_a, n_d, cg, ck, true, nullptr, nullptr, nullptr);
    // ac_validator.cpp:445-472
    for (int i = 0; i < n; ++i) {
      const bool base_ok = r.conv[static_cast<size_t>(i) * (K + 1)];
      int why = TG_AC_NONE;
      double lo = 0.0;
      if (!base_ok || r.nonconv[i] > ctx->cfg.nonconverged_fraction * K) {
        why = TG_AC_NONCONVERGENCE;
      } else {
        lo = r.fold_lambda_o[i];
        if (!(lo < ctx->base_lambda_o))
          why = TG_AC_OVERLOAD_NOT_IMPROVED;
        else if (r.fold_crit[i] > ctx->base_critical)
          why = TG_AC_CRITICAL_COUNT_INCREASED;
      }
      reason[i] = why;
      if (accepted) accepted[i] = why == TG_AC_NONE;
      if (ac_lambda_o) ac_lambda_o[i] = lo;
    }
  });
}

int64_t tg_ac_kernel_launches(tg_ac_context* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
