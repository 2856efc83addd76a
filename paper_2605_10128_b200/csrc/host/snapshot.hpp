// Host side of the snapshot hand-off:
//   HostSnapshot    make_snapshot (qd_optimizer.cpp:331-342) decoded from a
//                   device archive blob (tgb::BlobLayout) copied to pinned memory;
//   SnapshotChannel the reference's single-producer single-consumer queue
//                   (channel.hpp:15-79): a bounded channel never blocks the
//                   producer, when full the oldest non-final snapshot is dropped;
//                   capacity 0 = unbounded.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <memory>
#include <mutex>
#include <vector>

#include "../../../include/topopt_b200.h"

namespace tgb {

// One RepertoireSnapshot (qd_optimizer.hpp:83-95) owning its arrays; `view`
// points into them.
struct HostSnapshot {
  std::vector<int32_t> cell, genome, lc, lc0, ld, ls, lr, widx, wn;
  std::vector<double> fit, lo, lb, wval;
  tg_snapshot_view view{};

  void bind(int n_slots, int worst_k) {
    view.n_entries = static_cast<int32_t>(cell.size());
    view.n_slots = n_slots;
    view.worst_k = worst_k;
    view.cell = cell.data();
    view.genome = genome.data();
    view.fitness = fit.data();
    view.lambda_o = lo.data();
    view.lambda_c = lc.data();
    view.lambda_c0 = lc0.data();
    view.lambda_b = lb.data();
    view.lambda_d = ld.data();
    view.lambda_s = ls.data();
    view.lambda_r = lr.data();
    view.worst_idx = widx.data();
    view.worst_energy = wval.data();
    view.worst_n = wn.data();
  }

  // Entries in (cell, position) order, best = max over cells of the first
  // entry's fitness (Repertoire::best_fitness, qd_optimizer.cpp:317-322).
  // Blob sections as tgb::BlobLayout (cuda/qd.cuh); empty slots carry -inf.
  void from_blob(const uint8_t* blob, int cells, int cap, int ns, int wk, int epoch, int64_t evaluations,
                 bool final_snapshot) {
    const size_t S = static_cast<size_t>(cells) * cap;
    auto al = [](size_t x) { return (x + 7) & ~size_t{7}; };
    size_t o = 0;
    const double* b_fit = reinterpret_cast<const double*>(blob + o); o += al(S * 8);
    const double* b_lo = reinterpret_cast<const double*>(blob + o); o += al(S * 8);
    const double* b_lb = reinterpret_cast<const double*>(blob + o); o += al(S * 8);
    const double* b_wv = reinterpret_cast<const double*>(blob + o); o += al(S * wk * 8);
    const int32_t* b_gen = reinterpret_cast<const int32_t*>(blob + o); o += al(S * ns * 4);
    const int32_t* b_lc = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_lc0 = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_ld = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_ls = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_lr = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_wn = reinterpret_cast<const int32_t*>(blob + o); o += al(S * 4);
    const int32_t* b_wi = reinterpret_cast<const int32_t*>(blob + o);
    for (auto* v : {&cell, &genome, &lc, &lc0, &ld, &ls, &lr, &widx, &wn}) v->clear();
    for (auto* v : {&fit, &lo, &lb, &wval}) v->clear();
    double best = -std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < S; ++i) {
      const double f = b_fit[i];
      if (!(f > -std::numeric_limits<double>::infinity()) || f != f) continue;  // empty slot
      cell.push_back(static_cast<int32_t>(i / cap));
      genome.insert(genome.end(), b_gen + i * ns, b_gen + (i + 1) * ns);
      fit.push_back(f);
      lo.push_back(b_lo[i]);
      lb.push_back(b_lb[i]);
      lc.push_back(b_lc[i]);
      lc0.push_back(b_lc0[i]);
      ld.push_back(b_ld[i]);
      ls.push_back(b_ls[i]);
      lr.push_back(b_lr[i]);
      wn.push_back(b_wn[i]);
      widx.insert(widx.end(), b_wi + i * wk, b_wi + (i + 1) * wk);
      wval.insert(wval.end(), b_wv + i * wk, b_wv + (i + 1) * wk);
      if (i % cap == 0 && f > best) best = f;
    }
    view.epoch = epoch;
    view.evaluations = evaluations;
    view.best_fitness = best;
    view.final_snapshot = final_snapshot ? 1 : 0;
    bind(ns, wk);
  }

  // Deep copy of a caller's view (the channel stores its own snapshots).
  void from_view(const tg_snapshot_view& v) {
    const size_t n = static_cast<size_t>(std::max(v.n_entries, 0));
    const size_t ns = static_cast<size_t>(std::max(v.n_slots, 0)), wk = static_cast<size_t>(std::max(v.worst_k, 0));
    auto cp = [](auto& dst, const auto* src, size_t m) { dst.assign(src, src + (src ? m : 0)); };
    cp(cell, v.cell, n);
    cp(genome, v.genome, n * ns);
    cp(fit, v.fitness, n);
    cp(lo, v.lambda_o, n);
    cp(lc, v.lambda_c, n);
    cp(lc0, v.lambda_c0, n);
    cp(lb, v.lambda_b, n);
    cp(ld, v.lambda_d, n);
    cp(ls, v.lambda_s, n);
    cp(lr, v.lambda_r, n);
    cp(widx, v.worst_idx, n * wk);
    cp(wval, v.worst_energy, n * wk);
    cp(wn, v.worst_n, n);
    view = v;
    bind(static_cast<int>(ns), static_cast<int>(wk));
  }
};

// channel.hpp:15-79
class SnapshotChannel {
 public:
  explicit SnapshotChannel(size_t capacity) : capacity_(capacity) {}

  void push(std::unique_ptr<HostSnapshot> s) {
    {
      std::lock_guard<std::mutex> lock(mutex_);
      if (capacity_ > 0 && items_.size() >= capacity_) {
        for (auto it = items_.begin(); it != items_.end(); ++it)
          if (!(*it)->view.final_snapshot) {
            items_.erase(it);
            ++dropped_;
            break;
          }
      }
      items_.push_back(std::move(s));
    }
    ready_.notify_one();
  }
  void close() {
    {
      std::lock_guard<std::mutex> lock(mutex_);
      closed_ = true;
    }
    ready_.notify_all();
  }
  // blocking: waits until a snapshot arrives or the channel is closed and drained
  std::unique_ptr<HostSnapshot> pop(bool blocking) {
    std::unique_lock<std::mutex> lock(mutex_);
    if (blocking) ready_.wait(lock, [&] { return !items_.empty() || closed_; });
    if (items_.empty()) return nullptr;
    auto s = std::move(items_.front());
    items_.pop_front();
    return s;
  }
  size_t pending() const {
    std::lock_guard<std::mutex> lock(mutex_);
    return items_.size();
  }
  size_t dropped() const {
    std::lock_guard<std::mutex> lock(mutex_);
    return dropped_;
  }

 private:
  mutable std::mutex mutex_;
  std::condition_variable ready_;
  std::deque<std::unique_ptr<HostSnapshot>> items_;
  size_t capacity_;
  size_t dropped_ = 0;
  bool closed_ = false;
};

}  // namespace tgb
