// MapElites on the device (qd_optimizer.cpp:12-417).
//
// Offspring lanes replay the reference's RNG stream bit for bit: each lane
// seeds its own std::mt19937_64 (derive_seed(seed, iter, lane+1),
// qd_optimizer.cpp:382) and draws through restatements of the libstdc++-13
// distributions the reference calls (uniform_int_distribution's Lemire
// downscale, generate_canonical<double,53>, the mean<12 Poisson method). The
// engine state is generated lazily in place, so a lane only pays for the draws
// it makes. The archive insert replays the sequential per-lane insert order
// exactly with one warp per descriptor cell.
#include "qd.cuh"

namespace tgb {

namespace {

// ---------------------------------------------------------------- RNG (rng.hpp:9-21)
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ unsigned long long derive_seed(unsigned long long m, unsigned long long a,
                                                          unsigned long long b) {
  return mix64(mix64(m ^ mix64(a)) ^ mix64(b + 0x632be59bd9b4e019ull));
}

// std::mt19937_64 with the twist computed lazily, one word per draw, in place.
struct Mt64 {
  static constexpr int kN = 312, kM = 156;
  unsigned long long mt[kN];
  int i;
  __device__ void seed(unsigned long long s) {
    mt[0] = s;
    for (int k = 1; k < kN; ++k) mt[k] = 6364136223846793005ull * (mt[k - 1] ^ (mt[k - 1] >> 62)) + k;
    i = 0;
  }
  __device__ unsigned long long next() {
    const int k = i;
    const unsigned long long x = (mt[k] & 0xFFFFFFFF80000000ull) | (mt[k + 1 < kN ? k + 1 : 0] & 0x7FFFFFFFull);
    unsigned long long y = mt[k + kM < kN ? k + kM : k + kM - kN] ^ (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
    mt[k] = y;
    i = k + 1 < kN ? k + 1 : 0;
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
  }
};

// The same engine with its 312-word state in shared memory (k_offspring: the
// per-lane state in local memory spilled to L2, and every lazily twisted draw
// waited on it)
struct Mt64S {
  static constexpr int kN = Mt64::kN, kM = Mt64::kM;
  unsigned long long* mt;
  int i;
  __device__ void bind(unsigned long long* state) { mt = state; }
  __device__ void seed(unsigned long long s) {
    unsigned long long x = s;
    mt[0] = x;
    for (int k = 1; k < kN; ++k) {
      x = 6364136223846793005ull * (x ^ (x >> 62)) + k;
      mt[k] = x;
    }
    i = 0;
  }
  __device__ unsigned long long next() {
    const int k = i;
    const unsigned long long x = (mt[k] & 0xFFFFFFFF80000000ull) | (mt[k + 1 < kN ? k + 1 : 0] & 0x7FFFFFFFull);
    unsigned long long y = mt[k + kM < kN ? k + kM : k + kM - kN] ^ (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
    mt[k] = y;
    i = k + 1 < kN ? k + 1 : 0;
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
  }
};

// Philox4x32-10 (Salmon et al., SC'11): counter-based, stateless per draw; the
// lane key is the same derive_seed(seed, iter, lane + 1) the replay mode seeds
// mt19937_64 with, the counter is the draw index. Two 64-bit draws per block.
struct Philox {
  uint32_t k0, k1;
  uint32_t ctr = 0;
  unsigned long long buf = 0;
  bool have = false;
  __device__ void bind(unsigned long long*) {}
  __device__ void seed(unsigned long long s) {
    k0 = static_cast<uint32_t>(s);
    k1 = static_cast<uint32_t>(s >> 32);
    ctr = 0;
    have = false;
  }
  __device__ unsigned long long next() {
    if (have) {
      have = false;
      return buf;
    }
    uint32_t c0 = ctr++, c1 = 0x7f4a7c15u, c2 = 0, c3 = 0, a = k0, b = k1;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
      c0 = hi1 ^ c1 ^ a;
      c1 = lo1;
      c2 = hi0 ^ c3 ^ b;
      c3 = lo0;
      a += 0x9E3779B9u;
      b += 0xBB67AE85u;
    }
    buf = (static_cast<unsigned long long>(c3) << 32) | c2;
    have = true;
    return (static_cast<unsigned long long>(c1) << 32) | c0;
  }
};

// uniform_int_distribution<int>(a, b) over a 64-bit engine (uniform_int_dist.h:257-320)
template <class Rng>
__device__ int uniform_int(Rng& r, int a, int b) {
  const unsigned long long urange =
      static_cast<unsigned long long>(static_cast<long long>(b)) - static_cast<unsigned long long>(static_cast<long long>(a));
  const unsigned long long range = urange + 1ull;
  unsigned long long x = r.next();
  unsigned long long low = x * range;
  unsigned long long high = __umul64hi(x, range);
  if (low < range) {
    const unsigned long long threshold = (0ull - range) % range;
    while (low < threshold) {
      x = r.next();
      low = x * range;
      high = __umul64hi(x, range);
    }
  }
  return static_cast<int>(high + static_cast<unsigned long long>(static_cast<long long>(a)));
}

// generate_canonical<double, 53> (random.tcc:3349-3381): one 64-bit draw / 2^64
template <class Rng>
__device__ __forceinline__ double canonical(Rng& r) {
  double v = __dmul_rn(__ull2double_rn(r.next()), 0x1p-64);
  if (v >= 1.0) v = 1.0 - 0x1p-53;
  return v;
}

// uniform_real_distribution<double>(a, b): (u * (b - a)) + a, no contraction (random.h:1909)
template <class Rng>
__device__ __forceinline__ double uniform_real(Rng& r, double a, double b) {
  return __dadd_rn(__dmul_rn(canonical(r), __dsub_rn(b, a)), a);
}

// poisson_distribution<int>, mean < 12 branch (random.tcc:1401-1411)
template <class Rng>
__device__ int poisson(Rng& r, double thr) {
  int x = 0;
  double prod = 1.0;
  do {
    prod = __dmul_rn(prod, canonical(r));
    x += 1;
  } while (prod > thr);
  return x - 1;
}

// ---------------------------------------------------------------- operators
struct Ops {
  const DevGrid& g;
  const QdParams& p;
  __device__ int station(int a) const { return g.act_station[a]; }
  __device__ int lo(int a) const { return g.st_range_lo[station(a)]; }
  __device__ int hi(int a) const { return g.st_range_hi[station(a)]; }
};

// choose_feasible_op, qd_optimizer.cpp:100-113
template <class Rng>
__device__ int choose_op(const double* w, const bool* ok, Rng& r) {
  double total = 0.0;
  for (int i = 0; i < 4; ++i)
    if (ok[i]) total = __dadd_rn(total, w[i]);
  if (total <= 0.0) return 3;
  double draw = uniform_real(r, 0.0, total);
  for (int i = 0; i < 4; ++i) {
    if (!ok[i]) continue;
    if (draw < w[i]) return i;
    draw = __dsub_rn(draw, w[i]);
  }
  return 3;
}

__device__ void sort_small(int* v, int n) {
  for (int i = 1; i < n; ++i) {
    int x = v[i], j = i - 1;
    while (j >= 0 && v[j] > x) v[j + 1] = v[j], --j;
    v[j + 1] = x;
  }
}

// qd_optimizer.cpp:115-155
template <class Rng>
__device__ void mutate_actions_once(const Ops& o, int* g, Rng& r, int* trace) {
  const int na = o.p.n_a;
  // AddActionPool: excluded station ranges, sorted as pairs
  int elo[kMaxSplits], ehi[kMaxSplits], nex = 0, excluded = 0;
  for (int k = 0; k < na; ++k) {
    const int a = g[k];
    if (a < 0) continue;
    elo[nex] = o.lo(a);
    ehi[nex] = o.hi(a);
    excluded += ehi[nex] - elo[nex];
    ++nex;
  }
  for (int i = 1; i < nex; ++i) {
    const int xl = elo[i], xh = ehi[i];
    int j = i - 1;
    while (j >= 0 && (elo[j] > xl || (elo[j] == xl && ehi[j] > xh))) elo[j + 1] = elo[j], ehi[j + 1] = ehi[j], --j;
    elo[j + 1] = xl;
    ehi[j + 1] = xh;
  }
  const int add_size = o.p.n_actions - excluded;
  int empties[kMaxSplits], filled[kMaxSplits], ne = 0, nf = 0;
  for (int k = 0; k < na; ++k) (g[k] < 0 ? empties[ne++] : filled[nf++]) = k;
  // change pool: per filled slot (slot order), its station range minus the current set
  int cur[kMaxSplits], ncur = 0;
  for (int k = 0; k < na; ++k) {
    bool dup = false;
    for (int q = 0; q < ncur; ++q) dup = dup || cur[q] == g[k];
    if (!dup) cur[ncur++] = g[k];
  }
  sort_small(cur, ncur);
  int change_size = 0;
  for (int k = 0; k < na; ++k) {
    const int a = g[k];
    if (a < 0) continue;
    int in = 0;
    for (int q = 0; q < ncur; ++q) in += cur[q] >= o.lo(a) && cur[q] < o.hi(a);
    change_size += o.hi(a) - o.lo(a) - in;
  }
  const bool ok[4] = {ne > 0 && add_size > 0, nf > 0, change_size > 0, true};
  const int op = choose_op(o.p.p_action, ok, r);
  if (trace) *trace = op;
  if (op == 0) {
    const int slot = empties[uniform_int(r, 0, ne - 1)];
    int rank = uniform_int(r, 0, add_size - 1);
    int cursor = 0, pick = -1;
    for (int i = 0; i < nex && pick < 0; ++i) {
      const int gap = elo[i] - cursor;
      if (rank < gap) pick = cursor + rank;
      else rank -= gap, cursor = ehi[i];
    }
    g[slot] = pick >= 0 ? pick : cursor + rank;
  } else if (op == 1) {
    g[filled[uniform_int(r, 0, nf - 1)]] = -1;
  } else if (op == 2) {
    int idx = uniform_int(r, 0, change_size - 1), pick = -1;
    for (int k = 0; k < na && pick < 0; ++k) {
      const int a = g[k];
      if (a < 0) continue;
      const int lo = o.lo(a), hi = o.hi(a);
      int in = 0;
      for (int q = 0; q < ncur; ++q) in += cur[q] >= lo && cur[q] < hi;
      const int cnt = hi - lo - in;
      if (idx < cnt) {
        int cand = lo + idx;
        for (int q = 0; q < ncur; ++q)
          if (cur[q] >= lo && cur[q] < hi && cur[q] <= cand) ++cand;
        pick = cand;
      } else {
        idx -= cnt;
      }
    }
    const int st = o.station(pick);
    for (int k = 0; k < na; ++k)
      if (g[k] >= 0 && o.station(g[k]) == st) {
        g[k] = pick;
        break;
      }
  }
}

// qd_optimizer.cpp:157-198
template <class Rng>
__device__ void mutate_disconnections_once(const Ops& o, int* g, Rng& r, int* trace) {
  const int na = o.p.n_a, nd = o.p.n_d;
  int* d = g + na;
  int used[kMaxRemovedSweep], nu = 0;
  for (int k = 0; k < nd; ++k)
    if (d[k] >= 0) used[nu++] = d[k];
  sort_small(used, nu);
  const int pool = o.p.n_disc - nu;
  int empties[kMaxRemovedSweep], filled[kMaxRemovedSweep], ne = 0, nf = 0;
  for (int k = 0; k < nd; ++k) (d[k] < 0 ? empties[ne++] : filled[nf++]) = k;
  const bool ok[4] = {ne > 0 && pool > 0, nf > 0, nf > 0 && pool > 0, true};
  bool genome_empty = nf == 0;
  for (int k = 0; k < na; ++k) genome_empty = genome_empty && g[k] < 0;
  const int op = (genome_empty && ok[0]) ? 0 : choose_op(o.p.p_disc, ok, r);
  if (trace) *trace = 10 + op;
  auto pick_rank = [&](int rank) {
    for (int q = 0; q < nu; ++q)
      if (rank >= used[q]) ++rank;
    return rank;
  };
  if (op == 0) {
    const int slot = empties[uniform_int(r, 0, ne - 1)];
    d[slot] = pick_rank(uniform_int(r, 0, pool - 1));
  } else if (op == 1) {
    d[filled[uniform_int(r, 0, nf - 1)]] = -1;
  } else if (op == 2) {
    const int pick = pick_rank(uniform_int(r, 0, pool - 1));
    const int slot = filled[uniform_int(r, 0, nf - 1)];
    d[slot] = pick;
  }
}

// qd_optimizer.cpp:202-210
template <class Rng>
__device__ void mutate(const Ops& o, int* g, Rng& r, int* trace, int* n_trace) {
  int n = poisson(r, o.p.poisson_thr);
  const int hi = o.p.n_a > 1 ? o.p.n_a : 1;
  n = n < 1 ? 1 : (n > hi ? hi : n);
  int t = 0;
  for (int k = 0; k < n; ++k) mutate_actions_once(o, g, r, trace ? trace + t++ : nullptr);
  mutate_disconnections_once(o, g, r, trace ? trace + t++ : nullptr);
  if (n_trace) *n_trace = t;
}

// qd_optimizer.cpp:217-231
template <class Rng>
__device__ int union_draw(const int* p1, int n1, const int* p2, int n2, double pc1, Rng& r) {
  const double w1 = n1 == 0 ? 0.0 : pc1;
  const double w2 = n2 == 0 ? 0.0 : __dsub_rn(1.0, pc1);
  if (__dadd_rn(w1, w2) <= 0.0) return -1;
  bool first;
  if (w1 == 0.0)
    first = false;
  else if (w2 == 0.0)
    first = true;
  else
    first = uniform_real(r, 0.0, __dadd_rn(w1, w2)) < w1;
  return first ? p1[uniform_int(r, 0, n1 - 1)] : p2[uniform_int(r, 0, n2 - 1)];
}

__device__ bool contains(const int* v, int n, int x) {
  for (int i = 0; i < n; ++i)
    if (v[i] == x) return true;
  return false;
}

// qd_optimizer.cpp:235-277
template <class Rng>
__device__ void crossover(const Ops& o, const int* g1, const int* g2, int* child, Rng& r) {
  const int na = o.p.n_a, nd = o.p.n_d;
  for (int k = 0; k < na + nd; ++k) child[k] = -1;
  int a1[kMaxSplits], a2[kMaxSplits], n1 = 0, n2 = 0;
  for (int k = 0; k < na; ++k) {
    if (g1[k] >= 0) a1[n1++] = g1[k];
    if (g2[k] >= 0) a2[n2++] = g2[k];
  }
  sort_small(a1, n1);
  sort_small(a2, n2);
  int used_st[kMaxSplits], placed[kMaxSplits], nus = 0, npl = 0;
  for (int i = 0; i < na; ++i) {
    int q1[kMaxSplits], q2[kMaxSplits], m1 = 0, m2 = 0;
    for (int k = 0; k < n1; ++k)
      if (!contains(placed, npl, a1[k]) && !contains(used_st, nus, o.station(a1[k]))) q1[m1++] = a1[k];
    for (int k = 0; k < n2; ++k)
      if (!contains(placed, npl, a2[k]) && !contains(used_st, nus, o.station(a2[k])) && !contains(a1, n1, a2[k]))
        q2[m2++] = a2[k];
    const int pick = union_draw(q1, m1, q2, m2, o.p.p_c1, r);
    if (pick < 0) break;
    child[i] = pick;
    placed[npl++] = pick;
    used_st[nus++] = o.station(pick);
  }
  int d1[kMaxRemovedSweep], d2[kMaxRemovedSweep], e1 = 0, e2 = 0;
  for (int k = 0; k < nd; ++k) {
    if (g1[na + k] >= 0) d1[e1++] = g1[na + k];
    if (g2[na + k] >= 0) d2[e2++] = g2[na + k];
  }
  sort_small(d1, e1);
  sort_small(d2, e2);
  int pd[kMaxRemovedSweep], npd = 0;
  for (int i = 0; i < nd; ++i) {
    int q1[kMaxRemovedSweep], q2[kMaxRemovedSweep], m1 = 0, m2 = 0;
    for (int k = 0; k < e1; ++k)
      if (!contains(pd, npd, d1[k])) q1[m1++] = d1[k];
    for (int k = 0; k < e2; ++k)
      if (!contains(pd, npd, d2[k]) && !contains(d1, e1, d2[k])) q2[m2++] = d2[k];
    const int pick = union_draw(q1, m1, q2, m2, o.p.p_c1, r);
    if (pick < 0) break;
    child[na + i] = pick;
    pd[npd++] = pick;
  }
}

// Repertoire::member (qd_optimizer.cpp:305-315): flat cell-major index -> (cell, pos)
__device__ const int* member(const Archive& a, const QdParams& p, int ns, int flat) {
  int lo = 0, hi = p.cells;  // last cell with flat_start <= flat
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a.flat_start[mid] <= flat) lo = mid;
    else hi = mid;
  }
  const int pos = flat - a.flat_start[lo];
  return a.genome + (static_cast<size_t>(lo) * p.cap + pos) * ns;
}

// Block = kOffspringLanes lane threads + one extra warp whose first thread draws
// the iteration's mutation/crossover split, so that draw's engine seeding runs
// beside the lanes' own seeding instead of before it.
constexpr int kOffspringLanes = 64;

template <class Rng, int L = kOffspringLanes>
__global__ void k_offspring(DevGrid g, QdParams p, Archive a, int* genomes) {
  __shared__ int b_mc;
  extern __shared__ unsigned long long rng_state[];  // Mt64S: (L + 1) x 312 words
  const long long it = a.iter[0];
  const int lane = blockIdx.x * L + static_cast<int>(threadIdx.x);
  const bool is_lane = threadIdx.x < L && lane < p.batch;
  Rng r;
  r.bind(rng_state + static_cast<size_t>(threadIdx.x < L ? threadIdx.x : L) * Mt64::kN);
  if (threadIdx.x == L) {
    Rng ir;
    ir.bind(rng_state + static_cast<size_t>(L) * Mt64::kN);
    ir.seed(derive_seed(p.seed, 0x17e7ull, static_cast<unsigned long long>(it)));
    b_mc = uniform_int(ir, 0, p.batch);
  } else if (is_lane) {
    r.seed(derive_seed(p.seed, static_cast<unsigned long long>(it), static_cast<unsigned long long>(lane) + 1ull));
  }
  __syncthreads();
  if (!is_lane) return;
  const int ns = p.n_a + p.n_d;
  Ops o{g, p};
  const int total = a.flat_start[p.cells];
  int child[kMaxSlots];
  if (lane < b_mc) {
    const int* par = member(a, p, ns, uniform_int(r, 0, total - 1));
    for (int k = 0; k < ns; ++k) child[k] = par[k];
    mutate(o, child, r, nullptr, nullptr);
  } else {
    const int* p1 = member(a, p, ns, uniform_int(r, 0, total - 1));
    const int* p2 = member(a, p, ns, uniform_int(r, 0, total - 1));
    crossover(o, p1, p2, child, r);
  }
  for (int k = 0; k < ns; ++k) genomes[static_cast<size_t>(lane) * ns + k] = child[k];
}

template <class Rng>
__global__ void k_mutate_lanes(DevGrid g, QdParams p, const int* parents, const unsigned long long* seeds, int n,
                               int* children) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= n) return;
  const int ns = p.n_a + p.n_d;
  Ops o{g, p};
  Rng r;
  r.seed(seeds[lane]);
  int child[kMaxSlots];
  for (int k = 0; k < ns; ++k) child[k] = parents[static_cast<size_t>(lane) * ns + k];
  mutate(o, child, r, nullptr, nullptr);
  for (int k = 0; k < ns; ++k) children[static_cast<size_t>(lane) * ns + k] = child[k];
}

template <class Rng>
__global__ void k_crossover_lanes(DevGrid g, QdParams p, const int* p1, const int* p2,
                                  const unsigned long long* seeds, int n, int* children) {
  const int lane = blockIdx.x * blockDim.x + threadIdx.x;
  if (lane >= n) return;
  const int ns = p.n_a + p.n_d;
  Ops o{g, p};
  Rng r;
  r.seed(seeds[lane]);
  int child[kMaxSlots];
  crossover(o, p1 + static_cast<size_t>(lane) * ns, p2 + static_cast<size_t>(lane) * ns, child, r);
  for (int k = 0; k < ns; ++k) children[static_cast<size_t>(lane) * ns + k] = child[k];
}

// ---------------------------------------------------------------- archive insert
__device__ void canonical_key(const int* g, int na, int nd, int* key) {
  int n = 0;
  for (int k = 0; k < na; ++k)
    if (g[k] >= 0) key[n++] = g[k];
  sort_small(key, n);
  for (int k = n; k < na; ++k) key[k] = -1;
  n = 0;
  for (int k = 0; k < nd; ++k)
    if (g[na + k] >= 0) key[na + n++] = g[na + k];
  sort_small(key + na, n);
  for (int k = n; k < nd; ++k) key[na + k] = -1;
}

__device__ __forceinline__ int cell_of(const QdParams& p, int d, int s, int r) {
  d = d < p.d_max ? d : p.d_max;
  s = s < p.s_max ? s : p.s_max;
  r = r < p.r_max ? r : p.r_max;
  return d + (p.d_max + 1) * (s + (p.s_max + 1) * r);
}

// Cell of every finite-fitness lane (-1 otherwise); clears the insert results.
__global__ void k_lane_cell(QdParams p, Scores sc, int n, int* lane_cell, uint8_t* inserted) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double f = sc.fitness[c];
  lane_cell[c] = isfinite(f) ? cell_of(p, sc.lambda_d[c], sc.lambda_s[c], sc.lambda_r[c]) : -1;
  inserted[c] = 0;
}

// Moves one archive field of a cell after the register-level insert: lane i
// receives entry i from its source (old entry src >= 0 of the cell, or batch
// lane -src-1). Old entries only move to higher positions, so every lane reads
// its source before any lane writes.
template <typename T>
__device__ __forceinline__ void move_field(T* arr, const T* cand, size_t base, int width, bool moved, int src,
                                           int lane) {
  for (int k = 0; k < width; ++k) {
    T v{};
    if (moved) v = src >= 0 ? arr[(base + src) * width + k] : cand[static_cast<size_t>(-src - 1) * width + k];
    __syncwarp();
    if (moved) arr[(base + lane) * width + k] = v;
  }
  __syncwarp();
}

// One warp per cell replays Repertoire::insert (qd_optimizer.cpp:281-303) over
// the batch in lane order; cells are independent, so this equals the
// reference's sequential loop. Lane i of the warp holds entry i of the cell
// (fitness, canonical key, source) in registers: the duplicate test, the
// upper_bound position and the shift are warp votes and shuffles, and the
// payload is written once at the end.
__global__ void k_insert(QdParams p, Archive a, const int* genomes, Scores sc, const int* lane_cell, int n,
                         int worst_k, uint8_t* inserted) {
  const int cell = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cell >= p.cells) return;
  const int ns = p.n_a + p.n_d;
  const size_t base = static_cast<size_t>(cell) * p.cap;
  int cnt = a.count[cell];
  double efit = 0.0;
  int ekey[kMaxSlots];
  int esrc = lane;
#pragma unroll
  for (int k = 0; k < kMaxSlots; ++k) ekey[k] = -1;
  if (lane < cnt) {
    efit = a.fitness[base + lane];
#pragma unroll
    for (int k = 0; k < kMaxSlots; ++k)
      if (k < ns) ekey[k] = a.key[(base + lane) * ns + k];
  }
  bool changed = false;
  for (int c0 = 0; c0 < n; c0 += 128) {
    int lc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + 32 * j + lane;
      lc[j] = c < n ? lane_cell[c] : -1;
    }
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const bool mine = lc[j] == cell;
      unsigned m = __ballot_sync(0xffffffffu, mine);
      if (!m) continue;
      const int cbase = c0 + 32 * j;
      double cf = 0.0;
      int ck[kMaxSlots];
#pragma unroll
      for (int k = 0; k < kMaxSlots; ++k) ck[k] = -1;
      if (mine) cf = sc.fitness[cbase + lane];
      // a full cell only takes a strictly better entry and its worst never
      // decreases while it stays full: lanes not above the current worst are
      // rejected whatever comes before them
      if (cnt >= p.cap) {
        const double worst0 = __shfl_sync(0xffffffffu, efit, cnt - 1);
        m &= __ballot_sync(0xffffffffu, mine && cf > worst0);
        if (!m) continue;
      }
      if ((m >> lane) & 1u) canonical_key(genomes + static_cast<size_t>(cbase + lane) * ns, p.n_a, p.n_d, ck);
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const double fit = __shfl_sync(0xffffffffu, cf, bit);
        const double worst = __shfl_sync(0xffffffffu, efit, cnt > 0 ? cnt - 1 : 0);
        if (cnt >= p.cap && fit <= worst) continue;  // rejected before the duplicate test (same outcome)
        int key[kMaxSlots];
        bool same = lane < cnt;
#pragma unroll
        for (int k = 0; k < kMaxSlots; ++k) {
          key[k] = __shfl_sync(0xffffffffu, ck[k], bit);
          same = same && (k >= ns || ekey[k] == key[k]);
        }
        const bool ok = !__any_sync(0xffffffffu, same);
        if (ok) {
          const int pos = __popc(__ballot_sync(0xffffffffu, lane < cnt && !(fit > efit)));
          const double uf = __shfl_up_sync(0xffffffffu, efit, 1);
          const int us = __shfl_up_sync(0xffffffffu, esrc, 1);
#pragma unroll
          for (int k = 0; k < kMaxSlots; ++k) {
            const int uk = __shfl_up_sync(0xffffffffu, ekey[k], 1);
            if (lane > pos) ekey[k] = uk;
            if (lane == pos) ekey[k] = key[k];
          }
          if (lane > pos) {
            efit = uf;
            esrc = us;
          }
          if (lane == pos) {
            efit = fit;
            esrc = -(cbase + bit) - 1;
          }
          cnt = cnt < p.cap ? cnt + 1 : p.cap;
          changed = true;
        }
        if (lane == 0 && ok) inserted[cbase + bit] = 1;
      }
    }
  }
  if (!changed) return;
  if (lane == 0) a.count[cell] = cnt;
  const bool moved = lane < cnt && esrc != lane;
  if (moved) {
    a.fitness[base + lane] = efit;
    for (int k = 0; k < ns; ++k) a.key[(base + lane) * ns + k] = ekey[k];
  }
  move_field(a.genome, genomes, base, ns, moved, esrc, lane);
  move_field(a.lambda_o, sc.lambda_o, base, 1, moved, esrc, lane);
  move_field(a.lambda_c, sc.lambda_c, base, 1, moved, esrc, lane);
  move_field(a.lambda_c0, sc.lambda_c0, base, 1, moved, esrc, lane);
  move_field(a.lambda_b, sc.lambda_b, base, 1, moved, esrc, lane);
  move_field(a.lambda_d, sc.lambda_d, base, 1, moved, esrc, lane);
  move_field(a.lambda_s, sc.lambda_s, base, 1, moved, esrc, lane);
  move_field(a.lambda_r, sc.lambda_r, base, 1, moved, esrc, lane);
  move_field(a.worst_n, sc.worst_n, base, 1, moved, esrc, lane);
  move_field(a.worst_idx, sc.worst_idx, base, worst_k, moved, esrc, lane);
  move_field(a.worst_val, sc.worst_val, base, worst_k, moved, esrc, lane);
}

// Exclusive prefix of cell counts (member order) and the iteration counter.
__global__ void k_archive_prefix(QdParams p, Archive a, int advance) {
  __shared__ int part[1024];
  const int per = (p.cells + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(lo + per, p.cells);
  int s = 0;
  for (int c = lo; c < hi; ++c) s += a.count[c];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
      const int v = part[t];
      part[t] = run;
      run += v;
    }
    a.flat_start[p.cells] = run;
    if (advance) a.iter[0] += 1;
  }
  __syncthreads();
  int run = part[threadIdx.x];
  for (int c = lo; c < hi; ++c) {
    a.flat_start[c] = run;
    run += a.count[c];
  }
}

__global__ void k_archive_clear(QdParams p, Archive a, int reset_iter) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c <= p.cells; c += gridDim.x * blockDim.x) {
    if (c < p.cells) a.count[c] = 0;
    a.flat_start[c] = 0;
  }
  if (reset_iter && blockIdx.x == 0 && threadIdx.x == 0) a.iter[0] = 0;
}

// ---------------------------------------------------------------- island exchange
// One thread per archive slot: the slot's entry (or an empty marker with
// fitness -inf) into the island blob.
__global__ void k_archive_pack(QdParams p, Archive a, int wk, uint8_t* blob) {
  const int slots = p.cells * p.cap, ns = p.n_a + p.n_d;
  const BlobLayout L(slots, ns, wk);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= slots) return;
  const int cell = i / p.cap, pos = i % p.cap;
  const bool live = pos < a.count[cell];
  double* fit = reinterpret_cast<double*>(blob + L.fit);
  fit[i] = live ? a.fitness[i] : -CUDART_INF;
  reinterpret_cast<double*>(blob + L.lo)[i] = live ? a.lambda_o[i] : 0.0;
  reinterpret_cast<double*>(blob + L.lb)[i] = live ? a.lambda_b[i] : 0.0;
  reinterpret_cast<int*>(blob + L.lc)[i] = live ? a.lambda_c[i] : 0;
  reinterpret_cast<int*>(blob + L.lc0)[i] = live ? a.lambda_c0[i] : 0;
  reinterpret_cast<int*>(blob + L.ld)[i] = live ? a.lambda_d[i] : 0;
  reinterpret_cast<int*>(blob + L.ls)[i] = live ? a.lambda_s[i] : 0;
  reinterpret_cast<int*>(blob + L.lr)[i] = live ? a.lambda_r[i] : 0;
  const int wn = live ? min(a.worst_n[i], wk) : 0;
  reinterpret_cast<int*>(blob + L.wn)[i] = wn;
  for (int k = 0; k < ns; ++k)
    reinterpret_cast<int*>(blob + L.gen)[static_cast<size_t>(i) * ns + k] =
        live ? a.genome[static_cast<size_t>(i) * ns + k] : -1;
  for (int k = 0; k < wk; ++k) {
    const size_t at = static_cast<size_t>(i) * wk + k;
    reinterpret_cast<int*>(blob + L.widx)[at] = k < wn ? a.worst_idx[at] : 0;  // canonical: zeros past worst_n
    reinterpret_cast<double*>(blob + L.wval)[at] = k < wn ? a.worst_val[at] : 0.0;
  }
}

// Batch lanes [lo, lo + n) -> BlobLayout(n) blob (one thread per lane).
__global__ void k_scores_pack(QdParams p, int wk, const int* genomes, Scores sc, int lo, int n, uint8_t* blob) {
  const int ns = p.n_a + p.n_d;
  const BlobLayout L(n, ns, wk);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = lo + i;
  reinterpret_cast<double*>(blob + L.fit)[i] = sc.fitness[c];
  reinterpret_cast<double*>(blob + L.lo)[i] = sc.lambda_o[c];
  reinterpret_cast<double*>(blob + L.lb)[i] = sc.lambda_b[c];
  reinterpret_cast<int*>(blob + L.lc)[i] = sc.lambda_c[c];
  reinterpret_cast<int*>(blob + L.lc0)[i] = sc.lambda_c0[c];
  reinterpret_cast<int*>(blob + L.ld)[i] = sc.lambda_d[c];
  reinterpret_cast<int*>(blob + L.ls)[i] = sc.lambda_s[c];
  reinterpret_cast<int*>(blob + L.lr)[i] = sc.lambda_r[c];
  reinterpret_cast<int*>(blob + L.wn)[i] = sc.worst_n[c];
  for (int k = 0; k < ns; ++k)
    reinterpret_cast<int*>(blob + L.gen)[static_cast<size_t>(i) * ns + k] = genomes[static_cast<size_t>(c) * ns + k];
  for (int k = 0; k < wk; ++k) {
    reinterpret_cast<int*>(blob + L.widx)[static_cast<size_t>(i) * wk + k] = sc.worst_idx[static_cast<size_t>(c) * wk + k];
    reinterpret_cast<double*>(blob + L.wval)[static_cast<size_t>(i) * wk + k] =
        sc.worst_val[static_cast<size_t>(c) * wk + k];
  }
}

__global__ void k_scores_unpack(QdParams p, int wk, const uint8_t* blob, int lo, int n, Scores sc) {
  const int ns = p.n_a + p.n_d;
  const BlobLayout L(n, ns, wk);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = lo + i;
  sc.fitness[c] = reinterpret_cast<const double*>(blob + L.fit)[i];
  sc.lambda_o[c] = reinterpret_cast<const double*>(blob + L.lo)[i];
  sc.lambda_b[c] = reinterpret_cast<const double*>(blob + L.lb)[i];
  sc.lambda_c[c] = reinterpret_cast<const int*>(blob + L.lc)[i];
  sc.lambda_c0[c] = reinterpret_cast<const int*>(blob + L.lc0)[i];
  sc.lambda_d[c] = reinterpret_cast<const int*>(blob + L.ld)[i];
  sc.lambda_s[c] = reinterpret_cast<const int*>(blob + L.ls)[i];
  sc.lambda_r[c] = reinterpret_cast<const int*>(blob + L.lr)[i];
  sc.worst_n[c] = reinterpret_cast<const int*>(blob + L.wn)[i];
  for (int k = 0; k < wk; ++k) {
    sc.worst_idx[static_cast<size_t>(c) * wk + k] = reinterpret_cast<const int*>(blob + L.widx)[static_cast<size_t>(i) * wk + k];
    sc.worst_val[static_cast<size_t>(c) * wk + k] =
        reinterpret_cast<const double*>(blob + L.wval)[static_cast<size_t>(i) * wk + k];
  }
}

// Gathered blobs [island][BlobLayout] -> one insert batch, lane = island * S + slot.
__global__ void k_merge_unpack(QdParams p, int wk, const uint8_t* blobs, int n_islands, int* genomes, Scores sc) {
  const int slots = p.cells * p.cap, ns = p.n_a + p.n_d;
  const BlobLayout L(slots, ns, wk);
  const long n = static_cast<long>(slots) * n_islands;
  for (long lane = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; lane < n;
       lane += static_cast<long>(gridDim.x) * blockDim.x) {
    const int isl = static_cast<int>(lane / slots), i = static_cast<int>(lane % slots);
    const uint8_t* b = blobs + static_cast<size_t>(isl) * L.total;
    sc.fitness[lane] = reinterpret_cast<const double*>(b + L.fit)[i];
    sc.lambda_o[lane] = reinterpret_cast<const double*>(b + L.lo)[i];
    sc.lambda_b[lane] = reinterpret_cast<const double*>(b + L.lb)[i];
    sc.lambda_c[lane] = reinterpret_cast<const int*>(b + L.lc)[i];
    sc.lambda_c0[lane] = reinterpret_cast<const int*>(b + L.lc0)[i];
    sc.lambda_d[lane] = reinterpret_cast<const int*>(b + L.ld)[i];
    sc.lambda_s[lane] = reinterpret_cast<const int*>(b + L.ls)[i];
    sc.lambda_r[lane] = reinterpret_cast<const int*>(b + L.lr)[i];
    sc.worst_n[lane] = reinterpret_cast<const int*>(b + L.wn)[i];
    for (int k = 0; k < ns; ++k)
      genomes[lane * ns + k] = reinterpret_cast<const int*>(b + L.gen)[static_cast<size_t>(i) * ns + k];
    for (int k = 0; k < wk; ++k) {
      sc.worst_idx[lane * wk + k] = reinterpret_cast<const int*>(b + L.widx)[static_cast<size_t>(i) * wk + k];
      sc.worst_val[lane * wk + k] = reinterpret_cast<const double*>(b + L.wval)[static_cast<size_t>(i) * wk + k];
    }
  }
}

}  // namespace

void launch_archive_reset(const QdState& q, cudaStream_t s) {
  k_archive_clear<<<(q.p.cells + 256) / 256, 256, 0, s>>>(q.p, q.a, 1);
}

void launch_offspring(const DevGrid& g, const QdState& q, int* genomes, cudaStream_t s) {
  // lanes carry a 2.5 KB engine state in local memory
  const int blocks = (q.p.batch + kOffspringLanes - 1) / kOffspringLanes;
  if (q.p.rng == kRngPhilox)
    k_offspring<Philox><<<blocks, kOffspringLanes + 32, 0, s>>>(g, q.p, q.a, genomes);
  else
  {
    // replay engine: 32 lanes per block with their states in shared memory
    constexpr int kL = 32;
    const size_t smem = static_cast<size_t>(kL + 1) * Mt64::kN * sizeof(unsigned long long);
    static std::atomic<unsigned long long> configured{0};
    if (first_use_on_device(configured))
      cudaFuncSetAttribute(k_offspring<Mt64S, kL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_offspring<Mt64S, kL><<<(q.p.batch + kL - 1) / kL, kL + 32, smem, s>>>(g, q.p, q.a, genomes);
  }
}

namespace {
int insert_lanes(const QdState& q, const int* genomes, const Scores& sc, int n, int worst_k, bool advance_iter,
                 int* lane_cell, uint8_t* inserted, cudaStream_t s) {
  constexpr int kWarps = 4;
  if (n <= 0) return 0;
  k_lane_cell<<<(n + 255) / 256, 256, 0, s>>>(q.p, sc, n, lane_cell, inserted);
  k_insert<<<(q.p.cells + kWarps - 1) / kWarps, 32 * kWarps, 0, s>>>(q.p, q.a, genomes, sc, lane_cell, n, worst_k,
                                                                    inserted);
  k_archive_prefix<<<1, 256, 0, s>>>(q.p, q.a, advance_iter ? 1 : 0);
  return 3;
}
}  // namespace

int launch_insert(const QdState& q, const int* genomes, const Scores& sc, int n, int worst_k, bool advance_iter,
                  cudaStream_t s) {
  return insert_lanes(q, genomes, sc, n, worst_k, advance_iter, q.lane_cell, q.inserted, s);
}

void launch_archive_pack(const QdState& q, void* blob, cudaStream_t s) {
  const int slots = q.p.cells * q.p.cap;
  k_archive_pack<<<(slots + 255) / 256, 256, 0, s>>>(q.p, q.a, q.worst_k, static_cast<uint8_t*>(blob));
}

int launch_archive_merge(const QdState& q, const void* blobs, int n_islands, MergeBuffers& m, cudaStream_t s) {
  const int n = q.p.cells * q.p.cap * n_islands;
  k_merge_unpack<<<(n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024, 256, 0, s>>>(
      q.p, q.worst_k, static_cast<const uint8_t*>(blobs), n_islands, m.genomes, m.sc);
  k_archive_clear<<<(q.p.cells + 256) / 256, 256, 0, s>>>(q.p, q.a, 0);
  return 2 + insert_lanes(q, m.genomes, m.sc, n, q.worst_k, false, m.lane_cell, m.inserted, s);
}

void launch_scores_pack(const QdState& q, const int* genomes, const Scores& sc, int lo, int n, void* blob,
                        cudaStream_t s) {
  if (n > 0)
    k_scores_pack<<<(n + 255) / 256, 256, 0, s>>>(q.p, q.worst_k, genomes, sc, lo, n, static_cast<uint8_t*>(blob));
}

void launch_scores_unpack(const QdState& q, const void* blob, int lo, int n, const Scores& sc, cudaStream_t s) {
  if (n > 0)
    k_scores_unpack<<<(n + 255) / 256, 256, 0, s>>>(q.p, q.worst_k, static_cast<const uint8_t*>(blob), lo, n, sc);
}

void launch_mutate_lanes(const DevGrid& g, const QdState& q, const int* parents, const unsigned long long* seeds, int n,
                         int* children, cudaStream_t s) {
  if (q.p.rng == kRngPhilox)
    k_mutate_lanes<Philox><<<(n + 63) / 64, 64, 0, s>>>(g, q.p, parents, seeds, n, children);
  else
    k_mutate_lanes<Mt64><<<(n + 63) / 64, 64, 0, s>>>(g, q.p, parents, seeds, n, children);
}

void launch_crossover_lanes(const DevGrid& g, const QdState& q, const int* p1, const int* p2,
                            const unsigned long long* seeds, int n, int* children, cudaStream_t s) {
  if (q.p.rng == kRngPhilox)
    k_crossover_lanes<Philox><<<(n + 63) / 64, 64, 0, s>>>(g, q.p, p1, p2, seeds, n, children);
  else
    k_crossover_lanes<Mt64><<<(n + 63) / 64, 64, 0, s>>>(g, q.p, p1, p2, seeds, n, children);
}

}  // namespace tgb
