// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU reference of what the SVFusion hot path computes (arXiv 2601.08528,
// /root/reference/PAPER.md, cited as P:L<line>; the readings of ambiguous passages are SURVEY.md §8(c)
// I1..I18 and are listed again in DESIGN.md §"Readings").  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  It shares NO code, header,
// table or constant generator with the CUDA path in paper_2601_08528_b200/csrc/ (the counter-based
// init generator below is implemented independently on each side, as DESIGN.md states).
//
// Arithmetic: distances accumulate in fp64 from the fp32 inputs and are reported rounded to fp32;
// every ordering decision is taken on the (fp32 distance, id) pair, lower id first on ties (I5), in
// the paper's precision (fp32, uncompressed: P:L119).  -0.0 is canonicalised to +0.0.
//
// Pins (tests/test_oracle_pins.py): exhaustive enumeration on tiny inputs, SPEC worked examples,
// hand-traced searches in tests/golden/, "L >= live N  =>  search == exact kNN", invariants.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

constexpr uint32_t SENT = 0xFFFFFFFFu;            // empty adjacency slot / padded result id
const float INF = std::numeric_limits<float>::infinity();

// ---- distance: P:L162 (Euclidean; reported squared) and -<q,x> for inner product (I1) ----------
float dist(const float* q, const float* x, int D, int metric) {
  double acc = 0.0;
  if (metric == 0) {
    for (int i = 0; i < D; ++i) {
      double t = (double)q[i] - (double)x[i];
      acc += t * t;
    }
  } else {
    for (int i = 0; i < D; ++i) acc += (double)q[i] * (double)x[i];
    acc = -acc;
  }
  float f = (float)acc;
  return f + 0.0f;  // canonical +0
}

struct Entry {
  float d;
  uint32_t id;
  bool parented;
};
// total order on (distance, id): I5
bool key_less(const Entry& a, const Entry& b) { return a.d < b.d || (a.d == b.d && a.id < b.id); }

bool dead(const uint32_t* tomb, uint32_t id) { return tomb && ((tomb[id >> 5] >> (id & 31)) & 1u); }

// ---- I2: entry points along a seeded affine permutation of [0, n) ----------------------------------------
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void affine_params(uint64_t seed, uint64_t qidx, uint64_t n, uint64_t* a, uint64_t* b) {
  uint64_t h = splitmix64(seed ^ (qidx * 0x9E3779B97F4A7C15ull));
  uint64_t A = (h >> 1) % n;
  if (A == 0) A = 1;
  while (std::gcd(A, n) != 1) ++A;
  *a = A;
  *b = (h >> 33) % n;
}

template <class F>
void parallel_for(int64_t n, int threads, F f) {
  if (threads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&]() {
      for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& th : pool) th.join();
}

struct SearchCtx {
  const float* X;
  int D, metric;
  const uint32_t* graph;
  int R;
  const uint32_t* tomb;
  int64_t n_alloc;
  int L, p, n_init, max_iter;
  uint64_t seed;
};

struct Counters {
  int64_t n_dist = 0, n_exp = 0, iters = 0;
};

// ---- O2: greedy graph search, Algorithm 1 without the tiering split -----
// init_ids != nullptr replaces the random initialisation (test hook for hand-traced pins).
std::vector<Entry> graph_search_one(const SearchCtx& c, const float* q, uint64_t qidx, const uint32_t* init_ids,
                                    int n_init_ids, Counters& cnt) {
  std::unordered_set<uint32_t> V;  // exact visited set ("until C unchanged", no revisits: P:L361)
  std::vector<Entry> C;            // the candidate pool C_i
  // InitCandidatePool(G, L): random initialisation, reading I2.
  if (init_ids) {
    for (int j = 0; j < n_init_ids; ++j) {
      uint32_t id = init_ids[j];
      if (dead(c.tomb, id) || V.count(id)) continue;
      V.insert(id);
      C.push_back({dist(q, c.X + (size_t)id * c.D, c.D, c.metric), id, false});
      cnt.n_dist++;
    }
  } else if (c.n_alloc > 0) {
    uint64_t a, b;
    affine_params(c.seed, qidx, (uint64_t)c.n_alloc, &a, &b);
    for (uint64_t j = 0; j < (uint64_t)c.n_alloc && (int)C.size() < c.n_init; ++j) {
      uint32_t id = (uint32_t)((a * j + b) % (uint64_t)c.n_alloc);
      if (dead(c.tomb, id)) continue;  // deleted vertices are skipped
      V.insert(id);
      C.push_back({dist(q, c.X + (size_t)id * c.D, c.D, c.metric), id, false});
      cnt.n_dist++;
    }
  }
  std::sort(C.begin(), C.end(), key_less);
  if ((int)C.size() > c.L) C.resize(c.L);

  for (;;) {
    // GetNearest generalised to the first p unparented entries in pool order (I3).
    std::vector<uint32_t> par;
    for (auto& e : C)
      if (!e.parented && (int)par.size() < c.p) par.push_back(e.id);
    // "until C unchanged", reading I4: stop when every pool entry has been expanded.
    if (par.empty() || (c.max_iter > 0 && cnt.iters == c.max_iter)) break;
    for (auto& e : C)
      if (!e.parented && std::find(par.begin(), par.end(), e.id) != par.end()) e.parented = true;
    cnt.iters++;
    cnt.n_exp += (int64_t)par.size();
    std::vector<Entry> cand;
    for (uint32_t u : par) {
      // FetchNeighbors
      for (int s = 0; s < c.R; ++s) {
        uint32_t v = c.graph[(size_t)u * c.R + s];
        if (v == SENT || (int64_t)v >= c.n_alloc) continue;
        if (dead(c.tomb, v)) continue;  // P:L532 (I8)
        if (V.count(v)) continue;
        V.insert(v);
        // ParallelComputeDist
        cand.push_back({dist(q, c.X + (size_t)v * c.D, c.D, c.metric), v, false});
        cnt.n_dist++;
      }
    }
    // C.Update: keep the L best of C u cand
    C.insert(C.end(), cand.begin(), cand.end());
    std::sort(C.begin(), C.end(), key_less);
    if ((int)C.size() > c.L) C.resize(c.L);
  }
  return C;
}

void emit(const std::vector<Entry>& C, int n_out, uint32_t* ids, float* d) {
  for (int i = 0; i < n_out; ++i) {
    if (i < (int)C.size()) {
      ids[i] = C[i].id;
      d[i] = C[i].d;
    } else {
      ids[i] = SENT;  // I17: pad with (sentinel, +inf)
      d[i] = INF;
    }
  }
}

// ---- O3 (ii)+(iii): detour-ranked forward row + protected-prefix reverse edges ------------------------------
// Forward row of a new vertex v from its distance-ordered candidate list C (readings I10-I12).
void forward_row(const uint32_t* graph, int R, int P, const uint32_t* C_ids, const float* C_d, int nc,
                 uint32_t* row_ids, float* row_d) {
  int m = 0;
  while (m < nc && C_ids[m] != SENT) ++m;
  // count(i) = |{ j < i : C[i] in N_out(C[j]) }|  ("detourable paths")
  std::vector<int> count(m, 0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < i; ++j) {
      const uint32_t* rj = graph + (size_t)C_ids[j] * R;
      for (int s = 0; s < R; ++s)
        if (rj[s] == C_ids[i]) {
          count[i]++;
          break;
        }
    }
  // sort by detour count ascending, stable on original rank (I11); take the top R
  std::vector<int> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return count[a] < count[b]; });
  int sel = std::min(R, m);
  int npre = std::min(P, sel);
  for (int s = 0; s < R; ++s) {
    row_ids[s] = SENT;
    row_d[s] = INF;
  }
  for (int s = 0; s < npre; ++s) {  // protected prefix, detour order
    row_ids[s] = C_ids[order[s]];
    row_d[s] = C_d[order[s]];
  }
  std::vector<Entry> tail;
  for (int s = npre; s < sel; ++s) tail.push_back({C_d[order[s]], C_ids[order[s]], false});
  std::sort(tail.begin(), tail.end(), key_less);  // tail sorted by key(d,id)
  for (size_t s = 0; s < tail.size(); ++s) {
    row_ids[P + s] = tail[s].id;
    row_d[P + s] = tail[s].d;
  }
}

// Reverse-edge insertion (reading I12): tail(u) <- first (R-P) of sort_eff(tail(u) U requests(u)).
void apply_reverse(uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R, int P, uint32_t u,
                   const std::vector<Entry>& reqs) {
  if (dead(tomb, u)) return;  // deleted rows are frozen
  struct Eff {
    float eff;
    uint32_t id;
    float d;
  };
  std::vector<Eff> all;
  for (int s = P; s < R; ++s) {
    uint32_t id = graph[(size_t)u * R + s];
    float d = edge_dist[(size_t)u * R + s];
    float eff = (id == SENT || dead(tomb, id)) ? INF : d;  // tombstoned / empty count as +inf
    all.push_back({eff, id, id == SENT ? INF : d});
  }
  for (auto& r : reqs) all.push_back({r.d, r.id, r.d});
  std::sort(all.begin(), all.end(),
            [](const Eff& a, const Eff& b) { return a.eff < b.eff || (a.eff == b.eff && a.id < b.id); });
  for (int s = P; s < R; ++s) {
    const Eff& e = all[s - P];
    graph[(size_t)u * R + s] = e.id;
    edge_dist[(size_t)u * R + s] = e.d;
  }
}

// One sub-batch of links: new ids [first, first+n) with candidate lists (n x nc), all candidates < first.
void link_batch(uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R, int P, int64_t first, int64_t n,
                const uint32_t* cand_ids, const float* cand_d, int nc, int threads) {
  // (ii) forward rows, computed on snapshot rows (rows of ids < first are not modified until (iii))
  parallel_for(n, threads, [&](int64_t b) {
    forward_row(graph, R, P, cand_ids + b * nc, cand_d + b * nc, nc, graph + (size_t)(first + b) * R,
                edge_dist + (size_t)(first + b) * R);
  });
  // (iii) reverse requests (u, v, d) for every forward edge v -> u
  std::vector<std::pair<uint32_t, Entry>> req;
  for (int64_t b = 0; b < n; ++b) {
    uint32_t v = (uint32_t)(first + b);
    for (int s = 0; s < R; ++s) {
      uint32_t u = graph[(size_t)v * R + s];
      if (u == SENT) continue;
      req.push_back({u, Entry{edge_dist[(size_t)v * R + s], v, false}});
    }
  }
  std::sort(req.begin(), req.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  size_t i = 0;
  while (i < req.size()) {
    size_t j = i;
    std::vector<Entry> reqs;
    while (j < req.size() && req[j].first == req[i].first) reqs.push_back(req[j++].second);
    apply_reverse(graph, edge_dist, tomb, R, P, req[i].first, reqs);
    i = j;
  }
}

}  // namespace

extern "C" {

uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }

void orc_affine_params(uint64_t seed, uint64_t qidx, uint64_t n, uint64_t* a, uint64_t* b) {
  affine_params(seed, qidx, n, a, b);
}

float orc_dist(const float* q, const float* x, int D, int metric) { return dist(q, x, D, metric); }

// O1: exact k-NN over the live set (P:L160-162 definition; "exhaustive linear scan").
int orc_bf_knn(const float* X, int64_t n, int D, int metric, const uint32_t* tomb, const float* Q, int64_t nq, int k,
               uint32_t* out_ids, float* out_d, int threads) {
  if (k <= 0 || D <= 0 || n < 0 || nq < 0) return 1;
  parallel_for(nq, threads, [&](int64_t qi) {
    std::vector<Entry> all;
    all.reserve((size_t)n);
    for (int64_t i = 0; i < n; ++i)
      if (!dead(tomb, (uint32_t)i)) all.push_back({dist(Q + qi * D, X + i * D, D, metric), (uint32_t)i, false});
    size_t kk = std::min<size_t>((size_t)k, all.size());
    std::partial_sort(all.begin(), all.begin() + kk, all.end(), key_less);
    all.resize(kk);
    emit(all, k, out_ids + qi * k, out_d + qi * k);
  });
  return 0;
}

// O2: batched greedy graph search.  qidx[i] (or i when null) seeds query i's entry points (I18).
// insert_mode: emit the whole pool (L entries) instead of the first k.  counters: nq x {n_dist,n_exp,iters}.
int orc_graph_search(const float* X, int D, int metric, const uint32_t* graph, int R, const uint32_t* tomb,
                     int64_t n_alloc, const float* Q, int64_t nq, const int64_t* qidx, int k, int L, int p,
                     int n_init, int max_iter, uint64_t seed, int insert_mode, uint32_t* out_ids, float* out_d,
                     int64_t* counters, int threads) {
  if (k <= 0 || L < k || p <= 0 || n_init <= 0) return 1;
  SearchCtx c{X, D, metric, graph, R, tomb, n_alloc, L, p, n_init, max_iter, seed};
  int n_out = insert_mode ? L : k;
  parallel_for(nq, threads, [&](int64_t i) {
    Counters cnt;
    auto C = graph_search_one(c, Q + i * D, qidx ? (uint64_t)qidx[i] : (uint64_t)i, nullptr, 0, cnt);
    emit(C, n_out, out_ids + i * n_out, out_d + i * n_out);
    if (counters) {
      counters[i * 3 + 0] = cnt.n_dist;
      counters[i * 3 + 1] = cnt.n_exp;
      counters[i * 3 + 2] = cnt.iters;
    }
  });
  return 0;
}

// Test hook: O2 from explicit entry points (hand-traced golden pins).
int orc_graph_search_from(const float* X, int D, int metric, const uint32_t* graph, int R, const uint32_t* tomb,
                          int64_t n_alloc, const float* q, const uint32_t* init_ids, int n_init_ids, int k, int L,
                          int p, int max_iter, uint32_t* out_ids, float* out_d, int64_t* counters) {
  SearchCtx c{X, D, metric, graph, R, tomb, n_alloc, L, p, n_init_ids, max_iter, 0};
  Counters cnt;
  auto C = graph_search_one(c, q, 0, init_ids, n_init_ids, cnt);
  emit(C, k, out_ids, out_d);
  counters[0] = cnt.n_dist;
  counters[1] = cnt.n_exp;
  counters[2] = cnt.iters;
  return 0;
}

// O3 (ii)+(iii) only, from given candidate lists (the test entry svf_link_candidates mirrors this).
int orc_link_candidates(uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R, int P, int64_t first,
                        int64_t n_new, const uint32_t* cand_ids, const float* cand_d, int nc, int threads) {
  if (P < 0 || P > R) return 1;
  for (int64_t i = 0; i < n_new * nc; ++i)
    if (cand_ids[i] != SENT && (int64_t)cand_ids[i] >= first) return 1;
  link_batch(graph, edge_dist, tomb, R, P, first, n_new, cand_ids, cand_d, nc, threads);
  return 0;
}

// O3: batched insert of rows [n_alloc, n_alloc + n_new) of X (already placed), sub-batch snapshot semantics
// (I13: sub-batches of min(B_ins, n_current)).
int orc_insert(const float* X, int D, int metric, uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R,
               int P, int64_t n_alloc, int64_t n_new, int L_ins, int B_ins, int p, int n_init, int max_iter,
               uint64_t seed, int threads) {
  if (n_alloc <= 0 || B_ins <= 0 || P < 0 || P > R) return 1;
  int64_t done = 0;
  std::vector<uint32_t> cid;
  std::vector<float> cd;
  while (done < n_new) {
    int64_t snap = n_alloc + done;
    int64_t bsz = std::min<int64_t>({(int64_t)B_ins, snap, n_new - done});
    cid.assign((size_t)bsz * L_ins, SENT);
    cd.assign((size_t)bsz * L_ins, INF);
    std::vector<int64_t> qidx(bsz);
    for (int64_t b = 0; b < bsz; ++b) qidx[b] = snap + b;
    // (i) insert-mode search over the snapshot (ids < snap); the new rows are not reachable
    orc_graph_search(X, D, metric, graph, R, tomb, snap, X + snap * D, bsz, qidx.data(), 1, L_ins, p, n_init,
                     max_iter, seed, 1, cid.data(), cd.data(), nullptr, threads);
    link_batch(graph, edge_dist, tomb, R, P, snap, bsz, cid.data(), cd.data(), L_ins, threads);
    done += bsz;
  }
  return 0;
}

// O5: build = exact R-NN seed over the first min(n, seed_size) rows, then O3 growth (reading I15).
int orc_build(const float* X, int64_t n, int D, int metric, int R, int P, int L_ins, int B_ins, int seed_size,
              int p, int n_init, int max_iter, uint64_t seed, uint32_t* graph, float* edge_dist, int threads) {
  if (n <= 0 || seed_size <= 0 || P < 0 || P > R) return 1;
  int64_t n0 = std::min<int64_t>(n, seed_size);
  for (int64_t i = 0; i < n * R; ++i) {
    graph[i] = SENT;
    edge_dist[i] = INF;
  }
  parallel_for(n0, threads, [&](int64_t v) {
    std::vector<Entry> all;
    for (int64_t u = 0; u < n0; ++u)
      if (u != v) all.push_back({dist(X + v * D, X + u * D, D, metric), (uint32_t)u, false});
    size_t kk = std::min<size_t>((size_t)R, all.size());
    std::partial_sort(all.begin(), all.begin() + kk, all.end(), key_less);
    // prefix [0,P) = the P nearest, tail [P,R) = the rest: the key-sorted list fills both contiguously
    for (size_t s = 0; s < kk; ++s) {
      graph[v * R + s] = all[s].id;
      edge_dist[v * R + s] = all[s].d;
    }
  });
  if (n > n0)
    return orc_insert(X, D, metric, graph, edge_dist, nullptr, R, P, n0, n - n0, L_ins, B_ins, p, n_init, max_iter,
                      seed, threads);
  return 0;
}

// NEXT-1: localized topology-aware repair, reading R1' in DESIGN.md:
//   V^L = live v < n_alloc whose non-sentinel row entries are more than `threshold` deleted (strict);
//   for each v in V^L, for each deleted p in row(v) in slot order, take the first c members of N_out(p) in slot
//   order that are live, != v, not a live entry of row(v) and not already taken ("at most c vertices from
//   N_out(p)"); U = (live entries, stored distances) U (candidates, fresh distances) sorted by (dist, id)
//   and cut to its first `cap` (= insert_itopk); the new row is U's insertion selection (readings
//   I10-I12: detour counts on the call's starting rows, prefix P in detour order, tail sorted by key).
//   mode 0 (experiment hook, reading R1): the row is the R nearest of U instead.
// All rows are read from the state at the start of the call (rows of deleted p are frozen; only V^L rows change).
// hist[5] counts live rows by deleted fraction: 0, (0,0.1), [0.1,0.4], (0.4,threshold], >threshold (Fig. 5).
int orc_repair_mode(const float* X, int D, int metric, uint32_t* graph, float* edge_dist, const uint32_t* tomb,
                    int R, int P, int64_t n_alloc, int c, double threshold, int mode, int cap, int64_t* n_repaired,
                    int64_t* hist);
int orc_repair(const float* X, int D, int metric, uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R,
               int P, int64_t n_alloc, int c, double threshold, int cap, int64_t* n_repaired, int64_t* hist) {
  return orc_repair_mode(X, D, metric, graph, edge_dist, tomb, R, P, n_alloc, c, threshold, 1, cap, n_repaired, hist);
}
int orc_repair_mode(const float* X, int D, int metric, uint32_t* graph, float* edge_dist, const uint32_t* tomb,
                    int R, int P, int64_t n_alloc, int c, double threshold, int mode, int cap, int64_t* n_repaired,
                    int64_t* hist) {
  std::vector<uint32_t> snap(graph, graph + (size_t)n_alloc * R);
  std::vector<float> snapd(edge_dist, edge_dist + (size_t)n_alloc * R);
  int64_t repaired = 0;
  for (int i = 0; i < 5; ++i) hist[i] = 0;
  for (int64_t v = 0; v < n_alloc; ++v) {
    if (dead(tomb, (uint32_t)v)) continue;
    const uint32_t* row = snap.data() + (size_t)v * R;
    int total = 0, ndead = 0;
    for (int s = 0; s < R; ++s)
      if (row[s] != SENT) {
        total++;
        if (dead(tomb, row[s])) ndead++;
      }
    const double frac = total ? (double)ndead / total : 0.0;
    int bucket = ndead == 0 ? 0 : (frac < 0.1 ? 1 : (frac <= 0.4 ? 2 : (frac <= threshold ? 3 : 4)));
    hist[bucket]++;
    if (!(frac > threshold)) continue;
    std::vector<Entry> pool;
    std::unordered_set<uint32_t> taken;
    for (int s = 0; s < R; ++s)
      if (row[s] != SENT && !dead(tomb, row[s])) {
        pool.push_back({snapd[(size_t)v * R + s], row[s], false});
        taken.insert(row[s]);
      }
    for (int s = 0; s < R; ++s) {
      const uint32_t p = row[s];
      if (p == SENT || !dead(tomb, p)) continue;
      int got = 0;
      for (int t = 0; t < R && got < c; ++t) {
        const uint32_t x = snap[(size_t)p * R + t];
        if (x == SENT || dead(tomb, x) || x == (uint32_t)v || taken.count(x)) continue;
        taken.insert(x);
        pool.push_back({dist(X + (size_t)v * D, X + (size_t)x * D, D, metric), x, false});
        got++;
      }
    }
    std::sort(pool.begin(), pool.end(), key_less);
    if (mode == 1 && cap > 0 && (int)pool.size() > cap) pool.resize(cap);
    if (mode == 1) {
      std::vector<uint32_t> cid(pool.size());
      std::vector<float> cd(pool.size());
      for (size_t i = 0; i < pool.size(); ++i) {
        cid[i] = pool[i].id;
        cd[i] = pool[i].d;
      }
      forward_row(snap.data(), R, P, cid.data(), cd.data(), (int)pool.size(), graph + (size_t)v * R,
                  edge_dist + (size_t)v * R);
    } else {
      for (int s = 0; s < R; ++s) {
        graph[(size_t)v * R + s] = s < (int)pool.size() ? pool[s].id : SENT;
        edge_dist[(size_t)v * R + s] = s < (int)pool.size() ? pool[s].d : INF;
      }
    }
    repaired++;
  }
  *n_repaired = repaired;
  return 0;
}

// NEXT-4: global consolidation ("a global consolidation of all affected neighborhoods by aggregating
// candidates from the outgoing neighbors of deleted vertices"), reading C2 in DESIGN.md.  For every live v < n_alloc
// whose row holds at least one vacant entry (a tombstoned id), with all rows read from the call's starting state:
//   * live entries stay where they are (the protected prefix keeps its slots, the live tail entries are kept);
//   * U = live members of N_out(p) over the tombstoned p of row(v) (slot order), excluding v and the live entries of
//     row(v), without duplicates, each with its distance to v;
//   * each tombstoned PREFIX slot s (slot order) is refilled by the nearest (dist, id) member of N_out(p_s) in U not
//     taken by an earlier slot (the two-hop edge through the deleted p_s);
//   * the m tail vacancies (tombstoned tail entries plus empty tail slots) are refilled by the m nearest members of U
//     not taken by the prefix; the tail (kept live entries + refills) is re-sorted by key(d, id), empty slots last.
// A vacancy with no eligible candidate becomes an empty slot (sentinel, +inf).  Afterwards no live row references a
// deleted vertex; rows of deleted vertices and rows without deleted neighbours are unchanged.
int orc_consolidate(const float* X, int D, int metric, uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R,
                    int P, int64_t n_alloc, int64_t* n_rewritten) {
  if (P < 0 || P > R) return 1;
  std::vector<uint32_t> snap(graph, graph + (size_t)n_alloc * R);
  std::vector<float> snapd(edge_dist, edge_dist + (size_t)n_alloc * R);
  int64_t rewritten = 0;
  for (int64_t v = 0; v < n_alloc; ++v) {
    if (dead(tomb, (uint32_t)v)) continue;
    const uint32_t* row = snap.data() + (size_t)v * R;
    const float* rowd = snapd.data() + (size_t)v * R;
    bool affected = false;
    std::unordered_set<uint32_t> in_row;
    for (int s = 0; s < R; ++s) {
      if (row[s] == SENT) continue;
      if (dead(tomb, row[s])) affected = true;
      else in_row.insert(row[s]);
    }
    if (!affected) continue;
    // U with distances (first occurrence order is irrelevant: every choice below is by (dist, id))
    std::vector<Entry> U;
    std::unordered_set<uint32_t> seen;
    for (int s = 0; s < R; ++s) {
      const uint32_t p = row[s];
      if (p == SENT || !dead(tomb, p)) continue;
      for (int t = 0; t < R; ++t) {
        const uint32_t x = snap[(size_t)p * R + t];
        if (x == SENT || dead(tomb, x) || x == (uint32_t)v || in_row.count(x) || seen.count(x)) continue;
        seen.insert(x);
        U.push_back({dist(X + (size_t)v * D, X + (size_t)x * D, D, metric), x, false});
      }
    }
    std::unordered_set<uint32_t> taken;
    uint32_t* out = graph + (size_t)v * R;
    float* outd = edge_dist + (size_t)v * R;
    // prefix: slot by slot
    for (int s = 0; s < P; ++s) {
      out[s] = row[s];
      outd[s] = rowd[s];
      if (row[s] == SENT || !dead(tomb, row[s])) continue;
      const uint32_t p = row[s];
      const Entry* best = nullptr;
      for (const Entry& e : U) {
        if (taken.count(e.id)) continue;
        bool from_p = false;
        for (int t = 0; t < R && !from_p; ++t) from_p = snap[(size_t)p * R + t] == e.id;
        if (from_p && (!best || key_less(e, *best))) best = &e;
      }
      if (best) {
        out[s] = best->id;
        outd[s] = best->d;
        taken.insert(best->id);
      } else {
        out[s] = SENT;
        outd[s] = INF;
      }
    }
    // tail: kept live entries + the m nearest untaken members of U, sorted by key
    std::vector<Entry> tail;
    int m = 0;
    for (int s = P; s < R; ++s) {
      if (row[s] != SENT && !dead(tomb, row[s])) tail.push_back({rowd[s], row[s], false});
      else m++;
    }
    std::vector<Entry> rest;
    for (const Entry& e : U)
      if (!taken.count(e.id)) rest.push_back(e);
    std::sort(rest.begin(), rest.end(), key_less);
    for (int i = 0; i < m && i < (int)rest.size(); ++i) tail.push_back(rest[i]);
    std::sort(tail.begin(), tail.end(), key_less);
    for (int s = P; s < R; ++s) {
      const int i = s - P;
      out[s] = i < (int)tail.size() ? tail[i].id : SENT;
      outd[s] = i < (int)tail.size() ? tail[i].d : INF;
    }
    rewritten++;
  }
  *n_rewritten = rewritten;
  return 0;
}

// O6: merge of per-shard top-k lists (global ids) into the first k by key.
int orc_merge_topk(const uint32_t* ids, const float* d, int G, int64_t nq, int k, uint32_t* out_ids, float* out_d) {
  for (int64_t q = 0; q < nq; ++q) {
    std::vector<Entry> all;
    for (int g = 0; g < G; ++g)
      for (int i = 0; i < k; ++i) {
        size_t o = ((size_t)g * nq + q) * k + i;
        if (ids[o] != SENT) all.push_back({d[o], ids[o], false});
      }
    std::sort(all.begin(), all.end(), key_less);
    if ((int)all.size() > k) all.resize(k);
    emit(all, k, out_ids + q * k, out_d + q * k);
  }
  return 0;
}

}  // extern "C"
