// libsvf.so: the C ABI of include/svf.h — index state in HBM, host/device staging, validation, error handling.
// Every step of the method runs in the kernels of search.cu / link.cu / knn.cu; this file only marshals.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/svf.h"
#include "kernels.h"

using namespace svf;

struct svf_index {
  svf_params p{};
  int dev = 0, num_sms = 148, smem_optin = 227 * 1024, smem_sm = 228 * 1024;
  int D = 0, Dp = 0, dq = 0, R = 0, P = 0;
  int64_t cap = 0, n_alloc = 0, n_deleted = 0;
  float* vec = nullptr;
  uint32_t* graph = nullptr;
  float* edge_dist = nullptr;
  uint32_t* tomb = nullptr;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // [1] newly-deleted, [2] bad flag, [4] svf_search queue counter, [5] update-path (insert) queue counter,
  // [6] n_visible: ids whose insertion has completed on the device (the concurrent-search snapshot)
  unsigned long long* small = nullptr;
  void* sscratch = nullptr;             // svf_search staging (separate from the update path's scratch)
  size_t sscratch_bytes = 0;
  uint32_t* counters = nullptr;         // [nq][3] of the last search
  bool trace_on = false;                // per-query timeline of later searches (svf_set_trace)
  unsigned long long* trace = nullptr;
  int64_t trace_cap = 0, trace_nq = 0;
  int64_t counters_cap = 0, counters_nq = 0;
  cudaStream_t last_stream = nullptr;
  // streamed host queries (svf_search with a host Q): copy stream, chunk flags, pinned epoch ring
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_cs0 = nullptr, ev_cs1 = nullptr;
  unsigned int* q_flags = nullptr;
  unsigned int* h_epoch = nullptr;  // pinned ring of epoch values (copy sources)
  unsigned int epoch = 0;
  bool poisoned = false;
  int search_width = 1, n_init = 0, max_iter = 0, hash_bits = 0;
  int knn_mode = 0;                     // 0 auto (tcgen05 when supported), 1 FFMA only
  int wpq = 0;                          // warps per query: 0 auto, 1, 2
  double consolidate_ratio = 0.0;       // NEXT-4 trigger: deletions since the last consolidation / live then
  int64_t deleted_at_consolidation = 0;
  int64_t consolidations = 0;
  int last_launches = 0;                // kernels launched by the last run_search
  int ho_pct = -1;                      // pair-mode handoff threshold (% of one-warp warps): -1 auto, 0 off
  unsigned long long* ho = nullptr;     // handoff control words + slots of svf_search (handoff_words(), lazy)
  unsigned long long* ho_upd = nullptr; // the same for the update path's insert searches
  uint64_t knn_queries = 0, knn_fallbacks = 0, knn_tc_calls = 0;
  bool prof = false;
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_cnt[4] = {0, 0, 0, 0};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  struct ProfRec {
    cudaEvent_t a, b;
    int slot;
  };
  std::vector<ProfRec> prof_pending;  // recorded without synchronising; resolved by svf_profile_read
  std::vector<cudaEvent_t> ev_pool;
  std::mutex mu;
};

namespace {

thread_local std::string g_err;

svf_status fail(svf_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

svf_status cuda_fail(svf_index* idx, cudaError_t e, const char* what) {
  if (idx) idx->poisoned = true;
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return fail(e == cudaErrorMemoryAllocation ? SVF_ERR_OOM : SVF_ERR_CUDA, buf);
}

#define CK(idx, expr, what)                                \
  do {                                                     \
    cudaError_t e_ = (expr);                               \
    if (e_ != cudaSuccess) return cuda_fail(idx, e_, what); \
  } while (0)

bool is_device_ptr(const void* ptr) {
  if (ptr == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// grow-only scratch; reallocation synchronises the stream first (rare).  The update path (insert, delete, repair,
// build, exact kNN) uses `scratch`; svf_search stages through its own `sscratch`, so a search on one stream never
// shares a buffer with an update on another.
cudaError_t grow(void*& buf, size_t& have, size_t bytes, cudaStream_t st) {
  if (bytes <= have) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  if (buf) cudaFree(buf);
  buf = nullptr;
  have = 0;
  e = cudaMalloc(&buf, bytes);
  if (e != cudaSuccess) return e;
  have = bytes;
  return cudaSuccess;
}
cudaError_t ensure_sscratch(svf_index* idx, size_t bytes, cudaStream_t st) {
  return grow(idx->sscratch, idx->sscratch_bytes, std::max(bytes, (size_t)8 << 20), st);
}
cudaError_t ensure_scratch(svf_index* idx, size_t bytes, cudaStream_t st) {
  if (bytes <= idx->scratch_bytes) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  if (idx->scratch) cudaFree(idx->scratch);
  idx->scratch = nullptr;
  idx->scratch_bytes = 0;
  size_t want = std::max(bytes, (size_t)64 << 20);
  e = cudaMalloc(&idx->scratch, want);
  if (e != cudaSuccess) return e;
  idx->scratch_bytes = want;
  return cudaSuccess;
}

int pow2_at_least(int x) {
  int v = 1;
  while (v < x) v <<= 1;
  return v;
}

struct SearchCfg {
  int kpl, cpl, hbits, team, nv, n_init, wpq, lp, vc_bits, vc_slots;
  uint32_t vc_tmask;
  bool lp_auto;  // K-S-L cache sized by the launcher (no hash_bits / SVF_LP_BITS)
};

// K-S-L (shared-memory pool kernel) for pools of more than 64 keys; SVF_LP=0 keeps the register-pool kernel (A/B)
bool lp_enabled() {
  static const bool on = [] {
    const char* v = getenv("SVF_LP");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}
// SVF_LP_U32=1 forces u32 cache entries (A/B of the 16-bit tagged cache)
bool lp_u32_cache() {
  static const bool on = [] {
    const char* v = getenv("SVF_LP_U32");
    return v != nullptr && atoi(v) != 0;
  }();
  return on;
}
// K-S-L visited-cache size override (2^bits direct-mapped slots) for tuning; 0 = sized by lp_cache_slots
int lp_bits_env() {
  static const int env = [] {
    const char* v = getenv("SVF_LP_BITS");
    return v ? atoi(v) : 0;
  }();
  return env;
}
#ifndef SVF_MINB_LP
#define SVF_MINB_LP 7
#endif
// Default K-S-L visited-cache slots: pools of <= 256 keys run at SVF_MINB_LP blocks/SM (their register limit), so the
// cache gets whatever shared memory that residency leaves once the pool and buffers are placed (C2 L_insert 128: 3120
// 16-bit slots, C4 itopk 192: 2864; a power-of-two 2048 before round 2 recomputed 1.5x the oracle's distances, and
// 4096 cost two blocks/SM: profiles/r02_lp_cache.json); larger pools keep 4096 slots at lower residency.
int lp_cache_slots(const svf_index* idx, int L, int cpl, bool c16, int minb) {
  if (L > 256) return 4096;
  // 1 KB per block is reserved by the system; blocks are allocated in 128-byte units
  const long per_block = ((long)idx->smem_sm / minb - 1024) & ~127L;
  const long per_warp = (per_block / kSearchWarpsPerBlock) & ~15L;
  // all but the cache: the per-warp layout with an 8-slot cache, minus that cache region (which also stages the
  // query row, so it is at least Dp floats)
  const long c8 = ((std::max<long>(8L * (c16 ? 2 : 4), (long)idx->Dp * 4)) + 15) & ~15L;
  const long fixed = (long)search_smem_bytes(8, 0, cpl, L, 1, c16 ? 1 : 0, idx->Dp, 8) / kSearchWarpsPerBlock - c8;
  const long m = (per_warp - fixed) / (c16 ? 2 : 4);
  return (int)std::max(256L, m & ~7L);
}

// K-S-L visited cache of a configuration: 2^bits slots, or (bits = 0) sized for `minb` resident blocks per SM
void lp_cache_cfg(const svf_index* idx, int L, int cpl, int bits, int minb, SearchCfg& c) {
  // ids are < 2^B; 16-bit tags when a slot's run of hashed ids, ceil(2^B / M), fits 15 bits (DESIGN §6 K-S-L)
  int B = 1;
  while (B < 32 && ((int64_t)1 << B) < idx->cap) ++B;
  auto fits16 = [&](int M) {
    const uint64_t run = (((uint64_t)1 << B) + M - 1) / M;
    return B <= 31 && run <= 32768 && !lp_u32_cache();
  };
  int M = bits > 0 ? (1 << std::min(bits, 16)) : lp_cache_slots(idx, L, cpl, true, minb);
  c.vc_bits = fits16(M) ? B : 0;
  if (!c.vc_bits && bits == 0) M = lp_cache_slots(idx, L, cpl, false, minb);
  c.vc_slots = M;
  c.vc_tmask = 0;
  if (c.vc_bits) {
    const uint64_t run = (((uint64_t)1 << B) + M - 1) / M;
    int tb = 0;
    while (((uint64_t)1 << tb) < run) ++tb;
    c.vc_tmask = (1u << tb) - 1u;
  }
  c.hbits = 8;
  while ((1 << c.hbits) < M) ++c.hbits;  // reported only (svf_last_search_counters); K-S-L uses vc_slots
}

bool search_cfg(const svf_index* idx, int L, int p, int n_init, int hash_bits, SearchCfg& c, std::string& why) {
  if (p < 1 || p > 8) return why = "search_width must be in [1, 8]", false;
  const int LP = pow2_at_least(std::max(L, 32));
  const int MP = pow2_at_least(std::max(p * idx->R, 32));
  if (LP > 512) return why = "itopk must be <= 512", false;
  if (MP > 256) return why = "search_width * degree must be <= 256", false;
  c.kpl = LP / 32;
  c.cpl = MP / 32;
  int minbits = 1;
  while ((1 << minbits) < 4 * std::max(LP, MP)) ++minbits;  // forgetful-table invariant (I7)
  while ((1 << minbits) < idx->Dp) ++minbits;                  // the table also stages the query row
  // default: small tables buy occupancy (the search is latency-bound); forgetting costs ~10% extra distances
  // at small L (measured: C2 L=14, 1024 slots 9.9M QPS vs 2048 slots 9.5M vs 4096 slots 7.3M)
  // 2048 slots up to L = 128 (C3 10M x 96 at L = 96: 4.96 vs 5.40 ms with 4096 slots, C2 inserts at L = 128
  // 7.1 vs 7.2 ms; tools/param_sweep.py, tools/insert_rate.py)
  // 4096 slots for 128 < L <= 256 (C4 2M x 200, L_build 512: itopk 192 27.5 -> 15.4 ms, 256 37.6 -> 19.7 ms vs
  // 8192 slots, identical results; 2048 slots is 2% faster again but recomputes 1.6x; profiles/c4_2m_hash.json)
  // 1024 slots up to L = 32 (C3 itopk 20 cap 35, round 2: 1.050 -> 1.001 ms per 10K batch, 6 blocks/SM instead of 5;
  // 512 slots: 1.044 ms; C2 itopk 10: 512 slots 0.599 vs 0.573 ms; profiles/r02_ks_ab.json)
  const int autobits = L <= 32 ? 10 : (L <= 128 ? 11 : (L <= 256 ? 12 : 13));
  // K-S-L for pools of more than 64 keys (one warp per query): its direct-mapped visited cache needs no load
  // invariant, only room to stage the query row
  c.lp = LP > 64 && idx->wpq != 2 && lp_enabled();
  c.vc_bits = 0;
  c.vc_slots = 0;
  c.vc_tmask = 0;
  c.lp_auto = false;
  if (c.lp) {
    const int bits = hash_bits > 0 ? std::max(hash_bits, 8) : lp_bits_env();
    c.lp_auto = bits == 0;
    lp_cache_cfg(idx, L, c.cpl, bits, SVF_MINB_LP, c);
  } else {
    c.hbits = hash_bits > 0 ? std::max(hash_bits, minbits) : std::max(autobits, minbits);
  }
  if (c.hbits > 15) return why = "hash_bits too large", false;
  // a configuration whose block does not fit the opt-in shared memory is refused up front (INVALID, index intact)
  if (search_smem_bytes(c.hbits, c.kpl, c.cpl, L, c.lp, c.vc_bits, idx->Dp, c.vc_slots) > (size_t)idx->smem_optin)
    return why = "hash_bits too large: the search block's visited tables exceed the shared memory per block", false;
  c.team = pow2_at_least((idx->dq + 3) / 4);
  c.nv = (idx->dq + c.team - 1) / c.team;
  c.n_init = n_init > 0 ? n_init : L;
  c.wpq = idx->wpq == 2 ? 2 : 1;  // 0 (auto) is resolved per call from the batch size in run_search
  return true;
}

cudaEvent_t pool_event(svf_index* idx) {
  if (!idx->ev_pool.empty()) {
    cudaEvent_t e = idx->ev_pool.back();
    idx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_begin(svf_index* idx, cudaStream_t st, cudaEvent_t* a) {
  *a = nullptr;
  if (!idx->prof) return;
  *a = pool_event(idx);
  cudaEventRecord(*a, st);
}
void prof_end(svf_index* idx, cudaStream_t st, cudaEvent_t a, int slot) {
  if (!idx->prof || !a) return;
  cudaEvent_t b = pool_event(idx);
  cudaEventRecord(b, st);
  idx->prof_pending.push_back({a, b, slot});
}
void prof_resolve(svf_index* idx) {
  for (auto& r : idx->prof_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    idx->prof_ms[r.slot] += ms;
    idx->prof_cnt[r.slot] += 1;
    idx->ev_pool.push_back(r.a);
    idx->ev_pool.push_back(r.b);
  }
  idx->prof_pending.clear();
}

// Host queries are copied in chunks on the index's copy stream, each chunk followed by a 4-byte flag copy (copy
// engine only: no SM is needed to publish it, so a search grid spinning on the flags cannot starve it); the search
// starts at once and each query waits for its chunk.  Epochs make stale flags of earlier calls harmless.
struct StreamedQ {
  bool active;
  unsigned int* flags;
  unsigned int epoch;
  int chunk_log2;
};
constexpr int kMaxQChunks = 4096;
cudaError_t stream_queries(svf_index* idx, const float* Q, int64_t nq, char* dst, cudaStream_t st, StreamedQ& sq) {
  cudaError_t e;
  if (idx->cstream == nullptr) {
    if ((e = cudaStreamCreateWithFlags(&idx->cstream, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&idx->ev_cs0, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&idx->ev_cs1, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&idx->q_flags, kMaxQChunks * 4)) != cudaSuccess) return e;
    if ((e = cudaMemset(idx->q_flags, 0, kMaxQChunks * 4)) != cudaSuccess) return e;
    if ((e = cudaHostAlloc(&idx->h_epoch, 64 * 4, cudaHostAllocDefault)) != cudaSuccess) return e;
  }
  int lg = 9;  // 512 queries per chunk (256 KB at D = 128)
  while ((nq + (1LL << lg) - 1) >> lg > kMaxQChunks) ++lg;
  const int64_t nchunks = (nq + (1LL << lg) - 1) >> lg;
  // the previous call's chunk copies have run (normally long ago), so no pending copy still reads a ring slot
  if ((e = cudaEventSynchronize(idx->ev_cs1)) != cudaSuccess) return e;
  idx->epoch = idx->epoch + 1 == 0 ? 1 : idx->epoch + 1;
  unsigned int* src = idx->h_epoch + (idx->epoch & 63);
  *src = idx->epoch;
  // the copy stream starts after everything already queued on st (the staging buffer may still be in use)
  if ((e = cudaEventRecord(idx->ev_cs0, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(idx->cstream, idx->ev_cs0, 0)) != cudaSuccess) return e;
  const size_t row = (size_t)idx->D * 4;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t r0 = c << lg, r1 = std::min<int64_t>(nq, (c + 1) << lg);
    if ((e = cudaMemcpyAsync(dst + r0 * row, Q + r0 * idx->D, (size_t)(r1 - r0) * row, cudaMemcpyHostToDevice,
                             idx->cstream)) != cudaSuccess)
      return e;
    if ((e = cudaMemcpyAsync(idx->q_flags + c, src, 4, cudaMemcpyHostToDevice, idx->cstream)) != cudaSuccess) return e;
  }
  // later work on st (the next call's staging) waits for the copies
  if ((e = cudaEventRecord(idx->ev_cs1, idx->cstream)) != cudaSuccess) return e;
  sq = {true, idx->q_flags, idx->epoch, lg};
  return cudaSuccess;
}

// default handoff threshold: 45% of the one-warp grid's warps (C2, itopk 14, tools/tail_sweep.py: 10K batch
// 0.836 -> 0.758 ms, 20K 1.359 -> 1.313 ms, 40K 2.553 -> 2.479 ms; 25/35/55% were no better at any batch);
// SVF_HANDOFF overrides it for tuning
int handoff_auto() {
  static const int env = [] {
    const char* v = getenv("SVF_HANDOFF");
    return v ? atoi(v) : -1;
  }();
  return env >= 0 ? env : 45;
}

// run K-S on the index: Q (device) with row stride q_stride and q_dim valid floats
cudaError_t run_search(svf_index* idx, const float* Q, int64_t q_stride, int q_dim, int64_t nq, uint64_t n_snapshot,
                       uint64_t qidx_base, int L, int n_out, const SearchCfg& c, int p, int max_iter,
                       uint32_t* out_ids, float* out_d, uint32_t* counters, int prof_slot, cudaStream_t st,
                       bool update_path, const StreamedQ* sq = nullptr) {
  SearchArgs a{};
  a.vec = idx->vec;
  a.dq = idx->dq;
  a.graph = idx->graph;
  a.R = idx->R;
  a.rshift = (idx->R & (idx->R - 1)) == 0 ? __builtin_ctz((unsigned)idx->R) : -1;
  a.tomb = idx->n_deleted > 0 ? idx->tomb : nullptr;
  a.n_alloc = n_snapshot;
  a.Q = Q;
  a.q_stride = q_stride;
  a.q_dim = q_dim;
  a.nq = nq;
  a.qidx_base = qidx_base;
  a.L = L;
  a.p = p;
  a.n_init = c.n_init;
  a.max_iter = max_iter;
  a.metric = idx->p.metric;
  a.seed = idx->p.seed;
  a.team = c.team;
  a.nv = c.nv;
  a.hbits = c.hbits;
  a.n_out = n_out;
  a.out_ids = out_ids;
  a.out_d = out_d;
  a.counters = counters;
  a.trace = idx->trace_on && counters != nullptr && idx->trace_cap >= nq ? idx->trace : nullptr;
  a.q_flags = sq ? sq->flags : nullptr;
  a.q_epoch = sq ? sq->epoch : 0u;
  a.q_chunk_log2 = sq ? sq->chunk_log2 : 0;
  // the two paths own disjoint queue counters and handoff buffers, so an svf_search on one stream may overlap an
  // update on another; svf_search snapshots n at each query's start from n_visible
  a.work_counter = idx->small + (update_path ? 5 : 4);
  a.n_visible = update_path ? nullptr : idx->small + 6;
  // pair mode (2 warps per query, identical results) cuts per-query latency ~35% (C2 itopk 14: batch 1 p50
  // 0.151 -> 0.091 ms, batch 1024 0.348 -> 0.239 ms; profiles/r01_latency_c2.json) but costs throughput once the
  // batch fills the resident warps (4096: 0.51 vs 0.57 ms, 10K: 0.85 vs 1.20 ms).  Automatic: 2 while the batch
  // needs at most half of the resident warp slots (~24 per SM), else 1.
  a.wpq = c.wpq;
  if (idx->wpq == 0) a.wpq = (c.cpl >= 2 && c.kpl <= 4 && 2 * nq <= 24LL * idx->num_sms) ? 2 : 1;
  a.large_pool = c.lp && a.wpq == 1;
  SearchCfg cl = c;
  // wide rows (D >= 192: DRAM-bound, ncu C4 67% of DRAM peak) in a batch of more than ~1.25 waves of the 7-block
  // residency: the K-S-L cache is sized for 6 blocks/SM, trading residency for fewer recomputed 800-byte rows (C4
  // itopk 192 10K: 10.74-10.94 -> 10.52 ms, 6018 -> 5878 distances per query).  At D = 128 (38% of DRAM peak) the
  // same trade was slower (C2 itopk 128 10K 3.017 -> 3.049 ms), and a 4,096-query insert sub-batch keeps one wave.
  if (a.large_pool && c.lp_auto && idx->Dp >= 192 && nq * 4 > 5LL * SVF_MINB_LP * kSearchWarpsPerBlock * idx->num_sms)
    lp_cache_cfg(idx, L, c.cpl, 0, SVF_MINB_LP - 1, cl);
  a.vc_bits = cl.vc_bits;
  a.vc_slots = cl.vc_slots;
  a.vc_tmask = cl.vc_tmask;
  cudaError_t e = cudaMemsetAsync(a.work_counter, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  unsigned long long*& hob = update_path ? idx->ho_upd : idx->ho;
  // one-warp batches: stragglers are handed to a chained pair-mode grid once few warps are left (SearchArgs::ho)
  a.ho = nullptr;
  a.ho_thresh = a.wpq == 1 ? (idx->ho_pct >= 0 ? idx->ho_pct : handoff_auto()) : 0;
  if (a.ho_thresh > 0 && c.kpl <= kHandoffMaxKpl && c.cpl >= 2 && !a.large_pool) {
    if (hob == nullptr) {
      e = cudaMalloc(&hob, handoff_words() * 8);
      if (e != cudaSuccess) return e;
      e = cudaMemset(hob, 0, handoff_words() * 8);  // slot headers start free; resumed slots are re-freed
      if (e != cudaSuccess) return e;
    }
    a.ho = hob;
    e = cudaMemsetAsync(hob, 0, 8 * 8, st);       // control words
    if (e != cudaSuccess) return e;
  }
  idx->last_launches = a.ho != nullptr ? 2 : 1;
  if (e != cudaSuccess) return e;
  cudaEvent_t pa = nullptr;
  if (prof_slot >= 0) prof_begin(idx, st, &pa);
  e = launch_search(a, c.kpl, c.cpl, idx->num_sms, st);
  if (e != cudaSuccess) return e;
  prof_end(idx, st, pa, prof_slot);
  return cudaSuccess;
}

template <class F>
cudaError_t timed(svf_index* idx, int slot, cudaStream_t st, F f) {
  cudaEvent_t pa;
  prof_begin(idx, st, &pa);
  cudaError_t e = f();
  if (e != cudaSuccess) return e;
  prof_end(idx, st, pa, slot);
  return cudaSuccess;
}

// copy n rows (dim floats, contiguous, host or device) into vec rows [first, first+n), zero-padded to Dp
cudaError_t put_rows(svf_index* idx, const float* X, int64_t first, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  float* dst = idx->vec + (size_t)first * idx->Dp;
  if (X == nullptr) return cudaMemsetAsync(dst, 0, (size_t)n * idx->Dp * 4, st);
  if (idx->Dp == idx->D) return cudaMemcpyAsync(dst, X, (size_t)n * idx->D * 4, cudaMemcpyDefault, st);
  cudaError_t e = cudaMemsetAsync(dst, 0, (size_t)n * idx->Dp * 4, st);
  if (e != cudaSuccess) return e;
  return cudaMemcpy2DAsync(dst, (size_t)idx->Dp * 4, X, (size_t)idx->D * 4, (size_t)idx->D * 4, (size_t)n,
                           cudaMemcpyDefault, st);
}

svf_status validate_params(const svf_params* p) {
  if (!p) return fail(SVF_ERR_INVALID, "params is NULL");
  if (p->dim < 1 || p->dim > 512) return fail(SVF_ERR_INVALID, "dim must be in [1, 512]");
  if (p->degree < 2 || p->degree > 128) return fail(SVF_ERR_INVALID, "degree must be in [2, 128]");
  if (p->metric != SVF_L2 && p->metric != SVF_IP) return fail(SVF_ERR_INVALID, "metric must be SVF_L2 or SVF_IP");
  if (p->capacity < 1 || p->capacity > 0x7FFFFFFFll) return fail(SVF_ERR_INVALID, "capacity must be in [1, 2^31-1]");
  if (p->search_width < 1 || p->search_width > 8) return fail(SVF_ERR_INVALID, "search_width must be in [1, 8]");
  if (p->insert_itopk < 1 || p->insert_itopk > 512) return fail(SVF_ERR_INVALID, "insert_itopk must be in [1, 512]");
  if (p->build_itopk < 0 || p->build_itopk > 512) return fail(SVF_ERR_INVALID, "build_itopk must be in [0, 512]");
  if (p->protect_prefix < -1 || p->protect_prefix > p->degree) return fail(SVF_ERR_INVALID, "bad protect_prefix");
  if (p->insert_batch < 1) return fail(SVF_ERR_INVALID, "insert_batch must be >= 1");
  if (p->seed_size < 1) return fail(SVF_ERR_INVALID, "seed_size must be >= 1");
  if (p->n_init < 0 || p->max_iter < 0) return fail(SVF_ERR_INVALID, "n_init / max_iter must be >= 0");
  return SVF_OK;
}

svf_status alloc_index(const svf_params* p, svf_index** out) {
  svf_status s = validate_params(p);
  if (s != SVF_OK) return s;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SVF_ERR_CUDA, "no CUDA device available (libsvf has no CPU path)");
  }
  if (p->device < 0 || p->device >= ndev) return fail(SVF_ERR_INVALID, "device ordinal out of range");
  DeviceGuard g(p->device);
  svf_index* idx = new svf_index();
  idx->p = *p;
  idx->dev = p->device;
  cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, p->device);
  cudaDeviceGetAttribute(&idx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
  cudaDeviceGetAttribute(&idx->smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, p->device);
  idx->D = p->dim;
  idx->Dp = (p->dim + 3) / 4 * 4;
  idx->dq = idx->Dp / 4;
  idx->R = p->degree;
  idx->P = p->protect_prefix < 0 ? p->degree / 2 : p->protect_prefix;
  idx->cap = p->capacity;
  idx->search_width = p->search_width;
  idx->n_init = p->n_init;
  idx->max_iter = p->max_iter;
  idx->hash_bits = p->hash_bits;
  cudaError_t e;
  const size_t cap = (size_t)idx->cap;
  if ((e = cudaMalloc(&idx->vec, cap * idx->Dp * 4)) != cudaSuccess ||
      (e = cudaMalloc(&idx->graph, cap * idx->R * 4)) != cudaSuccess ||
      (e = cudaMalloc(&idx->edge_dist, cap * idx->R * 4)) != cudaSuccess ||
      (e = cudaMalloc(&idx->tomb, (cap + 31) / 32 * 4)) != cudaSuccess ||
      (e = cudaMalloc(&idx->small, 64)) != cudaSuccess || (e = cudaMemset(idx->small, 0, 64)) != cudaSuccess ||
      (e = cudaMemset(idx->tomb, 0, (cap + 31) / 32 * 4)) != cudaSuccess ||
      (e = cudaEventCreate(&idx->ev0)) != cudaSuccess || (e = cudaEventCreate(&idx->ev1)) != cudaSuccess) {
    svf_destroy(idx);
    return cuda_fail(nullptr, e, "allocating the index arenas");
  }
  *out = idx;
  return SVF_OK;
}

// insertion of rows [n_alloc, n_alloc + n) already present in vec (sub-batch snapshots, I13)
svf_status insert_present_rows(svf_index* idx, int64_t n, int L, cudaStream_t st) {
  SearchCfg c;
  std::string why;
  if (!search_cfg(idx, L, idx->p.search_width, idx->p.n_init, idx->hash_bits, c, why))
    return fail(SVF_ERR_INVALID, why);
  const int64_t B = std::min<int64_t>(idx->p.insert_batch, std::max<int64_t>(n, 1));
  const size_t cand_bytes = al((size_t)B * L * 4);
  const size_t rev_bytes = reverse_scratch_bytes(B, idx->R);
  CK(idx, ensure_scratch(idx, 2 * cand_bytes + al(rev_bytes), st), "allocating insert scratch");
  uint32_t* cid = static_cast<uint32_t*>(idx->scratch);
  float* cd = reinterpret_cast<float*>(static_cast<char*>(idx->scratch) + cand_bytes);
  void* rev = static_cast<char*>(idx->scratch) + 2 * cand_bytes;
  CK(idx, launch_fill_rows(idx->graph, idx->edge_dist, idx->n_alloc, n, idx->R, st), "fill rows");
  int64_t done = 0;
  while (done < n) {
    const int64_t snap = idx->n_alloc + done;
    const int64_t bsz = std::min<int64_t>({(int64_t)idx->p.insert_batch, snap, n - done});
    // (i) insert-mode search over the snapshot: the sub-batch's own rows are neither reachable nor sampled
    CK(idx,
       run_search(idx, idx->vec + (size_t)snap * idx->Dp, idx->Dp, idx->Dp, bsz, (uint64_t)snap, (uint64_t)snap, L,
                  L, c, idx->p.search_width, idx->p.max_iter, cid, cd, nullptr, 1, st, true),
       "insert search");
    // (ii) detour-ranked forward rows
    CK(idx, timed(idx, 2, st, [&] {
         return launch_detour_select(idx->graph, idx->edge_dist, idx->R, idx->P, snap, bsz, cid, cd, L, st);
       }), "detour select");
    // (iii) reverse edges
    CK(idx, timed(idx, 3, st, [&] {
         return launch_reverse(idx->graph, idx->edge_dist, idx->n_deleted > 0 ? idx->tomb : nullptr, idx->R, idx->P,
                               snap, bsz, rev, idx->scratch_bytes - 2 * cand_bytes, st);
       }), "reverse edges");
    done += bsz;
    // the sub-batch is linked: concurrent searches may now see it
    CK(idx, launch_store_u64(idx->small + 6, (uint64_t)(snap + bsz), st), "publish n_visible");
  }
  idx->n_alloc += n;
  return SVF_OK;
}

// the exact-kNN pruning bound from a short graph search (DESIGN §6 K-G); SVF_KNN_BOUND=0 keeps the sample pass (A/B)
bool knn_graph_bound() {
  static const bool on = [] {
    const char* v = getenv("SVF_KNN_BOUND");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}

// exact kNN over ids [0, n): tcgen05 TF32 path when supported, else the FFMA tile kernel.  With a built graph over
// those ids (svf_knn_exact), a capped K-S search first gives k live rows per query whose exact k-th distance bounds
// the true k-th from above: the tensor-core pass prunes with it (any such bound keeps the result exact: K-R's
// certificate and the FFMA fallback do not depend on it), replacing the slower sample pass.
cudaError_t run_knn(svf_index* idx, int64_t n, const uint32_t* tomb, const float* Q, int64_t q_stride, int q_dim,
                    int64_t nq, int k, int64_t self_base, uint32_t* oi, float* od, cudaStream_t st) {
  const bool tc = idx->knn_mode == 0 && knn_tc_supported(idx->dq, q_stride, Q, k);
  SearchCfg sc{};
  std::string why;
  const int Lb = std::max(k, 16);
  const bool bound = tc && self_base < 0 && n == idx->n_alloc && n >= 262144 && nq >= 512 && knn_graph_bound() &&
                     Lb <= 64 && search_cfg(idx, Lb, 1, 0, 0, sc, why);
  const size_t bb = bound ? 2 * al((size_t)nq * k * 4) : 0;
  const size_t need = bb + (tc ? knn_tc_scratch_bytes(nq, n, idx->dq, k) : knn_scratch_bytes(nq, k, std::max<int64_t>(n, 1)));
  cudaError_t e = ensure_scratch(idx, need, st);
  if (e != cudaSuccess) return e;
  idx->knn_queries += (uint64_t)nq;
  if (!tc)
    return launch_knn_exact(idx->vec, idx->dq, n, tomb, Q, q_stride, q_dim, nq, k, idx->p.metric, self_base, oi, od,
                            idx->scratch, idx->scratch_bytes, idx->num_sms, st);
  const float* bound_d = nullptr;
  if (bound) {
    uint32_t* b_ids = static_cast<uint32_t*>(idx->scratch);
    float* b_d = reinterpret_cast<float*>(static_cast<char*>(idx->scratch) + bb / 2);
    e = run_search(idx, Q, q_stride, q_dim, nq, (uint64_t)n, 0, Lb, k, sc, 1, 16, b_ids, b_d, nullptr, -1, st, true);
    if (e != cudaSuccess) return e;
    bound_d = b_d;
  }
  uint32_t fb = 0;
  e = launch_knn_tc(idx->vec, idx->dq, n, tomb, Q, q_stride, q_dim, nq, k, idx->p.metric, self_base, oi, od,
                    static_cast<char*>(idx->scratch) + bb, idx->scratch_bytes - bb, idx->num_sms, st, &fb, bound_d);
  idx->knn_fallbacks += fb;
  idx->knn_tc_calls += 1;
  return e;
}

svf_status enter(svf_index* idx) {
  if (!idx) return fail(SVF_ERR_INVALID, "index is NULL");
  if (idx->poisoned) return fail(SVF_ERR_POISONED, "index poisoned by an earlier CUDA failure");
  return SVF_OK;
}

}  // namespace

extern "C" {

void svf_default_params(svf_params* p, int32_t dim, int32_t degree) {
  std::memset(p, 0, sizeof *p);
  p->dim = dim;
  p->degree = degree;
  p->metric = SVF_L2;
  p->capacity = 0;
  p->search_width = 1;
  p->n_init = 0;
  p->max_iter = 0;
  p->insert_itopk = 128;
  p->protect_prefix = -1;
  p->insert_batch = 4096;
  p->seed_size = 4096;
  p->hash_bits = 0;
  p->seed = 42;
  p->device = 0;
}

const char* svf_last_error(void) { return g_err.c_str(); }

svf_status svf_build(const svf_params* p, const float* X, int64_t n, void* stream, svf_index** out) {
  if (!out || !X) return fail(SVF_ERR_INVALID, "NULL argument");
  if (n < 1) return fail(SVF_ERR_INVALID, "svf_build needs n >= 1");
  if (p && p->capacity < n) return fail(SVF_ERR_CAPACITY, "capacity < n");
  svf_index* idx = nullptr;
  svf_status s = alloc_index(p, &idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto bail = [&](svf_status s2) {
    svf_destroy(idx);
    return s2;
  };
  if (put_rows(idx, X, 0, n, st) != cudaSuccess) return bail(cuda_fail(nullptr, cudaGetLastError(), "copy X"));
  // seed: exact R-NN of the first n0 rows (self excluded), written straight into the rows (prefix|tail layout)
  const int64_t n0 = std::min<int64_t>(n, idx->p.seed_size);
  cudaError_t e = run_knn(idx, n0, nullptr, idx->vec, idx->Dp, idx->Dp, n0, idx->R, 0, idx->graph,
                          idx->edge_dist, st);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "seed exact R-NN"));
  idx->n_alloc = n0;
  if (n > n0) {
    s = insert_present_rows(idx, n - n0, idx->p.build_itopk ? idx->p.build_itopk : idx->p.insert_itopk, st);
    if (s != SVF_OK) return bail(s);
  }
  if ((e = launch_store_u64(idx->small + 6, (uint64_t)idx->n_alloc, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return bail(cuda_fail(nullptr, e, "build"));
  *out = idx;
  return SVF_OK;
}

svf_status svf_import(const svf_params* p, const float* vec, const uint32_t* graph, const float* edge_dist,
                      const uint32_t* tomb, int64_t n_alloc, svf_index** out) {
  if (!out || !vec || !graph) return fail(SVF_ERR_INVALID, "NULL argument");
  if (n_alloc < 0 || (p && n_alloc > p->capacity)) return fail(SVF_ERR_CAPACITY, "n_alloc > capacity");
  svf_index* idx = nullptr;
  svf_status s = alloc_index(p, &idx);
  if (s != SVF_OK) return s;
  DeviceGuard g(idx->dev);
  cudaError_t e;
  const size_t nr = (size_t)n_alloc * idx->R;
  if ((e = put_rows(idx, vec, 0, n_alloc, nullptr)) != cudaSuccess ||
      (e = cudaMemcpy(idx->graph, graph, nr * 4, cudaMemcpyDefault)) != cudaSuccess) {
    svf_destroy(idx);
    return cuda_fail(nullptr, e, "import copy");
  }
  if (edge_dist) {
    e = cudaMemcpy(idx->edge_dist, edge_dist, nr * 4, cudaMemcpyDefault);
  } else {
    std::vector<float> inf(nr, __builtin_inff());
    e = cudaMemcpy(idx->edge_dist, inf.data(), nr * 4, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && tomb) {
    const size_t words = ((size_t)n_alloc + 31) / 32;
    std::vector<uint32_t> h(words);
    e = cudaMemcpy(h.data(), tomb, words * 4, cudaMemcpyDefault);
    if (e == cudaSuccess) {
      if (n_alloc % 32) h[words - 1] &= (1u << (n_alloc % 32)) - 1u;
      int64_t cnt = 0;
      for (uint32_t w : h) cnt += __builtin_popcount(w);
      idx->n_deleted = cnt;
      e = cudaMemcpy(idx->tomb, h.data(), words * 4, cudaMemcpyHostToDevice);
    }
  }
  if (e == cudaSuccess) e = launch_store_u64(idx->small + 6, (uint64_t)n_alloc, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    svf_destroy(idx);
    return cuda_fail(nullptr, e, "import copy");
  }
  idx->n_alloc = n_alloc;
  *out = idx;
  return SVF_OK;
}

svf_status svf_search(svf_index* idx, const float* Q, int64_t nq, int32_t k, int32_t itopk, uint32_t* out_ids,
                      float* out_dists, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (nq < 0) return fail(SVF_ERR_INVALID, "nq < 0");
  if (nq == 0) return SVF_OK;
  if (!Q || !out_ids || !out_dists) return fail(SVF_ERR_INVALID, "NULL argument");
  if (k < 1 || itopk < k) return fail(SVF_ERR_INVALID, "need 1 <= k <= itopk");
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SearchCfg c;
  std::string why;
  if (!search_cfg(idx, itopk, idx->search_width, idx->n_init, idx->hash_bits, c, why))
    return fail(SVF_ERR_INVALID, why);
  const bool q_dev = is_device_ptr(Q), i_dev = is_device_ptr(out_ids), d_dev = is_device_ptr(out_dists);
  const size_t qb = q_dev ? 0 : al((size_t)nq * idx->D * 4);
  const size_t ob = al((size_t)nq * k * 4);
  CK(idx, ensure_sscratch(idx, qb + 2 * ob, st), "search scratch");
  char* sp = static_cast<char*>(idx->sscratch);
  const float* Qd = Q;
  StreamedQ sq{};
  if (!q_dev) {
    CK(idx, stream_queries(idx, Q, nq, sp, st, sq), "H2D queries");
    Qd = reinterpret_cast<const float*>(sp);
  }
  uint32_t* oi = i_dev ? out_ids : reinterpret_cast<uint32_t*>(sp + qb);
  float* od = d_dev ? out_dists : reinterpret_cast<float*>(sp + qb + ob);
  if (idx->counters_cap < nq) {
    if (idx->counters) cudaFree(idx->counters);
    idx->counters = nullptr;
    idx->counters_cap = 0;
    CK(idx, cudaMalloc(&idx->counters, (size_t)nq * 3 * 4), "counters");
    idx->counters_cap = nq;
  }
  idx->counters_nq = nq;
  if (idx->trace_on && idx->trace_cap < nq) {
    if (idx->trace) cudaFree(idx->trace);
    idx->trace = nullptr;
    idx->trace_cap = 0;
    CK(idx, cudaMalloc(&idx->trace, (size_t)nq * kTraceCols * 8), "trace");
    idx->trace_cap = nq;
  }
  if (idx->trace_on) idx->trace_nq = nq;
  idx->last_stream = st;
  CK(idx,
     run_search(idx, Qd, idx->D, idx->D, nq, (uint64_t)idx->n_alloc, 0, itopk, k, c, idx->search_width,
                idx->max_iter, oi, od, idx->counters, 0, st, false, sq.active ? &sq : nullptr),
     "search kernel");
  if (sq.active) CK(idx, cudaStreamWaitEvent(st, idx->ev_cs1, 0), "join copy stream");
  if (!i_dev) CK(idx, cudaMemcpyAsync(out_ids, oi, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
  if (!d_dev) CK(idx, cudaMemcpyAsync(out_dists, od, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H dists");
  if (!i_dev || !d_dev) CK(idx, cudaStreamSynchronize(st), "search sync");
  return SVF_OK;
}

svf_status svf_insert(svf_index* idx, const float* X, int64_t n, uint32_t* out_ids, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (n < 0) return fail(SVF_ERR_INVALID, "n < 0");
  if (n == 0) return SVF_OK;
  if (!X) return fail(SVF_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lk(idx->mu);
  if (idx->n_alloc < 1) return fail(SVF_ERR_INVALID, "insert into an empty index (build it first)");
  if (idx->n_alloc + n > idx->cap) return fail(SVF_ERR_CAPACITY, "n_alloc + n > capacity");
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t first = idx->n_alloc;
  CK(idx, put_rows(idx, X, first, n, st), "copy X");
  s = insert_present_rows(idx, n, idx->p.insert_itopk, st);
  if (s != SVF_OK) return s;
  if (out_ids) {
    std::vector<uint32_t> h((size_t)n);
    for (int64_t i = 0; i < n; ++i) h[i] = (uint32_t)(first + i);
    CK(idx, cudaMemcpyAsync(out_ids, h.data(), (size_t)n * 4, cudaMemcpyDefault, st), "ids");
    CK(idx, cudaStreamSynchronize(st), "insert sync");
  }
  return SVF_OK;
}

static svf_status consolidate_impl(svf_index* idx, int64_t* n_rewritten, cudaStream_t st);

svf_status svf_delete(svf_index* idx, const uint32_t* ids, int64_t n, int64_t* n_newly_deleted, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (n < 0) return fail(SVF_ERR_INVALID, "n < 0");
  if (n_newly_deleted) *n_newly_deleted = 0;
  if (n == 0) return SVF_OK;
  if (!ids) return fail(SVF_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint32_t* d_ids = ids;
  if (!is_device_ptr(ids)) {
    CK(idx, ensure_scratch(idx, al((size_t)n * 4), st), "delete scratch");
    CK(idx, cudaMemcpyAsync(idx->scratch, ids, (size_t)n * 4, cudaMemcpyHostToDevice, st), "H2D ids");
    d_ids = static_cast<const uint32_t*>(idx->scratch);
  }
  unsigned long long* newly = idx->small + 1;
  unsigned int* bad = reinterpret_cast<unsigned int*>(idx->small + 2);
  CK(idx, cudaMemsetAsync(idx->small + 1, 0, 16, st), "memset");
  CK(idx, launch_tomb_check(d_ids, n, (uint64_t)idx->n_alloc, bad, st), "tomb check");
  unsigned int hbad = 0;
  CK(idx, cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st), "D2H");
  CK(idx, cudaStreamSynchronize(st), "delete sync");
  if (hbad) return fail(SVF_ERR_NOT_FOUND, "delete of an id >= n_alloc (nothing deleted)");
  CK(idx, timed(idx, 3, st, [&] { return launch_tomb_set(d_ids, n, idx->tomb, newly, st); }), "tomb set");
  unsigned long long hn = 0;
  CK(idx, cudaMemcpyAsync(&hn, newly, 8, cudaMemcpyDeviceToHost, st), "D2H");
  CK(idx, cudaStreamSynchronize(st), "delete sync");
  idx->n_deleted += (int64_t)hn;
  if (n_newly_deleted) *n_newly_deleted = (int64_t)hn;
  // NEXT-4: global consolidation once the deletions since the last one pass the ratio ("e.g., 20%")
  if (idx->consolidate_ratio > 0.0) {
    const int64_t since = idx->n_deleted - idx->deleted_at_consolidation;
    const int64_t base = idx->n_alloc - idx->deleted_at_consolidation;
    if (since > 0 && (double)since > idx->consolidate_ratio * (double)base) return consolidate_impl(idx, nullptr, st);
  }
  return SVF_OK;
}

svf_status svf_knn_exact(svf_index* idx, const float* Q, int64_t nq, int32_t k, uint32_t* out_ids,
                         float* out_dists, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (nq < 0 || k < 1 || k > 256) return fail(SVF_ERR_INVALID, "need nq >= 0 and 1 <= k <= 256");
  if (nq == 0) return SVF_OK;
  if (!Q || !out_ids || !out_dists) return fail(SVF_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool q_dev = is_device_ptr(Q), i_dev = is_device_ptr(out_ids), d_dev = is_device_ptr(out_dists);
  const size_t qb = q_dev ? 0 : al((size_t)nq * idx->D * 4);
  const size_t ob = al((size_t)nq * k * 4);
  // staging lives in its own buffer: the kNN kernels use the scratch arena
  char* sp = nullptr;
  if (qb + 2 * ob > 0) CK(idx, cudaMallocAsync(reinterpret_cast<void**>(&sp), qb + 2 * ob, st), "knn staging");
  const float* Qd = Q;
  if (!q_dev) {
    CK(idx, cudaMemcpyAsync(sp, Q, (size_t)nq * idx->D * 4, cudaMemcpyHostToDevice, st), "H2D queries");
    Qd = reinterpret_cast<const float*>(sp);
  }
  uint32_t* oi = i_dev ? out_ids : reinterpret_cast<uint32_t*>(sp + qb);
  float* od = d_dev ? out_dists : reinterpret_cast<float*>(sp + qb + ob);
  CK(idx,
     run_knn(idx, idx->n_alloc, idx->n_deleted > 0 ? idx->tomb : nullptr, Qd, idx->D, idx->D, nq, k, -1, oi, od, st),
     "knn kernel");
  if (!i_dev) CK(idx, cudaMemcpyAsync(out_ids, oi, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
  if (!d_dev) CK(idx, cudaMemcpyAsync(out_dists, od, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st), "D2H dists");
  if (sp) CK(idx, cudaFreeAsync(sp, st), "knn staging free");
  if (!i_dev || !d_dev) CK(idx, cudaStreamSynchronize(st), "knn sync");
  return SVF_OK;
}

svf_status svf_merge_topk(const uint32_t* ids, const float* dists, int32_t G, int64_t nq, int32_t k,
                          uint32_t* out_ids, float* out_dists, void* stream) {
  if (G < 1 || nq < 0 || k < 1 || k > 256) return fail(SVF_ERR_INVALID, "need G >= 1, nq >= 0, 1 <= k <= 256");
  if (nq == 0) return SVF_OK;
  if (!ids || !dists || !out_ids || !out_dists) return fail(SVF_ERR_INVALID, "NULL argument");
  if (!is_device_ptr(ids) || !is_device_ptr(dists) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
    return fail(SVF_ERR_INVALID, "svf_merge_topk takes device pointers (the all-gather output)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_merge_topk(ids, dists, G, nq, k, out_ids, out_dists, st);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "merge kernel");
  return SVF_OK;
}

svf_status svf_shard_premerge(const uint32_t* ids, const float* dists, int32_t n_lists, int64_t nq, int32_t k,
                              uint32_t n_logical, const uint32_t* shard, uint64_t* out_pairs, void* stream) {
  if (n_lists < 1 || n_lists > 16 || nq < 0 || k < 1 || k > 256 || n_logical < 1)
    return fail(SVF_ERR_INVALID, "need 1 <= n_lists <= 16, nq >= 0, 1 <= k <= 256, n_logical >= 1");
  if (nq == 0) return SVF_OK;
  if (!ids || !dists || !shard || !out_pairs) return fail(SVF_ERR_INVALID, "NULL argument");
  if (!is_device_ptr(ids) || !is_device_ptr(dists) || !is_device_ptr(out_pairs))
    return fail(SVF_ERR_INVALID, "svf_shard_premerge takes device ids/dists/out_pairs");
  for (int i = 0; i < n_lists; ++i)
    if (shard[i] >= n_logical) return fail(SVF_ERR_INVALID, "shard index >= n_logical");
  cudaError_t e = launch_shard_premerge(ids, dists, n_lists, nq, k, n_logical, shard,
                                        reinterpret_cast<unsigned long long*>(out_pairs),
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "shard pre-merge kernel");
  return SVF_OK;
}

svf_status svf_merge_pairs(const uint64_t* pairs, int32_t G, int64_t nq, int32_t k, uint32_t* out_ids,
                           float* out_dists, void* stream) {
  if (G < 1 || nq < 0 || k < 1 || k > 256) return fail(SVF_ERR_INVALID, "need G >= 1, nq >= 0, 1 <= k <= 256");
  if (nq == 0) return SVF_OK;
  if (!pairs || !out_ids || !out_dists) return fail(SVF_ERR_INVALID, "NULL argument");
  if (!is_device_ptr(pairs) || !is_device_ptr(out_ids) || !is_device_ptr(out_dists))
    return fail(SVF_ERR_INVALID, "svf_merge_pairs takes device pointers (the all-gather output)");
  cudaError_t e = launch_merge_pairs(reinterpret_cast<const unsigned long long*>(pairs), G, nq, k, out_ids,
                                     out_dists, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "pair merge kernel");
  return SVF_OK;
}

svf_status svf_export(const svf_index* cidx, float* vec, uint32_t* graph, float* edge_dist, uint32_t* tomb,
                      int64_t* n_alloc) {
  svf_index* idx = const_cast<svf_index*>(cidx);
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  CK(idx, cudaDeviceSynchronize(), "sync");
  const int64_t n = idx->n_alloc;
  if (n_alloc) *n_alloc = n;
  if (vec && n > 0)
    CK(idx, cudaMemcpy2D(vec, (size_t)idx->D * 4, idx->vec, (size_t)idx->Dp * 4, (size_t)idx->D * 4, (size_t)n,
                         cudaMemcpyDefault), "export vec");
  if (graph && n > 0) CK(idx, cudaMemcpy(graph, idx->graph, (size_t)n * idx->R * 4, cudaMemcpyDefault), "export graph");
  if (edge_dist && n > 0)
    CK(idx, cudaMemcpy(edge_dist, idx->edge_dist, (size_t)n * idx->R * 4, cudaMemcpyDefault), "export edge_dist");
  if (tomb && n > 0) CK(idx, cudaMemcpy(tomb, idx->tomb, ((size_t)n + 31) / 32 * 4, cudaMemcpyDefault), "export tomb");
  return SVF_OK;
}

svf_status svf_link_candidates(svf_index* idx, const float* X, const uint32_t* cand_ids, const float* cand_d,
                               int64_t n_new, int32_t n_cand, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (n_new < 0 || n_cand < 1 || n_cand > 512) return fail(SVF_ERR_INVALID, "need n_new >= 0, 1 <= n_cand <= 512");
  if (n_new == 0) return SVF_OK;
  if (!cand_ids || !cand_d) return fail(SVF_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lk(idx->mu);
  if (idx->n_alloc + n_new > idx->cap) return fail(SVF_ERR_CAPACITY, "n_alloc + n_new > capacity");
  DeviceGuard g(idx->dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t m = (size_t)n_new * n_cand;
  std::vector<uint32_t> hid(m);
  CK(idx, cudaMemcpy(hid.data(), cand_ids, m * 4, cudaMemcpyDefault), "copy candidates");
  for (uint32_t v : hid)
    if (v != SVF_SENTINEL && (int64_t)v >= idx->n_alloc)
      return fail(SVF_ERR_INVALID, "candidate id >= n_alloc (candidates must be existing vertices)");
  const size_t cb = al(m * 4);
  const size_t rev = reverse_scratch_bytes(n_new, idx->R);
  CK(idx, ensure_scratch(idx, 2 * cb + al(rev), st), "link scratch");
  char* sp = static_cast<char*>(idx->scratch);
  CK(idx, cudaMemcpyAsync(sp, hid.data(), m * 4, cudaMemcpyHostToDevice, st), "H2D");
  CK(idx, cudaMemcpyAsync(sp + cb, cand_d, m * 4, cudaMemcpyDefault, st), "H2D");
  const int64_t first = idx->n_alloc;
  CK(idx, put_rows(idx, X, first, n_new, st), "copy X");
  CK(idx, launch_fill_rows(idx->graph, idx->edge_dist, first, n_new, idx->R, st), "fill rows");
  CK(idx,
     launch_detour_select(idx->graph, idx->edge_dist, idx->R, idx->P, first, n_new,
                          reinterpret_cast<uint32_t*>(sp), reinterpret_cast<float*>(sp + cb), n_cand, st),
     "detour select");
  CK(idx,
     launch_reverse(idx->graph, idx->edge_dist, idx->n_deleted > 0 ? idx->tomb : nullptr, idx->R, idx->P, first,
                    n_new, sp + 2 * cb, idx->scratch_bytes - 2 * cb, st),
     "reverse edges");
  CK(idx, launch_store_u64(idx->small + 6, (uint64_t)(first + n_new), st), "publish n_visible");
  CK(idx, cudaStreamSynchronize(st), "link sync");
  idx->n_alloc += n_new;
  return SVF_OK;
}

svf_status svf_set_search_params(svf_index* idx, int32_t search_width, int32_t n_init, int32_t max_iter,
                                 int32_t hash_bits) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (search_width < 1 || search_width > 8 || n_init < 0 || max_iter < 0 || hash_bits < 0 || hash_bits > 15)
    return fail(SVF_ERR_INVALID, "bad search params");
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->search_width = search_width;
  idx->n_init = n_init;
  idx->max_iter = max_iter;
  idx->hash_bits = hash_bits;
  return SVF_OK;
}

svf_status svf_last_search_counters(svf_index* idx, uint64_t out[5]) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  out[0] = out[1] = out[2] = 0;
  out[3] = (uint64_t)idx->counters_nq;
  out[4] = (uint64_t)idx->last_launches;
  if (idx->counters_nq == 0) return SVF_OK;
  CK(idx, cudaStreamSynchronize(idx->last_stream), "sync");
  std::vector<uint32_t> h((size_t)idx->counters_nq * 3);
  CK(idx, cudaMemcpy(h.data(), idx->counters, h.size() * 4, cudaMemcpyDeviceToHost), "D2H counters");
  for (int64_t q = 0; q < idx->counters_nq; ++q) {
    out[0] += h[q * 3 + 0];
    out[1] += h[q * 3 + 1];
    out[2] += h[q * 3 + 2];
  }
  return SVF_OK;
}

svf_status svf_set_trace(svf_index* idx, int32_t enable) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->trace_on = enable != 0;
  idx->trace_nq = 0;
  return SVF_OK;
}

svf_status svf_read_trace(svf_index* idx, uint64_t* out, int64_t cap, int64_t* nq) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  *nq = idx->trace_nq;
  if (idx->trace_nq == 0) return SVF_OK;
  if (cap < idx->trace_nq) return fail(SVF_ERR_INVALID, "trace buffer too small");
  CK(idx, cudaStreamSynchronize(idx->last_stream), "sync");
  CK(idx, cudaMemcpy(out, idx->trace, (size_t)idx->trace_nq * kTraceCols * 8, cudaMemcpyDeviceToHost), "D2H trace");
  return SVF_OK;
}

// NEXT-1 repair / NEXT-4 consolidation on the update path (caller holds the index lock)
static svf_status repair_impl(svf_index* idx, int c, double threshold, int64_t* n_repaired, uint64_t* hist, cudaStream_t st) {
  const uint32_t* tomb = idx->n_deleted > 0 ? idx->tomb : nullptr;
  CK(idx, ensure_scratch(idx, repair_mark_scratch_bytes(idx->n_alloc), st), "repair scratch");
  int64_t n_list = 0;
  uint64_t h[5];
  CK(idx, launch_repair_mark(idx->graph, tomb, idx->R, idx->n_alloc, threshold, idx->scratch, st, &n_list, h),
     "repair mark");
  if (n_list > 0) {
    int cap = idx->p.insert_itopk;  // U is cut to an insertion-sized candidate list (reading R1')
    if (const char* v = getenv("SVF_REPAIR_CAP")) cap = std::max(1, std::min(512, atoi(v)));  // experiment hook
    const size_t bytes = repair_apply_scratch_bytes(n_list, idx->R, cap);
    void* sp = nullptr;
    CK(idx, cudaMallocAsync(&sp, bytes, st), "repair apply scratch");
    CK(idx,
       launch_repair_apply(idx->graph, idx->edge_dist, idx->vec, idx->dq, idx->p.metric, tomb, idx->R, idx->P, c, cap,
                           idx->scratch, n_list, sp, bytes, idx->num_sms, st),
       "repair apply");
    CK(idx, cudaFreeAsync(sp, st), "repair free");
    CK(idx, cudaStreamSynchronize(st), "repair sync");
  }
  if (n_repaired) *n_repaired = n_list;
  if (hist)
    for (int i = 0; i < 5; ++i) hist[i] = h[i];
  return SVF_OK;
}

svf_status svf_repair(svf_index* idx, int32_t c, double threshold, int64_t* n_repaired, uint64_t hist[5],
                      void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (c < 1 || c > idx->R || !(threshold >= 0.0 && threshold < 1.0))
    return fail(SVF_ERR_INVALID, "need 1 <= c <= degree and 0 <= threshold < 1");
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  return repair_impl(idx, c, threshold, n_repaired, hist, static_cast<cudaStream_t>(stream));
}

// NEXT-4 global consolidation, reading C2: every live row holding a tombstoned id keeps its
// live entries and refills its vacancies from the live members of its deleted neighbours' lists
static svf_status consolidate_impl(svf_index* idx, int64_t* n_rewritten, cudaStream_t st) {
  int64_t n_list = 0;
  if (idx->n_deleted > 0) {
    CK(idx, ensure_scratch(idx, repair_mark_scratch_bytes(idx->n_alloc), st), "consolidation scratch");
    uint64_t h[5];
    CK(idx, launch_repair_mark(idx->graph, idx->tomb, idx->R, idx->n_alloc, 0.0, idx->scratch, st, &n_list, h),
       "consolidation mark");
    CK(idx,
       launch_consolidate(idx->graph, idx->edge_dist, idx->vec, idx->dq, idx->p.metric, idx->tomb, idx->R, idx->P,
                          idx->scratch, n_list, idx->num_sms, st),
       "consolidation");
    CK(idx, cudaStreamSynchronize(st), "consolidation sync");
  }
  if (n_rewritten) *n_rewritten = n_list;
  idx->deleted_at_consolidation = idx->n_deleted;
  idx->consolidations++;
  return SVF_OK;
}

svf_status svf_consolidate(svf_index* idx, int64_t* n_rewritten, void* stream) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  return consolidate_impl(idx, n_rewritten, static_cast<cudaStream_t>(stream));
}

svf_status svf_set_consolidation(svf_index* idx, double ratio) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (!(ratio >= 0.0 && ratio < 1.0)) return fail(SVF_ERR_INVALID, "consolidation ratio must be in [0, 1)");
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->consolidate_ratio = ratio;
  return SVF_OK;
}

svf_status svf_consolidation_stats(svf_index* idx, int64_t out[2]) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  out[0] = idx->consolidations;
  out[1] = idx->deleted_at_consolidation;
  return SVF_OK;
}

svf_status svf_set_warps_per_query(svf_index* idx, int32_t wpq) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (wpq < 0 || wpq > 2) return fail(SVF_ERR_INVALID, "warps_per_query must be 0 (auto), 1 or 2");
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->wpq = wpq;
  return SVF_OK;
}

svf_status svf_set_search_handoff(svf_index* idx, int32_t pct) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (pct < -1 || pct > 100) return fail(SVF_ERR_INVALID, "handoff threshold must be -1 (auto), 0 (off) or 1..100");
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->ho_pct = pct;
  return SVF_OK;
}

svf_status svf_set_knn_mode(svf_index* idx, int32_t mode) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  if (mode < 0 || mode > 1) return fail(SVF_ERR_INVALID, "knn mode must be 0 (auto) or 1 (FFMA)");
  std::lock_guard<std::mutex> lk(idx->mu);
  idx->knn_mode = mode;
  return SVF_OK;
}

svf_status svf_knn_stats(svf_index* idx, uint64_t out[3]) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  out[0] = idx->knn_queries;
  out[1] = idx->knn_fallbacks;
  out[2] = idx->knn_tc_calls;
  return SVF_OK;
}

svf_status svf_profile(svf_index* idx, int32_t enable) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  prof_resolve(idx);
  idx->prof = enable != 0;
  for (int i = 0; i < 4; ++i) {
    idx->prof_ms[i] = 0;
    idx->prof_cnt[i] = 0;
  }
  return SVF_OK;
}

svf_status svf_profile_read(svf_index* idx, double ms[4], int64_t cnt[4]) {
  svf_status s = enter(idx);
  if (s != SVF_OK) return s;
  std::lock_guard<std::mutex> lk(idx->mu);
  DeviceGuard g(idx->dev);
  prof_resolve(idx);
  for (int i = 0; i < 4; ++i) {
    ms[i] = idx->prof_ms[i];
    cnt[i] = idx->prof_cnt[i];
  }
  return SVF_OK;
}

svf_status svf_info(const svf_index* idx, int64_t* n_alloc, int64_t* n_deleted, int64_t* capacity) {
  if (!idx) return fail(SVF_ERR_INVALID, "index is NULL");
  if (n_alloc) *n_alloc = idx->n_alloc;
  if (n_deleted) *n_deleted = idx->n_deleted;
  if (capacity) *capacity = idx->cap;
  return SVF_OK;
}

svf_status svf_destroy(svf_index* idx) {
  if (!idx) return SVF_OK;
  DeviceGuard g(idx->dev);
  cudaDeviceSynchronize();
  cudaFree(idx->vec);
  cudaFree(idx->graph);
  cudaFree(idx->edge_dist);
  cudaFree(idx->tomb);
  cudaFree(idx->small);
  cudaFree(idx->scratch);
  if (idx->sscratch) cudaFree(idx->sscratch);
  cudaFree(idx->counters);
  if (idx->trace) cudaFree(idx->trace);
  if (idx->ho) cudaFree(idx->ho);
  if (idx->ho_upd) cudaFree(idx->ho_upd);
  if (idx->q_flags) cudaFree(idx->q_flags);
  if (idx->h_epoch) cudaFreeHost(idx->h_epoch);
  if (idx->ev_cs0) cudaEventDestroy(idx->ev_cs0);
  if (idx->ev_cs1) cudaEventDestroy(idx->ev_cs1);
  if (idx->cstream) cudaStreamDestroy(idx->cstream);
  if (idx->ev0) cudaEventDestroy(idx->ev0);
  if (idx->ev1) cudaEventDestroy(idx->ev1);
  for (auto& r : idx->prof_pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : idx->ev_pool) cudaEventDestroy(e);
  cudaGetLastError();
  delete idx;
  return SVF_OK;
}

}  // extern "C"
