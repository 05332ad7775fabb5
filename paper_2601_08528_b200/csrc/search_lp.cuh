// K-S-L: the search of SURVEY §8(a) S0-S8 (Algorithm 1) for LARGE candidate pools (L > 64: the insert
// search at L_insert = 128, C4's itopk 192, build searches at L_build 256-512).  Included by search_impl.cuh.
//
// Why a second kernel (DESIGN.md §6 "K-S-L"): the register-resident pool of K-S costs 4-16 u64 per lane plus an
// unrolled bitonic merge over L keys; at L >= 128 that is 113-128 registers (4 blocks/SM, ~14 warps), ~1360 warp
// instructions per iteration and a 2^11-2^12-slot probing visited table that is cleared and re-filled every ~40
// iterations (measured: 6.6 us per iteration, 1.83x recomputed distances at L = 128, profiles/r02_pool_probe.json).
// Here one warp still serves one query, but:
//  - the pool lives in shared memory as a sorted array of exactly L 64-bit keys (dist, id, parented flag; I6);
//    new keys are merged in place: each new key finds its insertion point by binary search, each moved pool key its
//    shift by binary search over the (few) new keys, and the moving suffix is rewritten back to front in 32-key
//    chunks (a merge is a bijection, so no position is written before it is read);
//  - parents are found from a cursor: every entry before it is parented, and a merge can only move the first
//    unparented entry up to the first inserted key;
//  - the visited set is a direct-mapped cache of ids (slot = hash(id), overwritten on collision, never cleared
//    mid-query, no atomics).  It may forget ids but never reports an unvisited one: reading I7 applies as for the
//    probing table (a forgotten non-pool id is rejected again by the L-th key, which never increases), and a
//    forgotten id that is still IN the pool is caught by an exact membership test (binary search) of the few keys
//    that pass the L-th-key threshold.  Results are therefore identical to the exact visited set (oracle O2);
//  - no per-lane pool registers: the gather engine keeps its registers, for more resident warps.
#pragma once

namespace svf {

namespace {

// SVF_LP_QSMEM = 1: the team gather (D = 96 / 128) reads the query from a shared-memory copy instead of 4 float4
// registers per lane, which removes the spills at the 72-register cap (C2 itopk 128: 4096 queries 1.438 -> 1.412 ms,
// 10K 3.057 -> 3.017 ms; itopk 96 10K 2.474 -> 2.428 ms; profiles/r02_lp_ab.json)
#ifndef SVF_LP_FILTER_PF
#define SVF_LP_FILTER_PF 1
#endif
// SVF_LP_FILTER_PF96 = 1 extends it to D = 96 (unrolled 3 lines): still slower there (C3 100K inserts, insert search
// 51.1 -> 55.9 ms)
#ifndef SVF_LP_FILTER_PF96
#define SVF_LP_FILTER_PF96 0
#endif
#ifndef SVF_LP_QSMEM
#define SVF_LP_QSMEM 1
#endif
// SVF_LP_WHOLE = 1: whole-warp rows at D = 200 (SVF_GATHER_W_LP / 2 rows per round); measured against teams of 16
// lanes with 2 rows each: C4 itopk 192 11.84 -> 11.00 ms; at D = 128 the 8-lane teams stay (whole-warp: 2.01 vs
// 1.89 ms for an itopk-128 4096-query batch), profiles/r02_lp_ab.json
#ifndef SVF_LP_WHOLE
#define SVF_LP_WHOLE 1
#endif
// per-warp shared memory: [visited cache M entries (u16 tags or u32 ids); the query row is staged here before the
// cache is cleared | pool Lp u64 | survivor ids MP u32 | keys MP u64 (compacted in place by C.Update) | query slot
// 2 u64 | parents 8 u32].  M need not be a power of two (slot = multiply-shift of a hashed id), so the launcher
// sizes the cache to whatever the target residency leaves (DESIGN.md §6 K-S-L).
struct LpLayout {
  int M, Lp, MP, c16, Dp;
  __host__ __device__ size_t cache_bytes() const {
    const size_t cb = (size_t)M * (c16 ? 2 : 4), qb = (size_t)Dp * 4;
    return ((cb > qb ? cb : qb) + 15) & ~(size_t)15;
  }
  // SVF_LP_QSMEM: a resident query copy for the team gather (the whole-warp gather at D = 200 keeps the query in
  // registers, so it stages the row through the cache region instead)
  __host__ __device__ bool qs_resident() const { return SVF_LP_QSMEM && !(SVF_LP_WHOLE && Dp == 200); }
  __host__ __device__ size_t qs_off() const { return cache_bytes(); }
  __host__ __device__ size_t pool_off() const {
    return qs_off() + (qs_resident() ? (((size_t)Dp * 4 + 15) & ~(size_t)15) : 0);
  }
  __host__ __device__ size_t sid_off() const { return pool_off() + (size_t)Lp * 8; }
  __host__ __device__ size_t skey_off() const { return sid_off() + (size_t)MP * 4; }
  __host__ __device__ size_t misc_off() const { return skey_off() + (size_t)MP * 8; }
  __host__ __device__ size_t warp_bytes() const { return (misc_off() + 48 + 15) & ~(size_t)15; }
};

#ifndef SVF_MINB_LP
#define SVF_MINB_LP 7
#endif

#ifndef SVF_GATHER_U_LP
#define SVF_GATHER_U_LP 2
#endif
#ifndef SVF_GATHER_W_LP
#define SVF_GATHER_W_LP 8
#endif
// SVF_LP_EARLY_ROW = 1: after each merge the exact next parent's row is loaded at once when the speculation missed
#ifndef SVF_LP_EARLY_ROW
#define SVF_LP_EARLY_ROW 1
#endif
// SVF_LP_ONE_WRITER = 1: one writer per cache slot per round (match_any) and a warp barrier between the round's cache
// reads and writes, so compute-sanitizer's racecheck sees no shared-memory hazard; 0: plain stores (the lossy cache
// tolerates the benign write/write and read/write races: any value a slot holds is a valid visited tag or empty)
#ifndef SVF_LP_ONE_WRITER
#define SVF_LP_ONE_WRITER 1
#endif

// Whole-warp gather for K-S-L at D = 128 / 200 (DQT = 32 / 50 float4): every lane holds NV = ceil(DQT / 32) float4 of
// each of U rows per round (the query costs NV float4 per lane instead of K-S's 4, so the registers go to rows in
// flight: 8 rows per round at D = 128, 4 at D = 200), and the U partial sums are reduced together by a transposing
// butterfly (at the step with offset 2^(4-j) each lane keeps half of its values and sends the other half: U - 1 + 5 -
// log2 U shuffles for U rows instead of 5 U), after which lane l holds row (l >> (5 - log2 U)).
template <int DQT, int U>
__device__ __forceinline__ void gather_keys_w(const SearchArgs& a, const uint32_t* sid, uint64_t* skey, int S,
                                              const float4 (&qv)[4], int lane, uint64_t pf) {
  static_assert(U == 1 || U == 2 || U == 4 || U == 8, "U must be a power of two <= 8");
  constexpr int NV = (DQT + 31) / 32;
  constexpr int LU = U == 1 ? 0 : U == 2 ? 1 : U == 4 ? 2 : 3;
  const float4* __restrict__ vec4 = reinterpret_cast<const float4*>(a.vec);
  __syncwarp();
  // every 128-byte line of the later rows (an exact-size cp.async.bulk.prefetch.L2 per 800-byte row avoids the line
  // overfetch but was slower: C4 10.52 vs 10.81 ms; prefetching each row at its filter, as the team gather does, was
  // slower here too: 7-8 lines per lane, 9.84 -> 10.11 ms)
  prefetch_rows_l2(vec4, sid, U, S, DQT, lane);
  for (int base = 0; base < S; base += U) {
    float4 xv[U][NV];
    uint32_t id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + u;
      id[u] = s < S ? sid[s] : kSent;
      const float4* row = vec4 + (size_t)(id[u] == kSent ? 0 : id[u]) * DQT;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = lane + 32 * v;
        xv[u][v] = (c < DQT && id[u] != kSent) ? __ldg(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t acc2 = 0ull;
#pragma unroll
      for (int v = 0; v < NV; ++v) acc2 = dist_acc4(acc2, xv[u][v], qv[v], a.metric);
      acc[u] = f2sum(acc2);
    }
    // transposing butterfly: after the step with offset 16 >> j, lane l holds the partial sums of rows whose index
    // bits (from the top) equal l's bits 4, 3, ... (U >> (j + 1) values left)
#pragma unroll
    for (int j = 0; j < LU; ++j) {
      const int off = 16 >> j;
      const bool hi = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < (U >> (j + 1)); ++i) {
        const float send = hi ? acc[i] : acc[i + (U >> (j + 1))];
        const float keep = hi ? acc[i + (U >> (j + 1))] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
#pragma unroll
    for (int off = 16 >> LU; off > 0; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
    const int r = lane >> (5 - LU), s = base + r;
    if ((lane & ((32 >> LU) - 1)) == 0 && s < S) {
      uint32_t idr = id[0];
#pragma unroll
      for (int u = 1; u < U; ++u)
        if (r == u) idr = id[u];
      const uint64_t key = make_key((a.metric == 0 ? acc[0] : -acc[0]) + 0.0f, idr);  // canonical +0
      skey[s] = key;
      if (key < pf) prefetch_graph_row(a.graph, a.R, idr);  // the likely next parent (gather_keys' PF)
    }
  }
  __syncwarp();
}

// Visited cache slot and tag of an id, for a cache of M slots.  vc_bits = B > 0: ids are < 2^B and h = id * odd mod
// 2^B is a bijection of [0, 2^B); slot = floor(h * M / 2^B), so the h of one slot form a contiguous run of at most
// ceil(2^B / M) <= 2^tb values and their low tb bits (tmask = 2^tb - 1) tell them apart: tag = (h & tmask) + 1 (0
// marks an empty slot), stored in 16 bits (tb <= 15).  Equal tags in a slot mean equal ids, so the cache stays exact
// while holding twice the entries of a u32 cache in the same shared memory.  B = 0: u32 entries holding the id itself
// (empty = 0xFFFFFFFF), slot = floor(h * M / 2^32) of the 32-bit hash.
__device__ __forceinline__ void cache_pos(uint32_t id, uint32_t M, int B, uint32_t tmask, uint32_t& slot,
                                          uint32_t& tag) {
  if (B) {
    const uint32_t h = (id * 0x9E3779B1u) & ((1u << B) - 1u);
    slot = (uint32_t)(((uint64_t)h * M) >> B);
    tag = (h & tmask) + 1u;
  } else {
    slot = (uint32_t)(((uint64_t)(id * 0x9E3779B1u) * M) >> 32);
    tag = id;
  }
}

// the same, with the quartile keys of a[0..n) read together first (three independent broadcast reads instead of two
// dependent probes), then a binary search inside the quarter
__device__ __forceinline__ int lower_bound_key_q(const uint64_t* a, int n, uint64_t k) {
  int lo = 0, hi = n;
  if (n >= 16) {
    const int q1 = n >> 2, q2 = n >> 1, q3 = q1 + q2;
    const uint64_t f1 = a[q1] & ~1ull, f2 = a[q2] & ~1ull, f3 = a[q3] & ~1ull;
    if (f2 < k) {
      lo = q2 + 1;
      if (f3 < k) lo = q3 + 1;
      else hi = q3;
    } else {
      hi = q2;
      if (f1 < k) lo = q1 + 1;
      else hi = q1;
    }
  }
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((a[mid] & ~1ull) < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// number of keys in sorted a[0..n) whose flag-stripped value is < k (k has its flag bit clear)
__device__ __forceinline__ int lower_bound_key(const uint64_t* a, int n, uint64_t k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((a[mid] & ~1ull) < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int CPL, int DQT>
__global__ void __launch_bounds__(kSearchWarpsPerBlock * 32, SVF_MINB_LP) search_lp_kernel(SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int MP = 32 * CPL;
  // whole-warp rows (gather_keys_w) at D = 200 (Geo<50> teams of 16 lanes leave 14 of 64 float4 slots idle and hold
  // 4 query float4 per lane); teams of Geo<DQT>::T lanes otherwise (D = 96 / 128: 8 lanes, no idle slots)
  constexpr bool kLpWhole = SVF_LP_WHOLE && DQT == 50;
  // survivors' rows prefetched at the filter instead of at the gather (SVF_LP_FILTER_PF), at D = 128 only: measured
  // faster there (C2 itopk 128 4096 q 1.277 -> 1.226 ms, C2G 2.21 -> 2.13 ms) but slower at D = 96 (C3 100K inserts
  // 51.1 -> 58.7 ms of insert search) and D = 200 (C4 9.84 -> 10.11 ms)
  constexpr bool kLpFilterPf = SVF_LP_FILTER_PF && (DQT == 32 || (SVF_LP_FILTER_PF96 && DQT == 24));
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int VB = a.vc_bits;  // 16-bit tagged cache when > 0
  const uint32_t M = (uint32_t)a.vc_slots, TM = a.vc_tmask;
  const LpLayout lay{a.vc_slots, (a.L + 31) & ~31, MP, VB > 0, a.dq * 4};
  unsigned char* base = smem + (size_t)wib * lay.warp_bytes();
  // the query is staged in the cache region (then the cache is cleared), or kept in its own region (SVF_LP_QSMEM)
  float4* qs = reinterpret_cast<float4*>(base + (lay.qs_resident() ? lay.qs_off() : 0));
  uint32_t* cache = reinterpret_cast<uint32_t*>(base);
  uint16_t* cache16 = reinterpret_cast<uint16_t*>(base);
  uint64_t* pool = reinterpret_cast<uint64_t*>(base + lay.pool_off());
  uint32_t* sid = reinterpret_cast<uint32_t*>(base + lay.sid_off());
  uint64_t* skey = reinterpret_cast<uint64_t*>(base + lay.skey_off());
  uint64_t* ck = skey;  // C.Update compacts the passing keys in place
  unsigned long long* qslot = reinterpret_cast<unsigned long long*>(base + lay.misc_off());
  uint32_t* spar = reinterpret_cast<uint32_t*>(base + lay.misc_off() + 16);
  const int L = a.L;

  for (;;) {
    if (lane == 0) {
      const unsigned long long f = atomicAdd(a.work_counter, 1ull);
      if (a.q_flags != nullptr && f < (unsigned long long)a.nq) {  // streamed host queries: wait for the chunk
        const volatile unsigned int* fl = a.q_flags + (f >> a.q_chunk_log2);
        while (*fl != a.q_epoch) __nanosleep(64);
        __threadfence();
      }
      unsigned long long nsnap = a.n_alloc;
      if (a.n_visible != nullptr)
        nsnap = min(nsnap, *reinterpret_cast<const volatile unsigned long long*>(a.n_visible));
      qslot[0] = f;
      qslot[1] = nsnap;
    }
    __syncwarp();
    const unsigned long long qf = qslot[0];
    const uint32_t n = (uint32_t)qslot[1];
    __syncwarp();
    if (qf >= (unsigned long long)a.nq) break;
    const unsigned long long qi = qf;
    unsigned long long t_start = 0;
    if (a.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    // S0: the query row through this warp's cache region (coalesced, zero-padded to Dp) into registers, then the
    // visited cache cleared
    const float* qg = a.Q + (size_t)qi * a.q_stride;
    float* qf32 = reinterpret_cast<float*>(qs);
    for (int i = lane; i < a.dq * 4; i += 32) qf32[i] = i < a.q_dim ? __ldcg(qg + i) : 0.f;
    __syncwarp();
    float4 qv[4];
    {
      const int T = kLpWhole ? 32 : (DQT ? Geo<DQT>::T : a.team), tl = lane & (T - 1);
      const int NV = kLpWhole ? (DQT + 31) / 32 : (DQT ? Geo<DQT>::NV : a.nv);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = tl + T * v;
        qv[v] = (v < NV && c < a.dq) ? qs[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    __syncwarp();
    if (VB) {
      for (uint32_t i = lane; i < (M >> 1); i += 32) cache[i] = 0u;
    } else {
      for (uint32_t i = lane; i < M; i += 32) cache[i] = kHashEmpty;
    }
    __syncwarp();

#if SVF_LP_QSMEM
#define QSRC QuerySmem{qs}
#else
#define QSRC QueryRegs{qv}
#endif
#define GATHER_LP(S_, PF_)                                                                                     \
  do {                                                                                                         \
    if constexpr (kLpWhole)                                                                                    \
      gather_keys_w<DQT, (DQT > 32 ? SVF_GATHER_W_LP / 2 : SVF_GATHER_W_LP)>(a, sid, skey, (S_), qv, lane, PF_); \
    else                                                                                                       \
      gather_keys<DQT, (DQT > 0 ? SVF_GATHER_U_LP : SVF_GATHER_U), true>(a, sid, skey, (S_), QSRC, lane, PF_);  \
  } while (0)
    int np = 0;  // entries in the pool (<= L)
    int fu = 0;  // every entry before fu is parented
    uint32_t n_dist = 0, iters = 0, n_exp = 0;

    // S6 C.Update for the keys skey[0..S): drop those not better than the L-th key, then, 32 at a time, drop repeated
    // keys and keys already in the pool and merge the rest in place.  No sort: a new key's final position is its
    // insertion point b (binary search in the pool) plus its rank among the kept new keys (a shuffle count), and a
    // pool key at position i moves up by the number of kept new keys with b <= i.
    auto update = [&](int S) {
      const uint64_t kth = np < L ? kEmptyKey : (pool[L - 1] & ~1ull);
      int S2 = 0;
#pragma unroll
      for (int r = 0; r < CPL; ++r) {
        const int e = r * 32 + lane;
        const uint64_t k = e < S ? skey[e] : kEmptyKey;
        const bool pass = k < kth;
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        if (pass) ck[S2 + __popc(m & ((1u << lane) - 1u))] = k;
        S2 += __popc(m);
      }
      __syncwarp();
      for (int base = 0; base < S2; base += 32) {
        const int nh = min(32, S2 - base);
        const uint64_t c = lane < nh ? ck[base + lane] : kEmptyKey;
        int b = L;
        bool keep = false;
        if (lane < nh) {
          b = lower_bound_key_q(pool, np, c);
          keep = !(b < np && (pool[b] & ~1ull) == c);  // already in the pool (the cache forgot it)
        }
        // the same id offered twice (p > 1): keep the first copy (lanes >= nh hold kEmptyKey and keep = false)
        if ((__match_any_sync(0xffffffffu, c) & ((1u << lane) - 1u)) != 0u) keep = false;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (km == 0u) continue;
        int rank = 0;
        for (unsigned mk = km; mk != 0u; mk &= mk - 1u) {  // over the kept keys only
          const uint64_t ci = __shfl_sync(0xffffffffu, c, __ffs(mk) - 1);
          rank += ci < c;
        }
        int b0 = keep ? b : L;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) b0 = min(b0, __shfl_xor_sync(0xffffffffu, b0, off));
        int* hist = reinterpret_cast<int*>(sid);  // 32 counters (sid is free between the gather and the filter)
        for (int s0 = b0 + ((np - b0 - 1) & ~31); np > b0 && s0 >= b0; s0 -= 32) {  // back to front
          const int i = s0 + lane;
          // cnt(i) = kept keys with b <= i: those below the chunk, plus an inclusive scan of the chunk's histogram
          int cnt = __popc(__ballot_sync(0xffffffffu, keep && b < s0));
          hist[lane] = 0;
          __syncwarp();
          if (keep && b >= s0 && b < s0 + 32) atomicAdd(hist + (b - s0), 1);
          __syncwarp();
          int h = hist[lane];
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, h, off);
            if (lane >= off) h += t;
          }
          cnt += h;
          const uint64_t pk = i < np ? pool[i] : 0ull;
          __syncwarp();
          if (i < np && i + cnt < L) pool[i + cnt] = pk;
          __syncwarp();
        }
        if (keep && b + rank < L) pool[b + rank] = c;
        __syncwarp();
        np = min(L, np + __popc(km));
        fu = min(fu, b0);
      }
    };

    // S1: the first n_init live ids along the seeded affine permutation (I2), scored and merged in chunks
    if (n > 0) {
      uint64_t pa = 0, pb = 0;
      if (lane == 0) perm_params(a.seed, a.qidx_base + qi, n, pa, pb);
      pa = __shfl_sync(0xffffffffu, pa, 0);
      pb = __shfl_sync(0xffffffffu, pb, 0);
      uint32_t cur = (uint32_t)((pa * (uint64_t)lane + pb) % n);
      const uint32_t step32 = (uint32_t)((pa * 32ull) % n);
      int taken = 0;
      for (uint64_t j0 = 0; j0 < n && taken < a.n_init; j0 += MP) {
        int running = 0;
#pragma unroll
        for (int r = 0; r < CPL; ++r) {
          const uint64_t j = j0 + (uint64_t)(r * 32 + lane);
          const uint32_t id = cur;
          cur += step32;
          if (cur >= n) cur -= n;
          bool ok = j < n;
          if (ok) ok = !tomb_dead(a.tomb, id);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const int pos = running + __popc(m & ((1u << lane) - 1u));
          const bool keep = ok && taken + pos < a.n_init;
          uint32_t slot = 0, tag = 0;
          if (keep) {
            sid[pos] = id;
            cache_pos(id, M, VB, TM, slot, tag);
            if (kLpFilterPf) prefetch_row_l2<DQT>(reinterpret_cast<const float4*>(a.vec), id, a.dq);
          }
          // one writer per slot (the lowest lane), so the cache never sees two stores to one slot at once
          const unsigned peers = SVF_LP_ONE_WRITER
                                     ? __match_any_sync(0xffffffffu, keep ? slot : (0x80000000u | (uint32_t)lane))
                                     : 0u;
          if (keep && (peers & ((1u << lane) - 1u)) == 0u) {
            if (VB) cache16[slot] = (uint16_t)tag;
            else cache[slot] = tag;
          }
          if (SVF_LP_ONE_WRITER) __syncwarp();
          running += __popc(m);
        }
        const int kept = min(running, a.n_init - taken);
        taken += kept;
        GATHER_LP(kept, 0ull);
        n_dist += kept;
        update(kept);
      }
    }

    // S2-S7: expand the first p unparented entries until every pool entry is parented (I3, I4)
    uint32_t spec_id = kSent;  // parent whose row sits in spec_row (speculative next-row load)
    uint32_t spec_row[CPL];
#ifdef SVF_PHASE_PROF
    unsigned long long ph[5] = {0, 0, 0, 0, 0};
    long long tp = clock64();
#define SVF_LPH(i)                  \
  {                                 \
    const long long tn = clock64(); \
    ph[i] += tn - tp;               \
    tp = tn;                        \
  }
#else
#define SVF_LPH(i)
#endif
    for (;;) {
      if (a.max_iter > 0 && (int)iters == a.max_iter) break;
      __syncwarp();  // the previous iteration's reads of spar are done before it is rewritten
      // S2 GetNearest: scan from the cursor, mark the first p unparented entries
      int npar = 0, last = -1;
      for (int s0 = fu; s0 < np && npar < a.p; s0 += 32) {
        const int i = s0 + lane;
        const uint64_t k = i < np ? pool[i] : kEmptyKey;
        unsigned m = __ballot_sync(0xffffffffu, (k & 1ull) == 0ull);
        while (m != 0u && npar < a.p) {
          const int l = __ffs(m) - 1;
          m &= m - 1u;
          if (lane == l) {
            pool[i] = k | 1ull;
            spar[npar] = key_id(k);
          }
          ++npar;
          last = s0 + l;
        }
      }
      if (npar == 0) break;
      __syncwarp();
      // the next unparented entry after the last parent: the likely next parent and the new cursor
      int nxt = np;
      for (int s0 = last + 1; s0 < np; s0 += 32) {
        const int i = s0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < np && (pool[i] & 1ull) == 0ull);
        if (m) {
          nxt = s0 + __ffs(m) - 1;
          break;
        }
      }
      fu = nxt;
      ++iters;
      n_exp += npar;
      SVF_LPH(0)
      const int ncand = npar * a.R;
      // S3: neighbour rows (from the speculative registers when the guess held), coalesced
      uint32_t rowv[CPL];
      const bool hit = npar == 1 && spar[0] == spec_id;
#pragma unroll
      for (int r = 0; r < CPL; ++r) {
        const int e = r * 32 + lane;
        rowv[r] = kSent;
        if (hit) {
          rowv[r] = spec_row[r];
        } else if (e < ncand) {
          const int pi = a.rshift >= 0 ? (e >> a.rshift) : e / a.R;
          rowv[r] = __ldg(a.graph + (size_t)spar[pi] * a.R + (e - pi * a.R));
        }
      }
      // the best unparented entry after this iteration's parents is the next parent unless a new key beats it: pull
      // its row toward L2 (no registers: the exact row is loaded after the merge, below)
      spec_id = kSent;
      if (nxt < np && lane < ((a.R * 4 + 127) >> 7))
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.graph + (size_t)key_id(pool[nxt]) * a.R + lane * 32));
      SVF_LPH(1)
      // S4: sentinel / snapshot / tombstone / visited-cache filters
      int running = 0;
#pragma unroll
      for (int r = 0; r < CPL; ++r) {
        const uint32_t id = rowv[r];
        bool ok = id != kSent && (uint64_t)id < n;
        if (ok) ok = !tomb_dead(a.tomb, id);
        uint32_t slot = 0, tag = 0;
        if (ok) {
          cache_pos(id, M, VB, TM, slot, tag);
          ok = VB ? cache16[slot] != (uint16_t)tag : cache[slot] != tag;
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          sid[running + __popc(m & ((1u << lane) - 1u))] = id;
          // the survivor's vector row toward L2 now, a filter round before the gather loads it (team gathers: C2
          // itopk 128 4096 queries 1.281 -> 1.245 ms, 10K 2.84 -> 2.70 ms; C2G 2.21 -> 2.13 ms)
          if (kLpFilterPf) prefetch_row_l2<DQT>(reinterpret_cast<const float4*>(a.vec), id, DQT ? DQT : a.dq);
        }
        if (SVF_LP_ONE_WRITER) __syncwarp();  // every lane's cache read of this round before any write
        // one writer per slot (the lowest lane); ids colliding in a slot are all scored, the cache keeps one
        const unsigned peers = SVF_LP_ONE_WRITER
                                   ? __match_any_sync(0xffffffffu, ok ? slot : (0x80000000u | (uint32_t)lane))
                                   : 0u;
        if (ok && (peers & ((1u << lane) - 1u)) == 0u) {
          if (VB) cache16[slot] = (uint16_t)tag;
          else cache[slot] = tag;
        }
        if (SVF_LP_ONE_WRITER) __syncwarp();
        running += __popc(m);
      }
      SVF_LPH(2)
      if (running > 0) {
        // S5 distances (a new key better than the best unparented entry prefetches its row), S6 merge
        GATHER_LP(running, fu < np ? (pool[fu] & ~1ull) : kEmptyKey);
        n_dist += running;
        SVF_LPH(3)
        update(running);
      }
      // p = 1: the next parent is now known exactly (pool[fu] is unparented whenever fu < np); load its row at once
      // (usually an L2 hit after the prefetches above), so the fetch overlaps the next select
      if (SVF_LP_EARLY_ROW && a.p == 1 && fu < np) {
        const uint32_t nid = key_id(pool[fu]);
        if (nid != spec_id) {
          spec_id = nid;
#pragma unroll
          for (int r = 0; r < CPL; ++r) {
            const int e = r * 32 + lane;
            spec_row[r] = e < a.R ? __ldg(a.graph + (size_t)nid * a.R + e) : kSent;
          }
        }
      }
      SVF_LPH(4)
    }

    // S8: emit the first n_out entries (k, or the whole pool in insert mode)
    for (int e = lane; e < a.n_out; e += 32) {
      const uint64_t k = e < np ? pool[e] : kEmptyKey;
      a.out_ids[(size_t)qi * a.n_out + e] = key_id(k);
      a.out_d[(size_t)qi * a.n_out + e] = key_dist(k);
    }
    if (lane == 0) {
      if (a.counters != nullptr) {
        a.counters[qi * 3 + 0] = n_dist;
        a.counters[qi * 3 + 1] = iters;
        a.counters[qi * 3 + 2] = n_exp;
      }
      if (a.trace != nullptr) {
        unsigned long long t_end;
        unsigned int smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* row = a.trace + qi * kTraceCols;
        row[0] = t_start;
        row[1] = t_end;
        row[2] = ((unsigned long long)smid << 32) | iters;
#ifdef SVF_PHASE_PROF
        for (int i = 0; i < 5; ++i) row[3 + i] = ph[i];
#else
        for (int i = 0; i < 5; ++i) row[3 + i] = 0;
#endif
      }
    }
    __syncwarp();
  }
}

}  // namespace

static inline size_t search_lp_smem_bytes(int slots, int L, int cpl, int c16, int Dp) {
  return kSearchWarpsPerBlock * LpLayout{slots, (L + 31) & ~31, 32 * cpl, c16, Dp}.warp_bytes();
}

template <int CPL, int DQT>
static cudaError_t launch_lp_cpl(SearchArgs a, int num_sms, cudaStream_t st) {
  auto kern = search_lp_kernel<CPL, DQT>;
  const size_t smem = search_lp_smem_bytes(a.vc_slots, a.L, CPL, a.vc_bits > 0, a.dq * 4);
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_per_sm = 0, cached_dev = -1;
  // the opt-in limit is only ever raised: a CUDA graph captured with the larger (6-block) cache must stay launchable
  // after a 7-block launch (an insert) on the same function
  static thread_local size_t attr_smem[16] = {};
  int dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  if (cached_smem == smem && cached_dev == dev) {
    per_sm = cached_per_sm;
  } else {
    cudaError_t e = cudaSuccess;
    if (smem > attr_smem[dev & 15]) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      // keep the L1 side large (in-flight gather lines), ask for just enough shared memory for the residency
      const int pct = (int)std::min<size_t>(100, (SVF_MINB_LP * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (e != cudaSuccess) return e;
      attr_smem[dev & 15] = smem;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSearchWarpsPerBlock * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    cached_smem = smem;
    cached_per_sm = per_sm;
    cached_dev = dev;
  }
  long long blocks = (long long)per_sm * num_sms;
  const long long need = (a.nq + kSearchWarpsPerBlock - 1) / kSearchWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kSearchWarpsPerBlock * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <int DQT>
cudaError_t launch_search_lp_dq(SearchArgs a, int cpl, int num_sms, cudaStream_t st) {
  switch (cpl) {
    case 1: return launch_lp_cpl<1, DQT>(a, num_sms, st);
    case 2: return launch_lp_cpl<2, DQT>(a, num_sms, st);
    case 4: return launch_lp_cpl<4, DQT>(a, num_sms, st);
    case 8: return launch_lp_cpl<8, DQT>(a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace svf
