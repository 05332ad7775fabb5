// K-S: batched greedy graph search on sm_100a (Algorithm 1).
//
// Design (DESIGN.md §6 "K-S"): persistent blocks of 4 warps pull query ids from an atomic counter; each query is
// served by WPQ warps (1, or 2 to halve per-query latency so a 10K batch does not end in a long tail).
//  - pool (the paper's candidate list C_i) lives in registers as 64-bit keys (dist, id, parent flag),
//    striped over the warp (element e = r*32 + lane), exact size L (I6) inside a power-of-two buffer.  With
//    WPQ = 2 both warps hold identical pools: every step that changes the pool is computed identically by both;
//  - visited set = per-query open-addressing table in shared memory, "forgetful": at half load it is cleared and
//    the pool ids are re-registered, which provably leaves results unchanged (I7);
//  - candidate slots are split between the query's warps (register r of the candidate array belongs to warp
//    r % WPQ): each warp filters, hashes and scores its slots (teams of T lanes per vector, coalesced 16-byte
//    gathers, FFMA, xor-shuffle reduction) and drops keys not better than the pool's L-th; one pair barrier per
//    iteration, then every warp sorts the union (bitonic) and merges it into its pool (bitonic merge).
#pragma once
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

// insert-if-absent (linear probing)
__device__ __forceinline__ bool hash_insert(uint32_t* tab, int hbits, uint32_t id) {
  const uint32_t mask = (1u << hbits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - hbits);
#ifdef SVF_HASH_READ_FIRST
  for (;;) {
    const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(tab + h);
    if (cur == id) return false;
    if (cur == kHashEmpty) {
      const uint32_t prev = atomicCAS(tab + h, kHashEmpty, id);
      if (prev == kHashEmpty) return true;
      if (prev == id) return false;
    }
    h = (h + 1) & mask;
  }
#else
  for (;;) {
    uint32_t prev = atomicCAS(tab + h, kHashEmpty, id);
    if (prev == kHashEmpty) return true;
    if (prev == id) return false;
    h = (h + 1) & mask;
  }
#endif
}

template <int WPQ>
__device__ __forceinline__ void qsync(int slot) {
  if (WPQ == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * WPQ) : "memory");
  }
}

// clear the table and re-register the pool ids (I7); identical decision in every warp of the query
template <int KPL, int WPQ>
__device__ __forceinline__ int hash_reset(uint32_t* tab, int hbits, const uint64_t (&pool)[KPL], int lane, int h,
                                          int slot) {
  const int H = 1 << hbits;
  for (int i = h * 32 + lane; i < H; i += 32 * WPQ) tab[i] = kHashEmpty;
  qsync<WPQ>(slot);
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < KPL; ++r) {
    const bool v = pool[r] != kEmptyKey;
    if (v && h == 0) hash_insert(tab, hbits, key_id(pool[r]));
    cnt += __popc(__ballot_sync(0xffffffffu, v));
  }
  qsync<WPQ>(slot);
  return cnt;
}

// Team geometry: DQT > 0 fixes the row length (float4 count) at compile time (the configs' D = 96 / 128 / 200);
// DQT == 0 is the generic path with the runtime geometry of SearchArgs.
template <int DQT>
struct Geo {
  static constexpr int T = DQT <= 4 ? 1 : DQT <= 8 ? 2 : DQT <= 16 ? 4 : DQT <= 32 ? 8 : DQT <= 64 ? 16 : 32;
  static constexpr int NV = (DQT + T - 1) / T;
};

// Gather depth (vectors per team per round): the one-warp kernel keeps 2 at small pools (more costs occupancy);
// pools of >= 128 keys run at 4 blocks/SM whatever the depth (their register limit is 128 either way), so they
// go as deep as fits without spills: 4 when a lane holds <= 3 float4 of a row (D = 96), else 3 (D = 128, 200);
// the pair-mode (latency) kernels use SVF_GATHER_U_PAIR at 32-key pools, 2 above.
template <int WPQ, int KPL, int DQT>
constexpr int gather_u() {
  return WPQ == 2 ? (KPL == 1 ? SVF_GATHER_U_PAIR : 2)  // deeper pair rounds spill once the pool is >= 64 keys
                  : (KPL >= 4 && DQT > 0) ? (Geo<DQT>::NV <= 3 ? 4 : 3) : SVF_GATHER_U;
}

// Pull every 128-byte line of the rows sid[first..S) toward L2 (prefetch.global.L2: no registers, nothing to wait
// for), so the gather rounds that load them later hit L2.  A row of DQ float4 spans up to DQ*16/128 + 1 lines when
// DQ*16 is not a multiple of 128 (D = 200: 800-byte rows start anywhere on a 32-byte sector, 7-8 lines).
// SVF_KS_FILTER_PF = 1: K-S prefetches each survivor's row at its filter (as K-S-L does) instead of at the gather;
// measured slower for K-S (C2 headline 0.5593 -> 0.5621 ms, C3 0.989 -> 1.289 ms), so off
#ifndef SVF_KS_FILTER_PF
#define SVF_KS_FILTER_PF 0
#endif
#ifndef SVF_LP_FILTER_PF
#define SVF_LP_FILTER_PF 1
#endif
#ifndef SVF_LP_FILTER_PF96
#define SVF_LP_FILTER_PF96 0
#endif
__device__ __forceinline__ void prefetch_rows_l2(const float4* __restrict__ vec4, const uint32_t* sid, int first,
                                                 int S, int DQ, int lane) {
  const int rb = DQ * 16;
  const int nl = (rb & 127) ? (rb >> 7) + 2 : (rb >> 7);  // lines a row may touch (aligned rows: exactly rb/128)
  for (int i = first * nl + lane; i < S * nl; i += 32) {
    const int s = i / nl, j = i - s * nl;
    const uintptr_t r0 = reinterpret_cast<uintptr_t>(vec4 + (size_t)sid[s] * DQ);
    const uintptr_t p = (r0 & ~(uintptr_t)127) + (uintptr_t)j * 128;
    if (p < r0 + rb) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

// One lane pulls every 128-byte line of vector row `id` toward L2 (the lane that found the survivor, at filter time)
template <int DQT>
__device__ __forceinline__ void prefetch_row_l2(const float4* __restrict__ vec4, uint32_t id, int DQ) {
  if constexpr (DQT > 0 && (DQT * 16) % 128 == 0) {  // rows are whole, aligned lines (D = 128: 4): unrolled
    const char* r0 = reinterpret_cast<const char*>(vec4 + (size_t)id * DQT);
#pragma unroll
    for (int j = 0; j < DQT * 16 / 128; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + j * 128));
  } else {
    const int rb = DQ * 16;
    const uintptr_t r0 = reinterpret_cast<uintptr_t>(vec4 + (size_t)id * DQ);
    for (uintptr_t p = r0 & ~(uintptr_t)127; p < r0 + rb; p += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

// Distances of the S ids sid[0..S) -> keys skey[0..S): teams of T lanes per vector, U vectors per team per round
// (U * 32/T rows in flight per warp), coalesced 16-byte gathers, FFMA, xor-shuffle reduction.
// PF (K-S-L): a key below `pf` (the best unparented pool key) makes its id the likely next parent, so the lane that
// computed it pulls that id's neighbour row toward L2 at once; the exact row load after the merge then hits L2.
__device__ __forceinline__ void prefetch_graph_row(const uint32_t* graph, int R, uint32_t id) {
  const char* p = reinterpret_cast<const char*>(graph + (size_t)id * R);
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  if (R > 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128));  // R = 64: two lines
  for (int b = 256; b < R * 4; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + b));
}

// Where a gather reads the query: this lane's NV float4 held in registers (K-S), or the row in shared memory (K-S-L
// with SVF_LP_QSMEM: 16 registers at D = 128 go to rows in flight instead)
struct QueryRegs {
  const float4 (&q)[4];
  __device__ __forceinline__ float4 operator()(int v, int) const { return q[v]; }
};
struct QuerySmem {
  const float4* q;
  __device__ __forceinline__ float4 operator()(int, int c) const { return q[c]; }
};

template <int DQT, int U, bool PF = false, class QF = QueryRegs>
__device__ __forceinline__ void gather_keys(const SearchArgs& a, const uint32_t* sid, uint64_t* skey, int S,
                                            const QF& qf, int lane, uint64_t pf = 0ull) {
  const int T = DQT ? Geo<DQT>::T : a.team, NV = DQT ? Geo<DQT>::NV : a.nv, DQ = DQT ? DQT : a.dq;
  const int tl = lane & (T - 1), team = lane / T, nteams = 32 / T;
  const float4* __restrict__ vec4 = reinterpret_cast<const float4*>(a.vec);
  __syncwarp();
#ifndef SVF_PREFETCH
#define SVF_PREFETCH 1
#endif
#if SVF_PREFETCH == 2
  // rows beyond the first gather round: one bulk L2 prefetch per row (TMA unit, no registers), so later rounds
  // hit L2 instead of waiting a full DRAM latency each
  for (int s = nteams * U + lane; s < S; s += 32)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vec4 + (size_t)sid[s] * DQ), "r"(DQ * 16)
                 : "memory");
#elif SVF_PREFETCH == 1
  // K-S-L (and K-S with SVF_KS_FILTER_PF) prefetched every survivor's row at its filter
  if (PF ? !(SVF_LP_FILTER_PF && (DQT == 32 || (SVF_LP_FILTER_PF96 && DQT == 24))) : !SVF_KS_FILTER_PF)
    prefetch_rows_l2(vec4, sid, nteams * U, S, DQ, lane);
#endif
  // the team geometry covers a row exactly at D = 96 / 128 (T * NV = DQ): rows load unconditionally (a slot past S
  // re-reads survivor 0's row, an L1 hit, and its key is never stored); other widths keep the per-lane guards
  constexpr bool kExact = PF && DQT > 0 && Geo<DQT>::T * Geo<DQT>::NV == DQT;  // K-S-L only (K-S keeps its guards)
  constexpr int NVC = DQT ? Geo<DQT>::NV : 4;  // float4 per lane per row (the generic path pads with zeros)
  for (int base = 0; base < S; base += nteams * U) {
    float4 xv[U][4];
    uint32_t id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + team + nteams * u;
      uint32_t rid;
      if (kExact) {  // one shared-memory read: slots past S re-read survivor 0
        rid = sid[s < S ? s : 0];
        id[u] = s < S ? rid : kSent;
      } else {
        id[u] = s < S ? sid[s] : kSent;
        rid = id[u] == kSent ? 0 : id[u];
      }
      const float4* row = vec4 + (size_t)rid * DQ;
#pragma unroll
      for (int v = 0; v < NVC; ++v) {
        const int c = tl + T * v;
        if (kExact)
          xv[u][v] = __ldg(row + c);
        else
          xv[u][v] = (v < NV && c < DQ && id[u] != kSent) ? __ldg(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    // one query float4 per v serves every row of the round (read once from shared memory in K-S-L)
    uint64_t acc2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc2[u] = 0ull;
#pragma unroll
    for (int v = 0; v < NVC; ++v) {
      const int c = tl + T * v;  // lanes past the row (generic / inexact geometries) hold zeros on both sides
      const float4 q = kExact || (v < NV && c < DQ) ? qf(v, c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u) acc2[u] = dist_acc4(acc2[u], xv[u][v], q, a.metric);
    }
    // every row's team reduction first (converged shuffles), then the divergent key stores
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = f2sum(acc2[u]);
      if (DQT) {
#pragma unroll
        for (int off = Geo<DQT>::T >> 1; off > 0; off >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], off);
      } else {
        for (int off = T >> 1; off > 0; off >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], off);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + team + nteams * u;
      if (tl == 0 && s < S) {
        float d = (a.metric == 0 ? acc[u] : -acc[u]) + 0.0f;  // canonical +0
        const uint64_t key = make_key(d, id[u]);
        skey[s] = key;
        if (PF && key < pf) prefetch_graph_row(a.graph, a.R, id[u]);
      }
    }
  }
  __syncwarp();
}

// Distances of this warp's S survivors sid[0..S) -> keys; keep those strictly better than the pool's current L-th
// key (the only ones that can enter: the pool keeps the L smallest of pool U cand), compacted into skey[0..S2).
template <int KPL, int CPL, int DQT, int U>
__device__ __forceinline__ int score_own(const SearchArgs& a, const uint64_t (&pool)[KPL], const uint32_t* sid,
                                         uint64_t* skey, int S, const float4 (&qv)[4], int lane) {
  gather_keys<DQT, U>(a, sid, skey, S, QueryRegs{qv}, lane);
  uint64_t kreg = kEmptyKey;
#pragma unroll
  for (int r = 0; r < KPL; ++r)
    if (r == ((a.L - 1) >> 5)) kreg = pool[r];
  const uint64_t kth = __shfl_sync(0xffffffffu, kreg, (a.L - 1) & 31);
  uint64_t c[CPL];
#pragma unroll
  for (int r = 0; r < CPL; ++r) {
    const int e = r * 32 + lane;
    c[r] = (e < S && skey[e] < kth) ? skey[e] : kEmptyKey;
  }
  __syncwarp();
  int S2 = 0;
#pragma unroll
  for (int r = 0; r < CPL; ++r) {
    const bool pass = c[r] != kEmptyKey;
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    if (pass) skey[S2 + __popc(m & ((1u << lane) - 1u))] = c[r];
    S2 += __popc(m);
  }
  return S2;
}

// Merge the union of the query's warps' surviving keys (list w = skeys[w][0..cnt[w])) into the pool.
template <int KPL, int CPL, int WPQ>
__device__ __forceinline__ void merge_all(const SearchArgs& a, uint64_t (&pool)[KPL], uint64_t* const (&lists)[WPQ],
                                          const int (&cnt)[WPQ], int total, int lane) {
  auto at = [&](int e) -> uint64_t {
    int off = 0;
#pragma unroll
    for (int w = 0; w < WPQ; ++w) {
      if (e - off < cnt[w]) return lists[w][e - off];
      off += cnt[w];
    }
    return kEmptyKey;
  };
  if (total <= 32) {
    uint64_t c1[1];
    c1[0] = lane < total ? at(lane) : kEmptyKey;
    warp_sort<1>(c1, lane);
    warp_merge_into<KPL, 1>(pool, c1, lane);
  } else {
    uint64_t c[CPL];
#pragma unroll
    for (int r = 0; r < CPL; ++r) {
      const int e = r * 32 + lane;
      c[r] = e < total ? at(e) : kEmptyKey;
    }
    warp_sort<CPL>(c, lane);
    warp_merge_into<KPL, CPL>(pool, c, lane);
  }
#pragma unroll
  for (int r = 0; r < KPL; ++r)
    if (r * 32 + lane >= a.L) pool[r] = kEmptyKey;  // exact pool size L (I6)
}

// Shared memory: one region per warp, [visited table 2^hbits | parents 8 | query id | survivor ids MP | keys 2xMP |
// counts].  A query served by W warps uses the first warp's table and query id and every warp's own parents,
// ids, keys and counts, so one-warp and two-warp (pair) processing share the layout.
// SVF_KS_TMA_ROW = 1: the one-warp kernel stages the speculative next parent's neighbour row in shared memory with a
// 1-D bulk copy (TMA unit, mbarrier completion) instead of holding it in registers (north star: "neighbour lists ...
// staged in shared memory via TMA"; A/B in DESIGN §6 K-S).  The tail then also holds [row buffer MP u32 | mbarrier].
#ifndef SVF_KS_TMA_ROW
#define SVF_KS_TMA_ROW 0
#endif
template <int CPL>
struct Smem {
  static constexpr int MP = 32 * CPL;
  static size_t __host__ __device__ head_bytes(int hbits) { return ((size_t)4 << hbits) + 32 + 16; }
  static constexpr size_t tail_bytes = (size_t)MP * 4 + (size_t)2 * MP * 8 + 16 + (SVF_KS_TMA_ROW ? (size_t)MP * 4 + 16 : 0);
  static size_t __host__ __device__ warp_bytes(int hbits) { return (head_bytes(hbits) + tail_bytes + 15) & ~(size_t)15; }
  static size_t __host__ __device__ block_bytes(int hbits) { return kSearchWarpsPerBlock * warp_bytes(hbits); }
};

// The table is cleared when an insertion round could push it past this load (numerator over 8); the host keeps
// H >= 4 * max(pool, round size), so any load <= 3/4 leaves room for a full round.
#ifndef SVF_HASH_LOAD8
#define SVF_HASH_LOAD8 4
#endif

// Resume kernel: the next suspended query's slot index, or ~0 once every one-warp warp has left and no reserved
// slot remains (lane 0 of the query's first warp).
__device__ __forceinline__ unsigned long long ho_take(const SearchArgs& a, size_t stride) {
  const unsigned long long i = atomicAdd(a.ho + 2, 1ull);
  if (i >= (unsigned long long)a.ho_total) return ~0ull;  // at most one suspension per one-warp warp
  volatile unsigned long long* hs = a.ho + 8 + i * stride;
  for (;;) {
    if (hs[0] >> 63) {
      __threadfence();
      return i;
    }
    if (*reinterpret_cast<volatile unsigned long long*>(a.ho + 3) >= (unsigned long long)a.ho_total) {
      // every one-warp warp has left (each published its slot before leaving): reservations are final
      __threadfence();
      if (i >= *reinterpret_cast<volatile unsigned long long*>(a.ho + 0)) return ~0ull;
    }
    __nanosleep(256);
  }
}

// Serve queries [base + fetched] while fetched < limit, W warps per query; `g0` = first warp of this group,
// h = this warp's rank in it, slot = the group's barrier slot.
template <int KPL, int CPL, int DQT, int W>
__device__ __forceinline__ void run_queries(const SearchArgs& a, unsigned char* smem, int g0, int h, int slot,
                                            unsigned long long* counter, int64_t base, int64_t limit, int lane) {
  constexpr int MP = 32 * CPL;
  using SM = Smem<CPL>;
  const size_t wb = SM::warp_bytes(a.hbits);
  unsigned char* lead = smem + (size_t)g0 * wb;
  uint32_t* tab = reinterpret_cast<uint32_t*>(lead);
  unsigned long long* qslot = reinterpret_cast<unsigned long long*>(lead + ((size_t)4 << a.hbits) + 32);
  unsigned char* wbase[W];
#pragma unroll
  for (int w = 0; w < W; ++w) wbase[w] = smem + (size_t)(g0 + w) * wb;
  uint32_t* spar = reinterpret_cast<uint32_t*>(wbase[h] + ((size_t)4 << a.hbits));  // this warp's parents
  uint32_t* sid = reinterpret_cast<uint32_t*>(wbase[h] + SM::head_bytes(a.hbits));
  const int H = 1 << a.hbits;
  const int T = DQT ? Geo<DQT>::T : a.team;
  const int tl = lane & (T - 1);
  auto keys_of = [&](int w, int par) {
    return reinterpret_cast<uint64_t*>(wbase[w] + SM::head_bytes(a.hbits) + (size_t)MP * 4) + par * MP;
  };
  auto cnts_of = [&](int w) {
    return reinterpret_cast<int*>(wbase[w] + SM::head_bytes(a.hbits) + (size_t)MP * 4 + (size_t)2 * MP * 8);
  };
  constexpr bool TMA_ROW = SVF_KS_TMA_ROW && W == 1;
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(cnts_of(h)) + 16);
  uint64_t* rowbar = reinterpret_cast<uint64_t*>(rowbuf + MP);
  uint32_t rphase = 0;
  bool rpending = false;  // a bulk copy into rowbuf may still be landing
  if (TMA_ROW) {
    if (lane == 0) bulk_mbar_init(rowbar);
    __syncwarp();
  }
  auto row_settle = [&]() {  // wait for the outstanding bulk copy (before reading or re-filling rowbuf, or leaving)
    if (TMA_ROW && rpending) {
      bulk_wait(rowbar, rphase);
      rphase ^= 1u;
      rpending = false;
    }
  };
  constexpr int WPQ = W;
  const bool resume = WPQ == 2 && a.is_tail;          // chained kernel: continue suspended queries
  const bool ho_on = WPQ == 1 && a.ho != nullptr;     // one-warp kernel that may suspend its stragglers
  // one slot layout for every pool size, so headers never alias pool keys left by a launch with another size
  constexpr size_t ho_stride = 4 + 32 * kHandoffMaxKpl;
  unsigned long long ho_ex = 0;                       // one-warp warps that have left (lane 0, loaded early)
  for (;;) {
    if (h == 0 && lane == 0) {
      const unsigned long long f = resume ? ho_take(a, ho_stride) : atomicAdd(counter, 1ull);
      // streamed host queries: wait until this query's chunk has landed (a resumed query's chunk already has)
      if (!resume && a.q_flags != nullptr && f < (unsigned long long)limit) {
        const volatile unsigned int* fl = a.q_flags + ((base + f) >> a.q_chunk_log2);
        while (*fl != a.q_epoch) __nanosleep(64);
        __threadfence();
      }
      qslot[0] = f;
      // the query's snapshot: ids below n exist (n_visible: inserts completed on another stream); resumed queries
      // keep the snapshot they started with
      unsigned long long nq = a.n_alloc;
      if (resume) {
        if (f != ~0ull) nq = __ldcg(a.ho + 8 + f * ho_stride + 2) >> 32;
      } else if (a.n_visible != nullptr) {
        nq = min(nq, *reinterpret_cast<const volatile unsigned long long*>(a.n_visible));
      }
      qslot[1] = nq;
    }
    qsync<WPQ>(slot);
    const unsigned long long qf = qslot[0];
    const uint32_t n = (uint32_t)qslot[1];  // ids are u32 below the sentinel: n < 2^32
    if (qf >= (unsigned long long)limit) break;
    unsigned long long* hs = resume ? a.ho + 8 + qf * ho_stride : nullptr;
    const unsigned long long qi = resume ? (__ldcg(hs) & 0xFFFFFFFFFFull) : (unsigned long long)base + qf;
    unsigned long long t_start = 0;
    if (a.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    // S0: the query fragment this lane needs (zero-padded to Dp), straight from global memory; clear the table
    // the query is staged (coalesced) through the visited table, which is cleared right after (H >= Dp: host)
    const float* qg = a.Q + (size_t)qi * a.q_stride;
    float* qstage = reinterpret_cast<float*>(tab);
    for (int i = h * 32 + lane; i < a.dq * 4; i += 32 * WPQ) qstage[i] = i < a.q_dim ? __ldcg(qg + i) : 0.f;
    qsync<WPQ>(slot);
    float4 qv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = tl + T * v;
      qv[v] = (v < (DQT ? Geo<DQT>::NV : a.nv) && c < a.dq) ? reinterpret_cast<const float4*>(qstage)[c]
                                                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    qsync<WPQ>(slot);
    for (int i = h * 32 + lane; i < H; i += 32 * WPQ) tab[i] = kHashEmpty;
    qsync<WPQ>(slot);
    uint64_t pool[KPL];
#pragma unroll
    for (int r = 0; r < KPL; ++r) pool[r] = kEmptyKey;
    int hcount = 0, par = 0;
    uint32_t n_dist = 0, iters = 0, n_exp = 0;
    uint32_t spec_id = kSent;  // parent whose row sits in spec_row (speculative next-row load)
    uint32_t spec_row[CPL];

    // exchange the warps' survivor lists and merge (one barrier per step)
    auto exchange_merge = [&](int S_own, int S2_own) {
      if (lane == 0) {
        cnts_of(h)[par * 2 + 0] = S_own;
        cnts_of(h)[par * 2 + 1] = S2_own;
      }
      qsync<WPQ>(slot);
      int cnt[WPQ];
      uint64_t* lists[WPQ];
      int total = 0, raw = 0;
#pragma unroll
      for (int w = 0; w < WPQ; ++w) {
        raw += cnts_of(w)[par * 2 + 0];
        cnt[w] = cnts_of(w)[par * 2 + 1];
        lists[w] = keys_of(w, par);
        total += cnt[w];
      }
      hcount += raw;
      n_dist += raw;
      if (total > 0) merge_all<KPL, CPL, WPQ>(a, pool, lists, cnt, total, lane);
      par ^= 1;
    };

    // S1: the first n_init live ids along the seeded affine permutation (I2), scored and merged in chunks
    if (resume) {
      // continue a suspended query: its pool (keys with parent flags) and counters; the visited table restarts
      // from the pool ids, which leaves the search unchanged (I7: a forgotten non-pool id is rejected again)
      const unsigned long long c1 = __ldcg(hs + 1);
      n_dist = (uint32_t)c1;
      iters = (uint32_t)(c1 >> 32);
      n_exp = (uint32_t)__ldcg(hs + 2);  // (high half: the snapshot n, read at the fetch)
      if (a.trace != nullptr) t_start = __ldcg(hs + 3);
#pragma unroll
      for (int r = 0; r < KPL; ++r) pool[r] = __ldcg(hs + 4 + r * 32 + lane);
      hcount = hash_reset<KPL, WPQ>(tab, a.hbits, pool, lane, h, slot);
      if (h == 0 && lane == 0) hs[0] = 0;  // both warps have read the slot: free for the next launch
    } else if (n > 0) {
      uint64_t pa = 0, pb = 0;
      if (lane == 0) perm_params(a.seed, a.qidx_base + qi, n, pa, pb);
      pa = __shfl_sync(0xffffffffu, pa, 0);
      pb = __shfl_sync(0xffffffffu, pb, 0);
      // lane's id for j = j0 + r*32 + lane, advanced by 32 permutation steps per register (32-bit adds)
      uint32_t cur = (uint32_t)((pa * (uint64_t)lane + pb) % n);
      const uint32_t step32 = (uint32_t)((pa * 32ull) % n);
      int taken = 0;
      for (uint64_t j0 = 0; j0 < n && taken < a.n_init; j0 += MP) {
        if (hcount + MP > H * SVF_HASH_LOAD8 / 8) hcount = hash_reset<KPL, WPQ>(tab, a.hbits, pool, lane, h, slot);
        int running = 0, mine = 0;
#pragma unroll
        for (int r = 0; r < CPL; ++r) {
          const uint64_t j = j0 + (uint64_t)(r * 32 + lane);
          const uint32_t id = cur;
          cur += step32;
          if (cur >= (uint32_t)n) cur -= (uint32_t)n;
          bool ok = j < n;
          if (ok) ok = !tomb_dead(a.tomb, id);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const int pos = running + __popc(m & ((1u << lane) - 1u));  // position among this chunk's live ids
          const bool keep = ok && taken + pos < a.n_init && ((pos >> 5) % WPQ) == h;
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          if (keep) {
            sid[mine + __popc(km & ((1u << lane) - 1u))] = id;
            hash_insert(tab, a.hbits, id);
            if (SVF_KS_FILTER_PF) prefetch_row_l2<DQT>(reinterpret_cast<const float4*>(a.vec), id, DQT ? DQT : a.dq);
          }
          mine += __popc(km);
          running += __popc(m);
        }
        const int kept = min(running, a.n_init - taken);
        taken += kept;
        const int S2 = score_own<KPL, CPL, DQT, gather_u<WPQ, KPL, DQT>()>(a, pool, sid, keys_of(h, par), mine, qv, lane);
        exchange_merge(mine, S2);
      }
    }

    // S2-S7: expand the first p unparented entries until every pool entry is parented (I3, I4)
#ifdef SVF_PHASE_PROF
    unsigned long long ph[5] = {0, 0, 0, 0, 0};
    long long tp = clock64();
#define SVF_PH(i)                 \
  {                               \
    const long long tn = clock64(); \
    ph[i] += tn - tp;             \
    tp = tn;                      \
  }
#else
#define SVF_PH(i)
#endif
    bool suspended = false;
    for (;;) {
      if (ho_on) {
        // the queue has drained and few one-warp warps are left: hand this query to the pair-mode kernel
        const unsigned long long ex = __shfl_sync(0xffffffffu, ho_ex, 0);
        if ((unsigned long long)a.ho_total - ex < (unsigned long long)a.ho_thresh) {
          unsigned long long si = 0;
          if (lane == 0) si = atomicAdd(a.ho + 0, 1ull);
          si = __shfl_sync(0xffffffffu, si, 0);
          unsigned long long* ws = a.ho + 8 + si * ho_stride;
#pragma unroll
          for (int r = 0; r < KPL; ++r) ws[4 + r * 32 + lane] = pool[r];
          if (lane == 0) {
            ws[1] = (unsigned long long)n_dist | ((unsigned long long)iters << 32);
            ws[2] = (unsigned long long)n_exp | ((unsigned long long)n << 32);
            ws[3] = t_start;
          }
          __threadfence();
          __syncwarp();
          if (lane == 0) {
            __threadfence();
            *reinterpret_cast<volatile unsigned long long*>(ws) = qi | (1ull << 63);
          }
          suspended = true;
          break;
        }
        if (lane == 0) ho_ex = *reinterpret_cast<volatile unsigned long long*>(a.ho + 3);  // used next iteration
      }
      if (a.max_iter > 0 && (int)iters == a.max_iter) break;
      __syncwarp();  // the previous iteration's reads of spar are done before it is rewritten
      int np = 0;
#pragma unroll
      for (int r = 0; r < KPL; ++r) {
        unsigned m = __ballot_sync(0xffffffffu, (pool[r] & 1ull) == 0ull);
        while (m != 0u && np < a.p) {
          const int l = __ffs(m) - 1;
          m &= m - 1u;
          const uint64_t kk = __shfl_sync(0xffffffffu, pool[r], l);
          if (lane == l) pool[r] |= 1ull;
          if (lane == 0) spar[np] = key_id(kk);
          ++np;
        }
      }
      if (np == 0) break;
      __syncwarp();
      SVF_PH(0)
      // The best still-unparented entry is the likely next parent (it stays first unless this iteration's
      // candidates beat it).  p == 1: load its row into registers now, consumed next iteration if the guess holds,
      // so the dependent row fetch overlaps this iteration's vector gathers.  p > 1: pull it toward L2.
      uint64_t nxt = kEmptyKey;
#pragma unroll
      for (int r = KPL - 1; r >= 0; --r) {
        const unsigned m = __ballot_sync(0xffffffffu, (pool[r] & 1ull) == 0ull);
        if (m) nxt = __shfl_sync(0xffffffffu, pool[r], __ffs(m) - 1);
      }
      ++iters;
      n_exp += np;
      const int ncand = np * a.R;
      if (hcount + ncand > H * SVF_HASH_LOAD8 / 8) hcount = hash_reset<KPL, WPQ>(tab, a.hbits, pool, lane, h, slot);
      // S3: this warp's neighbour-row slots (registers r with r % WPQ == h), coalesced; from the speculative
      // registers when the guess was right
      uint32_t rowv[CPL];
      const bool hit = np == 1 && spar[0] == spec_id;
      if (TMA_ROW && hit) row_settle();  // the bulk copy of the guessed row has landed in rowbuf
      for (int r = 0; r < CPL; ++r) {
        const int e = r * 32 + lane;
        rowv[r] = kSent;
        if ((r % WPQ) != h) continue;
        if (hit) {
          if (TMA_ROW) rowv[r] = e < a.R ? rowbuf[e] : kSent;
          else rowv[r] = spec_row[r];
        } else if (e < ncand) {
          const int pi = a.rshift >= 0 ? (e >> a.rshift) : e / a.R;
          rowv[r] = __ldg(a.graph + (size_t)spar[pi] * a.R + (e - pi * a.R));
        }
      }
      spec_id = kSent;
      if (nxt != kEmptyKey) {
        if (a.p == 1) {
          spec_id = key_id(nxt);
          if (TMA_ROW) {
            row_settle();
            __syncwarp();  // every lane's reads of rowbuf are done
            if (lane == 0) bulk_copy_g2s(rowbuf, a.graph + (size_t)spec_id * a.R, (uint32_t)a.R * 4u, rowbar);
            rpending = true;
          } else {
#pragma unroll
            for (int r = 0; r < CPL; ++r) {
              const int e = r * 32 + lane;
              if ((r % WPQ) == h) spec_row[r] = e < a.R ? __ldg(a.graph + (size_t)spec_id * a.R + e) : kSent;
            }
          }
        } else if (h == 0 && lane < ((a.R * 4 + 127) >> 7)) {
          const uint32_t* prow = a.graph + (size_t)key_id(nxt) * a.R + lane * 32;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(prow));
        }
      }
      SVF_PH(1)
      // S4: sentinel / snapshot / tombstone / visited filters on this warp's slots
      int running = 0;
#pragma unroll
      for (int r = 0; r < CPL; ++r) {
        if ((r % WPQ) != h) continue;
        const uint32_t id = rowv[r];
        bool ok = id != kSent && (uint64_t)id < n;
        if (ok) ok = !tomb_dead(a.tomb, id);
        if (ok) ok = hash_insert(tab, a.hbits, id);
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          sid[running + __popc(m & ((1u << lane) - 1u))] = id;
          if (SVF_KS_FILTER_PF) prefetch_row_l2<DQT>(reinterpret_cast<const float4*>(a.vec), id, DQT ? DQT : a.dq);
        }
        running += __popc(m);
      }
      SVF_PH(2)
      // S5: distances of this warp's survivors; S6: exchange + merge
      if (WPQ == 1 && running == 0) continue;
      const int S2 = score_own<KPL, CPL, DQT, gather_u<WPQ, KPL, DQT>()>(a, pool, sid, keys_of(h, par), running, qv, lane);
      SVF_PH(3)
      exchange_merge(running, S2);
      SVF_PH(4)
    }

    // S8: emit the first n_out entries (k, or the whole pool in insert mode)
    if (h == 0 && !suspended) {
#pragma unroll
      for (int r = 0; r < KPL; ++r) {
        const int e = r * 32 + lane;
        if (e < a.n_out) {
          a.out_ids[(size_t)qi * a.n_out + e] = key_id(pool[r]);
          a.out_d[(size_t)qi * a.n_out + e] = key_dist(pool[r]);
        }
      }
      if (a.counters != nullptr && lane == 0) {
        a.counters[qi * 3 + 0] = n_dist;
        a.counters[qi * 3 + 1] = iters;
        a.counters[qi * 3 + 2] = n_exp;
      }
      if (a.trace != nullptr && lane == 0) {
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
  row_settle();  // no bulk copy outlives the warp (its block's shared memory may be released)
}

template <int KPL, int CPL, int DQT, int WPQ>
__global__ void __launch_bounds__(kSearchWarpsPerBlock * 32, search_min_blocks(KPL, WPQ)) search_kernel(SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  if (WPQ == 2 && a.is_tail) {
    // chained resume kernel: continue the suspended queries, then wait for the one-warp grid so that stream order
    // (the next operation waits for this grid) also covers it
    run_queries<KPL, CPL, DQT, WPQ>(a, smem, wib - wib % WPQ, wib % WPQ, wib / WPQ, nullptr, 0, INT64_MAX, lane);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  // the chained resume kernel may be launched at once: its blocks take SM slots only as this grid's blocks exit,
  // i.e. after the queue has drained
  if (a.ho != nullptr) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  run_queries<KPL, CPL, DQT, WPQ>(a, smem, wib - wib % WPQ, wib % WPQ, wib / WPQ, a.work_counter, 0, a.nq, lane);
  if (WPQ == 1 && a.ho != nullptr && lane == 0) {
    __threadfence();  // this warp's suspended slot (if any) is published before it counts as gone
    atomicAdd(a.ho + 3, 1ull);
  }
}

}  // namespace

// resident blocks per SM of one instantiation (cached: keeps the launch path host-light) and its shared memory
template <int KPL, int CPL, int DQT, int WPQ>
static cudaError_t blocks_per_sm(const SearchArgs& a, int& per_sm, size_t& smem) {
  auto kern = search_kernel<KPL, CPL, DQT, WPQ>;
  smem = Smem<CPL>::block_bytes(a.hbits);
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_per_sm = 0;
  static thread_local int cached_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (cached_smem == smem && cached_dev == dev) {
    per_sm = cached_per_sm;
    return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // Carveout: the L1 part of the unified array holds the in-flight gather lines, so it must stay large (a max-
  // shared carveout measured 20% slower); ask for just enough shared memory for the register-limited residency.
  const int want = search_min_blocks(KPL, WPQ);
  const int pct = (int)std::min<size_t>(100, (want * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSearchWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  cached_smem = smem;
  cached_per_sm = per_sm;
  cached_dev = dev;
  return cudaSuccess;
}

template <int KPL, int CPL, int DQT, int WPQ>
static cudaError_t launch_kpl_cpl(SearchArgs a, int num_sms, cudaStream_t st) {
  int per_sm = 0;
  size_t smem = 0;
  cudaError_t e = blocks_per_sm<KPL, CPL, DQT, WPQ>(a, per_sm, smem);
  if (e != cudaSuccess) return e;
  long long blocks = (long long)per_sm * num_sms;
  constexpr int qpb = kSearchWarpsPerBlock / WPQ;
  const long long need = (a.nq + qpb - 1) / qpb;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  search_kernel<KPL, CPL, DQT, WPQ><<<(unsigned)blocks, kSearchWarpsPerBlock * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// One-warp grid + chained pair-mode resume grid (handoff of the batch's stragglers, see SearchArgs::ho).
// a.ho_thresh arrives as a percentage of the one-warp grid's warps.
template <int KPL, int CPL, int DQT>
static cudaError_t launch_handoff(SearchArgs a, int num_sms, cudaStream_t st) {
  int per_sm = 0, per_sm2 = 0;
  size_t smem = 0, smem2 = 0;
  cudaError_t e = blocks_per_sm<KPL, CPL, DQT, 1>(a, per_sm, smem);
  if (e != cudaSuccess) return e;
  e = blocks_per_sm<KPL, CPL, DQT, 2>(a, per_sm2, smem2);
  if (e != cudaSuccess) return e;
  long long blocks = (long long)per_sm * num_sms;
  const long long need = (a.nq + kSearchWarpsPerBlock - 1) / kSearchWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  a.ho_total = (int)(blocks * kSearchWarpsPerBlock);
  if (a.ho_total > kHandoffMaxWarps) return launch_kpl_cpl<KPL, CPL, DQT, 1>(a, num_sms, st);  // no slots
  a.ho_thresh = (int)((long long)a.ho_total * a.ho_thresh / 100);
  search_kernel<KPL, CPL, DQT, 1><<<(unsigned)blocks, kSearchWarpsPerBlock * 32, smem, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // programmatic dependent launch: the one-warp grid triggers at its start, so this grid's blocks are pending and
  // take SM slots as the one-warp grid's blocks exit
  long long blocks2 = (long long)per_sm2 * num_sms;
  // at most ho_thresh queries are still in flight when the warps start to suspend: two warps each
  const long long need2 = ((long long)a.ho_thresh * 2 + kSearchWarpsPerBlock - 1) / kSearchWarpsPerBlock + 1;
  if (blocks2 > need2) blocks2 = need2;
  a.is_tail = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)blocks2);
  cfg.blockDim = dim3(kSearchWarpsPerBlock * 32);
  cfg.dynamicSmemBytes = smem2;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, search_kernel<KPL, CPL, DQT, 2>, a);
}

template <int KPL, int CPL, int DQT>
static cudaError_t launch_wpq(SearchArgs a, int num_sms, cudaStream_t st) {
  // two warps per query only where the candidate slots split evenly (CPL >= 2) and pools are small
  if constexpr (CPL >= 2 && KPL <= 4) {
    if (a.wpq == 2) {
      a.ho = nullptr;
      return launch_kpl_cpl<KPL, CPL, DQT, 2>(a, num_sms, st);
    }
    if (a.ho != nullptr && a.ho_thresh > 0) return launch_handoff<KPL, CPL, DQT>(a, num_sms, st);
  }
  a.ho = nullptr;
  return launch_kpl_cpl<KPL, CPL, DQT, 1>(a, num_sms, st);
}

template <int KPL, int DQT>
static cudaError_t launch_kpl(SearchArgs a, int cpl, int num_sms, cudaStream_t st) {
  switch (cpl) {
    case 1: return launch_wpq<KPL, 1, DQT>(a, num_sms, st);
    case 2: return launch_wpq<KPL, 2, DQT>(a, num_sms, st);
    case 4: return launch_wpq<KPL, 4, DQT>(a, num_sms, st);
    case 8: return launch_wpq<KPL, 8, DQT>(a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

template <int DQT>
cudaError_t launch_search_lp_dq(SearchArgs a, int cpl, int num_sms, cudaStream_t st);

template <int DQT>
cudaError_t launch_search_dq(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
  if (a.large_pool) return launch_search_lp_dq<DQT>(a, cpl, num_sms, st);  // K-S-L (search_lp.cuh)
  switch (kpl) {
    case 1: return launch_kpl<1, DQT>(a, cpl, num_sms, st);
    case 2: return launch_kpl<2, DQT>(a, cpl, num_sms, st);
    case 4: return launch_kpl<4, DQT>(a, cpl, num_sms, st);
    case 8: return launch_kpl<8, DQT>(a, cpl, num_sms, st);
    case 16: return launch_kpl<16, DQT>(a, cpl, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace svf

#include "search_lp.cuh"
