// K-S: batched greedy graph search on sm_100a (Algorithm 1).
//
// Design (DESIGN.md §"K-S"): one WARP per query, persistent warps pulling queries from an atomic counter.
//  - pool (the paper's candidate list C_i) lives in registers as 64-bit keys (dist, id, parent flag),
//    striped over the warp (element e = r*32 + lane), exact size L (I6) inside a power-of-two buffer;
//  - visited set = per-warp open-addressing table in shared memory, "forgetful": when it reaches half load it
//    is cleared and the pool ids are re-registered, which provably leaves results unchanged (I7);
//  - distances: teams of T lanes per vector, each lane loads NV coalesced 16-byte chunks of the row, FFMA,
//    xor-shuffle reduction inside the team;
//  - merge: bitonic sort of the candidate keys + bitonic merge into the pool (warp shuffles only).
// No __syncthreads: the warps of a block are independent; all intra-query sync is __syncwarp.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

__device__ __forceinline__ bool hash_insert(uint32_t* tab, int hbits, uint32_t id) {
  const uint32_t mask = (1u << hbits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - hbits);
  for (;;) {
    uint32_t prev = atomicCAS(tab + h, kHashEmpty, id);
    if (prev == kHashEmpty) return true;
    if (prev == id) return false;
    h = (h + 1) & mask;
  }
}

template <int KPL>
__device__ __forceinline__ int hash_reset(uint32_t* tab, int hbits, const uint64_t (&pool)[KPL], int lane) {
  __syncwarp();
  const int H = 1 << hbits;
  for (int i = lane; i < H; i += 32) tab[i] = kHashEmpty;
  __syncwarp();
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < KPL; ++r) {
    const bool v = pool[r] != kEmptyKey;
    if (v) hash_insert(tab, hbits, key_id(pool[r]));
    cnt += __popc(__ballot_sync(0xffffffffu, v));
  }
  __syncwarp();
  return cnt;
}

// Team geometry: DQT > 0 fixes the row length (float4 count) at compile time (the configs' D = 96 / 128 / 200);
// DQT == 0 is the generic path with the runtime geometry of SearchArgs.
template <int DQT>
struct Geo {
  static constexpr int T = DQT <= 4 ? 1 : DQT <= 8 ? 2 : DQT <= 16 ? 4 : DQT <= 32 ? 8 : DQT <= 64 ? 16 : 32;
  static constexpr int NV = (DQT + T - 1) / T;
};

// Distances for the S survivors listed in sid[0..S) -> skey[0..S); then sort + merge into the pool.
template <int KPL, int CPL, int DQT>
__device__ __forceinline__ void score_and_merge(const SearchArgs& a, uint64_t (&pool)[KPL], const uint32_t* sid,
                                                uint64_t* skey, int S, const float4 (&qv)[4], int lane) {
  constexpr int U = 2;
  const int T = DQT ? Geo<DQT>::T : a.team, NV = DQT ? Geo<DQT>::NV : a.nv, DQ = DQT ? DQT : a.dq;
  const int tl = lane & (T - 1), team = lane / T, nteams = 32 / T;
  const float4* __restrict__ vec4 = reinterpret_cast<const float4*>(a.vec);
  __syncwarp();
  for (int base = 0; base < S; base += nteams * U) {
    float4 xv[U][4];
    uint32_t id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + team + nteams * u;
      id[u] = s < S ? sid[s] : kSent;
      const float4* row = vec4 + (size_t)(id[u] == kSent ? 0 : id[u]) * DQ;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = tl + T * v;
        xv[u][v] = (v < NV && c < DQ && id[u] != kSent) ? __ldg(row + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc = 0.f;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (a.metric == 0) {
          float dx = xv[u][v].x - qv[v].x, dy = xv[u][v].y - qv[v].y;
          float dz = xv[u][v].z - qv[v].z, dw = xv[u][v].w - qv[v].w;
          acc = fmaf(dx, dx, acc);
          acc = fmaf(dy, dy, acc);
          acc = fmaf(dz, dz, acc);
          acc = fmaf(dw, dw, acc);
        } else {
          acc = fmaf(xv[u][v].x, qv[v].x, acc);
          acc = fmaf(xv[u][v].y, qv[v].y, acc);
          acc = fmaf(xv[u][v].z, qv[v].z, acc);
          acc = fmaf(xv[u][v].w, qv[v].w, acc);
        }
      }
      if (DQT) {
#pragma unroll
        for (int off = Geo<DQT>::T >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      } else {
        for (int off = T >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      }
      const int s = base + team + nteams * u;
      if (tl == 0 && s < S) {
        float d = (a.metric == 0 ? acc : -acc) + 0.0f;  // canonical +0
        skey[s] = make_key(d, id[u]);
      }
    }
  }
  __syncwarp();
  // Only candidates strictly better than the pool's current L-th key can enter (exact: the pool keeps the L
  // smallest of pool U cand).  Drop the rest before sorting; most iterations keep only a handful.
  uint64_t kreg = kEmptyKey;
#pragma unroll
  for (int r = 0; r < KPL; ++r)
    if (r == ((a.L - 1) >> 5)) kreg = pool[r];
  const uint64_t kth = __shfl_sync(0xffffffffu, kreg, (a.L - 1) & 31);
  uint64_t c[CPL];
  int S2 = 0;
#pragma unroll
  for (int r = 0; r < CPL; ++r) {
    const int e = r * 32 + lane;
    c[r] = e < S ? skey[e] : kEmptyKey;
    const bool pass = c[r] < kth;
    c[r] = pass ? c[r] : kEmptyKey;
    S2 += __popc(__ballot_sync(0xffffffffu, pass));
  }
  if (S2 == 0) return;
  if (S2 <= 32) {
    // compact the survivors into one register (through shared memory) and use a 32-wide sort
    __syncwarp();
    int base2 = 0;
#pragma unroll
    for (int r = 0; r < CPL; ++r) {
      const bool pass = c[r] != kEmptyKey;
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) skey[base2 + __popc(m & ((1u << lane) - 1u))] = c[r];
      base2 += __popc(m);
    }
    __syncwarp();
    uint64_t c1[1];
    c1[0] = lane < S2 ? skey[lane] : kEmptyKey;
    warp_sort<1>(c1, lane);
    warp_merge_into<KPL, 1>(pool, c1, lane);
  } else {
    warp_sort<CPL>(c, lane);
    warp_merge_into<KPL, CPL>(pool, c, lane);
  }
#pragma unroll
  for (int r = 0; r < KPL; ++r)
    if (r * 32 + lane >= a.L) pool[r] = kEmptyKey;  // exact pool size L (I6)
}

template <int KPL, int CPL, int DQT>
__global__ void __launch_bounds__(kSearchWarpsPerBlock * 32, search_min_blocks(KPL)) search_kernel(SearchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int MP = 32 * CPL;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* base = smem + (size_t)wib * a.smem_per_warp;
  float4* qs = reinterpret_cast<float4*>(base);
  uint64_t* skey = reinterpret_cast<uint64_t*>(base + (size_t)a.dq * 16);
  uint32_t* sid = reinterpret_cast<uint32_t*>(skey + MP);
  uint32_t* spar = sid + MP;  // parents of the current iteration (<= 8)
  uint32_t* tab = spar + 8;
  const int H = 1 << a.hbits;
  const int T = DQT ? Geo<DQT>::T : a.team;
  const int tl = lane & (T - 1);

  for (;;) {
    unsigned long long qi = 0;
    if (lane == 0) qi = atomicAdd(a.work_counter, 1ull);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= (unsigned long long)a.nq) break;

    // S0: stage the query (zero-padded to Dp) and clear the visited table
    const float* qg = a.Q + (size_t)qi * a.q_stride;
    float* qsf = reinterpret_cast<float*>(qs);
    for (int i = lane; i < a.dq * 4; i += 32) qsf[i] = i < a.q_dim ? __ldg(qg + i) : 0.f;
    for (int i = lane; i < H; i += 32) tab[i] = kHashEmpty;
    __syncwarp();
    float4 qv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = tl + T * v;
      qv[v] = (v < (DQT ? Geo<DQT>::NV : a.nv) && c < a.dq) ? qs[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    uint64_t pool[KPL];
#pragma unroll
    for (int r = 0; r < KPL; ++r) pool[r] = kEmptyKey;
    int hcount = 0;
    uint32_t n_dist = 0, iters = 0, n_exp = 0;
    uint32_t spec_id = kSent;  // parent whose row sits in spec_row (speculative next-row load)
    uint32_t spec_row[CPL];

    // S1: the first n_init live ids along the seeded affine permutation (I2), scored and merged in chunks
    const uint64_t n = a.n_alloc;
    if (n > 0) {
      uint64_t pa = 0, pb = 0;
      if (lane == 0) perm_params(a.seed, a.qidx_base + qi, n, pa, pb);
      pa = __shfl_sync(0xffffffffu, pa, 0);
      pb = __shfl_sync(0xffffffffu, pb, 0);
      // lane's id for j = j0 + r*32 + lane, advanced by 32 permutation steps per register (32-bit adds)
      uint32_t cur = (uint32_t)((pa * (uint64_t)lane + pb) % n);
      const uint32_t step32 = (uint32_t)((pa * 32ull) % n);
      int taken = 0;
      for (uint64_t j0 = 0; j0 < n && taken < a.n_init; j0 += MP) {
        if (hcount + MP > H / 2) hcount = hash_reset<KPL>(tab, a.hbits, pool, lane);
        int running = 0;
#pragma unroll
        for (int r = 0; r < CPL; ++r) {
          const uint64_t j = j0 + (uint64_t)(r * 32 + lane);
          const uint32_t id = cur;
          cur += step32;
          if (cur >= (uint32_t)n) cur -= (uint32_t)n;
          bool ok = j < n;
          if (ok) ok = !tomb_dead(a.tomb, id);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const int rank = taken + running + __popc(m & ((1u << lane) - 1u));
          if (ok && rank < a.n_init) {
            sid[rank - taken] = id;
            hash_insert(tab, a.hbits, id);
          }
          running += __popc(m);
        }
        const int kept = min(running, a.n_init - taken);
        taken += kept;
        hcount += kept;
        n_dist += kept;
        score_and_merge<KPL, CPL, DQT>(a, pool, sid, skey, kept, qv, lane);
      }
    }

    // S2-S7: expand the first p unparented entries until every pool entry is parented (I3, I4)
    for (;;) {
      if (a.max_iter > 0 && (int)iters == a.max_iter) break;
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
      if (hcount + ncand > H / 2) hcount = hash_reset<KPL>(tab, a.hbits, pool, lane);
      // S3: neighbour rows (coalesced; from the speculative registers when the guess was right)
      uint32_t rowv[CPL];
      if (np == 1 && spar[0] == spec_id) {
#pragma unroll
        for (int r = 0; r < CPL; ++r) rowv[r] = spec_row[r];
      } else {
#pragma unroll
        for (int r = 0; r < CPL; ++r) {
          const int e = r * 32 + lane;
          rowv[r] = kSent;
          if (e < ncand) {
            const int pi = a.rshift >= 0 ? (e >> a.rshift) : e / a.R;
            rowv[r] = __ldg(a.graph + (size_t)spar[pi] * a.R + (e - pi * a.R));
          }
        }
      }
      spec_id = kSent;
      if (nxt != kEmptyKey) {
        if (a.p == 1) {
          spec_id = key_id(nxt);
#pragma unroll
          for (int r = 0; r < CPL; ++r) {
            const int e = r * 32 + lane;
            spec_row[r] = e < a.R ? __ldg(a.graph + (size_t)spec_id * a.R + e) : kSent;
          }
        } else if (lane < ((a.R * 4 + 127) >> 7)) {
          const uint32_t* prow = a.graph + (size_t)key_id(nxt) * a.R + lane * 32;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(prow));
        }
      }
      // S4: sentinel / snapshot / tombstone / visited filters
      int running = 0;
#pragma unroll
      for (int r = 0; r < CPL; ++r) {
        const uint32_t id = rowv[r];
        bool ok = id != kSent && (uint64_t)id < n;
        if (ok) ok = !tomb_dead(a.tomb, id);
        if (ok) ok = hash_insert(tab, a.hbits, id);
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) sid[running + __popc(m & ((1u << lane) - 1u))] = id;
        running += __popc(m);
      }
      hcount += running;
      n_dist += running;
      if (running > 0) score_and_merge<KPL, CPL, DQT>(a, pool, sid, skey, running, qv, lane);
    }

    // S8: emit the first n_out entries (k, or the whole pool in insert mode)
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
    __syncwarp();
  }
}

}  // namespace

template <int KPL, int CPL, int DQT>
static cudaError_t launch_kpl_cpl(SearchArgs a, int num_sms, cudaStream_t st) {
  auto kern = search_kernel<KPL, CPL, DQT>;
  const size_t smem = a.smem_per_warp * kSearchWarpsPerBlock;
  // per-instantiation cache of the (smem size -> resident blocks) query: keeps the launch path host-light
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_per_sm = 0;
  static thread_local int cached_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  cudaError_t e = cudaSuccess;
  if (cached_smem == smem && cached_dev == dev) {
    per_sm = cached_per_sm;
  } else {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSearchWarpsPerBlock * 32, smem);
    if (e != cudaSuccess) return e;
    cached_smem = smem;
    cached_per_sm = per_sm;
    cached_dev = dev;
  }
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long long blocks = (long long)per_sm * num_sms;
  const long long need = (a.nq + kSearchWarpsPerBlock - 1) / kSearchWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kSearchWarpsPerBlock * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <int KPL, int DQT>
static cudaError_t launch_kpl(SearchArgs a, int cpl, int num_sms, cudaStream_t st) {
  switch (cpl) {
    case 1: return launch_kpl_cpl<KPL, 1, DQT>(a, num_sms, st);
    case 2: return launch_kpl_cpl<KPL, 2, DQT>(a, num_sms, st);
    case 4: return launch_kpl_cpl<KPL, 4, DQT>(a, num_sms, st);
    case 8: return launch_kpl_cpl<KPL, 8, DQT>(a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

template <int DQT>
cudaError_t launch_search_dq(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st) {
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
