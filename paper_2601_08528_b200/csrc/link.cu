// K-L1 (detour select) and K-L2 (reverse edges): steps (ii) and (iii) of batched insertion (
// paper §5.1).  The paper runs both on the CPU with atomics + thread-local buffers;
// here both are GPU kernels and the reverse step is sort-then-apply, which makes it deterministic and equal to
// the order-independent definition "tail(u) <- first (R-P) of sort_eff(tail(u) U requests(u))" (reading I12).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

constexpr int kLinkWarps = 4;

// K-L1: snapshot rows of the candidate list in flight per warp (each lane holds two ids of each); 16 rows measured
// equal (10K inserts: detour 0.424 vs 0.436 ms), 32 slower (0.556 ms)
#ifndef SVF_DETOUR_JU
#define SVF_DETOUR_JU 8
#endif

__device__ __forceinline__ int map_find(const uint32_t* mid, const uint16_t* mpos, int mbits, uint32_t id) {
  const uint32_t mask = (1u << mbits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - mbits);
  for (;;) {
    const uint32_t v = mid[h];
    if (v == id) return mpos[h];
    if (v == kSent) return -1;
    h = (h + 1) & mask;
  }
}

// One warp per new vertex v = first + b.  Candidate list C = cand_ids[b][0..m) (distance order, SENT-padded).
// count(i) = |{ j < i : C[i] in row(C[j]) }| ("detourable paths"); stable sort by (count, i) (I11);
// select the first min(R, m): prefix [0,P) in detour order, tail [P,R) sorted by key(d, id) (I12).
// Rows are read from `graph` (the snapshot) and written to out_ids/out_d row b (disjoint from every row read).
//
// No sorting network (DESIGN.md §6 K-L1): the rank of i in (count, i) order is the number of entries with a smaller
// count (exclusive prefix of a count histogram) plus the entries with the same count and a smaller i (match_any
// peers in 32-wide chunks, in i order); and because C is in key order, the tail -- the selected entries past the
// prefix, sorted by key -- is simply those entries in i order (a ballot prefix).  A C that is not in key order (an
// svf_link_candidates caller's) falls back to a warp sort of the tail.
template <int E>
__global__ void __launch_bounds__(kLinkWarps * 32)
    detour_select_kernel(const uint32_t* __restrict__ graph, uint32_t* __restrict__ out_ids,
                         float* __restrict__ out_d, int R, int P, int64_t n_new,
                         const uint32_t* __restrict__ cand_ids, const float* __restrict__ cand_d, int nc, int mbits) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NC = 32 * E;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int M = 1 << mbits;
  const size_t per_warp = (size_t)NC * 4 * 4 + (size_t)M * 6 + 64;
  unsigned char* base = smem + ((per_warp + 15) & ~(size_t)15) * wib;
  uint32_t* sC = reinterpret_cast<uint32_t*>(base);
  uint32_t* cnt = sC + NC;
  uint32_t* hist = cnt + NC;   // count histogram -> exclusive prefix
  uint32_t* run = hist + NC;   // entries of each count already ranked
  uint32_t* mid = run + NC;
  uint16_t* mpos = reinterpret_cast<uint16_t*>(mid + M);
  const int64_t b = (int64_t)blockIdx.x * kLinkWarps + wib;
  if (b >= n_new) return;
  const uint32_t* C = cand_ids + b * nc;
  const float* Cd = cand_d + b * nc;
  const unsigned lt = (1u << lane) - 1u;

  for (int i = lane; i < M; i += 32) mid[i] = kSent;
  int m = nc;
  for (int i0 = 0; i0 < nc; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t c = i < nc ? C[i] : kSent;
    const unsigned s = __ballot_sync(0xffffffffu, i < nc && c == kSent);
    if (s) {
      m = i0 + __ffs(s) - 1;
      break;
    }
  }
  __syncwarp();
  // stage C (id -> position map) and check it is in key order
  bool sorted = true;
  for (int i = lane; i < NC; i += 32) {
    cnt[i] = 0;
    hist[i] = 0;
    run[i] = 0;
    if (i < m) {
      const uint32_t c = C[i];
      sC[i] = c;
      uint32_t h = (c * 0x9E3779B1u) >> (32 - mbits);
      while (atomicCAS(mid + h, kSent, c) != kSent) h = (h + 1) & (uint32_t)(M - 1);
      mpos[h] = (uint16_t)i;
      if (i > 0) {
        const float d0 = Cd[i - 1], d1 = Cd[i];
        sorted = sorted && (d0 < d1 || (d0 == d1 && C[i - 1] < c));
      }
    }
  }
  sorted = __all_sync(0xffffffffu, sorted);
  __syncwarp();
  // detour counts over the snapshot rows of C[0..m-2] (row m-1 can only precede nothing): JU rows in flight
  constexpr int JU = SVF_DETOUR_JU;
  const int nrow = m - 1;
  for (int j0 = 0; j0 < nrow; j0 += JU) {
    uint32_t u[JU][2];
#pragma unroll
    for (int t = 0; t < JU; ++t) {
      const int j = j0 + t;
      const uint32_t* row = graph + (size_t)(j < nrow ? sC[j] : 0) * R;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = h * 32 + lane;
        u[t][h] = (j < nrow && s < R) ? __ldg(row + s) : kSent;
      }
    }
#pragma unroll
    for (int t = 0; t < JU; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t x = u[t][h];
        if (x == kSent) continue;
        const int i = map_find(mid, mpos, mbits, x);
        if (i > j0 + t) atomicAdd(cnt + i, 1u);
      }
    // rows longer than 64 slots (R <= 128): the rest of each row
    for (int s0 = 64; s0 < R; s0 += 32)
      for (int t = 0; t < JU && j0 + t < nrow; ++t) {
        const int s = s0 + lane;
        const uint32_t x = s < R ? __ldg(graph + (size_t)sC[j0 + t] * R + s) : kSent;
        if (x == kSent) continue;
        const int i = map_find(mid, mpos, mbits, x);
        if (i > j0 + t) atomicAdd(cnt + i, 1u);
      }
  }
  __syncwarp();
  // rank in (count, i) order
  for (int i = lane; i < m; i += 32) atomicAdd(hist + cnt[i], 1u);
  __syncwarp();
  {
    uint32_t carry = 0;
    for (int c0 = 0; c0 < NC; c0 += 32) {  // exclusive prefix of the histogram
      const uint32_t hv = hist[c0 + lane];
      uint32_t x = hv;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      hist[c0 + lane] = carry + x - hv;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncwarp();
  uint32_t rank[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = r * 32 + lane;
    const uint32_t ci = i < m ? cnt[i] : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, ci);
    rank[r] = 0xFFFFFFFFu;
    if (i < m) rank[r] = hist[ci] + run[ci] + __popc(peers & lt);
    __syncwarp();
    if (i < m && (peers & lt) == 0u) run[ci] += __popc(peers);  // the group's lowest lane
    __syncwarp();
  }
  const int sel = min(R, m);
  const int npre = min(P, sel);
  uint32_t* row = out_ids + (size_t)b * R;
  float* rowd = out_d + (size_t)b * R;
  for (int s = lane; s < R; s += 32) {
    row[s] = kSent;
    rowd[s] = __int_as_float(0x7F800000);
  }
  __syncwarp();
  // prefix: detour order
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = r * 32 + lane;
    if (i < m && rank[r] < (uint32_t)npre) {
      row[rank[r]] = sC[i];
      rowd[rank[r]] = Cd[i];
    }
  }
  if (sorted) {
    // tail: the selected entries past the prefix, in i (= key) order
    int running = 0;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = r * 32 + lane;
      const bool tail = i < m && rank[r] >= (uint32_t)npre && rank[r] < (uint32_t)sel;
      const unsigned tm = __ballot_sync(0xffffffffu, tail);
      if (tail) {
        const int pos = P + running + __popc(tm & lt);
        row[pos] = sC[i];
        rowd[pos] = Cd[i];
      }
      running += __popc(tm);
    }
  } else {
    uint64_t tk[4];  // R - P <= 128
#pragma unroll
    for (int r = 0; r < 4; ++r) tk[r] = kEmptyKey;
    int running = 0;
    uint64_t* tkeys = reinterpret_cast<uint64_t*>(hist);  // hist + run: 2 * NC u32 = NC keys >= R - P
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = r * 32 + lane;
      const bool tail = i < m && rank[r] >= (uint32_t)npre && rank[r] < (uint32_t)sel;
      const unsigned tm = __ballot_sync(0xffffffffu, tail);
      if (tail) tkeys[running + __popc(tm & lt)] = make_key(Cd[i], sC[i]);
      running += __popc(tm);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = r * 32 + lane;
      tk[r] = e < running ? tkeys[e] : kEmptyKey;
    }
    warp_sort<4>(tk, lane);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = r * 32 + lane;
      if (e < running) {
        row[P + e] = key_id(tk[r]);
        rowd[P + e] = key_dist(tk[r]);
      }
    }
  }
}

// Reverse requests (u, key(d, v)) for every forward edge v -> u of the sub-batch.
// (empty slots get the key `none`, the largest value the sort's bit range holds; all targets are < first < none)
__global__ void reverse_emit_kernel(const uint32_t* __restrict__ graph, const float* __restrict__ edge_dist, int R,
                                    int64_t first, int64_t n_new, uint32_t none, uint32_t* __restrict__ ku,
                                    uint64_t* __restrict__ kv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_new * R) return;
  const int64_t b = t / R;
  const uint32_t v = (uint32_t)(first + b);
  const uint32_t u = graph[(size_t)v * R + (t - b * R)];
  ku[t] = u == kSent ? none : u;
  kv[t] = u == kSent ? kEmptyKey : make_key(edge_dist[(size_t)v * R + (t - b * R)], v);
}

__global__ void segment_heads_kernel(const uint32_t* __restrict__ ku, int64_t n, uint32_t none,
                                     uint32_t* __restrict__ heads, unsigned int* __restrict__ nseg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t u = ku[i];
  if (u != none && (i == 0 || ku[i - 1] != u)) heads[atomicAdd(nseg, 1u)] = (uint32_t)i;
}

// One warp per target u: tail(u) <- first (R-P) of sort_eff(tail(u) U requests(u)); prefix untouched; rows of
// deleted u are frozen.  Tombstoned / empty tail entries count as +inf but keep their stored distance.
// ET = registers per lane for the tail (R-P <= 32*ET); requests arrive in 32-wide chunks (typically 1-3 per target).
// a target with at most this many reverse requests inserts them one by one instead of sorting and merging them
constexpr int kFewRequests = 6;

template <int ET>
__global__ void __launch_bounds__(kLinkWarps * 32)
    reverse_apply_kernel(uint32_t* __restrict__ graph, float* __restrict__ edge_dist,
                         const uint32_t* __restrict__ tomb, int R, int P, const uint32_t* __restrict__ ku,
                         const uint64_t* __restrict__ kv, int64_t n, const uint32_t* __restrict__ heads,
                         const unsigned int* __restrict__ nseg) {
  __shared__ uint32_t old_id[kLinkWarps][32 * ET];
  __shared__ float old_d[kLinkWarps][32 * ET];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned int S = *nseg;
  const int TS = R - P;
  for (unsigned int w = blockIdx.x * kLinkWarps + wib; w < S; w += gridDim.x * kLinkWarps) {
    const int64_t start = heads[w];
    const uint32_t u = ku[start];
    if (tomb_dead(tomb, u)) continue;
    int64_t end = start;
    for (;;) {
      const int64_t i = end + lane;
      const unsigned same = __ballot_sync(0xffffffffu, i < n && ku[i] == u);
      if (same == 0xffffffffu) {
        end += 32;
        continue;
      }
      end += __ffs(~same) - 1;
      break;
    }
    uint64_t best[ET];
    bool sorted = true;
#pragma unroll
    for (int r = 0; r < ET; ++r) {
      const int e = r * 32 + lane;
      best[r] = kEmptyKey;
      if (e < TS) {
        const uint32_t id = graph[(size_t)u * R + P + e];
        const float d = edge_dist[(size_t)u * R + P + e];
        old_id[wib][e] = id;
        old_d[wib][e] = d;
        if (id != kSent) best[r] = make_key(tomb_dead(tomb, id) ? __int_as_float(0x7F800000) : d, id);
      }
    }
    // the tail is kept sorted; it only goes out of order when an entry was tombstoned since (then re-sort)
#pragma unroll
    for (int r = 0; r < ET; ++r) {
      uint64_t nx = __shfl_down_sync(0xffffffffu, best[r], 1);
      const uint64_t head_next = __shfl_sync(0xffffffffu, best[r + 1 < ET ? r + 1 : r], 0);
      if (lane == 31) nx = r + 1 < ET ? head_next : kEmptyKey;
      sorted = sorted && best[r] <= nx;
    }
    if (!__all_sync(0xffffffffu, sorted)) warp_sort<ET>(best, lane);
    __syncwarp();
    if (end - start <= kFewRequests) {
      // few requests (the common case): insert each by its rank in the sorted tail (one ballot per register) and
      // a one-slot shift, dropping the last -- the same first TS of tail U requests as the sort + merge below
      for (int64_t i = start; i < end; ++i) {
        const uint64_t c = kv[i];
        int pos = 0;
#pragma unroll
        for (int r = 0; r < ET; ++r) pos += __popc(__ballot_sync(0xffffffffu, best[r] < c));
        if (pos >= TS) continue;
#pragma unroll
        for (int r = ET - 1; r >= 0; --r) {
          const uint64_t carry = __shfl_sync(0xffffffffu, best[r > 0 ? r - 1 : 0], 31);
          uint64_t up = __shfl_up_sync(0xffffffffu, best[r], 1);
          if (lane == 0) up = carry;
          const int g = r * 32 + lane;
          best[r] = g >= TS ? kEmptyKey : (g > pos ? up : (g == pos ? c : best[r]));  // the last drops out
        }
      }
    } else {
      for (int64_t c0 = start; c0 < end; c0 += 32) {
        uint64_t cand[1];
        cand[0] = c0 + lane < end ? kv[c0 + lane] : kEmptyKey;
        warp_sort<1>(cand, lane);
        warp_merge_into<ET, 1>(best, cand, lane);
      }
    }
#pragma unroll
    for (int r = 0; r < ET; ++r) {
      const int e = r * 32 + lane;
      if (e < TS) {
        const uint32_t id = key_id(best[r]);
        float d = key_dist(best[r]);
        if (id != kSent && __float_as_uint(d) == 0x7F800000u) {  // a tombstoned old entry: keep its distance
          for (int s2 = 0; s2 < TS; ++s2)
            if (old_id[wib][s2] == id) d = old_d[wib][s2];
        }
        graph[(size_t)u * R + P + e] = id;
        edge_dist[(size_t)u * R + P + e] = d;
      }
    }
    __syncwarp();
  }
}

template <int E>
cudaError_t launch_detour_e(const uint32_t* graph, uint32_t* out_ids, float* out_d, int R, int P, int64_t n_new,
                            const uint32_t* cand_ids, const float* cand_d, int nc, cudaStream_t st) {
  int mbits = 1;
  while ((1 << mbits) < 4 * nc) ++mbits;  // id -> position map at load <= 1/4 (misses end at the first probe)
  const int M = 1 << mbits;
  const size_t per_warp = (((size_t)32 * E * 16 + (size_t)M * 6 + 64) + 15) & ~(size_t)15;
  const size_t smem = per_warp * kLinkWarps;
  auto kern = detour_select_kernel<E>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)((n_new + kLinkWarps - 1) / kLinkWarps);
  kern<<<blocks, kLinkWarps * 32, smem, st>>>(graph, out_ids, out_d, R, P, n_new, cand_ids, cand_d, nc, mbits);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_detour_rows(const uint32_t* graph, uint32_t* out_ids, float* out_d, int R, int P, int64_t n,
                               const uint32_t* cand_ids, const float* cand_d, int nc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (nc <= 32) return launch_detour_e<1>(graph, out_ids, out_d, R, P, n, cand_ids, cand_d, nc, st);
  if (nc <= 64) return launch_detour_e<2>(graph, out_ids, out_d, R, P, n, cand_ids, cand_d, nc, st);
  if (nc <= 128) return launch_detour_e<4>(graph, out_ids, out_d, R, P, n, cand_ids, cand_d, nc, st);
  if (nc <= 256) return launch_detour_e<8>(graph, out_ids, out_d, R, P, n, cand_ids, cand_d, nc, st);
  if (nc <= 512) return launch_detour_e<16>(graph, out_ids, out_d, R, P, n, cand_ids, cand_d, nc, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_detour_select(uint32_t* graph, float* edge_dist, int R, int P, int64_t first, int64_t n_new,
                                 const uint32_t* cand_ids, const float* cand_d, int nc, cudaStream_t st) {
  // new rows [first, first+n_new) are written; the candidates' rows (all < first) are read: disjoint
  return launch_detour_rows(graph, graph + (size_t)first * R, edge_dist + (size_t)first * R, R, P, n_new, cand_ids,
                            cand_d, nc, st);
}

static size_t cub_temp_bytes(int64_t m) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)m, 0, 32);
  return t;
}

size_t reverse_scratch_bytes(int64_t n_new, int R) {
  const int64_t m = n_new * R;
  return (size_t)m * (4 + 4 + 8 + 8 + 4) + 256 + cub_temp_bytes(m) + 1024;
}

cudaError_t launch_reverse(uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R, int P, int64_t first,
                           int64_t n_new, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (n_new <= 0 || P >= R) return cudaSuccess;
  const int64_t m = n_new * R;
  auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
  unsigned char* p = static_cast<unsigned char*>(scratch);
  uint64_t* kv = reinterpret_cast<uint64_t*>(p);
  p += align(m * 8);
  uint64_t* kv2 = reinterpret_cast<uint64_t*>(p);
  p += align(m * 8);
  uint32_t* ku = reinterpret_cast<uint32_t*>(p);
  p += align(m * 4);
  uint32_t* ku2 = reinterpret_cast<uint32_t*>(p);
  p += align(m * 4);
  uint32_t* heads = reinterpret_cast<uint32_t*>(p);
  p += align(m * 4);
  unsigned int* nseg = reinterpret_cast<unsigned int*>(p);
  p += 256;
  size_t temp = cub_temp_bytes(m);
  if ((size_t)(p - static_cast<unsigned char*>(scratch)) + temp > scratch_bytes) return cudaErrorInvalidValue;
  const unsigned blocks = (unsigned)((m + 255) / 256);
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) <= first) ++bits;  // 2^bits > first: every target id fits
  const uint32_t none = bits >= 32 ? 0xFFFFFFFFu : (uint32_t)(((uint64_t)1 << bits) - 1);
  reverse_emit_kernel<<<blocks, 256, 0, st>>>(graph, edge_dist, R, first, n_new, none, ku, kv);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(p, temp, ku, ku2, kv, kv2, (int)m, 0, bits, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(nseg, 0, 4, st);
  if (e != cudaSuccess) return e;
  segment_heads_kernel<<<blocks, 256, 0, st>>>(ku2, m, none, heads, nseg);
  const unsigned ablocks = (unsigned)std::min<int64_t>((m + kLinkWarps - 1) / kLinkWarps, 148 * 16);
  const int TS = R - P;
  if (TS <= 32)
    reverse_apply_kernel<1><<<ablocks, kLinkWarps * 32, 0, st>>>(graph, edge_dist, tomb, R, P, ku2, kv2, m, heads, nseg);
  else if (TS <= 64)
    reverse_apply_kernel<2><<<ablocks, kLinkWarps * 32, 0, st>>>(graph, edge_dist, tomb, R, P, ku2, kv2, m, heads, nseg);
  else
    reverse_apply_kernel<4><<<ablocks, kLinkWarps * 32, 0, st>>>(graph, edge_dist, tomb, R, P, ku2, kv2, m, heads, nseg);
  return cudaGetLastError();
}

// ---- K-D: tombstones (lazy deletion) ------------------------------------------------------------------
__global__ void tomb_check_kernel(const uint32_t* __restrict__ ids, int64_t n, uint64_t n_alloc, unsigned int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && (uint64_t)ids[i] >= n_alloc) *bad = 1u;
}
__global__ void tomb_set_kernel(const uint32_t* __restrict__ ids, int64_t n, uint32_t* tomb,
                                unsigned long long* newly) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool fresh = false;
  if (i < n) {
    const uint32_t id = ids[i];
    const uint32_t bit = 1u << (id & 31);
    fresh = (atomicOr(tomb + (id >> 5), bit) & bit) == 0u;
  }
  const unsigned m = __ballot_sync(0xffffffffu, fresh);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(newly, (unsigned long long)__popc(m));
}

cudaError_t launch_tomb_check(const uint32_t* ids, int64_t n, uint64_t n_alloc, unsigned int* bad, cudaStream_t st) {
  tomb_check_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ids, n, n_alloc, bad);
  return cudaGetLastError();
}
cudaError_t launch_tomb_set(const uint32_t* ids, int64_t n, uint32_t* tomb, unsigned long long* newly,
                            cudaStream_t st) {
  tomb_set_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ids, n, tomb, newly);
  return cudaGetLastError();
}

// ---- row helpers ---------------------------------------------------------------------------------------------------
__global__ void pad_rows_kernel(const float* __restrict__ src, int64_t n, int dim, float* __restrict__ dst, int dp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * dp) return;
  const int64_t r = t / dp;
  const int c = (int)(t - r * dp);
  dst[t] = c < dim ? src[r * dim + c] : 0.f;
}
__global__ void unpad_rows_kernel(const float* __restrict__ src, int64_t n, int dp, float* __restrict__ dst, int dim) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * dim) return;
  const int64_t r = t / dim;
  dst[t] = src[r * dp + (t - r * dim)];
}
__global__ void fill_rows_kernel(uint32_t* graph, float* edge_dist, int64_t first, int64_t n, int R) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * R) return;
  graph[first * R + t] = kSent;
  edge_dist[first * R + t] = __int_as_float(0x7F800000);
}

cudaError_t launch_pad_rows(const float* src, int64_t n, int dim, float* dst, int dq, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t t = n * dq * 4;
  pad_rows_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(src, n, dim, dst, dq * 4);
  return cudaGetLastError();
}
cudaError_t launch_unpad_rows(const float* src, int64_t n, int dq, float* dst, int dim, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t t = n * dim;
  unpad_rows_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(src, n, dq * 4, dst, dim);
  return cudaGetLastError();
}
cudaError_t launch_fill_rows(uint32_t* graph, float* edge_dist, int64_t first, int64_t n, int R, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fill_rows_kernel<<<(unsigned)((n * R + 255) / 256), 256, 0, st>>>(graph, edge_dist, first, n, R);
  return cudaGetLastError();
}

__global__ void store_u64_kernel(unsigned long long* p, unsigned long long v) {
  __threadfence();  // the stream's earlier writes (rows, edges) are visible before the published count
  *reinterpret_cast<volatile unsigned long long*>(p) = v;
}

cudaError_t launch_store_u64(unsigned long long* p, uint64_t v, cudaStream_t st) {
  store_u64_kernel<<<1, 1, 0, st>>>(p, (unsigned long long)v);
  return cudaGetLastError();
}

}  // namespace svf
