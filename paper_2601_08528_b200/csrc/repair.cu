// NEXT-1: localized topology-aware repair of severely affected vertices, reading R1'
// in DESIGN.md.  Every kernel reads the rows as they were at the start of the call (rows of deleted vertices are
// frozen, and repaired rows are staged in scratch and scattered only at the end):
//   repair_mark_kernel   warp per row: deleted fraction of the non-sentinel entries, histogram of Fig. 5 buckets,
//                        append v to V^L when the fraction exceeds the threshold (strict);
//   repair_union_kernel  warp per v in V^L: for each deleted p in row(v) in slot order take the first c members of
//                        N_out(p) in slot order that are live, != v, not a live entry of row(v) and not yet taken;
//                        U = (live entries, stored distances) U (candidates, FFMA distances), its `cap` smallest by
//                        (dist, id) -> a candidate list exactly like an insertion's;
//   K-L1 detour select   the insertion's neighbour selection over U into staged rows;
//   repair_scatter       staged rows -> graph / edge_dist.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

constexpr int kRepWarps = 4;

__global__ void repair_mark_kernel(const uint32_t* __restrict__ graph, const uint32_t* __restrict__ tomb, int R,
                                   int64_t n_alloc, double threshold, uint32_t* __restrict__ list,
                                   unsigned int* __restrict__ n_list, unsigned long long* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const int64_t v = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (v >= n_alloc || tomb_dead(tomb, (uint32_t)v)) return;
  int total = 0, ndead = 0;
  for (int s = lane; s < R; s += 32) {
    const uint32_t x = graph[(size_t)v * R + s];
    if (x != kSent) {
      ++total;
      if (tomb_dead(tomb, x)) ++ndead;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    total += __shfl_xor_sync(0xffffffffu, total, off);
    ndead += __shfl_xor_sync(0xffffffffu, ndead, off);
  }
  if (lane == 0) {
    const double frac = total ? (double)ndead / (double)total : 0.0;
    const int bucket = ndead == 0 ? 0 : (frac < 0.1 ? 1 : (frac <= 0.4 ? 2 : (frac <= threshold ? 3 : 4)));
    atomicAdd(hist + bucket, 1ull);
    if (frac > threshold) list[atomicAdd(n_list, 1u)] = (uint32_t)v;
  }
}

__device__ __forceinline__ bool set_has(const uint32_t* tab, int bits, uint32_t id) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - bits);
  for (;;) {
    const uint32_t x = tab[h];
    if (x == id) return true;
    if (x == kSent) return false;
    h = (h + 1) & mask;
  }
}
__device__ __forceinline__ void set_put(uint32_t* tab, int bits, uint32_t id) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - bits);
  while (atomicCAS(tab + h, kSent, id) != kSent && tab[h] != id) h = (h + 1) & mask;
}

// ER = registers per lane for a row (R <= 32*ER); EU = registers for the union's cap (cap <= 32*EU).
// Candidates are gathered in chunks of at most buf_cap (>= 2R) ids: a chunk is scored and merged into the running
// top-cap list whenever another deleted neighbour's row might not fit, so c may be as large as R (consolidation:
// every live member of every deleted neighbour's row) with a chunk buffer of 2R ids.  The union's cap smallest keys
// do not depend on the chunking (keys are distinct).
template <int ER, int EU>
__global__ void __launch_bounds__(kRepWarps * 32)
    repair_union_kernel(const uint32_t* __restrict__ graph, const float* __restrict__ edge_dist,
                        const float* __restrict__ vec, int dq, int metric, const uint32_t* __restrict__ tomb, int R,
                        int c, int cap, const uint32_t* __restrict__ list, int64_t n_list, int set_bits, int buf_cap,
                        uint32_t* __restrict__ u_ids, float* __restrict__ u_d) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t per_warp = (((size_t)4 << set_bits) + (size_t)buf_cap * 4 + (size_t)buf_cap * 8 + 15) & ~(size_t)15;
  unsigned char* base = smem + per_warp * wib;
  uint32_t* tab = reinterpret_cast<uint32_t*>(base);
  uint32_t* cid = tab + (1 << set_bits);
  uint64_t* ckey = reinterpret_cast<uint64_t*>(cid + buf_cap);
  const int wpb = blockDim.x >> 5;
  for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < n_list; w += (int64_t)gridDim.x * wpb) {
    const uint32_t v = list[w];
    for (int i = lane; i < (1 << set_bits); i += 32) tab[i] = kSent;
    __syncwarp();
    uint32_t rid[ER];
    uint64_t best[EU];
#pragma unroll
    for (int r = 0; r < EU; ++r) best[r] = kEmptyKey;
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      const int s = r * 32 + lane;
      rid[r] = s < R ? graph[(size_t)v * R + s] : kSent;
      const bool live = rid[r] != kSent && !tomb_dead(tomb, rid[r]);
      if (r < EU) best[r] = live ? make_key(edge_dist[(size_t)v * R + s], rid[r]) : kEmptyKey;
      if (live) set_put(tab, set_bits, rid[r]);
    }
    __syncwarp();
    warp_sort<EU>(best, lane);
    const float4* xv = reinterpret_cast<const float4*>(vec) + (size_t)v * dq;
    int ncand = 0;
    // score the buffered candidates (a lane per candidate, rows read as float4) and merge them into best
    auto flush = [&]() {
      for (int i = lane; i < ncand; i += 32) {
        const float4* xc = reinterpret_cast<const float4*>(vec) + (size_t)cid[i] * dq;
        float acc = 0.f;
        for (int j = 0; j < dq; ++j) {
          const float4 a = __ldg(xv + j), b = __ldg(xc + j);
          if (metric == 0) {
            const float d0 = b.x - a.x, d1 = b.y - a.y, d2 = b.z - a.z, d3 = b.w - a.w;
            acc = fmaf(d0, d0, acc);
            acc = fmaf(d1, d1, acc);
            acc = fmaf(d2, d2, acc);
            acc = fmaf(d3, d3, acc);
          } else {
            acc = fmaf(b.x, a.x, acc);
            acc = fmaf(b.y, a.y, acc);
            acc = fmaf(b.z, a.z, acc);
            acc = fmaf(b.w, a.w, acc);
          }
        }
        ckey[i] = make_key((metric == 0 ? acc : -acc) + 0.0f, cid[i]);
      }
      __syncwarp();
      for (int c0 = 0; c0 < ncand; c0 += 32) {
        uint64_t cc[1];
        cc[0] = c0 + lane < ncand ? ckey[c0 + lane] : kEmptyKey;
        warp_sort<1>(cc, lane);
        warp_merge_into<EU, 1>(best, cc, lane);
      }
      __syncwarp();
      ncand = 0;
    };
    // candidates: deleted p in slot order, first c qualifying members of N_out(p) in slot order
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      for (int l = 0; l < 32; ++l) {
        const uint32_t p = __shfl_sync(0xffffffffu, rid[r], l);
        if (r * 32 + l >= R || p == kSent || !tomb_dead(tomb, p)) continue;
        if (ncand + min(c, R) > buf_cap) flush();
        int got = 0;
#pragma unroll
        for (int r2 = 0; r2 < ER; ++r2) {
          const int t = r2 * 32 + lane;
          const uint32_t x = t < R ? graph[(size_t)p * R + t] : kSent;
          const bool ok = x != kSent && x != v && !tomb_dead(tomb, x) && !set_has(tab, set_bits, x);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const int rank = got + __popc(m & ((1u << lane) - 1u));
          const bool take = ok && rank < c;
          if (take) {
            cid[ncand + rank] = x;
            set_put(tab, set_bits, x);
          }
          got = min(got + __popc(m), c);
        }
        ncand += got;
        __syncwarp();
      }
    }
    flush();
#pragma unroll
    for (int r = 0; r < EU; ++r) {
      const int s = r * 32 + lane;
      if (s < cap) {
        u_ids[(size_t)w * cap + s] = key_id(best[r]);
        u_d[(size_t)w * cap + s] = key_dist(best[r]);
      }
    }
    __syncwarp();
  }
}

// insert-if-absent: true when id was not in the set (concurrent inserts of one id: exactly one lane wins)
__device__ __forceinline__ bool set_add(uint32_t* tab, int bits, uint32_t id) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = (id * 0x9E3779B1u) >> (32 - bits);
  for (;;) {
    const uint32_t prev = atomicCAS(tab + h, kSent, id);
    if (prev == kSent) return true;
    if (prev == id) return false;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ float row_dist(const float4* __restrict__ xv, const float4* __restrict__ xc, int dq,
                                          int metric) {
  float acc = 0.f;
  for (int j = 0; j < dq; ++j) {
    const float4 a = __ldg(xv + j), b = __ldg(xc + j);
    if (metric == 0) {
      const float d0 = b.x - a.x, d1 = b.y - a.y, d2 = b.z - a.z, d3 = b.w - a.w;
      acc = fmaf(d0, d0, acc);
      acc = fmaf(d1, d1, acc);
      acc = fmaf(d2, d2, acc);
      acc = fmaf(d3, d3, acc);
    } else {
      acc = fmaf(b.x, a.x, acc);
      acc = fmaf(b.y, a.y, acc);
      acc = fmaf(b.z, a.z, acc);
      acc = fmaf(b.w, a.w, acc);
    }
  }
  return (metric == 0 ? acc : -acc) + 0.0f;  // canonical +0
}

// NEXT-4 global consolidation, reading C2 (oracle orc_consolidate), warp per affected live vertex v (a
// row holding a tombstoned id).  Only tombstoned rows N_out(p) are read besides v's own row, and those are frozen,
// so every warp rewrites its row in place:
//   prefix: each tombstoned slot s < P (slot order) <- the nearest (dist, id) live member of N_out(p_s) that is not
//           v, not a live entry of row(v) and not taken by an earlier slot (empty when none);
//   tail:   the live tail entries stay; the m vacancies take the m nearest remaining members of the union of the
//           deleted neighbours' lists (deduplicated), streamed in chunks of <= buf_cap ids into a running top list;
//           the tail is re-sorted by key, empty slots last.
// tab holds row(v)'s live ids, the prefix refills and every union member seen (one set: all three are excluded).
template <int ER, int EU>
__global__ void __launch_bounds__(kRepWarps * 32)
    consolidate_kernel(uint32_t* __restrict__ graph, float* __restrict__ edge_dist, const float* __restrict__ vec,
                       int dq, int metric, const uint32_t* __restrict__ tomb, int R, int P,
                       const uint32_t* __restrict__ list, int64_t n_list, int set_bits, int buf_cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t per_warp = (((size_t)4 << set_bits) + (size_t)buf_cap * 4 + (size_t)buf_cap * 8 + 15) & ~(size_t)15;
  unsigned char* base = smem + per_warp * wib;
  uint32_t* tab = reinterpret_cast<uint32_t*>(base);
  uint32_t* cid = tab + (1 << set_bits);
  uint64_t* ckey = reinterpret_cast<uint64_t*>(cid + buf_cap);
  const int wpb = blockDim.x >> 5;
  const float4* v4 = reinterpret_cast<const float4*>(vec);
  for (int64_t w = (int64_t)blockIdx.x * wpb + wib; w < n_list; w += (int64_t)gridDim.x * wpb) {
    const uint32_t v = list[w];
    for (int i = lane; i < (1 << set_bits); i += 32) tab[i] = kSent;
    __syncwarp();
    uint32_t rid[ER], orig[ER];
    float rd[ER];
    bool dead_slot[ER];
    // slot s of a register-striped row (element s = r*32 + lane), without dynamic register indexing
    auto slot_of = [&](const uint32_t (&a)[ER], int s) {
      uint32_t x = kSent;
#pragma unroll
      for (int r = 0; r < ER; ++r) {
        const uint32_t y = __shfl_sync(0xffffffffu, a[r], s & 31);
        if (r == (s >> 5)) x = y;
      }
      return x;
    };
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      const int s = r * 32 + lane;
      rid[r] = s < R ? graph[(size_t)v * R + s] : kSent;
      orig[r] = rid[r];
      rd[r] = s < R ? edge_dist[(size_t)v * R + s] : 0.f;
      dead_slot[r] = rid[r] != kSent && tomb_dead(tomb, rid[r]);
      if (rid[r] != kSent && !dead_slot[r]) set_add(tab, set_bits, rid[r]);
    }
    __syncwarp();
    const float4* xv = v4 + (size_t)v * dq;
    // prefix slots in slot order
    for (int s = 0; s < P; ++s) {
      const uint32_t p = slot_of(orig, s);
      if (p == kSent || !tomb_dead(tomb, p)) continue;
      uint64_t bk = kEmptyKey;
#pragma unroll
      for (int r2 = 0; r2 < ER; ++r2) {
        const int t = r2 * 32 + lane;
        const uint32_t x = t < R ? graph[(size_t)p * R + t] : kSent;
        if (x != kSent && x != v && !tomb_dead(tomb, x) && !set_has(tab, set_bits, x)) {
          const uint64_t kk = make_key(row_dist(xv, v4 + (size_t)x * dq, dq, metric), x);
          bk = kk < bk ? kk : bk;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, bk, off);
        bk = o < bk ? o : bk;
      }
      __syncwarp();
      if (lane == 0 && bk != kEmptyKey) set_add(tab, set_bits, key_id(bk));
#pragma unroll
      for (int r = 0; r < ER; ++r)
        if (r == (s >> 5) && (s & 31) == lane) {  // the owning lane updates its register copy of the row
          rid[r] = key_id(bk);
          rd[r] = key_dist(bk);
        }
      __syncwarp();
    }
    // tail: m vacancies, refilled from the union of the deleted neighbours' lists
    int m = 0;
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      const int s = r * 32 + lane;
      m += __popc(__ballot_sync(0xffffffffu, s >= P && s < R && (rid[r] == kSent || dead_slot[r])));
    }
    uint64_t best[EU];
#pragma unroll
    for (int r = 0; r < EU; ++r) best[r] = kEmptyKey;
    int ncand = 0;
    auto flush = [&]() {
      for (int i = lane; i < ncand; i += 32) ckey[i] = make_key(row_dist(xv, v4 + (size_t)cid[i] * dq, dq, metric), cid[i]);
      __syncwarp();
      for (int c0 = 0; c0 < ncand; c0 += 32) {
        uint64_t cc[1];
        cc[0] = c0 + lane < ncand ? ckey[c0 + lane] : kEmptyKey;
        warp_sort<1>(cc, lane);
        warp_merge_into<EU, 1>(best, cc, lane);
      }
      __syncwarp();
      ncand = 0;
    };
    if (m > 0) {
      for (int s = 0; s < R; ++s) {
        // the original row's deleted entries (the prefix registers now hold the refills)
        const uint32_t p = slot_of(orig, s);
        if (p == kSent || !tomb_dead(tomb, p)) continue;
        if (ncand + R > buf_cap) flush();
#pragma unroll
        for (int r2 = 0; r2 < ER; ++r2) {
          const int t = r2 * 32 + lane;
          const uint32_t x = t < R ? graph[(size_t)p * R + t] : kSent;
          const bool ok = x != kSent && x != v && !tomb_dead(tomb, x) && set_add(tab, set_bits, x);
          const unsigned mk = __ballot_sync(0xffffffffu, ok);
          if (ok) cid[ncand + __popc(mk & ((1u << lane) - 1u))] = x;
          ncand += __popc(mk);
        }
        __syncwarp();
      }
      flush();
    }
    // new tail = kept live tail entries U the first m of best, sorted by key
    __syncwarp();
    int nk = 0;
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      const int s = r * 32 + lane;
      const bool keep = s >= P && s < R && rid[r] != kSent && !dead_slot[r];
      const unsigned mk = __ballot_sync(0xffffffffu, keep);
      if (keep) ckey[nk + __popc(mk & ((1u << lane) - 1u))] = make_key(rd[r], rid[r]);
      nk += __popc(mk);
    }
#pragma unroll
    for (int r = 0; r < EU; ++r) {
      const int e = r * 32 + lane;
      if (e < m) ckey[nk + e] = best[r];
    }
    __syncwarp();
    uint64_t tl[EU];
#pragma unroll
    for (int r = 0; r < EU; ++r) {
      const int e = r * 32 + lane;
      tl[r] = e < nk + m ? ckey[e] : kEmptyKey;
    }
    warp_sort<EU>(tl, lane);
    // the whole read of the starting row is done: write prefix (registers) and tail
#pragma unroll
    for (int r = 0; r < ER; ++r) {
      const int s = r * 32 + lane;
      if (s < P) {
        graph[(size_t)v * R + s] = rid[r];
        edge_dist[(size_t)v * R + s] = rid[r] == kSent ? __int_as_float(0x7F800000) : rd[r];
      }
    }
#pragma unroll
    for (int r = 0; r < EU; ++r) {
      const int e = r * 32 + lane;
      if (P + e < R) {
        graph[(size_t)v * R + P + e] = key_id(tl[r]);
        edge_dist[(size_t)v * R + P + e] = key_dist(tl[r]);
      }
    }
    __syncwarp();
  }
}

__global__ void repair_scatter_kernel(uint32_t* __restrict__ graph, float* __restrict__ edge_dist,
                                      const uint32_t* __restrict__ list, int64_t n_list, int R,
                                      const uint32_t* __restrict__ rows, const float* __restrict__ rows_d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_list * R) return;
  const int64_t b = t / R;
  const int s = (int)(t - b * R);
  graph[(size_t)list[b] * R + s] = rows[t];
  edge_dist[(size_t)list[b] * R + s] = rows_d[t];
}

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

size_t repair_mark_scratch_bytes(int64_t n_alloc) { return al256((size_t)n_alloc * 4) + 256; }

cudaError_t launch_repair_mark(const uint32_t* graph, const uint32_t* tomb, int R, int64_t n_alloc, double threshold,
                               void* scratch, cudaStream_t st, int64_t* n_list, uint64_t hist_out[5]) {
  uint32_t* list = static_cast<uint32_t*>(scratch);
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) +
                                                                   al256((size_t)n_alloc * 4));
  unsigned int* cnt = reinterpret_cast<unsigned int*>(hist + 5);
  cudaError_t e = cudaMemsetAsync(hist, 0, 64, st);
  if (e != cudaSuccess) return e;
  if (n_alloc > 0)
    repair_mark_kernel<<<(unsigned)((n_alloc + 7) / 8), 256, 0, st>>>(graph, tomb, R, n_alloc, threshold, list, cnt,
                                                                      hist);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  unsigned long long hh[6];
  if ((e = cudaMemcpyAsync(hh, hist, 48, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  for (int i = 0; i < 5; ++i) hist_out[i] = hh[i];
  *n_list = (int64_t)(hh[5] & 0xFFFFFFFFull);
  return cudaSuccess;
}

size_t repair_apply_scratch_bytes(int64_t n_list, int R, int cap) {
  return 2 * al256((size_t)n_list * cap * 4) + 2 * al256((size_t)n_list * R * 4);
}

cudaError_t launch_repair_apply(uint32_t* graph, float* edge_dist, const float* vec, int dq, int metric,
                                const uint32_t* tomb, int R, int P, int c, int cap, const void* mark_scratch,
                                int64_t n_list, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t st) {
  if (n_list <= 0) return cudaSuccess;
  if (scratch_bytes < repair_apply_scratch_bytes(n_list, R, cap) || cap > 512) return cudaErrorInvalidValue;
  const uint32_t* list = static_cast<const uint32_t*>(mark_scratch);
  char* sp = static_cast<char*>(scratch);
  uint32_t* u_ids = reinterpret_cast<uint32_t*>(sp);
  sp += al256((size_t)n_list * cap * 4);
  float* u_d = reinterpret_cast<float*>(sp);
  sp += al256((size_t)n_list * cap * 4);
  uint32_t* rows = reinterpret_cast<uint32_t*>(sp);
  sp += al256((size_t)n_list * R * 4);
  float* rows_d = reinterpret_cast<float*>(sp);
  // visited set for the row and every candidate (load <= 1/2; <= 2^13 slots: load <= 0.51 at c = R = 64)
  const int cand_total = std::min(c, R) * R;
  int set_bits = 1;
  while ((1 << set_bits) < 2 * (R + cand_total) && set_bits < 13) ++set_bits;
  while ((1 << set_bits) < (R + cand_total) * 5 / 4) ++set_bits;  // large sets: load <= 0.8
  const int buf_cap = 2 * R;                           // chunk buffer: room for one more deleted neighbour's row
  const size_t per_warp = (((size_t)4 << set_bits) + (size_t)buf_cap * 12 + 15) & ~(size_t)15;
  const int wpb = (int)std::max<size_t>(1, std::min<size_t>(kRepWarps, (200u << 10) / per_warp));
  const size_t smem = per_warp * wpb;
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    kern<<<(unsigned)(num_sms * 8), wpb * 32, smem, st>>>(graph, edge_dist, vec, dq, metric, tomb, R, c, cap,
                                                                list, n_list, set_bits, buf_cap, u_ids, u_d);
    return cudaGetLastError();
  };
  cudaError_t e;
  const bool big = cap > 128;
  if (R <= 32) e = big ? run(repair_union_kernel<1, 16>) : run(repair_union_kernel<1, 4>);
  else if (R <= 64) e = big ? run(repair_union_kernel<2, 16>) : run(repair_union_kernel<2, 4>);
  else e = big ? run(repair_union_kernel<4, 16>) : run(repair_union_kernel<4, 4>);
  if (e != cudaSuccess) return e;
  // the insertion's selection over U, counted on the (unmodified) starting rows, into staged rows
  if ((e = launch_detour_rows(graph, rows, rows_d, R, P, n_list, u_ids, u_d, cap, st)) != cudaSuccess) return e;
  repair_scatter_kernel<<<(unsigned)((n_list * R + 255) / 256), 256, 0, st>>>(graph, edge_dist, list, n_list, R, rows,
                                                                             rows_d);
  return cudaGetLastError();
}

cudaError_t launch_consolidate(uint32_t* graph, float* edge_dist, const float* vec, int dq, int metric,
                               const uint32_t* tomb, int R, int P, const void* mark_scratch, int64_t n_list, int num_sms,
                               cudaStream_t st) {
  if (n_list <= 0) return cudaSuccess;
  const uint32_t* list = static_cast<const uint32_t*>(mark_scratch);
  // one set for the row, the prefix refills and the union (<= R + R*R ids): load <= 1/2 up to 2^13 slots, else 0.8
  const int total = R + R * R;
  int set_bits = 1;
  while ((1 << set_bits) < 2 * total && set_bits < 13) ++set_bits;
  while ((1 << set_bits) < total * 5 / 4) ++set_bits;
  const int buf_cap = 2 * R;
  const size_t per_warp = (((size_t)4 << set_bits) + (size_t)buf_cap * 12 + 15) & ~(size_t)15;
  const int wpb = (int)std::max<size_t>(1, std::min<size_t>(kRepWarps, (200u << 10) / per_warp));
  const size_t smem = per_warp * wpb;
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    kern<<<(unsigned)(num_sms * 8), wpb * 32, smem, st>>>(graph, edge_dist, vec, dq, metric, tomb, R, P, list,
                                                                n_list, set_bits, buf_cap);
    return cudaGetLastError();
  };
  const int T = R - P;  // tail slots
  const int ER = R <= 32 ? 1 : R <= 64 ? 2 : 4;
  const int EU = T <= 32 ? 1 : T <= 64 ? 2 : 4;
  if (ER == 1) return run(consolidate_kernel<1, 1>);
  if (ER == 2) return EU == 1 ? run(consolidate_kernel<2, 1>) : run(consolidate_kernel<2, 2>);
  return EU == 1 ? run(consolidate_kernel<4, 1>) : EU == 2 ? run(consolidate_kernel<4, 2>) : run(consolidate_kernel<4, 4>);
}

}  // namespace svf
