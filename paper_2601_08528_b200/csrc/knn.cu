// K-G: exact k-NN ("ground truth computed via exhaustive linear scan"), and K-M: the
// top-k merge used after the multi-GPU all-gather.
//
// knn_tile_kernel: a block owns 64 queries x one split of the base rows; it streams 64-row tiles through shared
// memory in 32-float D chunks (register-tiled FFMA, 4x4 per thread, direct-difference L2 so values match the
// search kernel's arithmetic class), then each warp filters its 8 queries' tile rows against the running k-th
// key and merges survivors into a per-query sorted list (bitonic, warp shuffles).  Per-split lists are merged by
// merge_keys_kernel.  The tensor-core (tcgen05, TF32) scoring variant with exact re-rank is DESIGN.md's next step.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

constexpr int QB = 64, NB = 64, DK = 32;

template <int KPL>
__global__ void __launch_bounds__(256)
    knn_tile_kernel(const float* __restrict__ vec, int dp, int64_t n, const uint32_t* __restrict__ tomb,
                    const float* __restrict__ Q, int64_t q_stride, int q_dim, int64_t nq, int k, int metric,
                    int64_t self_base, int64_t rows_per_split, uint64_t* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t (*lists)[32 * KPL] = reinterpret_cast<uint64_t (*)[32 * KPL]>(smem);
  uint64_t* thr = reinterpret_cast<uint64_t*>(smem + (size_t)QB * 32 * KPL * 8);
  float (*qs)[QB + 1] = reinterpret_cast<float (*)[QB + 1]>(thr + QB);
  float (*xs)[NB + 1] = reinterpret_cast<float (*)[NB + 1]>(&qs[DK][0]);
  float (*dt)[NB + 1] = reinterpret_cast<float (*)[NB + 1]>(&xs[DK][0]);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t q0 = (int64_t)blockIdx.x * QB;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = std::min<int64_t>(n, r0 + rows_per_split);
  for (int i = tid; i < QB * 32 * KPL; i += 256) (&lists[0][0])[i] = kEmptyKey;
  for (int i = tid; i < QB; i += 256) thr[i] = kEmptyKey;
  __syncthreads();

  for (int64_t nb = r0; nb < r1; nb += NB) {
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int d0 = 0; d0 < dp; d0 += DK) {
      __syncthreads();
      for (int t = tid; t < QB * DK; t += 256) {
        const int qq = t / DK, dd = t % DK;
        const int64_t qi = q0 + qq;
        const int dglob = d0 + dd;
        qs[dd][qq] = (qi < nq && dglob < q_dim) ? __ldg(Q + qi * q_stride + dglob) : 0.f;
        const int64_t ri = nb + qq;
        xs[dd][qq] = (ri < r1 && dglob < dp) ? __ldg(vec + ri * dp + dglob) : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int dd = 0; dd < DK; ++dd) {
        float qv[4], xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = qs[dd][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) xv[j] = xs[dd][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (metric == 0) {
              const float df = xv[j] - qv[i];
              acc[i][j] = fmaf(df, df, acc[i][j]);
            } else {
              acc[i][j] = fmaf(xv[j], qv[i], acc[i][j]);
            }
          }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dt[ty + 16 * i][tx + 16 * j] = (metric == 0 ? acc[i][j] : -acc[i][j]) + 0.0f;
    __syncthreads();
    // epilogue: warp w filters queries w*8 .. w*8+7 against their running k-th key
    for (int qq = warp * 8; qq < warp * 8 + 8; ++qq) {
      const int64_t qi = q0 + qq;
      if (qi >= nq) break;
      uint64_t c[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        const int64_t ri = nb + col;
        bool ok = ri < r1 && !(self_base >= 0 && ri == self_base + qi);
        if (ok) ok = !tomb_dead(tomb, (uint32_t)ri);
        c[h] = ok ? make_key(dt[qq][col], (uint32_t)ri) : kEmptyKey;
      }
      const uint64_t t = thr[qq];
      if (__ballot_sync(0xffffffffu, c[0] < t || c[1] < t) == 0u) continue;
      uint64_t lst[KPL];
#pragma unroll
      for (int r = 0; r < KPL; ++r) lst[r] = lists[qq][r * 32 + lane];
      warp_sort<2>(c, lane);
      warp_merge_into<KPL, 2>(lst, c, lane);
#pragma unroll
      for (int r = 0; r < KPL; ++r) {
        if (r * 32 + lane >= k) lst[r] = kEmptyKey;
        lists[qq][r * 32 + lane] = lst[r];
      }
      uint64_t kreg = kEmptyKey;
#pragma unroll
      for (int r = 0; r < KPL; ++r)
        if (r == ((k - 1) >> 5)) kreg = lst[r];
      const uint64_t kth = __shfl_sync(0xffffffffu, kreg, (k - 1) & 31);
      __syncwarp();
      if (lane == 0) thr[qq] = kth;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int qq = warp; qq < QB; qq += 8) {
    const int64_t qi = q0 + qq;
    if (qi >= nq) continue;
    uint64_t* dst = part + ((size_t)blockIdx.y * nq + qi) * (32 * KPL);
#pragma unroll
    for (int r = 0; r < KPL; ++r) dst[r * 32 + lane] = lists[qq][r * 32 + lane];
  }
}

// lists [S][nq][32*KPL] of sorted keys -> first k per query
template <int KPL>
__global__ void merge_keys_kernel(const uint64_t* __restrict__ part, int S, int64_t nq, int k,
                                  uint32_t* __restrict__ out_ids, float* __restrict__ out_d) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  uint64_t best[KPL];
#pragma unroll
  for (int r = 0; r < KPL; ++r) best[r] = kEmptyKey;
  for (int s = 0; s < S; ++s) {
    uint64_t c[KPL];
    const uint64_t* src = part + ((size_t)s * nq + qi) * (32 * KPL);
#pragma unroll
    for (int r = 0; r < KPL; ++r) c[r] = src[r * 32 + lane];
    warp_merge_into<KPL, KPL>(best, c, lane);
  }
#pragma unroll
  for (int r = 0; r < KPL; ++r) {
    const int e = r * 32 + lane;
    if (e < k) {
      out_ids[qi * k + e] = key_id(best[r]);
      out_d[qi * k + e] = key_dist(best[r]);
    }
  }
}

// K-M: lists [G][nq][k] -> first k per query by (dist, id) (inputs need not be sorted).  Input entries are either
// separate (ids, d) arrays or packed pairs (distance bits << 32 | id); list g's ids may be mapped to global ids
// id * id_mul + add.v[g] (a rank's shards); the output is separate arrays or packed pairs.
struct IdAdd {
  uint32_t v[16];
};
template <int KPL, bool IN_PAIRS, bool OUT_PAIRS>
__global__ void merge_topk_kernel(const uint32_t* __restrict__ ids, const float* __restrict__ d,
                                  const unsigned long long* __restrict__ pairs, int G, int64_t nq, int k,
                                  uint32_t id_mul, IdAdd add, uint32_t* __restrict__ out_ids,
                                  float* __restrict__ out_d, unsigned long long* __restrict__ out_pairs) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  uint64_t best[KPL];
#pragma unroll
  for (int r = 0; r < KPL; ++r) best[r] = kEmptyKey;
  for (int g = 0; g < G; ++g) {
    uint64_t c[KPL];
    const size_t o = ((size_t)g * nq + qi) * k;
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
      const int e = r * 32 + lane;
      c[r] = kEmptyKey;
      if (e < k) {
        uint32_t id;
        float dist;
        if (IN_PAIRS) {
          const unsigned long long pr = pairs[o + e];
          id = (uint32_t)pr;
          dist = __uint_as_float((uint32_t)(pr >> 32));
        } else {
          id = ids[o + e];
          dist = d[o + e];
        }
        if (id != kSent) c[r] = make_key(dist + 0.0f, id_mul ? id * id_mul + add.v[g] : id);
      }
    }
    warp_sort<KPL>(c, lane);
    warp_merge_into<KPL, KPL>(best, c, lane);
  }
#pragma unroll
  for (int r = 0; r < KPL; ++r) {
    const int e = r * 32 + lane;
    if (e < k) {
      if (OUT_PAIRS) {
        out_pairs[qi * k + e] =
            ((unsigned long long)__float_as_uint(key_dist(best[r])) << 32) | (unsigned long long)key_id(best[r]);
      } else {
        out_ids[qi * k + e] = key_id(best[r]);
        out_d[qi * k + e] = key_dist(best[r]);
      }
    }
  }
}

int kpl_for(int k) {
  int kpl = 1;
  while (32 * kpl < k) kpl <<= 1;
  return kpl;
}

struct KnnPlan {
  int kpl;
  int64_t splits, rows_per_split, qtiles;
};
KnnPlan knn_plan(int64_t nq, int k, int64_t n, int num_sms) {
  KnnPlan p;
  p.kpl = kpl_for(k);
  p.qtiles = (nq + QB - 1) / QB;
  const int64_t want_blocks = (int64_t)num_sms * 4;
  int64_t s = (want_blocks + p.qtiles - 1) / p.qtiles;
  const int64_t max_s = std::max<int64_t>(1, (n + NB - 1) / NB);
  s = std::max<int64_t>(1, std::min(s, max_s));
  p.rows_per_split = ((n + s - 1) / s + NB - 1) / NB * NB;
  p.splits = std::max<int64_t>(1, (n + p.rows_per_split - 1) / p.rows_per_split);
  return p;
}

}  // namespace

size_t knn_scratch_bytes(int64_t nq, int k, int64_t n) {
  KnnPlan p = knn_plan(nq, k, n, 148);
  // plan depends on the SM count only through the split count; size for a generous SM count
  KnnPlan p2 = knn_plan(nq, k, n, 512);
  const int64_t s = std::max(p.splits, p2.splits);
  return (size_t)s * nq * 32 * p.kpl * 8 + 256;
}

template <int KPL>
static cudaError_t knn_launch(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                              int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                              uint32_t* out_ids, float* out_d, uint64_t* part, const KnnPlan& p, cudaStream_t st) {
  dim3 grid((unsigned)p.qtiles, (unsigned)p.splits);
  const size_t smem = (size_t)QB * 32 * KPL * 8 + QB * 8 + (size_t)DK * (QB + 1) * 4 + (size_t)DK * (NB + 1) * 4 +
                      (size_t)QB * (NB + 1) * 4;
  cudaError_t e0 = cudaFuncSetAttribute(knn_tile_kernel<KPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e0 != cudaSuccess) return e0;
  knn_tile_kernel<KPL><<<grid, 256, smem, st>>>(vec, dq * 4, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base,
                                             p.rows_per_split, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  merge_keys_kernel<KPL><<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(part, (int)p.splits, nq, k, out_ids, out_d);
  return cudaGetLastError();
}

cudaError_t launch_knn_exact(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                             int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                             uint32_t* out_ids, float* out_d, void* scratch, size_t scratch_bytes, int num_sms,
                             cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  KnnPlan p = knn_plan(nq, k, n, num_sms);
  if ((size_t)p.splits * nq * 32 * p.kpl * 8 > scratch_bytes) return cudaErrorInvalidValue;
  uint64_t* part = static_cast<uint64_t*>(scratch);
  switch (p.kpl) {
    case 1: return knn_launch<1>(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, part, p, st);
    case 2: return knn_launch<2>(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, part, p, st);
    case 4: return knn_launch<4>(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, part, p, st);
    case 8: return knn_launch<8>(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, part, p, st);
  }
  return cudaErrorInvalidValue;
}

template <bool IN_PAIRS, bool OUT_PAIRS>
static cudaError_t merge_launch(const uint32_t* ids, const float* d, const unsigned long long* pairs, int G, int64_t nq,
                                int k, uint32_t id_mul, const IdAdd& add, uint32_t* out_ids, float* out_d,
                                unsigned long long* out_pairs, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((nq + 7) / 8);
  switch (kpl_for(k)) {
    case 1: merge_topk_kernel<1, IN_PAIRS, OUT_PAIRS><<<blocks, 256, 0, st>>>(ids, d, pairs, G, nq, k, id_mul, add, out_ids, out_d, out_pairs); break;
    case 2: merge_topk_kernel<2, IN_PAIRS, OUT_PAIRS><<<blocks, 256, 0, st>>>(ids, d, pairs, G, nq, k, id_mul, add, out_ids, out_d, out_pairs); break;
    case 4: merge_topk_kernel<4, IN_PAIRS, OUT_PAIRS><<<blocks, 256, 0, st>>>(ids, d, pairs, G, nq, k, id_mul, add, out_ids, out_d, out_pairs); break;
    case 8: merge_topk_kernel<8, IN_PAIRS, OUT_PAIRS><<<blocks, 256, 0, st>>>(ids, d, pairs, G, nq, k, id_mul, add, out_ids, out_d, out_pairs); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_merge_topk(const uint32_t* ids, const float* d, int G, int64_t nq, int k, uint32_t* out_ids,
                              float* out_d, cudaStream_t st) {
  return merge_launch<false, false>(ids, d, nullptr, G, nq, k, 0, IdAdd{}, out_ids, out_d, nullptr, st);
}

cudaError_t launch_shard_premerge(const uint32_t* ids, const float* d, int n_lists, int64_t nq, int k,
                                  uint32_t n_logical, const uint32_t* shard, unsigned long long* out_pairs,
                                  cudaStream_t st) {
  if (n_lists < 1 || n_lists > 16) return cudaErrorInvalidValue;
  IdAdd add{};
  for (int i = 0; i < n_lists; ++i) add.v[i] = shard[i];
  return merge_launch<false, true>(ids, d, nullptr, n_lists, nq, k, n_logical, add, nullptr, nullptr, out_pairs, st);
}

cudaError_t launch_merge_pairs(const unsigned long long* pairs, int G, int64_t nq, int k, uint32_t* out_ids,
                               float* out_d, cudaStream_t st) {
  return merge_launch<true, false>(nullptr, nullptr, pairs, G, nq, k, 0, IdAdd{}, out_ids, out_d, nullptr, st);
}

}  // namespace svf
