// K-G on the 5th-generation tensor cores: exact k-NN ("ground truth via exhaustive linear scan", P:L695;
// SURVEY §8(a) G1) as a TF32 tcgen05 GEMM with a fused approximate top-k epilogue, followed by K-R, an exact
// fp32 re-rank with a certificate, and an exact FFMA fallback for the (rare) queries the certificate rejects.
//
// knn_tc_kernel (persistent, one CTA per SM, 192 threads):
//   warp 0      TMA producer: the 128-query A tile once per unit (K-major, SWIZZLE_128B, Dp/32 boxes of 128x32),
//               then 256-row x 32-float B boxes of the base vectors through an S-stage mbarrier ring;
//   warp 1      TMEM owner (512 columns = 2 accumulators of 128 lanes x 256 fp32) and single-thread MMA issuer:
//               4 x tcgen05.mma.kind::tf32 (M=128, N=256, K=8) per 32-float chunk; tcgen05.commit frees the stage
//               and, after the last chunk, publishes the accumulator;
//   warps 2..9  epilogue: thread = query row = TMEM lane; tcgen05.ld 32 columns at a time of the approximate
//               score s~ = ||x||^2 - 2 q.x (L2) or -q.x (IP), which the MMA produces directly: A rows are
//               [-2q | 0 | w] and B rows [x | 0 | p] with ||x||^2 = w.p split into pieces exact in TF32, one extra
//               K=8 MMA per tile; the epilogue keeps the KL smallest per (query, split, column half) in registers.
// knn_rerank_kernel (warp per query): merge the per-split lists to the best 64 approximate candidates, recompute
//   their distances exactly (direct-difference FFMA, the search kernel's arithmetic), sort, emit the top k, and
//   check the certificate  d_k < tau - E + ||q||^2  (tau = smallest score any excluded row can have, E = the
//   TF32 error bound; E = 0 when data and query are integers <= 2047 whose sums fit 2^24, as in C1/C2).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace svf {

namespace {

constexpr int TC_M = 128, TC_N = 256, TC_KC = 32, TC_LIST_MAX = 32;
constexpr int kTcEpiWarps = 8;                       // 2 per TMEM lane quarter, 128 columns each
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;
constexpr uint32_t kBStageBytes = TC_N * TC_KC * 4;  // 32 KB
constexpr uint32_t kAChunkBytes = TC_M * TC_KC * 4;  // 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// K-major operand, SWIZZLE_128B canonical layout: 128-byte rows, 8-row (1024 B) swizzle atoms, SBO = 1024 B
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address  [0,14)
  d |= (uint64_t)1 << 16;                    // LBO = 16 B      [16,30)  (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO = 1024 B    [32,46)
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // layout type: SWIZZLE_128B
  return d;
}
// instruction descriptor: D fp32, A/B tf32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                            ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// issue a 32-column TMEM load without waiting (pair with tmem_wait32 on the same registers)
__device__ __forceinline__ void tmem_issue32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// wait for the outstanding TMEM loads; the registers are in-out operands so no consumer is hoisted above it
__device__ __forceinline__ void tmem_wait32(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TcArgs {
  int64_t nq, n;         // queries, base rows (ids [0, n))
  int kc;                // 32-float K chunks (Dp / 32 rounded up)
  int stages;            // B ring depth
  int64_t rows_per_split;
  int64_t splits, units; // units = qtiles * splits
  const uint32_t* tomb;
  int64_t self_base;     // >= 0: exclude id == self_base + query
  int metric;
  uint64_t* cand;        // [splits*2][nq][KL] keys (approx score, id), sorted ascending
  int has_norm;          // L2: one more B chunk (the norm pieces) and one more K=8 MMA per tile
  const float* thr0;     // nullable: per-query pruning threshold in score space (from a sample pass)
};

// KL = per-thread (query row, split, column half) list length: 16 when k <= 16, else 32
template <bool kTomb, bool kSelf, int KL>
__global__ void __launch_bounds__(kTcThreads, 1)
    knn_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap xmap,
                  const __grid_constant__ CUtensorMap nmap, TcArgs a) {
  constexpr int TC_LIST = KL;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned operand area (SWIZZLE_128B atoms)
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int kca = a.kc + (a.has_norm ? 1 : 0);                // A chunks: the query tile + the norm weights
  unsigned char* sA = smem;                                   // kca x 16 KB
  unsigned char* sB = sA + (size_t)kca * kAChunkBytes;        // stages x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)a.stages * kBStageBytes);
  uint64_t* full = bars;                   // [stages]
  uint64_t* empty = full + a.stages;       // [stages]
  uint64_t* a_full = empty + a.stages;     // [1]
  uint64_t* a_empty = a_full + 1;          // [1]
  uint64_t* t_full = a_empty + 1;          // [2]
  uint64_t* t_empty = t_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, 32 * kTcEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    if (a.has_norm) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&nmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t qtiles = (a.nq + TC_M - 1) / TC_M;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      uint32_t stage = 0, phase = 0, aphase = 0;
      for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int64_t qt = u % qtiles, sp = u / qtiles;
        const int64_t r0 = sp * a.rows_per_split, r1 = min(a.n, r0 + a.rows_per_split);
        mbar_wait(a_empty, aphase ^ 1);
        aphase ^= 1;
        mbar_expect_tx(a_full, (uint32_t)kca * kAChunkBytes);
        for (int c = 0; c < kca; ++c)
          tma_load_2d(sA + (size_t)c * kAChunkBytes, &qmap, a_full, c * TC_KC, (int)(qt * TC_M));
        for (int64_t nb = r0; nb < r1; nb += TC_N) {
          for (int c = 0; c < kca; ++c) {
            mbar_wait(empty + stage, phase ^ 1);
            mbar_expect_tx(full + stage, kBStageBytes);
            if (c < a.kc)
              tma_load_2d(sB + (size_t)stage * kBStageBytes, &xmap, full + stage, c * TC_KC, (int)nb);
            else  // the norm pieces of the same 256 rows
              tma_load_2d(sB + (size_t)stage * kBStageBytes, &nmap, full + stage, 0, (int)nb);
            if (++stage == (uint32_t)a.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      uint32_t stage = 0, phase = 0, aphase = 0, acc = 0, tphase[2] = {0, 0};
      for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int64_t sp = u / qtiles;
        const int64_t r0 = sp * a.rows_per_split, r1 = min(a.n, r0 + a.rows_per_split);
        mbar_wait(a_full, aphase);
        aphase ^= 1;
        for (int64_t nb = r0; nb < r1; nb += TC_N) {
          mbar_wait(t_empty + acc, tphase[acc] ^ 1);
          tphase[acc] ^= 1;
          tc_fence_after();
          const uint32_t d = tmem_base + acc * TC_N;
          for (int c = 0; c < kca; ++c) {
            mbar_wait(full + stage, phase);
            tc_fence_after();
            const uint32_t abase = smem_u32(sA + (size_t)c * kAChunkBytes);
            const uint32_t bbase = smem_u32(sB + (size_t)stage * kBStageBytes);
            if (c < a.kc) {
#pragma unroll
              for (int kk = 0; kk < TC_KC / 8; ++kk)  // K = 8 tf32 (32 bytes) per MMA
                umma_tf32(d, sdesc(abase + kk * 32), sdesc(bbase + kk * 32), (c | kk) ? 1u : 0u);
            } else {
              umma_tf32(d, sdesc(abase), sdesc(bbase), 1u);  // + w . p = ||x||^2 (the pieces sit in K = 0..2)
            }
            umma_commit(empty + stage);
            if (++stage == (uint32_t)a.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(t_full + acc);
          acc ^= 1;
        }
        umma_commit(a_empty);  // the A tile may be replaced once every MMA of this unit is done
      }
    }
  } else {  // ---------------- epilogue: thread = query row = TMEM lane, half of the 256 columns ----------------
    const int lq = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;        // columns [half*128, half*128+128) of every tile
    const int row = lq * 32 + lane;
    uint32_t acc = 0, tphase[2] = {0, 0};
    for (int64_t u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int64_t qt = u % qtiles, sp = u / qtiles;
      const int64_t r0 = sp * a.rows_per_split, r1 = min(a.n, r0 + a.rows_per_split);
      const int64_t qi = qt * TC_M + row;
      float bv[TC_LIST];
      uint32_t bi[TC_LIST];
#pragma unroll
      for (int i = 0; i < TC_LIST; ++i) {
        bv[i] = __int_as_float(0x7F800000);
        bi[i] = kSent;
      }
      // rows scoring >= thr0 cannot be among the query's k nearest (a sample already holds k rows below it), so
      // the lists start with that bound: far fewer (warp-divergent) insertions
      const float thr0 = (a.thr0 != nullptr && qi < a.nq) ? a.thr0[qi] : __int_as_float(0x7F800000);
      float thr = fminf(bv[TC_LIST - 1], thr0);
      for (int64_t nb = r0; nb < r1; nb += TC_N) {
        mbar_wait(t_full + acc, tphase[acc]);
        tphase[acc] ^= 1;
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(lq * 32) << 16) + acc * TC_N + half * (TC_N / 2);
#ifdef SVF_KNN_NO_EPILOGUE
        if (true) {
          tc_fence_before();
          mbar_arrive(t_empty + acc);
          acc ^= 1;
          continue;
        }
#endif
        // one 32-column chunk: the MMA's scores, their minimum over 4 independent chains, (rarely) insertions
        auto process = [&](uint32_t(&v)[32], int c0) {
          const int64_t cb = nb + half * (TC_N / 2) + c0;
          // valid columns: inside the split, not deleted, not the query itself
          uint32_t valid = cb >= r1 ? 0u : (r1 - cb >= 32 ? 0xFFFFFFFFu : ((1u << (uint32_t)(r1 - cb)) - 1u));
          if (kTomb && cb < r1) valid &= ~__ldg(a.tomb + (cb >> 5));
          if (kSelf) {
            const int64_t sj = a.self_base + qi - cb;
            if (sj >= 0 && sj < 32) valid &= ~(1u << (uint32_t)sj);
          }
          float mn4[4] = {__int_as_float(0x7F800000), __int_as_float(0x7F800000), __int_as_float(0x7F800000),
                          __int_as_float(0x7F800000)};
#pragma unroll
          for (int j = 0; j < 32; ++j) mn4[j & 3] = fminf(mn4[j & 3], __uint_as_float(v[j]));
          const float mn = fminf(fminf(mn4[0], mn4[1]), fminf(mn4[2], mn4[3]));
          uint32_t pass = 0;
          if (mn < thr && valid != 0u) {
#pragma unroll
            for (int j = 0; j < 32; ++j) pass |= (__uint_as_float(v[j]) < thr ? 1u : 0u) << j;
            pass &= valid;
          }
          while (pass) {  // rare after warm-up: insert into the ascending register list
            const int jj = __ffs(pass) - 1;
            pass &= pass - 1u;
            float sc = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) sc = (j == jj) ? __uint_as_float(v[j]) : sc;
            if (sc < bv[TC_LIST - 1]) {
              const uint32_t id = (uint32_t)(cb + jj);
#pragma unroll
              for (int i = TC_LIST - 1; i > 0; --i) {
                const bool shift = bv[i - 1] > sc;
                const bool here = !shift && bv[i] > sc;
                bv[i] = shift ? bv[i - 1] : (here ? sc : bv[i]);
                bi[i] = shift ? bi[i - 1] : (here ? id : bi[i]);
              }
              if (bv[0] > sc) {
                bv[0] = sc;
                bi[0] = id;
              }
            }
          }
          thr = fminf(bv[TC_LIST - 1], thr0);
        };
        // software pipeline over the 4 chunks: the next chunk's TMEM load is in flight while one is processed
        uint32_t va[32], vb[32];
        __syncwarp();
        tmem_issue32(taddr + 0, va);
        tmem_wait32(va);
#pragma unroll 1
        for (int c0 = 0; c0 < TC_N / 2; c0 += 64) {
          tmem_issue32(taddr + c0 + 32, vb);
          process(va, c0);
          tmem_wait32(vb);
          if (c0 + 64 < TC_N / 2) tmem_issue32(taddr + c0 + 64, va);
          process(vb, c0 + 32);
          if (c0 + 64 < TC_N / 2) tmem_wait32(va);
        }
        tc_fence_before();
        mbar_arrive(t_empty + acc);
        acc ^= 1;
      }
      if (qi < a.nq) {
        uint64_t* dst = a.cand + ((size_t)(sp * 2 + half) * a.nq + qi) * TC_LIST;
#pragma unroll
        for (int i = 0; i < TC_LIST; ++i) dst[i] = bi[i] == kSent ? kEmptyKey : make_key(bv[i], bi[i]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ||x||^2 per row (fp32 FFMA) as the B operand's extra K chunk: pieces hi, mid, lo, each exact in TF32 (the top
// 11 significant bits of what remains), so that hi + mid + lo = ||x||^2 up to 2^-35 relative (exactly for integer
// norms < 2^24); plus dataset facts for the TF32 error bound: max ||x||, all values integer <= 2047
__global__ void row_norms_kernel(const float* __restrict__ vec, int dp, int64_t n, float* __restrict__ npieces,
                                 unsigned int* __restrict__ facts) {
  // grid-stride over rows, warp per row; the facts are reduced per warp and per block before one atomic per
  // block (a global atomic per row serialised on one address: 0.75 ms at 1M rows)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ unsigned int s_max[32], s_int[32];
  unsigned int wmax = 0u;
  bool wint = true;
  for (int64_t r = (int64_t)blockIdx.x * nw + wib; r < n; r += (int64_t)gridDim.x * nw) {
    float acc = 0.f;
    bool integral = true;
    for (int c = lane; c < dp; c += 32) {
      const float x = __ldg(vec + r * dp + c);
      acc = fmaf(x, x, acc);
      integral = integral && (x == rintf(x)) && fabsf(x) <= 2047.f;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    wint = wint && __all_sync(0xffffffffu, integral);
    const float hi = __uint_as_float(__float_as_uint(acc) & 0xFFFFE000u);
    const float rem = acc - hi;  // exact (Sterbenz)
    const float mid = __uint_as_float(__float_as_uint(rem) & 0xFFFFE000u);
    const float lo = __uint_as_float(__float_as_uint(rem - mid) & 0xFFFFE000u);
    npieces[r * 32 + lane] = lane == 0 ? hi : (lane == 1 ? mid : (lane == 2 ? lo : 0.f));
    wmax = max(wmax, __float_as_uint(sqrtf(acc)));  // positive floats order like their bit patterns
  }
  if (lane == 0) {
    s_max[wib] = wmax;
    s_int[wib] = wint ? 1u : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int m = 0u, in = 1u;
    for (int w = 0; w < nw; ++w) {
      m = max(m, s_max[w]);
      in &= s_int[w];
    }
    atomicMax(facts + 0, m);
    if (!in) atomicAnd(facts + 1, 0u);
  }
}

// Pruning threshold per query from the exact k-th distance d_s among a row sample (a valid upper bound of the
// true k-th): in score space (L2: s = d - ||q||^2, IP: s = d), raised by the TF32 error bound 2E of the
// approximate scores and a relative/absolute slack, so that every row of the true top k scores strictly below it.
__global__ void prune_threshold_kernel(const float* __restrict__ Q, int64_t q_stride, int q_dim, int64_t nq, int k,
                                       const float* __restrict__ d_sample, int metric, int D,
                                       const unsigned int* __restrict__ facts, float* __restrict__ thr0) {
  const int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  const float ds = d_sample[qi * k + k - 1];
  if (!(ds < __int_as_float(0x7F800000))) {
    thr0[qi] = __int_as_float(0x7F800000);
    return;
  }
  double qn = 0.0;
  bool qint = true;
  for (int c = 0; c < q_dim; ++c) {
    const float x = Q[(size_t)qi * q_stride + c];
    qn += (double)x * x;
    qint = qint && x == rintf(x) && fabsf(x) <= 2047.f;
  }
  const double xmax = (double)__uint_as_float(facts[0]);
  const double qnorm = sqrt(qn);
  // integer data (the K-R exactness condition): scores are exact integers, so +1 keeps the true top k strictly
  // below; otherwise the TF32 bound 2E plus the fp32 rounding of d_s and ||q||^2
  const bool exact = facts[1] != 0u && qint && xmax * xmax + 2.0 * qnorm * xmax < 16777216.0;
  const double u = 1.0 / 512.0 + (D + 9) * 2.384185791015625e-07;
  const double E = exact ? 0.0
                         : (metric == 0 ? 2.0 : 1.0) * u * qnorm * xmax +
                               (D + 4) * 5.9604644775390625e-08 * (xmax * xmax + qn);
  const double sc = (double)ds - (metric == 0 ? qn : 0.0);
  const double slack = (D + 4) * 1.1920928955078125e-07 * (fabs((double)ds) + qn) + (exact ? 1.0 : 1e-30);
  const double t = sc + 2.0 * E + slack;
  thr0[qi] = __double2float_ru(t + 1e-6 * fabs(t));  // rounded up: the bound never tightens
}

// A operand rows [s*q | 0 | w]: s = -2 (L2) or -1 (IP), exact in TF32 for the integer queries the exactness
// argument covers; w = (1, 1, 1) picks up the norm pieces (L2 only).  Row length (kc + 1) * 32 floats.
__global__ void stage_queries_kernel(const float* __restrict__ Q, int64_t q_stride, int q_dim, int64_t nq, int kc,
                                     int metric, float* __restrict__ qa) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int w = (kc + 1) * 32;
  if (t >= nq * w) return;
  const int64_t r = t / w;
  const int c = (int)(t - r * w);
  float v = 0.f;
  if (c < q_dim) v = (metric == 0 ? -2.f : -1.f) * Q[(size_t)r * q_stride + c];
  else if (c >= kc * 32 && c < kc * 32 + 3 && metric == 0) v = 1.f;
  qa[t] = v;
}

// K-R: exact re-rank of the approximate candidates + certificate (warp per query)
template <int KL>
__global__ void knn_rerank_kernel(const uint64_t* __restrict__ cand, int64_t splits, int64_t nq, int k,
                                  const float* __restrict__ vec, int dq, const float* __restrict__ Q,
                                  int64_t q_stride, int q_dim, int metric, const unsigned int* __restrict__ facts,
                                  uint32_t* __restrict__ out_ids, float* __restrict__ out_d,
                                  uint32_t* __restrict__ fail_list, unsigned int* __restrict__ n_fail,
                                  const float* __restrict__ thr0) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (qi >= nq) return;
  // merge the per-split approximate lists into the best 64; tau = least score an excluded row can have
  uint64_t best[2] = {kEmptyKey, kEmptyKey};
  float tau = __int_as_float(0x7F800000);
  for (int64_t s = 0; s < splits; ++s) {
    uint64_t c[1];
    c[0] = lane < KL ? cand[((size_t)s * nq + qi) * KL + lane] : kEmptyKey;
    const uint64_t last = __shfl_sync(0xffffffffu, c[0], KL - 1);
    if (last != kEmptyKey) tau = fminf(tau, key_dist(last));  // a full list excluded rows scoring >= its max
    warp_merge_into<2, 1>(best, c, lane);
  }
  const uint64_t m64 = __shfl_sync(0xffffffffu, best[1], 31);
  if (m64 != kEmptyKey) tau = fminf(tau, key_dist(m64));
  if (thr0 != nullptr) tau = fminf(tau, thr0[qi]);  // every list excluded rows scoring >= thr0
  // exact distances of the (up to) 64 candidates: lane handles 2, full row each (rows are L2/HBM gathers)
  const float* q = Q + (size_t)qi * q_stride;
  float qn = 0.f;
  for (int c = lane; c < q_dim; c += 32) qn = fmaf(q[c], q[c], qn);
  bool qint = true;
  for (int c = lane; c < q_dim; c += 32) qint = qint && (q[c] == rintf(q[c])) && fabsf(q[c]) <= 2047.f;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) qn += __shfl_xor_sync(0xffffffffu, qn, off);
  qint = __all_sync(0xffffffffu, qint);
  uint64_t ex[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t id = key_id(best[r]);
    ex[r] = kEmptyKey;
    if (id != kSent) {
      const float4* x4 = reinterpret_cast<const float4*>(vec + (size_t)id * dq * 4);
      float acc = 0.f;
      for (int c4 = 0; c4 < dq; ++c4) {
        const float4 x = __ldg(x4 + c4);
        const int c = c4 * 4;
        const float q0 = c < q_dim ? q[c] : 0.f, q1 = c + 1 < q_dim ? q[c + 1] : 0.f;
        const float q2 = c + 2 < q_dim ? q[c + 2] : 0.f, q3 = c + 3 < q_dim ? q[c + 3] : 0.f;
        if (metric == 0) {
          float d0 = x.x - q0, d1 = x.y - q1, d2 = x.z - q2, d3 = x.w - q3;
          acc = fmaf(d0, d0, acc);
          acc = fmaf(d1, d1, acc);
          acc = fmaf(d2, d2, acc);
          acc = fmaf(d3, d3, acc);
        } else {
          acc = fmaf(x.x, q0, acc);
          acc = fmaf(x.y, q1, acc);
          acc = fmaf(x.z, q2, acc);
          acc = fmaf(x.w, q3, acc);
        }
      }
      ex[r] = make_key((metric == 0 ? acc : -acc) + 0.0f, id);
    }
  }
  warp_sort<2>(ex, lane);
  if (lane < k) {
    out_ids[qi * k + lane] = key_id(ex[0]);
    out_d[qi * k + lane] = key_dist(ex[0]);
  }
  if (k > 32 && lane + 32 < k) {
    out_ids[qi * k + 32 + lane] = key_id(ex[1]);
    out_d[qi * k + 32 + lane] = key_dist(ex[1]);
  }
  // certificate: every excluded row has true score >= tau - E; accept if the exact k-th beats that strictly
  const uint64_t kk = __shfl_sync(0xffffffffu, k <= 32 ? ex[0] : ex[1], (k - 1) & 31);
  if (lane == 0 && tau != __int_as_float(0x7F800000)) {
    const double xmax = (double)__uint_as_float(facts[0]);
    const double qnorm = sqrt((double)qn);
    const int D = dq * 4;
    // integer data and queries: every product and partial sum of the MMA is an integer below 2^24 (partial dot
    // products are bounded by ||q|| ||x|| (Cauchy-Schwarz), the norm pieces by ||x||^2) -> scores are exact
    const bool exact = facts[1] != 0u && qint && xmax * xmax + 2.0 * qnorm * xmax < 16777216.0;
    double E = 0.0;
    if (!exact) {
      const double u = 1.0 / 512.0 + (D + 9) * 2.384185791015625e-07;  // 2^-9 + (D+9) 2^-22
      E = (metric == 0 ? 2.0 : 1.0) * u * qnorm * xmax + (D + 4) * 5.9604644775390625e-08 * (xmax * xmax + qn) +
          1e-30;
    }
    const double dk = (double)key_dist(kk) * (exact ? 1.0 : 1.0 + (D + 2) * 5.9604644775390625e-08);
    const double bound = (double)tau - E + (metric == 0 ? (double)qn : 0.0);
    if (kk == kEmptyKey || !(dk < bound)) fail_list[atomicAdd(n_fail, 1u)] = (uint32_t)qi;
  }
}

__global__ void gather_rows_kernel(const float* __restrict__ Q, int64_t q_stride, int q_dim,
                                   const uint32_t* __restrict__ rows, int64_t m, float* __restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * q_dim) return;
  const int64_t r = t / q_dim;
  dst[t] = Q[(size_t)rows[r] * q_stride + (t - r * q_dim)];
}
__global__ void scatter_results_kernel(const uint32_t* __restrict__ rows, int64_t m, int k,
                                       const uint32_t* __restrict__ src_ids, const float* __restrict__ src_d,
                                       uint32_t* __restrict__ out_ids, float* __restrict__ out_d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * k) return;
  const int64_t r = t / k;
  out_ids[(size_t)rows[r] * k + (t - r * k)] = src_ids[t];
  out_d[(size_t)rows[r] * k + (t - r * k)] = src_d[t];
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {TC_KC, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TcPlan {
  int kc, stages;
  int64_t splits, rows_per_split, units, qtiles;
  size_t smem;
};
TcPlan tc_plan(int64_t nq, int64_t n, int dq, int num_sms, int units_per_sm = 8) {
  TcPlan p;
  p.kc = (dq * 4 + TC_KC - 1) / TC_KC;
  const size_t a_bytes = (size_t)(p.kc + 1) * kAChunkBytes;  // + the norm-weight chunk
  const size_t budget = 227 * 1024 - 1024 - 512;
  p.stages = (int)std::min<size_t>(6, (budget - a_bytes) / kBStageBytes);
  p.qtiles = (nq + TC_M - 1) / TC_M;
  const int64_t ntiles = std::max<int64_t>(1, (n + TC_N - 1) / TC_N);
  int64_t s = std::max<int64_t>(1, ((int64_t)units_per_sm * num_sms + p.qtiles - 1) / p.qtiles);  // ~8 units/SM
  s = std::min(s, ntiles);
  p.rows_per_split = (ntiles + s - 1) / s * TC_N;
  p.splits = (n + p.rows_per_split - 1) / p.rows_per_split;
  if (p.splits < 1) p.splits = 1;
  p.units = p.qtiles * p.splits;
  p.smem = 1024 + a_bytes + (size_t)p.stages * kBStageBytes + 512;
  return p;
}

}  // namespace

bool knn_tc_supported(int dq, int64_t q_stride, const float* Q, int k) {
  const int kc = (dq * 4 + TC_KC - 1) / TC_KC;
  (void)q_stride;
  (void)Q;  // queries are restaged into the A layout
  return k <= 32 && (size_t)(kc + 1) * kAChunkBytes + 2 * kBStageBytes + 2048 <= 227 * 1024 && get_encode() != nullptr;
}

// the sample pass: enough rows that few rows of the full set beat its k-th (~ k n / S per query), few enough that
// it costs a few percent of the main pass
static int64_t sample_rows(int64_t n, int64_t nq) {
  static const int64_t div = [] {  // SVF_KNN_SAMPLE_DIV: tuning override of the sample fraction 1/div (0 = off)
    const char* v = getenv("SVF_KNN_SAMPLE_DIV");
    return v ? (int64_t)atoll(v) : (int64_t)32;  // n/32 rows (C2: 5.75 ms vs 5.83 at n/16, 7.2 without)
  }();
  if (div <= 0 || n < 262144 || nq < 512) return 0;
  return std::min<int64_t>(65536, std::max<int64_t>(8192, n / div)) / TC_N * TC_N;
}

size_t knn_tc_scratch_bytes(int64_t nq, int64_t n, int dq, int k) {
  const int64_t S = sample_rows(n, nq);
  const size_t sample = S ? knn_tc_scratch_bytes(nq, S, dq, k) + (size_t)nq * (k * 8 + 4) + 768 : 0;
  TcPlan p = tc_plan(nq, n, dq, 148);
  TcPlan p2 = tc_plan(nq, n, dq, 512);
  const int64_t s = std::max(p.splits, p2.splits);
  // cand + norm pieces + staged queries + facts + fail list + fallback buffers (rows, ids, dists) + FFMA scratch
  return (size_t)s * 2 * nq * TC_LIST_MAX * 8 + (size_t)n * 128 + (size_t)nq * (p.kc + 1) * 128 + 1024 +
         (size_t)nq * 4 + (size_t)nq * dq * 16 + (size_t)nq * k * 8 + knn_scratch_bytes(nq, k, n) + 10 * 256 +
         sample;
}

static cudaError_t knn_tc_impl(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                          int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                          uint32_t* out_ids, float* out_d, void* scratch, size_t scratch_bytes, int num_sms,
                          cudaStream_t st, uint32_t* n_fallback, bool inner, const float* bound_d) {
  if (nq <= 0) return cudaSuccess;
  // the sample pass: ~4 units per SM (C2: 5.75 vs 5.92 ms end to end at 8; 2 and 16 were no better)
  static const int inner_ups = [] {  // SVF_KNN_INNER_UPS: tuning override
    const char* v = getenv("SVF_KNN_INNER_UPS");
    return v ? atoi(v) : 4;
  }();
  TcPlan p = tc_plan(nq, n, dq, num_sms, inner ? inner_ups : 8);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  unsigned char* sp = static_cast<unsigned char*>(scratch);
  uint64_t* cand = reinterpret_cast<uint64_t*>(sp);
  const int KL = k <= 16 ? 16 : 32;
  sp += al((size_t)p.splits * 2 * nq * KL * 8);
  float* npieces = reinterpret_cast<float*>(sp);  // [n][32]: ||x||^2 pieces (B's extra K chunk)
  sp += al((size_t)n * 128);
  float* qa = reinterpret_cast<float*>(sp);       // [nq][(kc+1)*32]: the staged A rows
  sp += al((size_t)nq * (p.kc + 1) * 128);
  unsigned int* facts = reinterpret_cast<unsigned int*>(sp);  // [0] max norm bits, [1] integral, [2] n_fail
  sp += 256;
  uint32_t* fail_list = reinterpret_cast<uint32_t*>(sp);
  sp += al((size_t)nq * 4);
  float* fbQ = reinterpret_cast<float*>(sp);
  sp += al((size_t)nq * q_dim * 4);
  uint32_t* fb_ids = reinterpret_cast<uint32_t*>(sp);
  sp += al((size_t)nq * k * 4);
  float* fb_d = reinterpret_cast<float*>(sp);
  sp += al((size_t)nq * k * 4);
  float* thr0 = nullptr;
  // the pruning bound: the caller's k live rows per query (a graph search, DESIGN §6 K-G) or the sample pass
  const int64_t S = (self_base < 0 && !inner && bound_d == nullptr) ? sample_rows(n, nq) : 0;
  uint32_t* s_ids = nullptr;
  float* s_d = const_cast<float*>(bound_d);
  if (bound_d != nullptr) {
    thr0 = reinterpret_cast<float*>(sp);
    sp += al((size_t)nq * 4);
  }
  if (S > 0) {
    thr0 = reinterpret_cast<float*>(sp);
    sp += al((size_t)nq * 4);
    s_ids = reinterpret_cast<uint32_t*>(sp);
    sp += al((size_t)nq * k * 4);
    s_d = reinterpret_cast<float*>(sp);
    sp += al((size_t)nq * k * 4);
  }
  if ((size_t)(sp - static_cast<unsigned char*>(scratch)) > scratch_bytes) return cudaErrorInvalidValue;
  const size_t rest = scratch_bytes - (size_t)(sp - static_cast<unsigned char*>(scratch));
  if (S > 0) {
    // exact k-NN over the first S rows (same engine, no further sampling): its k-th distance bounds the true one
    // k distinct live rows with their exact distances bound the true k-th from above whether or not the
    // sample's own certificate holds, so the sample pass needs neither the fallback nor a host synchronisation
    cudaError_t es = knn_tc_impl(vec, dq, S, tomb, Q, q_stride, q_dim, nq, k, metric, -1, s_ids, s_d, sp, rest,
                                 num_sms, st, nullptr, true, nullptr);
    if (es != cudaSuccess) return es;
  }

  const uint64_t qa_w = (uint64_t)(p.kc + 1) * 32;
  CUtensorMap qmap, xmap, nmap;
  if (!make_map(&qmap, qa, qa_w, (uint64_t)nq, qa_w * 4, TC_M) ||
      !make_map(&xmap, vec, (uint64_t)dq * 4, (uint64_t)n, (uint64_t)dq * 16, TC_N) ||
      !make_map(&nmap, npieces, 32, (uint64_t)n, 128, TC_N))
    return cudaErrorInvalidValue;
  unsigned int init[3] = {0u, 1u, 0u};
  cudaError_t e = cudaMemcpyAsync(facts, init, sizeof init, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  row_norms_kernel<<<(unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)num_sms * 8), 256, 0, st>>>(vec, dq * 4, n,
                                                                                                   npieces, facts);
  stage_queries_kernel<<<(unsigned)((nq * (int64_t)qa_w + 255) / 256), 256, 0, st>>>(Q, q_stride, q_dim, nq, p.kc,
                                                                                       metric, qa);
  if (thr0 != nullptr)
    prune_threshold_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, st>>>(Q, q_stride, q_dim, nq, k, s_d, metric,
                                                                         dq * 4, facts, thr0);
  TcArgs a{nq, n, p.kc, p.stages, p.rows_per_split, p.splits, p.units, tomb, self_base, metric, cand,
           metric == 0 ? 1 : 0, thr0};
  auto launch = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    if (e2 != cudaSuccess) return e2;
    const unsigned grid = (unsigned)std::min<int64_t>(p.units, num_sms);
    kern<<<grid, kTcThreads, p.smem, st>>>(qmap, xmap, nmap, a);
    return cudaGetLastError();
  };
  if (KL == 16) {
    if (tomb && self_base >= 0) e = launch(knn_tc_kernel<true, true, 16>);
    else if (tomb) e = launch(knn_tc_kernel<true, false, 16>);
    else if (self_base >= 0) e = launch(knn_tc_kernel<false, true, 16>);
    else e = launch(knn_tc_kernel<false, false, 16>);
  } else {
    if (tomb && self_base >= 0) e = launch(knn_tc_kernel<true, true, 32>);
    else if (tomb) e = launch(knn_tc_kernel<true, false, 32>);
    else if (self_base >= 0) e = launch(knn_tc_kernel<false, true, 32>);
    else e = launch(knn_tc_kernel<false, false, 32>);
  }
  if (e != cudaSuccess) return e;
  if (KL == 16)
    knn_rerank_kernel<16><<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(cand, p.splits * 2, nq, k, vec, dq, Q, q_stride,
                                                                    q_dim, metric, facts, out_ids, out_d, fail_list,
                                                                    facts + 2, thr0);
  else
    knn_rerank_kernel<32><<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(cand, p.splits * 2, nq, k, vec, dq, Q, q_stride,
                                                                    q_dim, metric, facts, out_ids, out_d, fail_list,
                                                                    facts + 2, thr0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (inner) return cudaSuccess;
  // exact FFMA fallback for the queries the certificate rejected
  unsigned int hf = 0;
  if ((e = cudaMemcpyAsync(&hf, facts + 2, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (n_fallback) *n_fallback = hf;
  if (hf > 0) {
    if (self_base >= 0)  // seed build on non-integral data: redo the (small) seed exactly with FFMA
      return launch_knn_exact(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, sp,
                              rest, num_sms, st);
    gather_rows_kernel<<<(unsigned)((hf * (int64_t)q_dim + 255) / 256), 256, 0, st>>>(Q, q_stride, q_dim, fail_list,
                                                                                       hf, fbQ);
    e = launch_knn_exact(vec, dq, n, tomb, fbQ, q_dim, q_dim, hf, k, metric, -1, fb_ids, fb_d, sp, rest, num_sms, st);
    if (e != cudaSuccess) return e;
    scatter_results_kernel<<<(unsigned)((hf * (int64_t)k + 255) / 256), 256, 0, st>>>(fail_list, hf, k, fb_ids, fb_d,
                                                                                      out_ids, out_d);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_knn_tc(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                          int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                          uint32_t* out_ids, float* out_d, void* scratch, size_t scratch_bytes, int num_sms,
                          cudaStream_t st, uint32_t* n_fallback, const float* bound_d) {
  return knn_tc_impl(vec, dq, n, tomb, Q, q_stride, q_dim, nq, k, metric, self_base, out_ids, out_d, scratch,
                     scratch_bytes, num_sms, st, n_fallback, false, bound_d);
}

}  // namespace svf
