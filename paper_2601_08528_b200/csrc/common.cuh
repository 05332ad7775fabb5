// Device helpers shared by the sm_100a kernels of libsvf.so (NOT shared with oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace svf {

constexpr uint32_t kSent = 0xFFFFFFFFu;       // empty slot / padded id
constexpr uint64_t kEmptyKey = ~0ull;         // +inf key; flag bit set => never selected as a parent
constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;

// ---- 64-bit pool keys ------------------------------------------------------------------------------------------
// key = orderable(dist) << 32 | id << 1 | parented.  Ascending u64 order == (dist, id) order (I5) because ids in
// one pool are distinct, so the flag bit never decides an order.  orderable() is the sign-flip map that makes
// IEEE-754 order equal unsigned order (+0 canonical, see dist epilogues).
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t b = __float_as_uint(f);
  return b ^ ((b >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o ^ 0x80000000u) : ~o);
}
__device__ __forceinline__ uint64_t make_key(float d, uint32_t id) {
  return ((uint64_t)f2ord(d) << 32) | ((uint64_t)id << 1);
}
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return k == kEmptyKey ? kSent : (uint32_t)(k >> 1) & 0x7FFFFFFFu; }
__device__ __forceinline__ float key_dist(uint64_t k) {
  return k == kEmptyKey ? __int_as_float(0x7F800000) : ord2f((uint32_t)(k >> 32));
}

// ---- packed fp32 pairs (sm_100 FADD2 / FFMA2: two fp32 operations per issue slot) -------------------------------
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float f2sum(uint64_t r) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
  return a + b;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// acc += (x - q)^2 (metric 0, squared L2) or x * q (metric 1, inner product) over one float4, as two packed pairs:
// the low half accumulates components x, z and the high half y, w; f2sum(acc) is the lane's partial sum
__device__ __forceinline__ uint64_t dist_acc4(uint64_t acc, const float4& x, const float4& q, int metric) {
  const uint64_t x01 = f2pack(x.x, x.y), x23 = f2pack(x.z, x.w), q01 = f2pack(q.x, q.y), q23 = f2pack(q.z, q.w);
  if (metric == 0) {
    const uint64_t d01 = f2sub(x01, q01), d23 = f2sub(x23, q23);
    return f2fma(d23, d23, f2fma(d01, d01, acc));
  }
  return f2fma(x23, q23, f2fma(x01, q01, acc));
}

__device__ __forceinline__ bool tomb_dead(const uint32_t* __restrict__ tomb, uint32_t id) {
  return tomb != nullptr && ((__ldg(tomb + (id >> 5)) >> (id & 31)) & 1u);
}

// ---- entry-point law (reading I2): seeded affine permutation of [0, n) --------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t s) {
  s += 0x9E3779B97F4A7C15ull;
  s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ull;
  s = (s ^ (s >> 27)) * 0x94D049BB133111EBull;
  return s ^ (s >> 31);
}
__device__ __forceinline__ uint64_t gcd64(uint64_t x, uint64_t y) {
  while (y) {
    uint64_t t = x % y;
    x = y;
    y = t;
  }
  return x;
}
// a coprime with n, b in [0, n): id_j = (a*j + b) mod n
__device__ __forceinline__ void perm_params(uint64_t seed, uint64_t qidx, uint64_t n, uint64_t& a, uint64_t& b) {
  uint64_t h = mix64(seed ^ (qidx * 0x9E3779B97F4A7C15ull));
  a = (h >> 1) % n;
  if (a == 0) a = 1;
  while (gcd64(a, n) != 1) ++a;
  b = (h >> 33) % n;
}

// ---- warp bitonic network over a striped register array (element e = r*32 + lane) -----------------------------
template <int E>
__device__ __forceinline__ void cmpx(uint64_t (&v)[E], int j, int k, int lane) {
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int e = r * 32 + lane;
    const bool up = (k == 0) || ((e & k) == 0);
    if (j >= 32) {
      const int rj = j >> 5;
      if ((r & rj) == 0) {
        const int r2 = r | rj;
        uint64_t a = v[r], b = v[r2];
        const bool sw = up ? (a > b) : (a < b);
        v[r] = sw ? b : a;
        v[r2] = sw ? a : b;
      }
    } else {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
      const bool lower = (lane & j) == 0;
      v[r] = (lower == up) ? (v[r] < o ? v[r] : o) : (v[r] > o ? v[r] : o);
    }
  }
}
// full ascending sort of 32*E keys
template <int E>
__device__ __forceinline__ void warp_sort(uint64_t (&v)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) cmpx<E>(v, j, k, lane);
}
// ascending merge of a bitonic sequence of 32*E keys
template <int E>
__device__ __forceinline__ void warp_bitonic_merge(uint64_t (&v)[E], int lane) {
#pragma unroll
  for (int j = 16 * E; j > 0; j >>= 1) cmpx<E>(v, j, 0, lane);
}
// pool <- the 32*EP smallest of pool (sorted asc) U cand (sorted asc, 32*EC keys), sorted asc
template <int EP, int EC>
__device__ __forceinline__ void warp_merge_into(uint64_t (&pool)[EP], const uint64_t (&cand)[EC], int lane) {
#pragma unroll
  for (int r = 0; r < EP; ++r) {
    const int rr = EP - 1 - r;  // element e = r*32+lane pairs with reversed element (EP*32-1-e)
    uint64_t b = kEmptyKey;
    if (rr < EC) b = __shfl_sync(0xffffffffu, cand[rr < EC ? rr : 0], 31 - lane);
    pool[r] = pool[r] < b ? pool[r] : b;
  }
  warp_bitonic_merge<EP>(pool, lane);
}

// ---- 1-D bulk copies (TMA unit) into shared memory, completed on an mbarrier --------------------------------------
__device__ __forceinline__ uint32_t bulk_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bulk_smem_u32(b)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// dst, src 16-byte aligned, bytes a multiple of 16; one thread issues; the mbarrier's phase completes on arrival
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of dst before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bulk_smem_u32(b)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   bulk_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(bulk_smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BW_%=;\n}" ::"r"(bulk_smem_u32(b)),
      "r"(parity)
      : "memory");
}

}  // namespace svf
