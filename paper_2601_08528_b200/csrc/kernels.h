// Internal launchers of libsvf.so (below the C ABI in include/svf.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace svf {

constexpr int kSearchWarpsPerBlock = 4;
constexpr int kTraceCols = 8;  // per-query trace row: start ns, end ns, smid << 32 | iters, 5 phase cycle sums
constexpr int kHandoffMaxWarps = 148 * 64;  // handoff slots: one per warp of the one-warp grid
constexpr int kHandoffMaxKpl = 4;           // pools of <= 128 keys (the pair-mode instantiations)
constexpr size_t handoff_words() { return 8 + (size_t)kHandoffMaxWarps * (4 + 32 * kHandoffMaxKpl); }
// register cap per pool size: small pools -> more resident warps (latency-bound gathers want occupancy)
#ifndef SVF_MINB1
#define SVF_MINB1 6
#endif
#ifndef SVF_MINB_PAIR
#define SVF_MINB_PAIR 4
#endif
#ifndef SVF_MINB4
#define SVF_MINB4 4
#endif
constexpr int search_min_blocks(int kpl, int wpq = 1) {
  return wpq == 2 ? SVF_MINB_PAIR : kpl <= 1 ? SVF_MINB1 : kpl <= 2 ? 5 : kpl <= 4 ? SVF_MINB4 : kpl <= 8 ? 3 : 2;
}
// vectors per distance team per gather round: the throughput (one-warp) kernel keeps 2 (more costs occupancy);
// the latency kernels (pair mode: small batches and the batch tail) gather deeper per round
#ifndef SVF_GATHER_U
#define SVF_GATHER_U 2
#endif
#ifndef SVF_GATHER_U_PAIR
#define SVF_GATHER_U_PAIR 4
#endif


struct SearchArgs {
  const float* vec;        // [cap][dq*4]
  int dq;                  // float4 per row (Dp / 4)
  const uint32_t* graph;   // [cap][R]
  int R;
  int rshift;              // log2(R) if R is a power of two, else -1
  const uint32_t* tomb;    // nullable (no deletions)
  uint64_t n_alloc;        // snapshot: ids >= n_alloc are not sampled nor followed
  const float* Q;          // query rows
  int64_t q_stride;        // floats between query rows
  int q_dim;               // valid floats per query row (zero-padded to dq*4)
  int64_t nq;
  uint64_t qidx_base;      // query i seeds its entry points with qidx_base + i (I18)
  int L, p, n_init, max_iter, metric;
  uint64_t seed;
  int team, nv;            // lanes per distance, float4 per lane (team * nv >= dq, nv <= 4)
  int hbits;               // visited table slots = 2^hbits per warp
  int n_out;               // k (search) or L (insert mode)
  uint32_t* out_ids;
  float* out_d;
  uint32_t* counters;      // nullable: [nq][3] = n_dist, iters, n_exp
  unsigned long long* work_counter;  // query queue counter, zeroed before launch
  int wpq;                 // warps per query: 1, or 2 (pair mode; used when the candidate slots split evenly)
  // Pair-mode handoff (one-warp batches): once the query queue has drained and fewer than ho_thresh of the grid's
  // ho_total warps are still serving queries, each of them suspends its query (pool keys + counters) into a slot
  // of `ho`; a pair-mode kernel chained by programmatic dependent launch resumes the suspended queries on the SM
  // slots the first grid frees, two warps per query, so the batch does not end with long single-warp stragglers.
  // ho: nullable; [0] slots reserved, [1] unused, [2] slots taken, [3] warps exited, slots from word 8.
  unsigned long long* ho;
  int ho_thresh, ho_total;
  int is_tail;             // set by the launcher on the chained pair-mode (resume) kernel
  unsigned long long* trace;  // nullable: [nq][kTraceCols] (svf_set_trace, include/svf.h)
  // nullable: device word holding the ids whose insertion has completed; each query snapshots
  // n = min(n_alloc, *n_visible) at its start (svf_search overlapping an insert on another stream)
  const unsigned long long* n_visible;
  // nullable: host queries streamed in chunks of 2^q_chunk_log2 rows on a copy stream; q_flags[c] == q_epoch once
  // chunk c has landed (its flag is copied after it, in copy-stream order), so the search overlaps the H2D copy
  const unsigned int* q_flags;
  unsigned int q_epoch;
  int q_chunk_log2;
  int large_pool;          // 1: K-S-L, the shared-memory pool kernel (search_lp.cuh; one warp per query, no handoff)
  int vc_bits;             // K-S-L visited cache: B > 0 = 16-bit tags over ids < 2^B, 0 = u32 ids
  int vc_slots;            // K-S-L visited cache slots M (any even count >= 8; search_lp.cuh cache_pos)
  uint32_t vc_tmask;       // K-S-L 16-bit tags: 2^tb - 1 with 2^tb >= ceil(2^vc_bits / M), tb <= 15
};
cudaError_t launch_search(SearchArgs a, int kpl, int cpl, int num_sms, cudaStream_t st);
// dynamic shared memory of one search block for a configuration (search_d0.cu); large_pool: K-S-L's layout
size_t search_smem_bytes(int hbits, int kpl, int cpl, int L, int large_pool, int vc_bits, int Dp, int lp_slots);

// K-L1: detour-ranked forward rows for new ids [first, first + n_new) from candidates [n_new][nc]
// (reads the snapshot rows of the candidates, writes rows first..first+n_new-1; disjoint by construction)
cudaError_t launch_detour_select(uint32_t* graph, float* edge_dist, int R, int P, int64_t first, int64_t n_new,
                                 const uint32_t* cand_ids, const float* cand_d, int nc, cudaStream_t st);
// K-L1 into an arbitrary output buffer (row b -> out + b*R), counting detours on `graph` (used by repair)
cudaError_t launch_detour_rows(const uint32_t* graph, uint32_t* out_ids, float* out_d, int R, int P, int64_t n,
                               const uint32_t* cand_ids, const float* cand_d, int nc, cudaStream_t st);
// K-L2: reverse edges.  Scratch must hold 2*n_new*R u32 + 2*n_new*R u64 + n_new*R u32 + cub temp bytes.
size_t reverse_scratch_bytes(int64_t n_new, int R);
cudaError_t launch_reverse(uint32_t* graph, float* edge_dist, const uint32_t* tomb, int R, int P, int64_t first,
                           int64_t n_new, void* scratch, size_t scratch_bytes, cudaStream_t st);

// *p = v in stream order (publishes n_visible after an insert sub-batch is linked)
cudaError_t launch_store_u64(unsigned long long* p, uint64_t v, cudaStream_t st);

// K-D: tombstones.  check pass: *bad = 1 if any id >= n_alloc.  set pass: *newly += newly set bits.
cudaError_t launch_tomb_check(const uint32_t* ids, int64_t n, uint64_t n_alloc, unsigned int* bad, cudaStream_t st);
cudaError_t launch_tomb_set(const uint32_t* ids, int64_t n, uint32_t* tomb, unsigned long long* newly,
                            cudaStream_t st);

// K-G (+K-R): exact k-NN over ids [0, n) of vec (live only).  self_base >= 0 excludes id == self_base + query.
size_t knn_scratch_bytes(int64_t nq, int k, int64_t n);
cudaError_t launch_knn_exact(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                             int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                             uint32_t* out_ids, float* out_d, void* scratch, size_t scratch_bytes, int num_sms,
                             cudaStream_t st);

// K-G on tcgen05 (TF32) + K-R exact re-rank + certificate + exact FFMA fallback (knn_tc.cu).  bound_d (nullable):
// [nq][k] exact distances of k live rows per query (ascending; +inf padded) whose k-th bounds the true k-th from
// above, used as the main pass's pruning threshold instead of the sample pass
bool knn_tc_supported(int dq, int64_t q_stride, const float* Q, int k);
size_t knn_tc_scratch_bytes(int64_t nq, int64_t n, int dq, int k);
cudaError_t launch_knn_tc(const float* vec, int dq, int64_t n, const uint32_t* tomb, const float* Q,
                          int64_t q_stride, int q_dim, int64_t nq, int k, int metric, int64_t self_base,
                          uint32_t* out_ids, float* out_d, void* scratch, size_t scratch_bytes, int num_sms,
                          cudaStream_t st, uint32_t* n_fallback,
                          const float* bound_d = nullptr);

// K-M: merge G lists [G][nq][k] (ids/dists) -> first k per query by (dist, id)
cudaError_t launch_merge_topk(const uint32_t* ids, const float* d, int G, int64_t nq, int k, uint32_t* out_ids,
                              float* out_d, cudaStream_t st);
// K-M variants of the sharded search: a rank's pre-merge of its shards' LOCAL-id lists into packed
// (distance bits << 32 | global id) pairs, g = local * n_logical + shard[i]; and the merge of the all-gathered pairs
cudaError_t launch_shard_premerge(const uint32_t* ids, const float* d, int n_lists, int64_t nq, int k,
                                  uint32_t n_logical, const uint32_t* shard, unsigned long long* out_pairs,
                                  cudaStream_t st);
cudaError_t launch_merge_pairs(const unsigned long long* pairs, int G, int64_t nq, int k, uint32_t* out_ids,
                               float* out_d, cudaStream_t st);

// NEXT-1 localized repair (repair.cu)
// phase 1: V^L list + histogram (returns |V^L| after a sync); phase 2: rewrite those rows (reading R1')
size_t repair_mark_scratch_bytes(int64_t n_alloc);
cudaError_t launch_repair_mark(const uint32_t* graph, const uint32_t* tomb, int R, int64_t n_alloc, double threshold,
                               void* scratch, cudaStream_t st, int64_t* n_list, uint64_t hist_out[5]);
size_t repair_apply_scratch_bytes(int64_t n_list, int R, int cap);
cudaError_t launch_repair_apply(uint32_t* graph, float* edge_dist, const float* vec, int dq, int metric,
                                const uint32_t* tomb, int R, int P, int c, int cap, const void* mark_scratch,
                                int64_t n_list, void* scratch, size_t scratch_bytes, int num_sms, cudaStream_t st);

// NEXT-4 global consolidation (reading C2): rewrite, in place, every row of the mark list (threshold 0 = every live
// row holding a tombstoned id)
cudaError_t launch_consolidate(uint32_t* graph, float* edge_dist, const float* vec, int dq, int metric,
                               const uint32_t* tomb, int R, int P, const void* mark_scratch, int64_t n_list, int num_sms,
                               cudaStream_t st);

// small helpers
cudaError_t launch_pad_rows(const float* src, int64_t n, int dim, float* dst, int dq, cudaStream_t st);
cudaError_t launch_fill_rows(uint32_t* graph, float* edge_dist, int64_t first, int64_t n, int R, cudaStream_t st);
cudaError_t launch_unpad_rows(const float* src, int64_t n, int dq, float* dst, int dim, cudaStream_t st);

}  // namespace svf
