/* svf.h — C ABI of the B200 hot path of SVFusion (arXiv 2601.08528): batched graph-based ANNS over a
 * fixed-out-degree proximity graph, with batched insertion and tombstoned deletion.
 *
 * Citations: P:L<n> = /root/reference/PAPER.md line n (the paper), S:L<n> = SPEC.md line n.  The operations
 * follow the paper's statement of the streaming ANNS problem, Build / Search / Insert / Delete (§2.2,
 * P:L195-211), the search loop of Algorithm 1, insertion (§5.1) and lazy deletion
 * (§5.2.1).  Readings of ambiguous passages are SURVEY.md §8(c) I1..I18, restated in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Pointers may be HOST or DEVICE memory (detected with cudaPointerGetAttributes).  The caller owns every
 *    buffer; the library copies inputs during the call and keeps no caller pointer.  Device outputs are ready
 *    when `stream` (a cudaStream_t, NULL = legacy default stream) completes; when an output pointer is host
 *    memory the call synchronises `stream` before returning.
 *  - Distances: metric SVF_L2 reports the SQUARED Euclidean distance sum_i (q_i - x_i)^2 (order-
 *    equivalent to P:L162); SVF_IP reports -<q, x>, so ascending order always means "nearer" (reading I1).
 *    fp32 inputs, fp32 arithmetic (the paper keeps vectors uncompressed fp32: P:L119).
 *  - Ordering and ties: results are sorted ascending by (distance, id); equal distances -> lower id (I5).
 *  - Ids: 0-based uint32, allocated by the library in insertion order, never reused (reading I14).
 *    Ids must stay below 2^31 (capacity <= 2^31 - 1).  0xFFFFFFFF (SVF_SENTINEL) pads results (I17) and
 *    marks empty adjacency slots.
 *  - Errors: status codes only, never exceptions.  Validation failures (SVF_ERR_INVALID / CAPACITY /
 *    NOT_FOUND) leave the index unchanged.  A CUDA failure poisons the index: every later call returns
 *    SVF_ERR_POISONED.  svf_last_error() returns a thread-local message for the last failure.
 *  - Calls on one index are serialised by an internal mutex (no concurrency control beyond that: SURVEY A29).
 *
 * Layout in HBM (owned by the index, sized at `capacity` when built/imported):
 *    vec      float [capacity][Dp]   Dp = D rounded up to a multiple of 4 (16-byte rows, zero padding)
 *    graph    uint32[capacity][R]    slots [0,P) protected prefix (detour order), [P,R) tail sorted by
 *                                    (edge_dist, id) with tombstoned entries counted as +inf
 *    edge_dist float[capacity][R]    distance of each edge (+inf for empty slots)
 *    tomb     uint32[capacity/32]    deletion bitset, bit (id % 32) of word (id / 32)
 */
#ifndef SVF_H_
#define SVF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVF_SENTINEL 0xFFFFFFFFu

typedef struct svf_index svf_index; /* opaque; owns all device memory */

typedef enum {
  SVF_OK = 0,
  SVF_ERR_INVALID = 1,   /* bad argument (k > itopk, n <= 0, unsupported dim/degree, ...) */
  SVF_ERR_CAPACITY = 2,  /* n_alloc + n would exceed capacity; nothing inserted */
  SVF_ERR_NOT_FOUND = 3, /* delete of an id >= n_alloc */
  SVF_ERR_CUDA = 4,      /* CUDA runtime failure (index poisoned) */
  SVF_ERR_OOM = 5,       /* device allocation failed */
  SVF_ERR_NCCL = 6,      /* reserved for the sharded layer */
  SVF_ERR_POISONED = 7   /* an earlier CUDA failure poisoned this index */
} svf_status;

typedef enum { SVF_L2 = 0, SVF_IP = 1 } svf_metric;

typedef struct {
  int32_t dim;            /* D >= 1, <= 512 */
  int32_t degree;         /* R: fixed out-degree (KNNG with uniform degree); 2 <= R <= 128 */
  int32_t metric;         /* svf_metric */
  int64_t capacity;       /* max ids ever allocated (ids are never reused) */
  int32_t search_width;   /* p >= 1 parents expanded per iteration (1 = Alg. 1 GetNearest; I3) */
  int32_t n_init;         /* random entry points per query (I2); 0 = use itopk */
  int32_t max_iter;       /* iteration cap; 0 = run to convergence (I4) */
  int32_t insert_itopk;   /* L_insert: candidate-list size of the insert search (I9; default 128) */
  int32_t protect_prefix; /* P protected forward slots per row (I12); -1 = R/2; 0 = SPEC drop-farthest */
  int32_t insert_batch;   /* B_ins: insert sub-batch size (I13; default 4096, <= 2^13 per P:L1067) */
  int32_t seed_size;      /* n0 rows built as the exact R-NN seed by svf_build (I15; default 4096) */
  int32_t hash_bits;      /* visited-table slots per query = 2^hash_bits (I7); 0 = automatic */
  uint64_t seed;          /* entry-point seed (I2, I18) */
  int32_t device;         /* CUDA ordinal the index lives on */
  int32_t build_itopk;    /* L_build: candidate-list size of svf_build's growth inserts (I15); 0 = insert_itopk.
                           * A larger L_build buys graph quality once, at build time; later svf_insert calls use
                           * insert_itopk.  <= 512. */
} svf_params;

/* Fill *p with the defaults above for dimension `dim` and degree `degree` (metric L2, capacity 0). */
void svf_default_params(svf_params* p, int32_t dim, int32_t degree);

/* Build(X_init): allocate the index at p->capacity (>= n), copy X (n x dim, row-major), build the
 * graph as the exact R-NN of the first min(n, seed_size) rows, then grow it by batched insertion of the rest
 * (reading I15 / SURVEY O5).  n >= 1.  On success *out owns the new index (free with svf_destroy). */
svf_status svf_build(const svf_params* p, const float* X, int64_t n, void* stream, svf_index** out);

/* Search(q, k) (Algorithm 1) for a batch of nq queries (nq x dim, row-major).
 * itopk = L, the internal candidate-pool size (k <= L <= 512; "L >= k").  Writes out_ids[nq][k] and
 * out_dists[nq][k], sorted ascending, padded with (SVF_SENTINEL, +inf) when fewer than k live vectors are
 * reachable.  Deleted vectors are never returned.  Query i seeds its entry points with qidx = i.
 * Two-stream overlap ("multiple search streams plus one update stream"): svf_search on
 * one stream may run on the GPU concurrently with ONE svf_insert / svf_delete / svf_repair on another stream
 * (the two paths own disjoint scratch, queue counters and handoff buffers).  Visibility rule: each query
 * snapshots n at its start as the ids whose insertion sub-batch has completed on the device, so it never reaches
 * or samples a partially linked vertex; a row being rewritten concurrently may be read before or after its
 * update (every id it holds is < n or filtered); a concurrent delete is seen or not, per word.  Results of a
 * concurrent search are therefore valid but timing-dependent; with no update in flight they are deterministic.
 * svf_build, svf_knn_exact, svf_import/export and svf_link_candidates must not overlap other calls. */
svf_status svf_search(svf_index* idx, const float* Q, int64_t nq, int32_t k, int32_t itopk, uint32_t* out_ids,
                      float* out_dists, void* stream);

/* Insert(x) (§5.1) for a batch of n vectors: ids n_alloc .. n_alloc+n-1 are assigned and
 * written to out_ids (nullable).  Sub-batches of min(insert_batch, n_current) vertices run: (i) insert-mode
 * search over the sub-batch-start snapshot (L = insert_itopk), (ii) detour-ranked forward rows, (iii) reverse
 * edges into the targets' row tails.  CAPACITY if n_alloc + n > capacity (nothing inserted). */
svf_status svf_insert(svf_index* idx, const float* X, int64_t n, uint32_t* out_ids, void* stream);

/* Delete(x) (lazy deletion P:L529-533): set the tombstone bit of each id.  Idempotent; deleting a
 * deleted id is OK.  *n_newly_deleted (nullable) = ids whose bit was newly set.  NOT_FOUND if any id >= n_alloc
 * (then nothing is deleted).  Visible to every search issued after the call's stream work completes. */
svf_status svf_delete(svf_index* idx, const uint32_t* ids, int64_t n, int64_t* n_newly_deleted, void* stream);

/* Exact k-NN over the live set (ground truth "via exhaustive linear scan"): out_ids[nq][k],
 * out_dists[nq][k] sorted by (distance, id).  Tensor-core scoring + exact fp32 re-rank. k <= 256. */
svf_status svf_knn_exact(svf_index* idx, const float* Q, int64_t nq, int32_t k, uint32_t* out_ids,
                         float* out_dists, void* stream);

/* Localized topology-aware repair (reading R1' in DESIGN.md; 1 <= c <= degree): every live vertex whose
 * non-empty neighbour slots are more than `threshold` (paper: 0.5) deleted gets, for each deleted neighbour p (slot
 * order), the first c (paper: 8) live members of N_out(p) that are not itself and not already its neighbours;
 * its row is rebuilt by the insertion's selection rule (detour counts, protected prefix + sorted tail) over the
 * insert_itopk nearest of its live neighbours and those candidates.  Only those rows change.  *n_repaired = rows rewritten; hist (nullable) = live rows by deleted-neighbour fraction in buckets
 * {0, (0,0.1), [0.1,0.4], (0.4,threshold], >threshold} (the distribution of Fig. 5).  Synchronous. */
svf_status svf_repair(svf_index* idx, int32_t c, double threshold, int64_t* n_repaired, uint64_t hist[5],
                      void* stream);

/* Global consolidation (reading C2 in DESIGN.md): "a global consolidation of all affected
 * neighborhoods by aggregating candidates from the outgoing neighbors of deleted vertices".  Every live row holding a
 * tombstoned id keeps its live entries (prefix entries in their slots) and refills its vacancies from the live
 * members of its deleted neighbours' lists: a deleted prefix slot takes the nearest member of that deleted
 * neighbour's own list, the tail vacancies take the nearest of the remaining union; the tail is re-sorted by
 * (edge_dist, id).  Afterwards no live row references a deleted vertex.  *n_rewritten (nullable) = rows rewritten.
 * Synchronous; may overlap an svf_search on another stream (see svf_search). */
svf_status svf_consolidate(svf_index* idx, int64_t* n_rewritten, void* stream);

/* Automatic consolidation: after an svf_delete, when the vertices deleted since the last consolidation exceed
 * `ratio` times the vertices that were live then ("e.g., 20%"), the delete call consolidates on its
 * stream.  0 = off (default), else in (0, 1). */
svf_status svf_set_consolidation(svf_index* idx, double ratio);

/* out[0] = consolidations run so far (explicit + automatic), out[1] = n_deleted at the last one. */
svf_status svf_consolidation_stats(svf_index* idx, int64_t out[2]);

/* Merge G per-shard top-k lists (ids/dists laid out [G][nq][k], GLOBAL ids) into the first k by (dist, id)
 * per query (the step after the NCCL all-gather).  Uses the current device. */
svf_status svf_merge_topk(const uint32_t* ids, const float* dists, int32_t G, int64_t nq, int32_t k,
                          uint32_t* out_ids, float* out_dists, void* stream);

/* Sharded search, SURVEY §8(e) (the dataset is split into n_logical shards, global id g -> shard g mod n_logical,
 * local id g div n_logical; a rank holds several shards).  Step 2, a rank's pre-merge: merge n_lists (<= 16) shard
 * results ids/dists [n_lists][nq][k] (device, LOCAL ids, SVF_SENTINEL padded) into the first k per query by
 * (dist, id) with GLOBAL ids g = local * n_logical + shard[i] (shard: HOST array of n_lists values < n_logical),
 * written to out_pairs[nq][k] (device) as packed u64 pairs (float bits of the distance << 32 | global id; padding
 * = (+inf, SVF_SENTINEL)), ready for one all_gather_into_tensor.  Global ids must stay below 2^31.  Uses the current
 * device; INVALID on bad sizes or non-device buffers. */
svf_status svf_shard_premerge(const uint32_t* ids, const float* dists, int32_t n_lists, int64_t nq, int32_t k,
                              uint32_t n_logical, const uint32_t* shard, uint64_t* out_pairs, void* stream);

/* Step 4: merge G gathered pair lists pairs[G][nq][k] (device, as written by svf_shard_premerge) into out_ids /
 * out_dists [nq][k] (device), the first k per query by (dist, id).  Merging is associative over this total order, so
 * the result does not depend on how the shards were grouped into ranks. */
svf_status svf_merge_pairs(const uint64_t* pairs, int32_t G, int64_t nq, int32_t k, uint32_t* out_ids,
                           float* out_dists, void* stream);

/* Copy the index state out (any pointer may be NULL to skip): vec[n_alloc][dim] (unpadded), graph[n_alloc][R],
 * edge_dist[n_alloc][R], tomb[ceil(n_alloc/32)], *n_alloc.  Synchronous. */
svf_status svf_export(const svf_index* idx, float* vec, uint32_t* graph, float* edge_dist, uint32_t* tomb,
                      int64_t* n_alloc);

/* Create an index from given state (same layouts as svf_export; edge_dist/tomb may be NULL = +inf / none). */
svf_status svf_import(const svf_params* p, const float* vec, const uint32_t* graph, const float* edge_dist,
                      const uint32_t* tomb, int64_t n_alloc, svf_index** out);

/* TEST ENTRY: steps (ii)+(iii) of insertion from GIVEN candidate lists (n_new x n_cand ids/dists, distance-
 * ordered, SVF_SENTINEL-padded, all ids < n_alloc) for new vertices n_alloc .. n_alloc+n_new-1 whose vectors
 * are X (n_new x dim; NULL = zeros).  Lets tests check the integer adjacency update bit-exactly. */
svf_status svf_link_candidates(svf_index* idx, const float* X, const uint32_t* cand_ids, const float* cand_d,
                               int64_t n_new, int32_t n_cand, void* stream);

/* Warps serving one query in svf_search / svf_insert's search: 1, 2 (both warps keep identical pools and split the
 * candidate slots; used when degree * search_width > 32 and itopk <= 128: ~35% lower per-query latency, lower
 * throughput once the batch fills the GPU), or 0 = automatic (2 while 2*nq <= 24 * SM count, else 1).  Results
 * are identical for every setting (NEXT-2 low-latency path). */
svf_status svf_set_warps_per_query(svf_index* idx, int32_t wpq);

/* Pair-mode handoff of one-warp batches (NEXT-2 latency path, applied to the batch tail): once the
 * query queue has drained and fewer than `pct`% of the one-warp grid's warps are still searching, each suspends its
 * query (pool keys with parent flags + counters) and a second grid, chained by programmatic dependent launch onto
 * the SM slots the first frees, resumes it with two warps per query.  The visited table restarts from the pool ids,
 * which leaves the search unchanged (reading I7), so results are identical for every setting.  -1 = automatic,
 * 0 = off, 1..100.  Applies to pools of <= 128 entries with degree * search_width > 32. */
svf_status svf_set_search_handoff(svf_index* idx, int32_t pct);

/* Exact-kNN engine: mode 0 = automatic (tcgen05 TF32 scoring + exact FFMA re-rank with a certificate, exact FFMA
 * fallback for rejected queries; used when k <= 32 and query rows are 16-byte aligned), 1 = FFMA tiles only. */
svf_status svf_set_knn_mode(svf_index* idx, int32_t mode);

/* Exact-kNN counters since creation: out[0] = queries, out[1] = queries that took the FFMA fallback after the
 * tensor-core certificate rejected them, out[2] = tensor-core launches. */
svf_status svf_knn_stats(svf_index* idx, uint64_t out[3]);

/* Search-time knobs (overrides the build params): search_width, n_init (0 = itopk), max_iter, hash_bits. */
svf_status svf_set_search_params(svf_index* idx, int32_t search_width, int32_t n_init, int32_t max_iter,
                                 int32_t hash_bits);

/* Counters of the last svf_search on this index (synchronises its stream):
 * out[0] = distance computations, out[1] = iterations, out[2] = parents expanded, out[3] = queries,
 * out[4] = kernels launched (1, or 2 with the pair-mode handoff grid). */
svf_status svf_last_search_counters(svf_index* idx, uint64_t out[5]);

/* Per-query timeline of svf_search calls (diagnostics for the batch-tail analysis): after
 * svf_set_trace(idx, 1), each search records an 8-word row per query i: out[8i] = start and out[8i+1] = end
 * (device %globaltimer, ns), out[8i+2] = SM id << 32 | iterations, out[8i+3..8i+7] = SM cycles spent in the
 * select / row-fetch / filter / distance / merge phases (zero unless built with -DSVF_PHASE_PROF).
 * svf_read_trace copies the last search's rows into the host buffer `out` (cap >= nq rows, else INVALID;
 * synchronises) and sets *nq (0 if none).  Off by default. */
svf_status svf_set_trace(svf_index* idx, int32_t enable);
svf_status svf_read_trace(svf_index* idx, uint64_t* out, int64_t cap, int64_t* nq);

/* Device-time profiling of the main kernel of each call (CUDA events on the caller's stream).
 * svf_profile(idx, 1) enables and resets; svf_profile_read fills ms[0..3] = total ms of
 * {search kernel, insert-search kernel, detour kernel, reverse-apply kernels} and cnt[0..3] launch counts. */
svf_status svf_profile(svf_index* idx, int32_t enable);
svf_status svf_profile_read(svf_index* idx, double ms[4], int64_t cnt[4]);

/* State: *n_alloc, *n_deleted (live = n_alloc - n_deleted), *capacity (any may be NULL). */
svf_status svf_info(const svf_index* idx, int64_t* n_alloc, int64_t* n_deleted, int64_t* capacity);

svf_status svf_destroy(svf_index* idx);

/* Thread-local message describing the last non-OK status on this thread ("" if none). */
const char* svf_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SVF_H_ */
