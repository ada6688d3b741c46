/*
 * louiskv.h — C ABI of the B200-native LouisKV KV-retrieval hot path.
 *
 * Method: LouisKV (arXiv 2510.11292). Citations: P:n = PAPER.md line n.
 *   cluster_prompt  = kvm.store_cache(K, V, 'prefill')   Alg. 1, §4.2
 *   should_retrieve = is_new_segment / r_t vs tau        Alg. 1, §4.1
 *   retrieve        = kvm.Retrieve(q_t, B)               Alg. 1, App. B
 *   append_output   = kvm.store_cache(k_t, v_t,'decode') Alg. 1, §4.2
 *   sparse_attn     = o_t over [KV_critical : KV_local]  Alg. 1, §3.1
 *
 * Conventions (all entry points):
 *  - Pointers named d_* or documented "device" are CUDA device pointers; "host"
 *    pointers are ordinary host memory. The library never takes ownership of
 *    caller memory; device inputs are borrowed for the stream-ordered duration
 *    of the call (the library copies what it keeps).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Hot calls only ENQUEUE work; none of should_retrieve / retrieve /
 *    append_output / sparse_attn synchronises with the host, so a whole decode
 *    step is CUDA-graph capturable (the one exception: retrieve with
 *    fetch_mode LOUISKV_FETCH_BATCHED_DMA, documented there).
 *  - Layout: head_dim d must be 128. K/V/q/out elements are bf16 (uint16 bits),
 *    d contiguous. Strides are in ELEMENTS.
 *  - Errors: argument/state errors return synchronously and enqueue nothing.
 *    An asynchronous CUDA fault surfaces as LOUISKV_ERR_CUDA on a later call
 *    and is sticky: the context must be destroyed. louiskv_last_error() gives
 *    a message. Degenerate inputs are not errors: P <= S gives zero prompt
 *    units, B = 0 gives an empty selection, a zero query has cosine 0.
 *  - There is no CPU fallback: every computation runs in sm_100a kernels.
 *  - A context is single-owner and used from one stream at a time.
 */
#ifndef LOUISKV_H_
#define LOUISKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct louiskv_ctx louiskv_ctx; /* opaque, library-owned */

typedef enum {
  LOUISKV_OK = 0,
  LOUISKV_ERR_INVALID_ARG = 1,
  LOUISKV_ERR_STATE = 2,
  LOUISKV_ERR_CAPACITY = 3,
  LOUISKV_ERR_OOM_DEVICE = 4,
  LOUISKV_ERR_OOM_HOST = 5,
  LOUISKV_ERR_CUDA = 6,
  LOUISKV_ERR_NOT_IMPLEMENTED = 7
} louiskv_status;

enum { LOUISKV_TRIG_PREV_STEP = 0, LOUISKV_TRIG_LAST_RETRIEVAL = 1 };
enum { LOUISKV_BOUNDARY_PER_LAYER = 0, LOUISKV_BOUNDARY_SHARED = 1 };
/* gather of the selected units' rows ("transfer data from specific rows"):
 * ZERO_COPY   — the select kernel's own threads read the pinned pool through its device mapping with
 *               16-B vector loads (no host involvement; graph-capturable; the default);
 * BATCHED_DMA — select writes per-unit copy spans (K rows, V rows) into mapped pinned memory; the
 *               host waits for them (louiskv_retrieve synchronises its stream), merges spans that are
 *               contiguous at both ends and enqueues one cudaMemcpyAsync per span on the copy engines
 *               (host pool -> working set for new units, device -> device for kept units). Not
 *               graph-capturable (retrieve returns STATE inside a capture); louiskv_decode_layer then
 *               issues the per-call sequence. */
enum { LOUISKV_FETCH_ZERO_COPY = 0, LOUISKV_FETCH_BATCHED_DMA = 1 };
enum { LOUISKV_KMEANS_TC = 0, LOUISKV_KMEANS_SIMT = 1 };
/* prompt units: semantic k-means clusters (the method) or contiguous pages (the page units of
 * the paper's comparison systems, §3.1 P:63 "partition the entire key cache ... into m fixed-size
 * pages", page size 16 at P:143) */
enum { LOUISKV_UNITS_KMEANS = 0, LOUISKV_UNITS_PAGES = 1 };
enum { LOUISKV_ATTN_TC = 0, LOUISKV_ATTN_SIMT = 1 };
/* element type of the KV rows in the pinned host pool (config pool_dtype). BF16: the rows as given
 * (the paper's pool, "All KV cache is stored in FP16"). FP8_E4M3 (a
 * variant the paper does not have): every row entering the pool (prompt offload, segment eviction)
 * is stored as E4M3, round-to-nearest-even, saturating at +-448 — half the host-link bytes of every
 * offload and gather; the gather converts back to bf16 (exactly) into the working set. Sinks, the
 * local buffer, centroids and full-cache layers stay bf16 / fp32. Not combinable with BATCHED_DMA. */
enum { LOUISKV_POOL_BF16 = 0, LOUISKV_POOL_FP8_E4M3 = 1 };

typedef struct {
  int32_t num_layers, num_q_heads, num_kv_heads, head_dim; /* head_dim must be 128; num_q_heads <= 64;
                                                              g = num_q_heads/num_kv_heads in {1,2,4,8};
                                                              num_layers <= 64 */
  int32_t kv_head_begin, kv_head_count;                    /* KV-head shard owned by this ctx */
  int32_t max_batch;
  int64_t max_prompt_len, max_output_len;                  /* fix every capacity at create */
  int32_t budget_tokens;     /* B: retrieved tokens per (b, layer, kv-head) */
  int32_t sink_tokens;       /* S */
  int32_t window_tokens;     /* W: local-buffer tokens */
  double tau;                /* boundary threshold */
  int32_t avg_cluster_size;  /* c: k = ceil((P-S)/c) clusters */
  int32_t kmeans_iters;      /* Lloyd iterations (fixed count, no early exit) */
  int32_t kmeans_impl;       /* LOUISKV_KMEANS_TC (tcgen05) | LOUISKV_KMEANS_SIMT */
  uint64_t full_cache_layers; /* bitmask of layers that keep the full cache (0b11) */
  int32_t trigger_ref;       /* LOUISKV_TRIG_PREV_STEP | _LAST_RETRIEVAL */
  int32_t boundary_mode;     /* LOUISKV_BOUNDARY_PER_LAYER | _SHARED */
  int32_t shared_layer;      /* designated layer for SHARED mode */
  int32_t max_open_segment;  /* force-seal bound on the open segment (0 -> window_tokens) */
  int32_t fetch_mode;        /* LOUISKV_FETCH_ZERO_COPY (default) | LOUISKV_FETCH_BATCHED_DMA; other
                                values: INVALID_ARG at create */
  int32_t device;            /* CUDA device ordinal */
  int32_t attn_impl;         /* full-cache attention: LOUISKV_ATTN_TC (mma.sync + TMA tensor maps,
                                default) | LOUISKV_ATTN_SIMT (CUDA cores) */
  int32_t trigger_stride;    /* 0 (default): the semantic-boundary trigger, flag = (t == 1) || r_t < tau
                                (Alg. 1). k >= 1: the fixed-stride retrieval of the paper's
                                ablation ("retrieves every 5 / 16 steps"): flag = (t - 1) % k == 0;
                                r_t is still computed and reported, segments then span k tokens.
                                Negative: INVALID_ARG at create. */
  int32_t prompt_units;      /* LOUISKV_UNITS_KMEANS (default) | LOUISKV_UNITS_PAGES: cluster_prompt
                                splits [S, P) into k = ceil((P-S)/c) contiguous pages of c =
                                avg_cluster_size tokens (the last one shorter), centroid = mean of the
                                page's keys (fp32), no Lloyd iterations; everything downstream (offload,
                                scoring, selection, gather) is unchanged. Other values: INVALID_ARG. */
  int32_t index_offload;     /* 0 (default): the unit index (fp32 centroids + their bf16 scoring copy,
                                [units][d] per instance) in device memory. 1: the index in pinned,
                                device-mapped host memory — the paper's future work ("memory
                                consumption could be further reduced by offloading KV cache indices to
                                CPU DRAM"): scoring reads the centroid rows over the host link, segment
                                evictions write them there, and cluster_prompt runs k-means on one
                                layer's device scratch and copies that layer's centroids out. Results are
                                bit-identical to 0; device memory drops by ~6*d bytes per unit-table
                                row. Other values: INVALID_ARG. */
  int32_t pool_dtype;        /* LOUISKV_POOL_BF16 (default) | LOUISKV_POOL_FP8_E4M3; other values, or FP8
                                with fetch_mode BATCHED_DMA: INVALID_ARG */
} louiskv_config;

typedef struct {
  uint64_t retrievals;        /* flagged (b, layer) retrieve events */
  uint64_t units_scored;      /* units scored over all flagged (b, layer, kv-head) */
  uint64_t units_selected;
  uint64_t units_reused;      /* selected units already resident (D2D copy) */
  uint64_t units_fetched;     /* selected units read from the host pool */
  uint64_t bytes_h2d;         /* host-pool bytes read by the gather */
  uint64_t bytes_d2h;         /* bytes written to the host pool (prompt offload + evictions) */
  uint64_t segments_evicted;
  uint64_t kmeans_tc_iters;   /* Lloyd assignment passes run on the tcgen05 kernel */
  uint64_t kmeans_simt_iters; /* ... on the SIMT kernel (impl SIMT, or TMA-incompatible strides) */
  uint64_t dma_copies;        /* fetch_mode BATCHED_DMA: copy-engine copies issued by retrieve */
} louiskv_stats;

/* Allocates every device buffer and the pinned, device-mapped host pool.
 * Errors: INVALID_ARG (bad geometry / head_dim != 128 / shard out of range),
 * OOM_DEVICE, OOM_HOST, CUDA. *out is NULL on failure. */
louiskv_status louiskv_create(const louiskv_config* cfg, louiskv_ctx** out);
/* Synchronises the device, frees everything. NULL is a no-op. */
void louiskv_destroy(louiskv_ctx* ctx);

/* kvm.store_cache(K, V, 'prefill') for one layer.
 * k, v: device bf16, element (b, t, h, e) at base + b*stride_b + t*stride_t + h*stride_h + e,
 *   h in [0, kv_head_count) (the owned heads), t in [0, prompt_len).
 * Retrieval layer: per (b, h) k-means of keys [S, P) into k = ceil((P-S)/c) clusters
 *   (kmeans_iters Lloyd iterations, strided init, empty-cluster repair), centroids kept on
 *   the device (fp32 + bf16), KV rows offloaded cluster-major to the host pool, sinks kept.
 * Full-cache layer: K, V copied to the device cache.
 * Must be called once per layer before the first decode step; resets that layer's decode
 * state. Asynchronous: the KV offload runs on a library-owned copy stream (device staging ->
 * pinned pool), overlapping later calls; every decode-path call on this layer makes its stream
 * wait for it (inside a graph capture as an external event-wait node), and the introspection
 * calls synchronise it. Errors: INVALID_ARG (layer, batch > max_batch,
 * prompt_len > max_prompt_len, batch differing from an earlier call), STATE. */
louiskv_status louiskv_cluster_prompt(louiskv_ctx* ctx, int32_t layer, const void* k, const void* v,
                                      int64_t stride_b, int64_t stride_t, int64_t stride_h,
                                      int32_t batch, int64_t prompt_len, void* stream);

/* Makes `stream` wait for every prompt offload still in flight ("offload (K, V) to CPU
 * memory pool asynchronously"): after it, the whole prefill of every layer is complete in
 * stream order. Enqueues event waits only. Errors: INVALID_ARG, CUDA. */
louiskv_status louiskv_prompt_fence(louiskv_ctx* ctx, void* stream);

/* Same as cluster_prompt but with the clustering supplied by the caller (external or
 * reference clustering): h_assign host int32 [batch][kv_head_count][P-S] cluster ids in
 * [0, k); h_centroids host fp32 [batch][kv_head_count][k][d]; every cluster non-empty.
 * Synchronous (copies host arrays). Errors: INVALID_ARG, STATE. */
louiskv_status louiskv_set_prompt_units(louiskv_ctx* ctx, int32_t layer, const void* k, const void* v,
                                        int64_t stride_b, int64_t stride_t, int64_t stride_h,
                                        int32_t batch, int64_t prompt_len, int32_t n_clusters,
                                        const int32_t* h_assign, const float* h_centroids, void* stream);

/* Decode step t (1-based, advanced by this call) of one layer: r_t and the retrieval flag
 * (P:101-106). q_all: device bf16 [batch][num_q_heads][d] (ALL query heads),
 * sequence b at q_all + b*stride_b. d_flag_out (uint8 [batch]) and d_r_out (double [batch])
 * are optional DEVICE outputs. Per-step call order per layer:
 * should_retrieve -> retrieve -> append_output -> sparse_attn. Full-cache layers write flag 0.
 * Errors: INVALID_ARG, STATE (order broken, cluster_prompt missing, SHARED designated layer
 * not yet called this step, more than max_output_len steps). */
louiskv_status louiskv_should_retrieve(louiskv_ctx* ctx, int32_t layer, const void* q_all, int64_t stride_b,
                                       uint8_t* d_flag_out, double* d_r_out, void* stream);

/* kvm.Retrieve(q_t, B) for every flagged sequence: group-consistent scores
 * A = mean_j softmax(q^j C^T / sqrt(d)) over all host-resident units of each owned KV head
 * (App. B), greedy budgeted selection in (A desc, unit id asc) order, and the gather of
 * the selected units' KV rows (new units from the pinned host pool over the host link, kept
 * units device-to-device) into the working set. Unflagged sequences are untouched.
 * q_own: device bf16 [batch][g*kv_head_count][d] (owned query heads). No-op on full-cache
 * layers. fetch_mode BATCHED_DMA: the call synchronises `stream` after the selection (the span lists
 * must reach the host) and enqueues one batched copy; STATE when `stream` is capturing.
 * Errors: INVALID_ARG, STATE, CUDA. */
louiskv_status louiskv_retrieve(louiskv_ctx* ctx, int32_t layer, const void* q_own, int64_t stride_b, void* stream);

/* kvm.store_cache(k_t, v_t, 'decode'): seal the open segment at a boundary
 * (or at max_open_segment), append (k_t, v_t), evict the oldest sealed segments while the
 * local buffer holds more than W tokens (centroid = mean of its keys, rows offloaded to the
 * host pool, appended as a new unit). k_t, v_t: device bf16 [batch][kv_head_count][d].
 * Errors: INVALID_ARG, STATE, CAPACITY (pool full; sticky). */
louiskv_status louiskv_append_output(louiskv_ctx* ctx, int32_t layer, const void* k_t, const void* v_t,
                                     int64_t stride_b, void* stream);

/* o = softmax(q K_I^T / sqrt(d)) V_I for every owned query head over
 * I = sinks ∪ working set ∪ local buffer (incl. this step's k_t); full-cache layers attend
 * to all P+t rows. q_own as in retrieve. out: device bf16
 * [batch][g*kv_head_count][d] contiguous; out_f32 optional device fp32, same shape.
 * Errors: INVALID_ARG, STATE. */
louiskv_status louiskv_sparse_attn(louiskv_ctx* ctx, int32_t layer, const void* q_own, int64_t stride_b,
                                   void* out, float* out_f32, void* stream);

/* Fused equivalent of louiskv_append_output followed by louiskv_sparse_attn (identical results):
 * on a retrieval layer one clustered launch (8 CTAs per (b, owned head); rank 0 runs the
 * seal/append/evict of store_cache, the cluster barrier publishes the local buffer, all ranks
 * attend their split, rank 0 merges the partials through distributed shared memory). On a
 * full-cache layer it issues the two calls. Arguments as in the two calls. Errors: as there. */
louiskv_status louiskv_append_attn(louiskv_ctx* ctx, int32_t layer, const void* k_t, const void* v_t,
                                   int64_t stride_kv, const void* q_own, int64_t stride_q, void* out,
                                   float* out_f32, void* stream);

/* One whole decode step of one layer (Algorithm 1: trigger, retrieve when flagged,
 * store_cache, attention), identical in results to should_retrieve -> retrieve ->
 * append_output -> sparse_attn with q_own = q_all + kv_head_begin*g*d (same stride). On a
 * retrieval layer it is ONE clustered launch of CL CTAs per (b, owned head) — CL = 8 when every
 * instance's cluster fits one wave of one CTA per SM, else 4 while two waves suffice, else 2 (env
 * LOUISKV_LAYER_CL overrides): every rank recomputes r_t (recipe R1), the flagged instances score
 * with their units split over the CL ranks and every
 * rank runs the budgeted selection on the replicated scores (exchanged through distributed shared
 * memory; instances with more than 8192 LIVE units keep the per-unit select arrays in global
 * scratch instead — same launch, decided on the device per step), the ranks gather the new working
 * set, the last rank appends, all ranks attend one split each. A full-cache layer is one launch
 * too (dense attention with the store_cache fused). Budgets with min(B, unit capacity) > 1024
 * issue the multi-kernel sequence instead, and so does fetch_mode BATCHED_DMA. Arguments: q_all
 * as in should_retrieve (stride_q), k_t/v_t as in append_output (stride_kv), out/out_f32 as in
 * sparse_attn, d_flag_out/d_r_out optional device outputs as in should_retrieve.
 * Errors: INVALID_ARG, STATE (as should_retrieve), CUDA. */
louiskv_status louiskv_decode_layer(louiskv_ctx* ctx, int32_t layer, const void* q_all, int64_t stride_q,
                                    const void* k_t, const void* v_t, int64_t stride_kv, void* out,
                                    float* out_f32, uint8_t* d_flag_out, double* d_r_out, void* stream);

/* ---- introspection (synchronous: they synchronise the device) ---- */
/* Current working-set unit ids of (layer, b, owned head h), ascending. */
louiskv_status louiskv_get_selection(louiskv_ctx* ctx, int32_t layer, int32_t b, int32_t h,
                                     int32_t* ids, int32_t cap, int32_t* n);
/* Unit table of (layer, b, h): up to cap units. Any output pointer may be NULL.
 * centroids_f32 host [cap][d]; sizes host [cap]; first_pos host [cap] (lowest member
 * position); n_units receives the number of units (prompt clusters first, then evicted
 * segments in eviction order). */
louiskv_status louiskv_get_units(louiskv_ctx* ctx, int32_t layer, int32_t b, int32_t h, int32_t cap,
                                 float* centroids_f32, int32_t* sizes, int32_t* first_pos, int32_t* n_units);
/* Token positions of the host-pool rows of (layer, b, h) in pool order (unit after unit,
 * members ascending), up to cap. */
louiskv_status louiskv_get_unit_positions(louiskv_ctx* ctx, int32_t layer, int32_t b, int32_t h,
                                          int32_t* positions, int64_t cap, int64_t* n);
/* Copies the current working set (K rows then V rows, bf16 bits) of (layer, b, h) to host
 * arrays [cap][d]; *n_rows receives the row count. */
louiskv_status louiskv_get_working_set(louiskv_ctx* ctx, int32_t layer, int32_t b, int32_t h,
                                       uint16_t* k_rows, uint16_t* v_rows, int32_t cap, int32_t* n_rows);
louiskv_status louiskv_get_stats(louiskv_ctx* ctx, louiskv_stats* out);
/* Memory held by the context (the paper's memory comparison, Table 3 / P:404-425): device bytes
 * of every device allocation made at create (sinks, working sets, local buffers, centroids, unit
 * tables, full-cache layers, scratch) and the pinned host bytes (the KV pool, plus the unit index
 * when index_offload = 1). Either pointer may be NULL.
 * No synchronisation. Errors: INVALID_ARG (null ctx). */
louiskv_status louiskv_get_memory(const louiskv_ctx* ctx, uint64_t* device_bytes, uint64_t* host_pool_bytes);
/* NUMA placement of the pinned host pool: on hosts with more than one NUMA node the pool is
 * allocated on the GPU's own node (sysfs numa_node of its PCI device; anonymous mmap bound with mbind,
 * then pinned and mapped with cudaHostRegister), so each GPU's host-link traffic stays on its socket;
 * otherwise cudaHostAlloc. Env LOUISKV_POOL_NUMA=0 disables, =1 forces the bound allocation on a
 * single-node host. *node = the bound node, or -1 (cudaHostAlloc). Errors: INVALID_ARG. */
louiskv_status louiskv_get_pool_numa_node(const louiskv_ctx* ctx, int32_t* node);

/* ---- prefill phase timer (the per-phase breakdown of cluster_prompt; SURVEY §5 tracing) ----
 * When enabled, every later cluster_prompt records stream-ordered CUDA events between its phases:
 * init (sinks, centroid init), assign (the tcgen05 assignment GEMM + fused argmax, one per Lloyd
 * iteration), sort (cluster histogram, scan, empty-cluster repair, stable scatter), update (centroid
 * means), stage (cluster-major permute into the device staging buffer + unit table) and, on the
 * library's copy stream, the D2H copies into the pinned pool. Times are device elapsed times between
 * consecutive marks (the phases run back to back on the caller's stream). Costs one event record per
 * phase boundary; off by default. */
typedef struct {
  double init_ms, assign_ms, sort_ms, update_ms, stage_ms, d2h_ms;
  uint64_t assign_flops;   /* algorithmic: 2 * N * k * d per instance per assignment pass */
  uint64_t keys;           /* clustered keys (N per instance per cluster_prompt call) */
  uint64_t d2h_bytes;      /* bytes copied into the host pool */
  uint64_t assign_passes;  /* assignment passes (Lloyd iterations x calls) */
  int32_t calls;           /* cluster_prompt calls timed */
} louiskv_prefill_times;
/* Enable (1) / disable (0) the timer and reset its accumulators. Synchronises the device.
 * Errors: INVALID_ARG, CUDA. */
louiskv_status louiskv_set_prefill_timing(louiskv_ctx* ctx, int32_t enable);
/* Accumulated phase times since the last set_prefill_timing. Synchronises the device.
 * Errors: INVALID_ARG (null out), CUDA. */
louiskv_status louiskv_get_prefill_times(louiskv_ctx* ctx, louiskv_prefill_times* out);

/* ---- decode-state checkpoint (device resident) ----
 * state_save copies, stream-ordered on `stream`, every device buffer the decode path mutates
 * (instance states, selections, both working-set buffers, local buffers and segment FIFOs, q_ref,
 * flags, r, step counters, pending gather jobs, stats counters) into checkpoint buffers owned by the
 * context (allocated on the first save). state_restore copies them back and restores the host-side
 * step counters, so the decode continues exactly from the saved step (rows appended to unit tables,
 * the host pool or the full cache after the save are beyond the restored counters and get rewritten).
 * Use: replaying the same decode steps (e.g. A/B measurement, speculative-decoding rollback).
 * Must be called between steps (every layer's step complete) after cluster_prompt on every layer.
 * Errors: STATE (no prefill / inside a step / restore without save), OOM_DEVICE, CUDA. */
louiskv_status louiskv_state_save(louiskv_ctx* ctx, void* stream);
louiskv_status louiskv_state_restore(louiskv_ctx* ctx, void* stream);

const char* louiskv_last_error(const louiskv_ctx* ctx);
/* Library build string (arch, version). */
const char* louiskv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LOUISKV_H_ */
