/*
 * trinity_b200.h -- C-ABI of the B200-native Trinity vector-search pool.
 *
 * Plain pointers and sizes only.  Each entry point replaces one reference
 * interface (citations are path:line under the reference's pkg/src/trinity/);
 * the reference is pure Python, so the "FFI" a maintainer binds is ctypes --
 * see INTEGRATION.md for the binding and for the Python shim that keeps the
 * reference's API (paper_2512_02281_b200/).
 *
 * Status codes: TRI_OK, TRI_EINVAL (-> ValueError: bad shape / k / dim /
 * non-finite input, the reference's ann_graph.py:131-134, engine.py:158-163),
 * TRI_EINTERNAL (-> RuntimeError: internal consistency, engine.py:196-198,
 * 249-250), TRI_ECUDA (CUDA failure).  tri_last_error() returns the message of
 * the calling thread's last failure.
 *
 * Handles own their device memory.  Functions without the _dev suffix take
 * HOST buffers and synchronise the stream before returning; _dev functions
 * take DEVICE buffers (per-query k / nprobe stay host arrays) and are
 * asynchronous on `stream` (NULL = the handle's own stream).  A handle is
 * single-owner: the reference's engine is a single-owner stepper
 * (engine.py:313-319) and so is every handle here.
 *
 * Numerics: returned distances are float64 squared L2 computed in the
 * reference's exact operation order (bit-identical to
 * ann_graph.rowwise_sq_dists); ids are ordered by (dist, id) as
 * ann_graph.py:136.  Candidates are generated in fp32 and certified (see
 * DESIGN.md); uncertified queries are recomputed exactly on the device.
 */
#ifndef TRINITY_B200_H
#define TRINITY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TRI_OK 0
#define TRI_EINVAL 1
#define TRI_EINTERNAL 2
#define TRI_ECUDA 3

#define TRI_MAX_K 1638 /* largest k of the candidate-scan path: IVF k and nprobe are capped at it; brute force
                        * beyond it runs the exhaustive path (every exact distance + a device radix sort),
                        * so tri_knn_bruteforce accepts any k <= n like brute_force_knn (ann_graph.py:131) */

typedef struct tri_store tri_store;
typedef struct tri_ivf tri_ivf;

/* Library ------------------------------------------------------------------ */
const char* tri_last_error(void);
int tri_version(void);
/* Process-wide counts of whole-search executions: eager (host-planned
 * launches), graph captures and graph replays.  Ragged batches replay
 * fixed-shape padded graphs keyed by (bucket(B), max k, max nprobe); option
 * "ragged_graphs" = 0 restores exact-shape keys. */
int tri_graph_counters(int64_t* eager, int64_t* captured, int64_t* replayed);
int tri_device_count(int32_t* count);
/* Debug/test knobs: "force_fixup" (1 = treat every query as uncertified),
 * "kp_extra" (extra over-fetch added to k), "scan_kernel" (0 auto: IVF
 * lists on the fp16 tensor-core scan, stores on TF32 when it fits; 1 fp32
 * SIMT scan; 2 TF32 tensor-core scan, no fp16), "dense_off" (1 = no dense
 * small-store path), "tc_stages" (cap on the tensor-core scan ring depth,
 * 0 = deepest that fits), "scan_reserve" (SMs the IVF list scan leaves free
 * for batches on other streams; -1 default = 8 once an index runs on more
 * than one stream), "scan_abufs" (1 default / 2 append-list buffers of the IVF
 * tensor-core scan), "scan_qbufs" (1 / 2 default query tiles), "scan_l2hint"
 * (IVF scan row loads: 0 default policy, 1 default = L2 evict_first, 2
 * evict_last), "pack_mixed" (1 default: tensor-core scan groups mix k classes),
 * "gthr" (1 default: cross-item thresholds), "fx_slice_rows" (fix-up: minimum
 * rows per slice, default 256), "graphs" (1 default: CUDA graph replay of
 * repeated search shapes), "scan_debug" (timing experiments only: results are
 * invalid while set).  Every option changes scheduling or tuning only; results
 * stay bit-identical. */
int tri_set_option(const char* name, int64_t value);

/* Vector store: replaces ann_graph.VectorStore (ann_graph.py:21-48).
 * x is n x d row-major float32 on the host; no float64 copy is kept. */
int tri_store_create(const float* x, int64_t n, int32_t d, int32_t device, tri_store** out);
int tri_store_destroy(tri_store* s);
int tri_store_info(const tri_store* s, int64_t* n, int32_t* d, double* max_norm);
/* Global id of row 0 (shards of a larger database). */
int tri_store_set_id_offset(tri_store* s, int64_t id_offset);

/* Exact kNN: replaces ann_graph.brute_force_knn (ann_graph.py:124-137),
 * batched with a per-query k.  q: B x d float64.  Outputs B x ldo, row i holds
 * k[i] results sorted by (dist, id). */
int tri_knn_bruteforce(tri_store* s, const double* q, int32_t B, const int32_t* k, int32_t ldo, int64_t* ids,
                       double* dists, void* stream);
int tri_knn_bruteforce_dev(tri_store* s, const double* q, int32_t B, const int32_t* k, int32_t ldo, int64_t* ids,
                           double* dists, void* stream);

/* Row distances: replaces ann_graph.rowwise_sq_dists (ann_graph.py:97-105)
 * for the rows of the store named by `rows` (host buffers). */
int tri_rowwise_sq_dists(tri_store* s, const double* q, const int64_t* rows, int64_t n, double* out, void* stream);

/* rowwise_sq_dists on arbitrary float64 rows (ann_graph.py:97-105), host
 * buffers: q is 1 x d (broadcast) or n x d (row i paired with query i, numpy
 * broadcasting), rows n x d float64; same operation order, computed on
 * `device`.  Used when the rows do not come from a float32 store. */
int tri_rowwise_sq_dists_f64(const double* q, int32_t q_rows, const double* rows, int64_t n, int32_t d, int32_t device,
                             double* out);

/* Fixed-shape distance batch: replaces engine.execute_distance_batch
 * (engine.py:229-256).  Task i pairs query row owner[i] of `queries`
 * (n_queries x d float64) with store row cand[i]; returns TRI_EINTERNAL if a
 * candidate is out of range (engine.py:249-250).  Host buffers. */
int tri_distance_tasks(tri_store* s, const int32_t* owner, const int64_t* cand, int32_t n_tasks,
                       const double* queries, int32_t n_queries, double* out, void* stream);

/* IVF-Flat (new component; the reference has no IVF).
 * train: GPU Lloyd k-means from the host-chosen init rows, `iters` updates
 * (exact assignment, float64 ascending-id centroid sums: deterministic).
 * create: from a shared artifact (fp32 centroids + the list id of each row),
 * `id_offset` = global id of the store's row 0 (shards). */
int tri_ivf_train(tri_store* s, int32_t nlist, int32_t iters, const int64_t* init_rows, tri_ivf** out);
/* Exact nearest-centroid assignment of every store row (host centroids
 * nlist x d float32 -> host assign[n]): brute_force_knn over the centroids
 * with k = 1 (ann_graph.py:124-137), ties to the smaller centroid id.  It is
 * also the assignment step of tri_ivf_train, whose Lloyd update sums each
 * list's rows in ascending id order in float64 -- so training is
 * deterministic and reproducible on the CPU (oracle.kmeans). */
int tri_kmeans_assign(tri_store* s, const float* centroids, int32_t nlist, int32_t* assign);
int tri_ivf_create(tri_store* s, const float* centroids, int32_t nlist, const int32_t* assign, int64_t id_offset,
                   tri_ivf** out);
int tri_ivf_destroy(tri_ivf* v);
int tri_ivf_info(const tri_ivf* v, int32_t* nlist, int64_t* n, int32_t* d);
/* centroids: nlist x d float32; assign: n int32 (either may be NULL). */
int tri_ivf_export(tri_ivf* v, float* centroids, int32_t* assign);
int tri_ivf_list_sizes(tri_ivf* v, int64_t* sizes);

/* Ragged batched IVF search: query i wants k[i] results over its nprobe[i]
 * closest lists (coarse step = exact kNN over the centroids).  This is the
 * continuous-batch entry: prefill (large k / nprobe) and decode (small)
 * queries share one launch sequence.  Outputs B x ldo; entries past the
 * results (probed lists hold fewer than k[i] vectors, or columns >= k[i]) are
 * id -1 / distance +inf. */
int tri_ivf_search(tri_ivf* v, const double* q, int32_t B, const int32_t* k, const int32_t* nprobe, int32_t ldo,
                   int64_t* ids, double* dists, void* stream);
int tri_ivf_search_dev(tri_ivf* v, const double* q, int32_t B, const int32_t* k, const int32_t* nprobe,
                       int32_t ldo, int64_t* ids, double* dists, void* stream);
/* Probed list ids of the last search (B x ld, host), for inspection: the
 * exact top-nprobe SET of centroids by (dist, id) (brute_force_knn over the
 * centroids, ann_graph.py:124-137).  The fine step scans their union, so with
 * option coarse_set (default) the set comes in approximate-distance order;
 * coarse_set = 0 returns the exact (dist, id) order. */
int tri_ivf_last_probes(tri_ivf* v, int64_t* probes, int32_t ld);
/* Queries of the last search that needed the exact fix-up (host int). */
int tri_ivf_last_fixups(tri_ivf* v, int32_t* n);
int tri_store_last_fixups(tri_store* s, int32_t* n);
/* Profiling: when enabled, CUDA events bracket every pipeline stage of each
 * search (read back lazily, no synchronisation inside a timed loop).
 * scan_time: accumulated list-scan kernel time and number of searches;
 * stage_times: ms[6] = coarse step, packer, list scan, merge, exact re-rank,
 * certified fix-up. */
int tri_ivf_set_profiling(tri_ivf* v, int32_t on);
int tri_ivf_scan_time(tri_ivf* v, double* total_ms, int32_t* launches);
int tri_ivf_stage_times(tri_ivf* v, double* ms, int32_t* searches);
/* Algorithmic bytes of the last search's list scan: every probed list read
 * once (d*4 + 4 bytes per vector).  Also returns the number of scanned
 * (query, vector) pairs. */
int tri_ivf_last_scan_bytes(tri_ivf* v, int64_t* bytes, int64_t* pairs);

/* Arithmetic of the last search's list scan: 2 = fp16 tensor-core
 * candidates (certified), 1 = fp32/TF32 candidates, 0 = no search yet. */
int tri_ivf_last_scan_kind(tri_ivf* v, int32_t* kind);

/* Device-resident continuous-batching graph search: replaces
 * engine.ContinuousBatchEngine (engine.py:312-422).  adjacency: n x degree
 * uint32 (NeighborGraph, ann_graph.py:51-70); the config mirrors EngineConfig
 * (engine.py:39-66; m <= 4096, p * degree <= 8192).  Requests are seeded,
 * extended, merged and finalized on the device with the reference's exact
 * float64 distances; results and batch accounting are bit-identical. */
typedef struct tri_engine tri_engine;
int tri_engine_create(tri_store* s, const uint32_t* adjacency, int32_t degree, int32_t m, int32_t p,
                      int32_t entry_count, int32_t batch_capacity, int32_t stop_streak, int32_t max_extends,
                      tri_engine** out);
int tri_engine_destroy(tri_engine* e);
/* ContinuousBatchEngine.submit (engine.py:337-345): q is one float64 row of
 * the store's dimension; queued until the next step admits it. */
int tri_engine_submit(tri_engine* e, const double* q, int32_t k, int64_t* rid);
/* Batched submit (B rows, per-request k); same validation, all or nothing. */
int tri_engine_submit_batch(tri_engine* e, const double* q, int32_t B, const int32_t* k, int64_t* rids);
/* Accumulated device time of the step launches (CUDA events) and steps run. */
int tri_engine_device_time(tri_engine* e, double* ms, int64_t* steps);
/* active_count / pending_admissions (engine.py:347-353). */
int tri_engine_counts(tri_engine* e, int32_t* active, int32_t* pending);
/* One active request's state (white-box; synchronises the engine stream):
 * found = 0 if rid is not active.  top_d / top_i / top_e (capacity m) get the
 * top-M list in (dist, id) order with expanded flags, visited (capacity
 * ceil(n / 32) words) the visited bitmap (bit i of word i / 32 = row i);
 * any output may be NULL.  Replaces reading ContinuousBatchEngine._active
 * (engine.py:330, SearchRequestState engine.py:70-83). */
int tri_engine_request_state(tri_engine* e, int64_t rid, int32_t* found, int32_t* n_top, double* top_d,
                             int32_t* top_i, uint8_t* top_e, uint32_t* visited, int32_t* extends, int32_t* streak);
/* Up to max_steps steps (engine.py:369-411); step 0 admits the pending
 * requests.  until_idle != 0 stops after the first step that leaves no
 * active request (run_to_completion, engine.py:413-422).  Per-step outputs
 * (arrays of max_steps, may be NULL): total emissions (batch accounting:
 * ceil(E / batch_capacity) batches), admissions, retirements. */
int tri_engine_run(tri_engine* e, int32_t max_steps, int32_t until_idle, int32_t* steps_done,
                   int64_t* emissions, int32_t* admitted, int32_t* retired);
/* Drain up to cap retired results (retirement order: step, then request id):
 * request id, extends, k, step index of the run, and k ids / float64
 * distances per row (row stride ld). */
int tri_engine_retired(tri_engine* e, int32_t cap, int32_t ld, int32_t* n, int64_t* rids, int32_t* extends,
                       int32_t* ks, int32_t* steps, int64_t* ids, double* dists);
/* Same results scattered by request id into caller arrays indexed [rid]
 * (rows of ld for ids/dists; capacity = rows available): the form a
 * long-lived server keeps.  rids (optional, length = retired count) lists the
 * drained ids in retirement order. */
int tri_engine_retired_by_id(tri_engine* e, int64_t capacity, int32_t ld, int32_t* n, int64_t* rids, int32_t* ids,
                             double* dists, int32_t* extends, int32_t* ks);
int tri_engine_pending_retired(tri_engine* e, int32_t* n);

/* Test hooks for the certificate.  debug_bound: the error
 * model constants cdot, csum of |D~ - D| <= cdot 2|q||x| + csum (|q| + |x|)^2
 * for a scan arithmetic (0 fp32 SIMT, 1 TF32, 2 fp16, 3 split fp16 coarse).
 * ivf_debug_keys: the last search's candidate keys ((fp32 order bits of D~)
 * << 32 | row position), which = 0 the fine partial lists (layout[3 i ..] =
 * part_off, kp, slots of query i; slot j holds probe j's list), which = 1 the
 * coarse step's merged lists (layout[0] = row stride).  keys may be NULL to
 * query the size. */
int tri_debug_bound(int32_t d, int32_t mode, double* cdot, double* csum);
int tri_ivf_debug_keys(tri_ivf* v, int32_t which, uint64_t* keys, int64_t cap, int64_t* n, int64_t* layout);
/* Timeline probe of the tensor-core scan (option scan_debug & 8): per CTA
 * (up to 256) eight globaltimer stamps: entry, setup done, first item
 * published, first query tile staged, first chunk's MMAs issued, first chunk
 * read by the epilogue, last TMA issued, epilogue done.  Synchronises the device.
 * n = 4 instead reads and resets the scan_debug & 16 selection counters. */
int tri_debug_scan_ts(uint64_t* out, int32_t n);

/* Exact merge of G per-shard result lists (device buffers, G x B x k_in,
 * id -1 = empty) into the global top-k_out by (dist, id). */
int tri_merge_topk(const double* dists, const int64_t* ids, int32_t G, int32_t B, int32_t k_in, int32_t k_out,
                   double* out_dists, int64_t* out_ids, void* stream);
/* Strided form for packed shard results: element (g, b, j) of the input lists
 * is at [g * g_stride + b * ld_in + j], output row b at [b * ld_out].  A rank
 * that writes its top-k ids and then its dists into ONE [2, B, k] block (ids
 * at p, dists at p + B*k, ldo = k) gathers a single tensor per batch and the
 * merge reads the gathered [G, 2, B, k] in place (output columns [k_out, ld_out)
 * get id -1 / +inf): ids = p, dists = p + B*k,
 * ld_in = k, g_stride = 2*B*k.  The per-shard merge SURVEY.md 8(e) adds (the
 * reference has none); tie rule of ann_graph.py:136. */
int tri_merge_topk_ld(const double* dists, const int64_t* ids, int32_t G, int32_t B, int32_t k_in, int32_t ld_in,
                      int64_t g_stride, int32_t k_out, double* out_dists, int64_t* out_ids, int32_t ld_out,
                      void* stream);

/* Native sharded search over NCCL (C4; the reference has no sharding,
 * SPEC.md:536, and SURVEY.md 8(b) asks for tri_comm_init).  NCCL is loaded at
 * run time (libnccl.so.2).  Rank 0 makes a 128-byte unique id, the caller
 * distributes it (e.g. a torch.distributed broadcast), every rank calls
 * tri_comm_init with it.  tri_ivf_search_sharded then runs one batch on
 * `stream`: the rank's local search (global ids, shard offset folded in) into
 * a packed [2, B, k] block, one ncclAllGather of B*k*16 bytes per rank, and
 * the exact (dist, id) merge into ids / dists (device, row stride ldo) on every
 * rank.  Stream-ordered and CUDA-graph capturable; one communicator per
 * concurrently used stream is the caller's choice (collectives on one
 * communicator must be issued in the same order on every rank). */
typedef struct tri_comm tri_comm;
int tri_comm_unique_id(uint8_t* id128);
int tri_comm_init(const uint8_t* id128, int32_t world, int32_t rank, int32_t device, tri_comm** out);
int tri_comm_destroy(tri_comm* c);
int tri_ivf_search_sharded(tri_ivf* v, tri_comm* c, const double* q, int32_t B, int32_t k, const int32_t* nprobe,
                           int32_t ldo, int64_t* ids, double* dists, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TRINITY_B200_H */
