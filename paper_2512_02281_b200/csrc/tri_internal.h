// Internal host/device interface of libtrinity_b200 (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace tri {

// Hot-path kernels launch with programmatic stream serialization (option
// "pdl", default off: measured no gain): the launch of kernel N+1 may overlap the tail of kernel N;
// every such kernel starts with pdl_wait() (tri_common.cuh).
extern long long g_pdl;
template <typename... P, typename... A>
inline cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

// One unit of scan work: a contiguous row range of a (list-major) vector
// matrix scanned against a group of <= gmax queries that share a candidate
// capacity kp.  Produced on the host for brute force, on the device (the
// continuous-batch packer) for IVF.
struct WorkItem {
  long long row_begin;
  int row_count;
  int member_begin;
  int member_count;
  int kp;
  int pad0, pad1;
};

// A (query, partial-list slot) pair; slot is a key offset into the partial buffer.
struct Member {
  int q;
  int pad;  // the query's kp (tensor-core scan: per-member threshold / output size)
  long long slot;
};

// Per-query plan metadata.
struct QueryMeta {
  int k;           // results wanted
  int kp;          // candidate capacity (power of two >= over-fetch(k))
  int n_slots;     // partial lists to merge
  int cls;         // capacity class index (log2(kp) - 5)
  long long part_off;  // first key of this query's partial lists
  long long n_total;   // candidates the query scans (all rows / probed-list rows)
};

constexpr int kNumCls = 7;    // kp in {32 .. 2048}
constexpr int kMinKp = 32;
constexpr int kMaxKp = 2048;

struct ScanLaunch {
  const void* tmap;     // CUtensorMap over X: 64-row x 16-float boxes, 64B swizzle (SIMT scan)
  const void* tmap_tc;  // CUtensorMap over X (fp32 or the fp16 copy): box_rows x 128-byte boxes, 128B swizzle
  const void* tmap_tc_tail;  // same tensor, 32-row boxes (partial last chunk of a work item)
  const float* X;
  long long ldx;
  const float* xnorm;
  const float* Q;
  int qld;
  const float* qnorm;
  const WorkItem* items;
  const int* n_items;
  int* counter;
  const Member* members;
  unsigned long long* part;
  int dp;
  int gmax;
  int cap;      // selection buffer per query (>= 2 * max kp, power of two)
  int grid;
  int dbg;      // experiment switches (0 in production): 1 skip selection, 2 skip MMA
  // fp16 tensor-core scan (f16 != 0): tmap_tc maps the fp16 copy of X, queries
  // come from Qh (row stride qldh halves) and dots are scaled by qinv[query].
  int f16;
  int stages;   // tensor-core scan: shared-memory ring depth (tc_scan_stages)
  int box_rows; // tensor-core scan: rows per TMA box of tmap_tc (32, 64 or 128; full chunks)
  const void* Qh;
  int qldh;
  const float* qinv;
  // per-query cross-item threshold (B keys, TRI_KEY_MAX at start; nullptr =
  // off): the tensor-core scan publishes each full partial list's kp-th key
  // with atomicMin and filters against the smallest one seen
  unsigned long long* gthr;
  int qbufs;  // tensor-core scan: query tiles (2 = next item staged during this one; 1 frees a ring stage)
  int abufs;  // tensor-core scan: append-list buffers (2 = one barrier per chunk; 1 = two barriers, frees a ring stage)
  int l2hint;  // tensor-core scan TMA loads: 0 default, 1 L2 evict_first, 2 L2 evict_last
  int nq;      // tensor-core scan query-group width (MMA N): kTcGroup or kTcGroupWide
  // brute force (nq = kTcGroupWide): items of consecutive queries load their
  // query tile with TMA through tmap_q (a CUtensorMap over Q: 32-float x 64-row
  // SW128 boxes); seed = 1 runs the seed pass (items <= kTcWideMaxChunks chunks)
  int q_tma;
  const void* tmap_q;
  int seed;            // 1: per-item seed; 2: cross-item seed (one item per CTA, seed_items <= kTcSeedItems)
  int early;           // launched as a programmatic dependent of the prep kernel: the row producer streams
                       // before the prep's results are visible (fixed item assignment only), the other roles wait
  uint32_t* seed_min;  // seed 2: B x seed_items fp32 order bits of each item's smallest distance (0xff.. = none)
  int* seed_ctr;       // seed 2: items that published (zeroed before the launch)
  int seed_items;
  // seed 2: each item appends at most kp survivors per query, unsorted, at the
  // front of the query's partial region (part + meta part_off), counted here
  // (B ints, zeroed before the launch); merged by launch_merge_compact
  int* compact_cnt;
  // list scan, wide members (kp >= 128): at the end of each item the member's
  // 32 smallest keys join the query's pool (pool + q * pool_cap), and the
  // kp-th smallest key in the pool tightens the query's cross-item bound gthr
  unsigned long long* pool;  // B x pool_cap keys, all ones = empty
  int* pool_cnt;             // B: slots reserved so far
  int pool_cap;              // multiple of 32, <= kPoolMax
  int pool_pub;              // 1: item ends publish; 2: first chunks too
  int pool_minkp;            // members with kp >= this use the pool
  const QueryMeta* meta;
};
constexpr int kTcSeedItems = 160;
constexpr int kTcWideMaxChunks = 8;  // 8 x 64 TMEM columns: a wide item's every chunk stays resident

size_t scan_smem_bytes(int gmax, int qld, int cap);
int scan_gmax(int qld, int cap, int smem_limit);
cudaError_t launch_scan(const ScanLaunch& s, cudaStream_t st);

// tensor-core scan (tri_tcscan.cu): fixed groups of 16 queries, qld <= kTcMaxQld
constexpr int kTcMaxQld = 1024;
constexpr int kTcGroup = 16;
constexpr int kTcGroupWide = 64;   // brute force: one row pass per 64 queries (MMA N = 64)
constexpr int kTcWideMaxKp = 64;   // ... with register lists of at most 64 keys
constexpr int kTcMaxKp = 256;  // register-resident top-kp lists in the epilogue
constexpr int kTcMinStages = 4;
// minimum (kTcMinStages ring) shared memory; row_bytes = qld*4 or qldh*2, nq = query-group width
size_t tc_scan_smem_bytes(int row_bytes, int nq);
// deepest ring that fits (want > 0 caps it)
int tc_scan_stages(int row_bytes, int smem_limit, int want, int qbufs, int abufs, int nq);
cudaError_t launch_scan_tc(const ScanLaunch& s, cudaStream_t st);
cudaError_t read_scan_ts(unsigned long long* out, int n);  // dbg & 8 timeline stamps (256 CTAs x 8)

// Up to six 32-bit fills the prep kernel performs on the side (the search's
// counters and seed buffers), replacing one cudaMemsetAsync each.
struct ClearList {
  static constexpr int kMax = 6;
  void* p[kMax];
  long long words[kMax];
  uint32_t val[kMax];
  int n;
  void add(void* ptr, long long w, uint32_t v) {
    p[n] = ptr;
    words[n] = w;
    val[n] = v;
    ++n;
  }
};
// fp64 queries -> fp32 rows + norms; with Qh != nullptr also the fp16 scan
// copy (scale sx of the index's fp16 rows) in the same kernel.
cudaError_t launch_prep(const double* q64, int B, int d, float* Q32, int qld, float* qn32, double* qn64,
                        int* bad, cudaStream_t st, float sx = 1.f, void* Qh = nullptr, int ldh = 0,
                        float* qinv = nullptr, void* Ql = nullptr, const ClearList* clears = nullptr);
cudaError_t launch_absmax(const float* X, long long n, int d, long long ldx, unsigned int* bits, cudaStream_t st);
cudaError_t launch_to_half(const float* X, long long n, int d, long long ldx, float sx, void* Xh, int ldh,
                           cudaStream_t st);
cudaError_t launch_prep_half(const float* Q32, int B, int qld, int d, float sx, void* Qh, int ldh, float* qinv,
                             cudaStream_t st);
cudaError_t launch_norms(const float* X, long long n, int d, long long ldx, float* xnorm,
                         unsigned long long* xmax_bits, cudaStream_t st);

// dense small-store brute force (tri_dense.cu): distances to D (B x ldd fp32),
// then per-query top-kp (kp <= kDenseMaxKp) straight into `merged`.
constexpr long long kDenseMaxN = 4096;
constexpr int kDenseMaxKp = 256;
constexpr int kDenseSlices = 16;  // max split-K slices of the distance GEMM (D holds up to this many B x ldd partials)
extern int g_dense_slices;       // slices used (option "dense_slices", <= kDenseSlices)
cudaError_t launch_dense(const float* Q, int qld, const float* qn, int B, const float* X, long long ldx,
                         const float* xn, long long n, int dp, float* D, long long ldd, const QueryMeta* meta,
                         unsigned long long* merged, int ld_merged, int kp_max, cudaStream_t st);

// tensor-core coarse GEMM (tri_coarse.cu): split-fp16 operands, K-split
// TMEM accumulators; writes the fp32 dot of every (query, centroid) to P.
struct CoarseLaunch {
  const void* map_h;  // CUtensorMap over the centroids' fp16 hi copy (64-half x 128-row SW128 boxes)
  const void* map_l;  // ... and the lo copy
  const void* Qh;     // B x ldq fp16 hi of the scaled queries (prep)
  const void* Ql;     // ... lo
  int ldq;            // halves per query row (multiple of 64)
  const float* qinv;  // 1 / (s_q * s_list) per query (< 0: unscalable)
  float ratio;        // s_list / s_centroid (power of two): qinv * ratio = 1 / (s_q * s_centroid)
  int B;
  long long n;        // centroids
  int nslab;          // ldq / 64
  float* P;           // coarse_tc_slices(nslab) x B x ldd partial dots (split-K)
  long long ldd;
  int slab_cap;       // set by launch_coarse_tc
  int tmem_cols;      // set by launch_coarse_tc
};
extern int g_coarse_split;
int coarse_tc_slices(int nslab);
size_t coarse_tc_smem(int slab_cap);
cudaError_t launch_coarse_tc(const CoarseLaunch& a, cudaStream_t st);
cudaError_t launch_to_half_lo(const float* X, long long n, int d, long long ldx, float sx, void* Xl, int ldh,
                              cudaStream_t st);

// per-query top-kp of nsl summed dot slices (D: nsl x B x ldd fp32)
extern long long g_dense_fold;  // dense select: warp-list folds (1) or bisection (0)
cudaError_t launch_dense_select(const float* D, int nsl, long long ldd, int B, const float* qn, const float* xn,
                                long long n, const QueryMeta* meta, unsigned long long* merged, int ld_merged,
                                int kp_max, cudaStream_t st);

cudaError_t launch_merge(const unsigned long long* part, const QueryMeta* meta, unsigned long long* merged,
                         int ld_merged, int B, int kp_max, cudaStream_t st);
// cnt[q] unsorted keys at part + meta[q].part_off (ScanLaunch::compact_cnt)
cudaError_t launch_merge_compact(const unsigned long long* part, const int* cnt, const QueryMeta* meta,
                                 unsigned long long* merged, int ld_merged, int B, int kp_max, cudaStream_t st);

struct Exact;

struct RerankLaunch {
  const unsigned long long* merged;
  Exact* exact;             // B x ld_merged scratch
  int ld_merged;
  const QueryMeta* meta;
  const double* q64;
  int d;
  const double* qn64;
  const float* X;
  long long ldx;
  const long long* idmap;   // position -> id (nullptr: id = position)
  long long id_offset;
  double xmax;              // max row norm (sqrt of squared norm)
  double cdot;              // |approx - exact| <= cdot*2|q||x| + csum*(|q|+|x|)^2
  double csum;
  long long* out_ids;
  double* out_d;
  int ldo;
  int* n_flag;
  int* flag_list;
  unsigned long long* fx_thr;  // per flagged query: the fix-up's exact k-th bound (set to +inf when flagged)
  int skip_far;                // fused re-rank: skip candidates 2E above the k-th approx key (option "rerank_skip")
  int B;
  int kp_max;
  int lpt;                  // fused re-rank: CTAs take queries in descending capacity class (wide lists first)
  int lpt_cls;              // fused re-rank split: 0 = every class, 1 = class 0 only (kp 32), 2 = classes >= 1
  const float* qinv;        // fp16 scan: qinv[q] < 0 marks a query the scan could not scale (never certified)
  // brute force with a cross-item seed: the scan's unsorted compact lists
  // (cnt[q] keys at part + part_off); the re-rank merges them itself
  const unsigned long long* part;
  const int* compact_cnt;
  const float* xnorm;  // squared row norms of X (coarse_set_kernel's per-candidate bound)
};
cudaError_t launch_rerank(const RerankLaunch& r, cudaStream_t st);
// IVF coarse step, set semantics: exact distances only for candidates whose top-k
// membership the error bound leaves open (tri_select.cu coarse_set_kernel).
cudaError_t launch_coarse_set(const RerankLaunch& r, cudaStream_t st);
extern long long g_rerank_smem_cap;  // bytes; 0 = no cap
extern long long g_rerank_f2f;
extern long long g_rerank_skip;
extern long long g_rerank_wide_slab;
extern long long g_rerank_split;
extern long long g_merge_split;
extern long long g_rerank_lpt;  // kp >= 128: ring up to the SM's shared memory
extern long long g_fx_slice_rows;  // fix-up: minimum rows per slice       // 1: hardware F2F conversions in the re-rank (else integer bit moves)

struct FixupLaunch {
  const int* n_flag;
  const int* flag_list;
  const QueryMeta* meta;
  const double* q64;
  int d;
  const float* X;
  long long ldx;
  long long n_rows;             // brute-force mode: rows [0, n_rows)
  const long long* probes;      // IVF mode: probed list ids (nullptr = brute force)
  int ld_probes;
  const int* nprobe;            // per-query probe count (IVF mode)
  const long long* list_off;    // IVF list offsets (nlist + 1)
  const long long* idmap;
  long long id_offset;
  long long* out_ids;
  double* out_d;
  int ldo;
  int B;
  int k_max;
  Exact* scratch;  // per-(flagged query, slice) partial top-k (fixup_part_bytes(B, k_max) from fixup_scratch)
  unsigned long long* fx_thr;  // per flagged query: smallest slice k-th exact distance (double bits)
  int* fx_cnt;                 // per (flagged query, slice): entries in its partial list
  int max_units;               // partial lists the scratch holds (slices x flagged queries)
  int slice_rows;              // minimum rows per slice (option "fx_slice_rows")
  // fp32 pre-filter: a row's exact distance is computed only when its fp32
  // distance (the SIMT scan's arithmetic) is within 4x the SIMT error bound of
  // the current fix-up bound
  const float* Q32;
  int qld;
  const float* qn32;
  const double* qn64;
  const float* xnorm;  // norms of the rows of X
  double xmax;
  double cdot, csum;   // bound_for(d, kSimt)
};
// Fix-up scratch: fx_thr (B x 8 bytes), fx_cnt (max_units ints), each
// 256-aligned, then the partial lists.
size_t fixup_scratch_bytes(int B, int k_max);
size_t fixup_thr_bytes(int B);
size_t fixup_cnt_bytes(int B, int k_max);
int fixup_max_units(int B, int k_max);
cudaError_t launch_fixup(const FixupLaunch& f, cudaStream_t st);

cudaError_t launch_distance_tasks(const int* owner, const long long* cand, int n_tasks, const double* q64, int d,
                                  const float* X, long long ldx, long long n_rows, double* out, int* err,
                                  cudaStream_t st);

cudaError_t launch_rowwise_f64(const double* q, long long q_stride, const double* X, long long n, int d, double* out,
                               cudaStream_t st);
cudaError_t launch_merge_exact(const double* dists, const long long* ids, int G, int B, int k_in, int k_out,
                               double* out_d, long long* out_ids, cudaStream_t st, int ld_in, int ld_out,
                               long long g_stride);

// IVF packer ------------------------------------------------------------------
struct PackLaunch {
  const long long* probes;
  int ld_probes;
  const int* nprobe;
  QueryMeta* meta;
  int B;
  const long long* list_off;
  const int* list_by_size;   // lists in descending size order
  int nlist;
  int cls_mask;              // capacity classes present in the batch
  int* counts;               // nlist * kNumCls
  int* fill;                 // nlist * kNumCls
  int* member_base;          // nlist * kNumCls
  WorkItem* items;
  int* n_items;
  Member* members;
  int gmax;
  int mixed;  // 1: one group sequence per list for all capacity classes (item kp = members' max)
};
// Fixed-shape ragged batches (tri_ivf.cu): device-side plan of a padded batch.
struct RaggedPlan {
  const int* in;          // [B, unused, (k, nprobe) x Bc]
  int Bc;
  int f16, tc, f16_div, kp_extra;  // the host's over-fetch rule (kp_for / kp_for_f16)
  QueryMeta* meta;
  int* nprobe;
  long long* total_keys;  // sum of nprobe * kp
};
cudaError_t launch_ragged_plan(const RaggedPlan& r, cudaStream_t st);
cudaError_t launch_fill_keys(unsigned long long* p, const long long* count, int grid, cudaStream_t st);
cudaError_t launch_pad_rows(const double* src, double* dst, const int* nB, int Bc, int d, cudaStream_t st);
cudaError_t launch_pack(const PackLaunch& p, cudaStream_t st);

// k-means / index layout --------------------------------------------------------
cudaError_t launch_rows_to_f64(const float* X, long long ldx, long long n, int d, double* out, cudaStream_t st);
cudaError_t launch_narrow_ids(const long long* ids, long long n, int* out, cudaStream_t st);
cudaError_t launch_counts(const int* assign, long long n, int nlist, int* counts, cudaStream_t st);
cudaError_t launch_list_members(const int* assign, long long n, int nlist, const long long* offsets,
                                long long* perm, cudaStream_t st);
cudaError_t launch_centroid_update(const float* X, long long ldx, int d, const long long* perm,
                                   const long long* offsets, int nlist, float* C, long long ldc, cudaStream_t st);
cudaError_t launch_gather_rows(const float* X, long long ldx, const long long* perm, long long n, int dp,
                               float* out, cudaStream_t st);

// Engine support (tri_engine.cu): a read-only view of a store's device rows and
// the library's per-thread error slot.
struct StoreView {
  const float* X;
  long long ldx;
  long long n;
  int d;
  int device;
};

}  // namespace tri

struct tri_store;
namespace tri {
int store_view(const tri_store* s, StoreView* v);
// Exhaustive exact kNN for k > TRI_MAX_K (tri_exhaustive.cu): exact distances to
// every row + a stable radix sort by (dist, id); q64 is B x d on the device.
size_t exhaustive_scratch_bytes(long long n);
cudaError_t launch_exhaustive_knn(const StoreView& sv, long long id_offset, const double* q64, int B, const int* k,
                                  int ldo, long long* ids, double* dists, void* scratch, cudaStream_t st);
int set_error(int code, const char* fmt, ...);
}  // namespace tri
