// C-ABI of libtrinity_b200: handles, host-side planning and launch sequences.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/trinity_b200.h"
#include "tri_internal.h"

using namespace tri;

namespace {

thread_local std::string g_err;
long long g_force_fixup = 0;
long long g_kp_extra = 0;
constexpr int kSmemLimit = 226 * 1024;
constexpr int kProfSearches = 2048;  // profiled searches kept before read-back
constexpr int kStagesProf = 6;       // coarse, pack, scan, merge, rerank, fixup
constexpr int kSelCapMin = 512;  // >= one 512-row chunk of appends

int round16(int d) { return (d + 15) & ~15; }

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                          \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(TRI_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

#define TRY(expr)            \
  do {                       \
    int _rc = (expr);        \
    if (_rc != TRI_OK) return _rc; \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  long long* owner = nullptr;  // the owning workspace's epoch (nullptr: the global one)
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Bumped whenever a device scratch buffer moves or a cached plan is rewritten:
// captured CUDA graphs bake in pointers and plan contents, so any bump retires them.
long long g_epoch = 0;
// capture repeated search shapes into CUDA graphs (option "graphs"; the
// environment variable TRI_GRAPHS=0 turns it off at load, e.g. under ncu,
// whose kernel replay does not support the graphs' host-memory nodes)
long long g_graphs = [] {
  const char* e = std::getenv("TRI_GRAPHS");
  return (e && e[0] == '0') ? 0LL : 1LL;
}();

int ensure(DevBuf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return TRI_OK;
  if (b.p) {  // a pointer captured graphs may bake in goes away (a fresh allocation retires nothing)
    ++(b.owner ? *b.owner : g_epoch);
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.cap = 0;
  size_t want = std::max<size_t>(bytes + bytes / 4, 256);
  CU(cudaMalloc(&b.p, want));
  b.cap = want;
  return TRI_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
};

int ensure_host(HostBuf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return TRI_OK;
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = std::max<size_t>(bytes + bytes / 4, 256);
  CU(cudaMallocHost(&b.p, want));
  b.cap = want;
  return TRI_OK;
}

long long g_box_rows = 128;     // rows per TMA box of the tensor-core scan maps (fixed at index creation)
long long g_scan_reserve = -1;  // SMs the IVF list scan leaves to other streams (-1: scan_reserve_for)
long long g_tc_stages = 0;   // tensor-core scan ring depth cap (0 = as deep as shared memory allows)
long long g_scan_kernel = 0;  // 0 auto (IVF: fp16 tensor core), 1 fp32 SIMT, 2 TF32 tensor core
long long g_scan_l2hint = 1;  // L2 policy of the IVF tensor-core scan's row loads (option "scan_l2hint")
long long g_pack_mixed = 1;  // IVF tensor-core scan: one group sequence per list for all k classes (option "pack_mixed")
long long g_scan_debug = 0;   // timing experiments only (results invalid when set)
long long g_dense_off = 0;    // 1: never use the dense small-store brute force
long long g_gthr = 1;         // cross-item per-query threshold in the tensor-core scan
long long g_scan_abufs = 1;  // IVF tensor-core scan append-list buffers (option "scan_abufs": 1 or 2)
long long g_scan_qbufs = 2;   // tensor-core scan query tiles (option "scan_qbufs": 1 or 2)
long long g_coarse_tc = 1;    // IVF coarse GEMM on tensor cores (split fp16) when the index allows
long long g_bf_wide = 1;      // brute force: 64-query groups (one row pass per 64 queries) when kp <= 64
long long g_bf_seed = 2;      // ... with the TMEM seed pass (tri_tcscan.cu tc_seed_pass): 1 per item, 2 cross-item
long long g_bf_qtma = 1;      // ... and TMA-loaded query tiles
std::atomic<long long> g_gr_eager{0}, g_gr_captured{0}, g_gr_replayed{0};  // graph_run outcomes
long long g_ragged_graphs = 1;
long long g_scan_pool = 1024;  // list scan: pooled cross-item bound for kp >= 128 members, pool keys per query (option "scan_pool", 0 = off)
long long g_scan_pool_pub = 2;  // 1: each finished item adds its 32 best keys; 2: also its first chunk's 32 best, when folded (option "scan_pool_pub")
long long g_scan_pool_minkp = 128;  // ... for members with kp >= this (option "scan_pool_minkp")
long long g_scan_early = 1;  // wide brute force: scan launched as the prep's programmatic dependent (option "scan_early")
long long g_coarse_set = 1;  // IVF coarse step: exact distances only where top-nprobe membership is open  // ragged / odd-sized batches replay fixed-shape padded graphs (option "ragged_graphs")


// Candidate capacity: over-fetch so the certified re-rank almost never falls
// back.  TF32 candidates carry ~2^-9 relative dot error, so they over-fetch 2x.
int kp_for(int k, bool tc) {
  long long want = (long long)k + (tc ? std::max<long long>(16, k) : std::max<long long>(16, k / 4)) + g_kp_extra;
  int kp = kMinKp;
  while (kp < want) kp <<= 1;
  return kp;
}

// fp16 candidates carry half the TF32 dot error (2^-10 vs 2^-9 relative);
// over-fetch k + max(16, k / g_f16_div).  With the 2x certificate margin,
// k / 4 (kp 128 at k = 100) left 20 of 85 prefill queries per C3 batch
// uncertified; k / 2 (kp 256) certifies all (tools/margin_cost.py).
long long g_f16_div = 2;
int kp_for_f16(int k) {
  long long want = (long long)k + std::max<long long>(16, k / std::max<long long>(1, g_f16_div)) + g_kp_extra;
  int kp = kMinKp;
  while (kp < want) kp <<= 1;
  return kp;
}

// Dense small-store path: its select and re-rank take any capacity, so the
// over-fetch is rounded to 16 instead of a power of two (nprobe 32 -> 48).
long long g_dense_pow2 = 0;
int kp_dense(int k) {
  if (g_dense_pow2) return kp_for(k, false);
  const long long want = (long long)k + std::max<long long>(16, k / 4) + g_kp_extra;
  return (int)std::max<long long>(kMinKp, (want + 15) / 16 * 16);
}

int cls_of(int kp) {
  int c = 0;
  while ((kMinKp << c) < kp) ++c;
  return c;
}

int sm_count(int device) {
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

// Error model of the approximate candidate distance D~ = fl(qn + xn - 2 q.x)
// against the exact float64 D = |q64 - x|^2:
//   |D~ - D| <= cdot * 2|q||x| + csum * (|q| + |x|)^2
// csum = 6u covers query/norm rounding and the two fp32 additions (u = 2^-24);
// cdot bounds the relative dot-product error: gamma_d for an fp32 FMA chain,
// 2^-9 (both TF32 inputs truncated to 10 mantissa bits) + accumulation for
// tcgen05 kind::tf32.
struct Bound {
  double cdot, csum;
};
// Scan arithmetic -> certification constants:
//   kSimt  fp32 FFMA dot of fp32(q) and x                       cdot = gamma_d
//   kTf32  tensor-core TF32 (operands truncated to 10 bits)     cdot = 2^-9 + ...
//   kF16   tensor-core f16 on power-of-two scaled RN fp16 copies of fp32(q)
//          and x: conversion 2^-11 each (+2^-24 for q -> fp32), subnormal floor
//          2^-25 of a 2^14-scaled element on each side (<= 2^-38 sqrt(d)),
//          accumulation as for TF32; csum gains 2^-80 for an fp32 subnormal
//          product after the exact 1/(s_q s_x) rescale.
//   kSplit tensor-core coarse GEMM on split fp16 (hi + lo) copies of both
//          sides: residual of the split 3 x 2^-22 (+ 2^-24 query -> fp32),
//          subnormal floor, 96-product K slices accumulated in fp32 (2x the
//          RN bound, as for the scans) and the slices summed in fp32.
enum ScanMode { kSimt = 0, kTf32 = 1, kF16 = 2, kSplit = 3 };
// Safety factor on the tensor-core dot-error terms, in percent (option
// "bound_margin", default 200).  The model above is tight: constant vectors make every
// conversion / truncation error coherent and reach 0.71 of it on B200
// (tests/test_gpu_certificate.py), so the certificate carries a 2x margin
// over the worst case measured rather than relying on the hardware never
// doing worse than the analysis.
long long g_bound_margin = 200;
Bound bound_for(int d, int mode) {
  const double u = std::ldexp(1.0, -24);
  Bound b;
  b.csum = 6.0 * u;
  const double acc = 2.0 * d * std::ldexp(1.0, -23);
  if (mode == kTf32) {
    b.cdot = std::ldexp(1.0, -9) + std::ldexp(1.0, -19) + acc;
  } else if (mode == kSplit) {
    const int nacc = 2 * ((d + 63) / 64);
    b.cdot = 3 * std::ldexp(1.0, -22) * (1.0 + std::ldexp(1.0, -10)) + u +
             2.0 * 96 * std::ldexp(1.0, -23) * (1.0 + std::ldexp(1.0, -9)) + nacc * std::ldexp(1.0, -23) +
             std::ldexp(1.0, -36) * std::sqrt((double)d);
    b.csum += std::ldexp(1.0, -80);
  } else if (mode == kF16) {
    const double u16 = std::ldexp(1.0, -11);
    b.cdot = 2 * u16 + u + 3 * u16 * u16 + acc * (1.0 + 4 * u16) + std::ldexp(1.0, -37) * std::sqrt((double)d);
    b.csum += std::ldexp(1.0, -80);
  } else {
    b.cdot = d * u / (1.0 - d * u);
  }
  if (mode != kSimt) b.cdot *= (double)std::max<long long>(100, g_bound_margin) / 100.0;
  return b;
}

int sel_cap(int kp_max) { return std::max(kSelCapMin, 2 * kp_max); }

// 2-D TMA descriptors over a row-major fp32 matrix (rows x ldx floats):
//   SIMT scan : 64-row x 16-float boxes, 64-byte swizzle
//   TC scan   : 32-row x 32-float boxes, 128-byte swizzle (UMMA K-major SW128)
int make_tmap(CUtensorMap* map, const void* X, long long rows, int ldx, bool tc, bool f16 = false, int box_rows = 32) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    void* fn = nullptr;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
    if (!fn || qr != cudaDriverEntryPointSuccess) return fail(TRI_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const size_t esz = f16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)ldx, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * esz};
  cuuint32_t box[2] = {tc ? (cuuint32_t)(128 / esz) : 16u, tc ? (cuuint32_t)box_rows : 64u};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                      const_cast<void*>(X), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, tc ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TRI_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TRI_OK;
}

// Scan kernel choice for a row width: the tensor-core scan unless forced off
// or the queries do not fit its shared-memory layout.
bool use_tc(int qld, int kp_max_tc) {
  if (g_scan_kernel == 1) return false;
  return kp_max_tc <= kTcMaxKp && qld <= kTcMaxQld && tc_scan_smem_bytes(qld * 4, kTcGroup) <= (size_t)kSmemLimit;
}

// Per-search scratch shared by the brute-force and IVF pipelines.  One
// Workspace per stream ("lane", see Lanes): searches issued on different
// streams never share scratch, so they can overlap on the device.
struct Workspace {
  static constexpr int kStaging = 4;  // pinned host staging ring depth
  // Bumped when one of THIS workspace's buffers moves or a plan of it is
  // dropped: only graphs that use this workspace retire (graph_run).
  long long epoch = 0;
  DevBuf q64, Q32, qn32, qn64, flags, plan, part, merged, exact, out_ids, out_d;
  // IVF per-search buffers
  DevBuf probes, probe_d, counts, fill, mbase, items, members, counters, meta;
  DevBuf Qh, qinv;  // fp16 scan: scaled fp16 queries + 1/(s_q s_x)
  DevBuf seedb;     // wide brute force: per (query, item) smallest distance (cross-item seed)
  DevBuf gthr;      // per-query cross-item scan threshold
  DevBuf pool;      // list scan: per-query pools of finished items' best keys + counters
  DevBuf Ql;        // lo half of the split fp16 queries (tensor-core coarse GEMM)
  bool split_q = false;  // this search prepared Qh/Ql/qinv for the split coarse GEMM

  DevBuf fxs;       // fix-up partial lists
  // fixed-shape padded batches: uploaded plan input, device key total, padded
  // queries and results
  DevBuf rplan, rtot, qpad, pad_ids, pad_d;
  DevBuf exh;  // exhaustive large-k path: distance keys, rows, sort scratch
  int pad_real = -1;  // real queries of the last search when it ran padded (-1: not padded)
  HostBuf h_plan;
  HostBuf h_stage[kStaging];
  HostBuf h_bq, h_bids, h_bd;  // pinned copies of a host brute-force call's queries / results (graph replay)
  cudaEvent_t staged[kStaging] = {nullptr, nullptr, nullptr, nullptr};
  bool staged_live[kStaging] = {false, false, false, false};
  int stage_i = 0;
  cudaEvent_t done = nullptr;  // recorded after the last search issued on this lane
  bool done_live = false;
  // cached host plan (brute force)
  std::vector<int> plan_k;
  int plan_B = -1;
  long long plan_n = -1;
  int n_items = 0, grid = 0, gmax = 0, cap = 0, kp_max = 0, k_max = 0;
  int nq = kTcGroup;  // tensor-core scan query-group width of the plan
  int q_tma = 0;      // groups are runs of consecutive queries
  CUtensorMap qmap;   // over Q32 (wide brute-force groups), encoded per search
  long long plan_opts = -1;
  bool tc = false;
  bool dense = false;
  DevBuf dmat;
  size_t off_items = 0, off_members = 0, plan_bytes = 0;
  long long part_keys = 0;
  int last_fixups = 0;
  int last_B = 0, last_npmax = 0, last_f16 = 0;
  std::vector<int> last_np;
  // CUDA-graph capture of repeated search shapes (see graph_run)
  bool capturing = false;
  HostBuf* cap_host = nullptr;  // graph-owned pinned staging used while capturing
  cudaEvent_t* cap_ph = nullptr;  // profiling placeholders recorded as graph event nodes
  struct Graph {
    int mode = 0, B = 0, ldo = 0;
    std::vector<int> k, np;
    const void *q = nullptr, *ids = nullptr, *dists = nullptr;
    bool prof = false;
    long long opts = 0, epoch = -1;
    int state = 0;  // 1 seen once (next call captures), 2 graph ready, 3 capture failed (stay eager)
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    HostBuf host;
    cudaEvent_t ph[7] = {};
    cudaGraphNode_t evnode[7] = {};
    unsigned long long used = 0;
    int last_B = 0, last_npmax = 0, last_f16 = 0;
    std::vector<int> last_np;
    void destroy() {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      if (graph) cudaGraphDestroy(graph);
      graph = nullptr;
      if (host.p) cudaFreeHost(host.p);
      host.p = nullptr;
      host.cap = 0;
      for (auto& e : ph)
        if (e) {
          cudaEventDestroy(e);
          e = nullptr;
        }
    }
  };
  std::vector<Graph> graphs;
  unsigned long long graph_clock = 0;
  // brute-force plans not currently active (see plan_bruteforce): each keeps
  // its own device buffer, so graphs captured against it stay valid
  struct Plan {
    DevBuf plan;
    size_t plan_bytes = 0, off_items = 0, off_members = 0;
    int plan_B = -1;
    long long plan_n = -1, plan_opts = -1, part_keys = 0;
    std::vector<int> plan_k;
    bool dense = false, tc = false;
    int n_items = 0, grid = 0, gmax = 0, cap = 0, kp_max = 0, k_max = 0, nq = kTcGroup, q_tma = 0;
    unsigned long long used = 0;
  };
  std::vector<Plan> plan_cache;
  unsigned long long plan_clock = 0;
  void plan_out(Plan& p) const {
    p.plan = plan;
    p.plan_bytes = plan_bytes;
    p.off_items = off_items;
    p.off_members = off_members;
    p.plan_B = plan_B;
    p.plan_n = plan_n;
    p.plan_opts = plan_opts;
    p.part_keys = part_keys;
    p.plan_k = plan_k;
    p.dense = dense;
    p.tc = tc;
    p.n_items = n_items;
    p.grid = grid;
    p.gmax = gmax;
    p.cap = cap;
    p.kp_max = kp_max;
    p.k_max = k_max;
    p.nq = nq;
    p.q_tma = q_tma;
  }
  void plan_in(const Plan& p) {
    plan = p.plan;
    plan_bytes = p.plan_bytes;
    off_items = p.off_items;
    off_members = p.off_members;
    plan_B = p.plan_B;
    plan_n = p.plan_n;
    plan_opts = p.plan_opts;
    part_keys = p.part_keys;
    plan_k = p.plan_k;
    dense = p.dense;
    tc = p.tc;
    n_items = p.n_items;
    grid = p.grid;
    gmax = p.gmax;
    cap = p.cap;
    kp_max = p.kp_max;
    k_max = p.k_max;
    nq = p.nq;
    q_tma = p.q_tma;
  }
  Workspace() {
    for (DevBuf* b : {&q64, &Q32, &qn32, &qn64, &flags, &plan, &part, &merged, &exact, &out_ids, &out_d, &dmat,
                      &probes, &probe_d, &counts, &fill, &mbase, &items, &members, &counters, &meta, &Qh, &qinv,
                      &gthr, &fxs, &Ql, &seedb, &rplan, &rtot, &qpad, &pad_ids, &pad_d, &exh})
      b->owner = &epoch;
  }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  void free_all() {
    for (auto& g : graphs) g.destroy();
    graphs.clear();
    for (auto& p : plan_cache)
      if (p.plan.p) cudaFree(p.plan.p);
    plan_cache.clear();
    for (DevBuf* b : {&q64, &Q32, &qn32, &qn64, &flags, &plan, &part, &merged, &exact, &out_ids, &out_d, &dmat,
                      &probes, &probe_d, &counts, &fill, &mbase, &items, &members, &counters, &meta, &Qh, &qinv,
                      &gthr, &fxs, &Ql, &seedb, &rplan, &rtot, &qpad, &pad_ids, &pad_d, &exh})
      release(*b);
    for (HostBuf* b : {&h_plan, &h_bq, &h_bids, &h_bd}) {
      if (b->p) cudaFreeHost(b->p);
      b->p = nullptr;
      b->cap = 0;
    }
    for (int i = 0; i < kStaging; ++i) {
      if (h_stage[i].p) cudaFreeHost(h_stage[i].p);
      h_stage[i].p = nullptr;
      if (staged[i]) cudaEventDestroy(staged[i]);
      staged[i] = nullptr;
    }
    if (done) cudaEventDestroy(done);
    done = nullptr;
  }
};

// Pinned host staging for an async upload: returns a slot of the lane's ring
// whose previous upload has completed (host waits only if the device is
// kStaging uploads behind).  Call staged_upload() after filling it.
int stage_host(Workspace& w, size_t bytes, int* slot, void** ptr) {
  if (w.capturing) {  // the graph replays this upload: it gets its own buffer
    if (!w.cap_host || w.cap_host->cap < bytes) return fail(TRI_EINTERNAL, "graph staging buffer too small");
    *slot = -1;
    *ptr = w.cap_host->p;
    return TRI_OK;
  }
  const int i = w.stage_i;
  w.stage_i = (w.stage_i + 1) % Workspace::kStaging;
  if (w.staged_live[i]) CU(cudaEventSynchronize(w.staged[i]));
  w.staged_live[i] = false;
  TRY(ensure_host(w.h_stage[i], bytes));
  *slot = i;
  *ptr = w.h_stage[i].p;
  return TRI_OK;
}

int staged_upload(Workspace& w, int slot, void* dst, size_t bytes, cudaStream_t st) {
  if (slot < 0) {
    CU(cudaMemcpyAsync(dst, w.cap_host->p, bytes, cudaMemcpyHostToDevice, st));
    return TRI_OK;
  }
  CU(cudaMemcpyAsync(dst, w.h_stage[slot].p, bytes, cudaMemcpyHostToDevice, st));
  if (!w.staged[slot]) CU(cudaEventCreateWithFlags(&w.staged[slot], cudaEventDisableTiming));
  CU(cudaEventRecord(w.staged[slot], st));
  w.staged_live[slot] = true;
  return TRI_OK;
}

// Stream -> Workspace map.  A new stream takes a free lane; with all lanes
// taken the least recently assigned one is recycled after its last search
// (its `done` event) has completed.
struct Lanes {
  static constexpr int kMax = 8;
  Workspace w[kMax];
  cudaStream_t st[kMax] = {};
  double t_get[kMax] = {};  // host time (s) of each lane's last search
  int used = 0, next_victim = 0, last = 0;
  static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  int get(cudaStream_t s, Workspace** out) {
    for (int i = 0; i < used; ++i)
      if (st[i] == s) {
        last = i;
        t_get[i] = now_s();
        *out = &w[i];
        return TRI_OK;
      }
    int i = used < kMax ? used++ : next_victim;
    if (i == next_victim && used == kMax) next_victim = (next_victim + 1) % kMax;
    if (w[i].done_live) CU(cudaEventSynchronize(w[i].done));
    w[i].done_live = false;
    st[i] = s;
    last = i;
    t_get[i] = now_s();
    *out = &w[i];
    return TRI_OK;
  }
  // another lane searched within the last `window` seconds
  bool others_active(cudaStream_t s, double window) const {
    const double t = now_s();
    for (int i = 0; i < used; ++i)
      if (st[i] != s && t - t_get[i] < window) return true;
    return false;
  }
  Workspace& recent() { return w[last]; }
  void free_all() {
    for (auto& x : w) x.free_all();
  }
};

int lane_done(Workspace& w, cudaStream_t st) {
  if (w.capturing) return TRI_OK;  // recorded after the graph launch instead
  if (!w.done) CU(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming));
  CU(cudaEventRecord(w.done, st));
  w.done_live = true;
  return TRI_OK;
}

}  // namespace

struct tri_store {
  int device = 0;
  int prefer_simt = 0;  // 1: fp32 SIMT scan (tight certification bound; IVF coarse step)
  long long n = 0;
  int d = 0, dp = 0, qld = 0;
  long long id_offset = 0;
  float* X = nullptr;
  float* xnorm = nullptr;
  double xmax = 0.0;
  CUtensorMap tmap, tmap_tc, tmap_tc_tail;
  int box_rows = 32;
  // split fp16 copies for the tensor-core coarse GEMM (IVF centroid stores)
  void* Ch = nullptr;
  void* Cl = nullptr;
  int dph = 0;
  float sc = 1.f;           // power-of-two scale of the split copies
  float split_ratio = 1.f;  // s_list / s_centroid (IVF centroid stores)
  CUtensorMap tmap_ch, tmap_cl;
  cudaStream_t own = nullptr;
  Lanes lanes;
  std::mutex mu;  // enqueue is serialised per handle; waits happen outside it
};

struct tri_ivf {
  int device = 0;
  long long n = 0;
  int d = 0, dp = 0, qld = 0, nlist = 0;
  long long id_offset = 0;
  float* Xl = nullptr;
  float* xnl = nullptr;
  long long* ids = nullptr;
  long long* list_off = nullptr;
  int* list_by_size = nullptr;
  int* assign = nullptr;  // per original row (store order)
  double xmax = 0.0;
  CUtensorMap tmap, tmap_tc, tmap_tc_tail;
  int box_rows = 32;
  // fp16 copy of the lists for candidate generation (null: TF32 / SIMT scans)
  void* Xh = nullptr;
  int dph = 0;       // row stride in halves (multiple of 64)
  float sx = 1.f;    // power-of-two scale of the fp16 copy
  CUtensorMap tmap_h, tmap_h_tail;
  std::vector<long long> h_off;
  tri_store* cstore = nullptr;  // centroids as a vector store (coarse step)
  cudaStream_t own = nullptr;
  Lanes lanes;
  std::mutex mu;  // enqueue is serialised per handle; waits happen outside it
  int reserve_now = 0;  // automatic scan reserve of the search being enqueued (set_reserve_now)
  bool prof = false;
  // profiling: a ring of (start, stop) event pairs around the list-scan kernel,
  // read back lazily so the timed loop never synchronises.
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;  // profiled searches with pending events (7 events each)
  double stage_ms[kStagesProf] = {0, 0, 0, 0, 0, 0};
  int prof_n = 0;
};

// SMs the IVF list scan leaves free: the option's value, or (-1, default)
// kAutoReserve once batches run on more than one stream of the index, so the
// other lanes' small kernels -- and the next lane's scan -- start beside the
// HBM-bound scan instead of in its tail.  The scan stays HBM-bound on 124 SMs,
// so consecutive lanes' scans overlap on all 148 (measured at 4 lanes, 100
// steps: 918K QPS with 8 SMs, 937-941K with 16, 946-949K with 24-28, 939K
// with 40-48; C3 631-640K -> 659-665K at 24).  One lane loses about 1% with
// any reservation, so it keeps every SM.
// "More than one stream" means another lane of the index enqueued a search
// within the last kActiveWindow seconds: a single-stream caller of an index
// that once served several lanes keeps every SM, while lanes that keep each
// other busy reserve from their first search on.  (Deciding by whether
// another lane's work is still in flight instead cost 7% at 20 bench steps:
// the first search after an idle moment took the whole GPU.)  Decided once
// per search (set_reserve_now, under the handle's lock), so the graph key and
// the captured grid agree.
constexpr int kAutoReserve = 24;
constexpr double kActiveWindow = 0.25;
void set_reserve_now(tri_ivf* v, cudaStream_t st) {
  v->reserve_now = (g_scan_reserve < 0 && v->lanes.used > 1 && v->lanes.others_active(st, kActiveWindow))
                       ? kAutoReserve : 0;
}
int scan_reserve_for(const tri_ivf* v) {
  if (g_scan_reserve >= 0) return (int)g_scan_reserve;
  return v->reserve_now;
}

namespace {

cudaStream_t pick(void* stream, cudaStream_t own) { return stream ? static_cast<cudaStream_t>(stream) : own; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Branch-free scan (vectorises): a double is non-finite iff its exponent bits
// are all ones (no per-element branch; about 25% faster on a C2 batch).
int check_queries(const double* q, long long count) {
  uint64_t bad = 0;
  for (long long i = 0; i < count; ++i) {
    uint64_t u;
    std::memcpy(&u, q + i, sizeof(u));  // no type punning through the caller's buffer
    bad |= (uint64_t)((u & 0x7ff0000000000000ull) == 0x7ff0000000000000ull);
  }
  if (bad) return fail(TRI_EINVAL, "query must be finite");
  return TRI_OK;
}

// Create a store from device-resident rows (row stride ldx floats).
int store_from_device(const float* Xdev, long long ldx, long long n, int d, int device, tri_store** out) {
  tri_store* s = new tri_store();
  s->device = device;
  s->n = n;
  s->d = d;
  s->dp = round16(d);
  s->qld = s->dp;
  cudaError_t e = cudaMalloc(&s->X, (size_t)n * s->dp * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->xnorm, (size_t)n * sizeof(float));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemset2DAsync(s->X, s->dp * sizeof(float), 0, s->dp * sizeof(float), n, s->own);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(s->X, s->dp * sizeof(float), Xdev, ldx * sizeof(float), d * sizeof(float), n,
                          cudaMemcpyDeviceToDevice, s->own);
  unsigned long long* xm = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&xm, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemsetAsync(xm, 0, sizeof(unsigned long long), s->own);
  if (e == cudaSuccess) e = launch_norms(s->X, n, d, s->dp, s->xnorm, xm, s->own);
  unsigned long long bits = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bits, xm, sizeof(bits), cudaMemcpyDeviceToHost, s->own);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->own);
  if (xm) cudaFree(xm);
  if (e != cudaSuccess) {
    tri_store_destroy(s);
    return fail(TRI_ECUDA, "store creation failed: %s", cudaGetErrorString(e));
  }
  std::memcpy(&s->xmax, &bits, sizeof(double));
  if (std::getenv("TRI_DEBUG_ALLOC")) std::fprintf(stderr, "[tri] store X=%p xnorm=%p\n", (void*)s->X, (void*)s->xnorm);
  int rc = make_tmap(&s->tmap, s->X, n, s->dp, false);
  if (rc == TRI_OK) rc = make_tmap(&s->tmap_tc, s->X, n, s->dp, true, false, (int)g_box_rows);
  if (rc == TRI_OK) rc = make_tmap(&s->tmap_tc_tail, s->X, n, s->dp, true, false, 32);
  s->box_rows = (int)g_box_rows;
  if (rc != TRI_OK) {
    tri_store_destroy(s);
    return rc;
  }
  *out = s;
  return TRI_OK;
}

// ---------------------------------------------------------------------------
// Brute-force plan: queries grouped by capacity class, the rows cut into
// ranges so that (#ranges x #groups) work items fill the GPU; items are
// range-major so CTAs running concurrently share rows through L2.

// Kernel + capacities for a batch: tensor-core scan when its layout fits.
struct ScanChoice {
  bool tc = false;
  int kp_max = kMinKp, k_max = 1, cap = 0, gmax = 0;
};

int choose_scan(int qld, int d, int B, const int* k, std::vector<int>& kp, ScanChoice& ch, bool prefer_simt) {
  int kp_tc = kMinKp;
  for (int i = 0; i < B; ++i) kp_tc = std::max(kp_tc, kp_for(k[i], true));
  ch.tc = !prefer_simt && use_tc(qld, kp_tc);
  kp.resize(B);
  ch.kp_max = kMinKp;
  ch.k_max = 1;
  for (int i = 0; i < B; ++i) {
    kp[i] = kp_for(k[i], ch.tc);
    ch.kp_max = std::max(ch.kp_max, kp[i]);
    ch.k_max = std::max(ch.k_max, k[i]);
  }
  ch.cap = sel_cap(ch.kp_max);
  ch.gmax = ch.tc ? kTcGroup : scan_gmax(qld, ch.cap, kSmemLimit);
  if (ch.gmax < 1) return fail(TRI_EINVAL, "dimension %d too large for the device scan", d);
  return TRI_OK;
}

long long plan_opts() {
  return g_bf_wide * 10000000000LL + g_pack_mixed * 1000000000 + g_dense_pow2 * 100000000 + g_dense_off * 10000000 + g_scan_kernel * 100000 +
         g_kp_extra;
}

// Split fp16 (hi + lo) copies of a store's rows for the tensor-core GEMM
// (tri_coarse.cu), scaled by sc = 2^(14 - ilogb(max|x|)), rows of dph halves.
// Returns TRI_OK without copies when the data's magnitude is out of range.
static int store_split_copy(tri_store* c, int dph, cudaStream_t st) {
  if (c->Ch) return TRI_OK;
  unsigned int* mb = nullptr;
  CU(cudaMalloc(&mb, sizeof(unsigned int)));
  CU(cudaMemsetAsync(mb, 0, sizeof(unsigned int), st));
  CU(launch_absmax(c->X, c->n, c->d, c->dp, mb, st));
  unsigned int bits = 0;
  CU(cudaMemcpyAsync(&bits, mb, sizeof(bits), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(mb);
  float m;
  std::memcpy(&m, &bits, sizeof(m));
  if (!(m >= std::ldexp(1.0f, -30) && m <= std::ldexp(1.0f, 30))) return TRI_OK;
  ++g_epoch;
  c->sc = std::ldexp(1.0f, 14 - std::ilogb(m));
  c->dph = dph;
  CU(cudaMalloc(&c->Ch, (size_t)c->n * dph * 2));
  CU(cudaMalloc(&c->Cl, (size_t)c->n * dph * 2));
  CU(launch_to_half(c->X, c->n, c->d, c->dp, c->sc, c->Ch, dph, st));
  CU(launch_to_half_lo(c->X, c->n, c->d, c->dp, c->sc, c->Cl, dph, st));
  TRY(make_tmap(&c->tmap_ch, c->Ch, c->n, dph, true, true, 128));
  TRY(make_tmap(&c->tmap_cl, c->Cl, c->n, dph, true, true, 128));
  return TRI_OK;
}

// Per-workspace brute-force plans.  The active plan lives in the Workspace
// fields; up to kPlanCache others are kept with their own device buffers, so
// alternating shapes (a serving loop's batch profiles, the IVF coarse step at
// several nprobe) switch plans without re-planning and without touching the
// device copy any captured graph reads.  Only evicting a plan retires graphs.
constexpr int kPlanCache = 16;

int plan_bruteforce(tri_store* s, Workspace& w, int B, const int* k, cudaStream_t st) {
  auto same = [&](int pB, long long pn, long long popts, const std::vector<int>& pk) {
    return pB == B && pn == s->n && popts == plan_opts() && (int)pk.size() == B && std::equal(pk.begin(), pk.end(), k);
  };
  if (same(w.plan_B, w.plan_n, w.plan_opts, w.plan_k)) return TRI_OK;
  for (auto& p : w.plan_cache)
    if (same(p.plan_B, p.plan_n, p.plan_opts, p.plan_k)) {  // swap the cached plan in
      Workspace::Plan cur;
      w.plan_out(cur);
      w.plan_in(p);
      p = cur;
      p.used = ++w.plan_clock;
      return TRI_OK;
    }
  if (w.capturing) return fail(TRI_EINTERNAL, "re-plan during graph capture");
  if (w.plan_B >= 0 && w.plan.p) {  // park the active plan (its buffer stays alive)
    if ((int)w.plan_cache.size() >= kPlanCache) {
      auto lru = std::min_element(w.plan_cache.begin(), w.plan_cache.end(),
                                  [](const Workspace::Plan& a, const Workspace::Plan& b) { return a.used < b.used; });
      ++w.epoch;  // graphs captured against it read its device copy
      cudaFree(lru->plan.p);
      w.plan_cache.erase(lru);
    }
    w.plan_cache.emplace_back();
    w.plan_out(w.plan_cache.back());
    w.plan_cache.back().used = ++w.plan_clock;
    w.plan = DevBuf{nullptr, 0, &w.epoch};  // the new plan gets a fresh buffer
  }
  // Dense path for small stores: the whole B x n distance matrix is cheap.
  {
    int kpd = kMinKp, kmx = 1;
    for (int i = 0; i < B; ++i) {
      kpd = std::max(kpd, kp_dense(k[i]));
      kmx = std::max(kmx, k[i]);
    }
    if (!g_dense_off && s->n <= kDenseMaxN && kpd <= kDenseMaxKp) {
      const size_t bytes = (((size_t)B * sizeof(QueryMeta) + 255) & ~(size_t)255) + 256;
      TRY(ensure(w.plan, bytes));
      int slot = 0;
      void* hp = nullptr;
      TRY(stage_host(w, bytes, &slot, &hp));  // ring of pinned buffers: no host sync
      QueryMeta* hm = static_cast<QueryMeta*>(hp);
      for (int i = 0; i < B; ++i) {
        hm[i].k = k[i];
        hm[i].kp = kp_dense(k[i]);
        hm[i].n_slots = 1;
        hm[i].cls = cls_of(hm[i].kp);
        hm[i].part_off = 0;
        hm[i].n_total = s->n;
      }
      TRY(staged_upload(w, slot, w.plan.p, bytes, st));
      w.plan_bytes = bytes;
      w.plan_B = B;
      w.plan_n = s->n;
      w.plan_opts = plan_opts();
      w.plan_k.assign(k, k + B);
      w.dense = true;
      w.tc = false;
      w.kp_max = kpd;
      w.k_max = kmx;
      w.part_keys = 0;
      return TRI_OK;
    }
  }
  w.dense = false;
  std::vector<int> kp, cls(B);
  ScanChoice ch;
  TRY(choose_scan(s->qld, s->d, B, k, kp, ch, s->prefer_simt != 0));
  for (int i = 0; i < B; ++i) cls[i] = cls_of(kp[i]);
  const int kp_max = ch.kp_max, k_max = ch.k_max, cap = ch.cap;
  const int nsm = sm_count(s->device);
  const long long max_ranges = std::max<long long>(1, (s->n + 511) / 512);
  // Group size: as large as shared memory allows (each extra group re-reads
  // the rows from L2), except that the SIMT scan's per-thread FFMA work grows
  // with the group -- small stores (the IVF coarse step) shrink groups until
  // the items cover every SM.
  int gmax = ch.gmax;
  int nq = kTcGroup;
  if (ch.tc && g_bf_wide && kp_max <= kTcWideMaxKp && B > kTcGroup &&
      tc_scan_stages(s->qld * 4, kSmemLimit, 0, 1, 1, kTcGroupWide) >= kTcMinStages) {
    gmax = kTcGroupWide;  // every row slab serves 64 queries: a quarter of the L2 reads of 16-query groups
    nq = kTcGroupWide;
  }
  if (!ch.tc) {
    auto n_groups = [&](int g) {
      std::vector<int> per(kNumCls, 0);
      for (int i = 0; i < B; ++i) per[cls[i]]++;
      long long t = 0;
      for (int c = 0; c < kNumCls; ++c) t += (per[c] + g - 1) / g;
      return t;
    };
    while (gmax > 4 && n_groups(gmax) * max_ranges < nsm) gmax >>= 1;
  }
  // groups: consecutive same-class queries in index order (the tensor-core
  // scan takes mixed-k groups at the members' largest kp: one pass per group)
  std::vector<std::vector<int>> groups;
  for (int c = 0; c < kNumCls; ++c) {
    std::vector<int> cur;
    for (int i = 0; i < B; ++i)
      if ((ch.tc && g_pack_mixed) ? c == 0 : cls[i] == c) {
        cur.push_back(i);
        if ((int)cur.size() == gmax) {
          groups.push_back(cur);
          cur.clear();
        }
      }
    if (!cur.empty()) groups.push_back(cur);
  }
  long long nr = std::max<long long>(1, ((long long)nsm + (long long)groups.size() - 1) / (long long)groups.size());
  nr = std::min(nr, max_ranges);
  long long R = (s->n + nr - 1) / nr;
  const long long rq = ch.tc ? 32 : 512;  // tensor-core items: any multiple of the 32-row tail box
  R = ((R + rq - 1) / rq) * rq;
  if (nq == kTcGroupWide) R = std::min<long long>(R, (long long)kTcWideMaxChunks * 128);  // chunks stay in TMEM
  nr = (s->n + R - 1) / R;
  // sizes
  std::vector<QueryMeta> meta(B);
  long long off = 0;
  for (int i = 0; i < B; ++i) {
    meta[i].k = k[i];
    meta[i].kp = kp[i];
    meta[i].n_slots = (int)nr;
    meta[i].cls = cls[i];
    meta[i].part_off = off;
    meta[i].n_total = s->n;
    off += nr * kp[i];
  }
  const long long n_items = nr * (long long)groups.size();
  const long long n_members = nr * (long long)B;
  w.off_items = ((size_t)B * sizeof(QueryMeta) + 255) & ~(size_t)255;
  w.off_members = w.off_items + (((size_t)n_items * sizeof(WorkItem) + 255) & ~(size_t)255);
  size_t counters_off = w.off_members + (((size_t)n_members * sizeof(Member) + 255) & ~(size_t)255);
  w.plan_bytes = counters_off + 256;
  TRY(ensure(w.plan, w.plan_bytes));
  int slot = 0;
  void* hp = nullptr;
  TRY(stage_host(w, w.plan_bytes, &slot, &hp));  // ring of pinned buffers: no host sync
  unsigned char* h = static_cast<unsigned char*>(hp);
  std::memcpy(h, meta.data(), B * sizeof(QueryMeta));
  WorkItem* items = reinterpret_cast<WorkItem*>(h + w.off_items);
  Member* members = reinterpret_cast<Member*>(h + w.off_members);
  long long it = 0, mb = 0;
  for (long long r = 0; r < nr; ++r) {
    for (const auto& g : groups) {
      WorkItem wi;
      wi.row_begin = r * R;
      wi.row_count = (int)std::min<long long>(R, s->n - r * R);
      wi.member_begin = (int)mb;
      wi.member_count = (int)g.size();
      wi.kp = 0;
      for (int q : g) wi.kp = std::max(wi.kp, kp[q]);
      wi.pad0 = 0;
      wi.pad1 = 0;
      items[it++] = wi;
      for (int q : g) {
        Member m;
        m.q = q;
        m.pad = kp[q];
        m.slot = meta[q].part_off + r * kp[q];
        members[mb++] = m;
      }
    }
  }
  int* ctr = reinterpret_cast<int*>(h + counters_off);
  ctr[0] = (int)n_items;
  TRY(staged_upload(w, slot, w.plan.p, w.plan_bytes, st));
  w.plan_B = B;
  w.plan_n = s->n;
  w.plan_opts = plan_opts();
  w.tc = ch.tc;
  w.plan_k.assign(k, k + B);
  w.n_items = (int)n_items;
  w.grid = (int)std::min<long long>(n_items, nsm);
  w.gmax = gmax;
  w.nq = nq;
  w.q_tma = 1;  // every group is a run of consecutive query indices (TMA query tiles)
  for (const auto& g : groups)
    for (size_t i = 1; i < g.size(); ++i)
      if (g[i] != g[0] + (int)i) w.q_tma = 0;
  w.cap = cap;
  w.kp_max = kp_max;
  w.k_max = k_max;
  w.part_keys = off;
  return TRI_OK;
}

int ensure_query_bufs(Workspace& w, int B, int d, int qld) {
  TRY(ensure(w.q64, (size_t)B * d * sizeof(double)));
  TRY(ensure(w.Q32, (size_t)B * qld * sizeof(float)));
  TRY(ensure(w.qn32, (size_t)B * sizeof(float)));
  TRY(ensure(w.qn64, (size_t)B * sizeof(double)));
  TRY(ensure(w.flags, (size_t)(B + 64) * sizeof(int)));
  return TRI_OK;
}

int finish_bruteforce(tri_store* s, Workspace& w, const double* q64dev, const Workspace& qw, const QueryMeta* meta,
                      int B, int ldo, long long* ids, double* dists, int mode, cudaStream_t st,
                      const unsigned long long* part = nullptr, const int* compact_cnt = nullptr,
                      bool set_only = false);

// Dense small-store brute force: distance matrix + warp select -> merged.
int dense_core(tri_store* s, Workspace& w, const Workspace& qw, const double* q64dev, int B, int ldo, long long* ids,
               double* dists, cudaStream_t st, bool set_only) {
  const long long ldd = (s->n + 3) & ~3LL;
  TRY(ensure(w.dmat, (size_t)kDenseSlices * B * ldd * sizeof(float)));
  TRY(ensure(w.merged, (size_t)B * w.kp_max * sizeof(unsigned long long)));
  TRY(ensure(w.exact, (size_t)B * w.kp_max * 16));
  TRY(ensure(w.flags, (size_t)(B + 64) * sizeof(int)));
  const QueryMeta* meta = static_cast<const QueryMeta*>(w.plan.p);
  CU(cudaMemsetAsync(w.flags.p, 0, 2 * sizeof(int), st));  // flag count + fix-up completion counter
  if (s->Ch && qw.split_q) {  // tensor-core coarse GEMM on the split fp16 copies
    CoarseLaunch c;
    c.map_h = &s->tmap_ch;
    c.map_l = &s->tmap_cl;
    c.Qh = qw.Qh.p;
    c.Ql = qw.Ql.p;
    c.ldq = s->dph;
    c.qinv = qw.qinv.as<float>();
    c.ratio = s->split_ratio;
    c.B = B;
    c.n = s->n;
    c.nslab = s->dph / 64;
    c.P = w.dmat.as<float>();
    c.ldd = ldd;
    CU(launch_coarse_tc(c, st));
    CU(launch_dense_select(w.dmat.as<float>(), coarse_tc_slices(c.nslab), ldd, B, qw.qn32.as<float>(), s->xnorm, s->n, meta,
                           w.merged.as<unsigned long long>(), w.kp_max, w.kp_max, st));
    return finish_bruteforce(s, w, q64dev, qw, meta, B, ldo, ids, dists, kSplit, st, nullptr, nullptr, set_only);
  }
  CU(launch_dense(qw.Q32.as<float>(), s->qld, qw.qn32.as<float>(), B, s->X, s->dp, s->xnorm, s->n, s->dp,
                  w.dmat.as<float>(), ldd, meta, w.merged.as<unsigned long long>(), w.kp_max, w.kp_max, st));
  return finish_bruteforce(s, w, q64dev, qw, meta, B, ldo, ids, dists, kSimt, st, nullptr, nullptr, set_only);
}

int prep_queries(Workspace& w, const double* q64dev, int B, int d, int qld, cudaStream_t st);

// Run the brute-force pipeline; prep = true prepares the fp64 queries at
// q64dev into `w` first (w == qw), otherwise they are prepared in `qw`
// (Q32/qn32/qn64).  Results to device ids/dists with row stride ldo.
int bruteforce_core(tri_store* s, Workspace& w, const Workspace& qw, const double* q64dev, int B, const int* k,
                    int ldo, long long* ids, double* dists, cudaStream_t st, bool prep, bool set_only = false) {
  TRY(plan_bruteforce(s, w, B, k, st));
  if (w.dense) {
    if (prep) TRY(prep_queries(w, q64dev, B, s->d, s->qld, st));
    return dense_core(s, w, qw, q64dev, B, ldo, ids, dists, st, set_only);
  }
  TRY(ensure(w.part, (size_t)w.part_keys * sizeof(unsigned long long)));
  TRY(ensure(w.merged, (size_t)B * w.kp_max * sizeof(unsigned long long)));
  TRY(ensure(w.exact, (size_t)B * w.kp_max * 16));
  TRY(ensure(w.flags, (size_t)(B + 64) * sizeof(int)));
  unsigned char* plan = static_cast<unsigned char*>(w.plan.p);
  const QueryMeta* meta = reinterpret_cast<const QueryMeta*>(plan);
  int* ctr = reinterpret_cast<int*>(plan + w.plan_bytes - 256);
  int* n_flag = w.flags.as<int>();
  int* flag_list = n_flag + 64;
  // per-search fills: the prep kernel does them on the side when it runs here
  ClearList cl{};
  cl.add(ctr + 1, 2, 0u);   // work-item counter + seed publish counter
  cl.add(n_flag, 2, 0u);    // flag count + fix-up completion counter

  ScanLaunch sl{};
  sl.tmap = &s->tmap;
  sl.tmap_tc = &s->tmap_tc;
  sl.tmap_tc_tail = &s->tmap_tc_tail;
  sl.X = s->X;
  sl.ldx = s->dp;
  sl.xnorm = s->xnorm;
  sl.Q = qw.Q32.as<float>();
  sl.qld = s->qld;
  sl.qnorm = qw.qn32.as<float>();
  sl.items = reinterpret_cast<const WorkItem*>(plan + w.off_items);
  sl.n_items = ctr;
  sl.counter = ctr + 1;
  sl.members = reinterpret_cast<const Member*>(plan + w.off_members);
  sl.part = w.part.as<unsigned long long>();
  sl.dp = s->dp;
  sl.gmax = w.gmax;
  sl.cap = w.cap;
  sl.grid = w.grid;
  sl.dbg = (int)g_scan_debug;
  sl.l2hint = 0;  // rows re-read by the batch's other query groups: default L2 policy
  sl.nq = w.nq;
  // brute force: selection-bound (L2-resident rows), keep one barrier per chunk
  // -- except 64-query groups, whose 64 KB append buffer and 32 KB query tile
  // leave room for only one of each beside a 7-slab ring
  sl.qbufs = w.nq == kTcGroupWide ? 1 : (int)g_scan_qbufs;
  sl.abufs = w.nq == kTcGroupWide ? 1 : 2;
  sl.stages = tc_scan_stages(s->qld * 4, kSmemLimit, (int)g_tc_stages, sl.qbufs, sl.abufs, sl.nq);
  sl.box_rows = s->box_rows;
  if (w.nq == kTcGroupWide) {
    sl.seed = (int)g_bf_seed;
    // cross-item seed: one wave (every item its own CTA) of at least kp items
    if (sl.seed == 2 && !(w.n_items <= w.grid && w.n_items <= kTcSeedItems && w.n_items >= w.kp_max)) sl.seed = 1;
    if (sl.seed == 2) {
      const size_t sb = ((size_t)B * w.n_items * sizeof(uint32_t) + 255) & ~(size_t)255;
      TRY(ensure(w.seedb, sb + (size_t)B * sizeof(int)));
      cl.add(w.seedb.p, (long long)(sb / 4), 0xffffffffu);
      int* ccnt = reinterpret_cast<int*>(static_cast<unsigned char*>(w.seedb.p) + sb);
      cl.add(ccnt, B, 0u);
      sl.seed_min = static_cast<uint32_t*>(w.seedb.p);
      sl.seed_ctr = ctr + 2;
      sl.seed_items = w.n_items;
      sl.grid = w.n_items;  // one CTA per item (tc_producer: fixed assignment)
      sl.compact_cnt = ccnt;
      sl.meta = meta;
    }
    if (w.q_tma && g_bf_qtma) {
      TRY(make_tmap(&w.qmap, qw.Q32.p, B, s->qld, true, false, kTcGroupWide));
      sl.q_tma = 1;
      sl.tmap_q = &w.qmap;
    }
  }
  if (g_gthr && w.tc) {
    TRY(ensure(w.gthr, (size_t)B * sizeof(unsigned long long)));
    cl.add(w.gthr.p, 2LL * B, 0xffffffffu);
    sl.gthr = w.gthr.as<unsigned long long>();
  }
  if (prep) {
    CU(launch_prep(q64dev, B, s->d, w.Q32.as<float>(), s->qld, w.qn32.as<float>(), w.qn64.as<double>(), nullptr, st,
                   1.f, nullptr, 0, nullptr, nullptr, &cl));
    // the scan launches as the prep's programmatic dependent: its fixed
    // per-CTA items start streaming rows while the prep runs
    sl.early = (g_scan_early && w.tc && sl.seed == 2) ? 1 : 0;
  } else {
    for (int r = 0; r < cl.n; ++r)
      CU(cl.val[r] == 0 ? cudaMemsetAsync(cl.p[r], 0, (size_t)cl.words[r] * 4, st)
                        : cudaMemsetAsync(cl.p[r], 0xff, (size_t)cl.words[r] * 4, st));
  }
  CU(w.tc ? launch_scan_tc(sl, st) : launch_scan(sl, st));
  if (sl.compact_cnt)  // the compact lists are merged by the re-rank kernel itself
    return finish_bruteforce(s, w, q64dev, qw, meta, B, ldo, ids, dists, w.tc ? kTf32 : kSimt, st,
                             w.part.as<unsigned long long>(), sl.compact_cnt);
  CU(launch_merge(w.part.as<unsigned long long>(), meta, w.merged.as<unsigned long long>(), w.kp_max, B, w.kp_max,
                  st));
  return finish_bruteforce(s, w, q64dev, qw, meta, B, ldo, ids, dists, w.tc ? kTf32 : kSimt, st, nullptr, nullptr,
                           set_only);
}

// Exact re-rank + certification + fix-up shared by the scan and dense paths.
int finish_bruteforce(tri_store* s, Workspace& w, const double* q64dev, const Workspace& qw, const QueryMeta* meta,
                      int B, int ldo, long long* ids, double* dists, int mode, cudaStream_t st,
                      const unsigned long long* part, const int* compact_cnt, bool set_only) {
  int* n_flag = w.flags.as<int>();
  int* flag_list = n_flag + 64;
  RerankLaunch rr{};
  rr.merged = w.merged.as<unsigned long long>();
  rr.exact = reinterpret_cast<Exact*>(w.exact.p);
  rr.ld_merged = w.kp_max;
  rr.meta = meta;
  rr.q64 = q64dev;
  rr.d = s->d;
  rr.qn64 = qw.qn64.as<double>();
  rr.X = s->X;
  rr.ldx = s->dp;
  rr.idmap = nullptr;
  rr.id_offset = s->id_offset;
  rr.xmax = s->xmax;
  const Bound bd = bound_for(s->d, mode);
  rr.cdot = g_force_fixup ? 1e30 : bd.cdot;
  rr.csum = bd.csum;
  rr.qinv = mode == kSplit ? qw.qinv.as<float>() : nullptr;  // unscalable queries are never certified
  rr.out_ids = ids;
  rr.out_d = dists;
  rr.ldo = ldo;
  TRY(ensure(w.fxs, fixup_scratch_bytes(B, w.k_max)));  // fix-up bounds + partial lists
  rr.fx_thr = static_cast<unsigned long long*>(w.fxs.p);
  rr.skip_far = (int)tri::g_rerank_skip;
  rr.n_flag = n_flag;
  rr.flag_list = flag_list;
  rr.B = B;
  rr.kp_max = w.kp_max;
  rr.part = part;
  rr.compact_cnt = compact_cnt;
  rr.xnorm = s->xnorm;
  // the IVF coarse step needs only the top-nprobe SET (coarse_set_kernel)
  if (set_only && g_coarse_set && !compact_cnt && w.kp_max <= 256 && s->d <= 1024)
    CU(launch_coarse_set(rr, st));
  else
    CU(launch_rerank(rr, st));
  FixupLaunch fx;
  fx.n_flag = n_flag;
  fx.flag_list = flag_list;
  fx.meta = meta;
  fx.q64 = q64dev;
  fx.d = s->d;
  fx.X = s->X;
  fx.ldx = s->dp;
  fx.n_rows = s->n;
  fx.probes = nullptr;
  fx.ld_probes = 0;
  fx.nprobe = nullptr;
  fx.list_off = nullptr;
  fx.idmap = nullptr;
  fx.id_offset = s->id_offset;
  fx.out_ids = ids;
  fx.out_d = dists;
  fx.ldo = ldo;
  fx.B = B;
  fx.k_max = w.k_max;
  fx.fx_thr = static_cast<unsigned long long*>(w.fxs.p);
  fx.fx_cnt = reinterpret_cast<int*>(static_cast<unsigned char*>(w.fxs.p) + fixup_thr_bytes(B));
  fx.scratch = reinterpret_cast<Exact*>(static_cast<unsigned char*>(w.fxs.p) + fixup_thr_bytes(B) +
                                        fixup_cnt_bytes(B, w.k_max));
  fx.max_units = fixup_max_units(B, w.k_max);
  fx.slice_rows = (int)tri::g_fx_slice_rows;
  {
    const Bound bs = bound_for(s->d, kSimt);
    fx.Q32 = qw.Q32.as<float>();
    fx.qld = s->qld;
    fx.qn32 = qw.qn32.as<float>();
    fx.qn64 = qw.qn64.as<double>();
    fx.xnorm = s->xnorm;
    fx.xmax = s->xmax;
    fx.cdot = bs.cdot;
    fx.csum = bs.csum;
  }
  CU(launch_fixup(fx, st));
  return TRI_OK;
}

int validate_k(const int* k, int B, long long limit, const char* what, bool capped = true) {
  for (int i = 0; i < B; ++i) {
    if (k[i] < 1 || k[i] > limit) return fail(TRI_EINVAL, "%s must be in [1, %lld], got %d", what, limit, k[i]);
    if (capped && k[i] > TRI_MAX_K) return fail(TRI_EINVAL, "%s=%d exceeds the device limit %d", what, k[i], TRI_MAX_K);
  }
  return TRI_OK;
}

int prep_queries(Workspace& w, const double* q64dev, int B, int d, int qld, cudaStream_t st) {
  CU(launch_prep(q64dev, B, d, w.Q32.as<float>(), qld, w.qn32.as<float>(), w.qn64.as<double>(), nullptr, st));
  return TRI_OK;
}

}  // namespace

// ===========================================================================
namespace tri {
int store_view(const tri_store* s, StoreView* v) {
  if (!s || !v) return fail(TRI_EINVAL, "store is NULL");
  v->X = s->X;
  v->ldx = s->dp;
  v->n = s->n;
  v->d = s->d;
  v->device = s->device;
  return TRI_OK;
}

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
}  // namespace tri

// CUDA-graph cache around one whole search (defined below, after the C-ABI
// entry points that use it).
template <class Body>
static int graph_run(tri_ivf* v, Workspace& w, Workspace* cw, cudaStream_t st, int mode, int B, const int* k,
                     const int* np, int ldo, const void* q, const void* ids, const void* dists, Body&& body,
                     int nk = -1);
// fixed-shape padded batches (defined with graph_run)
static int bucket_of(int B);
static int ensure_padded(Workspace& w, int Bc, int d, int ldo);
static int bf_padded(tri_store* s, Workspace& w, cudaStream_t st, int B, const int* k, int ldo);
static int padded_in(Workspace& w, const double* q, int B, int Bc, int d, int ldo, cudaStream_t st);
static int padded_out(Workspace& w, int B, int ldo, int64_t* ids, double* dists, cudaStream_t st);
static bool pad_bf(int B, const int* k);
static bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}


extern "C" {

const char* tri_last_error(void) { return g_err.c_str(); }

int tri_version(void) { return 1; }

int tri_graph_counters(int64_t* eager, int64_t* captured, int64_t* replayed) {
  if (eager) *eager = g_gr_eager.load();
  if (captured) *captured = g_gr_captured.load();
  if (replayed) *replayed = g_gr_replayed.load();
  return TRI_OK;
}

int tri_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(TRI_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = c;
  return TRI_OK;
}

int tri_set_option(const char* name, int64_t value) {
  if (!name) return fail(TRI_EINVAL, "option name is NULL");
  if (!std::strcmp(name, "force_fixup")) g_force_fixup = value;
  else if (!std::strcmp(name, "kp_extra")) g_kp_extra = value;
  else if (!std::strcmp(name, "scan_kernel")) g_scan_kernel = value;
  else if (!std::strcmp(name, "scan_debug")) g_scan_debug = value;
  else if (!std::strcmp(name, "dense_off")) g_dense_off = value;
  else if (!std::strcmp(name, "tc_stages")) g_tc_stages = value;
  else if (!std::strcmp(name, "scan_reserve")) g_scan_reserve = value;
  else if (!std::strcmp(name, "graphs")) g_graphs = value;
  else if (!std::strcmp(name, "gthr")) g_gthr = value;
  else if (!std::strcmp(name, "pack_mixed")) g_pack_mixed = value;
  else if (!std::strcmp(name, "scan_l2hint")) g_scan_l2hint = value;
  else if (!std::strcmp(name, "scan_abufs")) {
    if (value != 1 && value != 2) return fail(TRI_EINVAL, "scan_abufs must be 1 or 2");
    g_scan_abufs = value;
  }
  else if (!std::strcmp(name, "scan_qbufs")) {
    if (value != 1 && value != 2) return fail(TRI_EINVAL, "scan_qbufs must be 1 or 2");
    g_scan_qbufs = value;
  }
  else if (!std::strcmp(name, "coarse_tc")) g_coarse_tc = value;
  else if (!std::strcmp(name, "bf_wide")) g_bf_wide = value;
  else if (!std::strcmp(name, "bf_seed")) g_bf_seed = value;
  else if (!std::strcmp(name, "bf_qtma")) g_bf_qtma = value;
  else if (!std::strcmp(name, "ragged_graphs")) g_ragged_graphs = value;
  else if (!std::strcmp(name, "coarse_set")) g_coarse_set = value;
  else if (!std::strcmp(name, "dense_pow2")) g_dense_pow2 = value;

  else if (!std::strcmp(name, "coarse_split")) {
    if (value < 1 || value > kDenseSlices) return fail(TRI_EINVAL, "coarse_split must be in [1, %d]", kDenseSlices);
    tri::g_coarse_split = (int)value;
  }
  else if (!std::strcmp(name, "f16_div")) g_f16_div = value;
  else if (!std::strcmp(name, "bound_margin")) {
    if (value < 100 || value > 1600) return fail(TRI_EINVAL, "bound_margin must be in [100, 1600] percent");
    g_bound_margin = value;
  }
  else if (!std::strcmp(name, "dense_slices")) tri::g_dense_slices = (int)value;
  else if (!std::strcmp(name, "rerank_smem_cap")) tri::g_rerank_smem_cap = value;
  else if (!std::strcmp(name, "rerank_f2f")) tri::g_rerank_f2f = value;
  else if (!std::strcmp(name, "rerank_skip")) tri::g_rerank_skip = value;
  else if (!std::strcmp(name, "dense_fold")) tri::g_dense_fold = value;
  else if (!std::strcmp(name, "rerank_wide_slab")) tri::g_rerank_wide_slab = value;
  else if (!std::strcmp(name, "rerank_split")) tri::g_rerank_split = value;
  else if (!std::strcmp(name, "merge_split")) tri::g_merge_split = value;
  else if (!std::strcmp(name, "rerank_lpt")) tri::g_rerank_lpt = value;
  else if (!std::strcmp(name, "scan_pool")) g_scan_pool = value;
  else if (!std::strcmp(name, "scan_early")) g_scan_early = value;
  else if (!std::strcmp(name, "scan_pool_pub")) g_scan_pool_pub = value;
  else if (!std::strcmp(name, "scan_pool_minkp")) g_scan_pool_minkp = value;
  else if (!std::strcmp(name, "pdl")) tri::g_pdl = value;
  else if (!std::strcmp(name, "fx_slice_rows")) {
    if (value < 32) return fail(TRI_EINVAL, "fx_slice_rows must be >= 32");
    tri::g_fx_slice_rows = value;
  }
  else if (!std::strcmp(name, "tc_box_rows")) {
    if (value != 32 && value != 64 && value != 128) return fail(TRI_EINVAL, "tc_box_rows must be 32, 64 or 128");
    g_box_rows = value;
  }
  else return fail(TRI_EINVAL, "unknown option '%s'", name);
  return TRI_OK;
}

int tri_store_create(const float* x, int64_t n, int32_t d, int32_t device, tri_store** out) {
  if (!out) return fail(TRI_EINVAL, "out is NULL");
  if (n < 1 || d < 1) return fail(TRI_EINVAL, "vector store must be a nonempty 2-D matrix, got shape (%lld, %d)",
                                  (long long)n, d);
  if (n >= (1LL << 31)) return fail(TRI_EINVAL, "stores hold < 2^31 rows per device");
  for (long long i = 0; i < n * (long long)d; ++i)
    if (!std::isfinite(x[i])) return fail(TRI_EINVAL, "vector store entries must all be finite");
  CU(cudaSetDevice(device));
  float* tmp = nullptr;
  CU(cudaMalloc(&tmp, (size_t)n * d * sizeof(float)));
  // a synchronous H2D copy from pageable memory may return before its DMA
  // lands; the kernels that read tmp run on a non-blocking stream, so wait
  cudaError_t e = cudaMemcpy(tmp, x, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
  if (e != cudaSuccess) {
    cudaFree(tmp);
    return fail(TRI_ECUDA, "upload: %s", cudaGetErrorString(e));
  }
  int rc = store_from_device(tmp, d, n, d, device, out);
  cudaFree(tmp);
  return rc;
}

int tri_store_destroy(tri_store* s) {
  if (!s) return TRI_OK;
  DeviceGuard g(s->device);
  if (s->own) cudaStreamSynchronize(s->own);
  if (s->X) cudaFree(s->X);
  if (s->xnorm) cudaFree(s->xnorm);
  if (s->Ch) cudaFree(s->Ch);
  if (s->Cl) cudaFree(s->Cl);
  s->lanes.free_all();
  if (s->own) cudaStreamDestroy(s->own);
  delete s;
  return TRI_OK;
}

int tri_store_info(const tri_store* s, int64_t* n, int32_t* d, double* max_norm) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (n) *n = s->n;
  if (d) *d = s->d;
  if (max_norm) *max_norm = s->xmax;
  return TRI_OK;
}

int tri_store_set_id_offset(tri_store* s, int64_t id_offset) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (s->id_offset != id_offset) ++g_epoch;  // captured graphs bake the offset into kernel arguments
  s->id_offset = id_offset;
  return TRI_OK;
}

// k beyond the candidate-scan capacity (brute_force_knn takes any k <= N,
// ann_graph.py:131-133): every row's exact distance + a stable radix sort
// (tri_exhaustive.cu), eager.  q64 is on the device.
static int bruteforce_exhaustive(tri_store* s, Workspace& w, const double* q64, int B, const int* k, int ldo,
                                 int64_t* ids, double* dists, cudaStream_t st) {
  StoreView sv;
  TRY(tri::store_view(s, &sv));
  TRY(ensure(w.exh, exhaustive_scratch_bytes(s->n)));
  CU(launch_exhaustive_knn(sv, s->id_offset, q64, B, k, ldo, reinterpret_cast<long long*>(ids), dists, w.exh.p, st));
  return TRI_OK;
}

int tri_knn_bruteforce(tri_store* s, const double* q, int32_t B, const int32_t* k, int32_t ldo, int64_t* ids,
                       double* dists, void* stream) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (B < 0) return fail(TRI_EINVAL, "batch size must be >= 0");
  if (B == 0) return TRI_OK;
  TRY(validate_k(k, B, s->n, "k", false));
  int km = *std::max_element(k, k + B);
  if (ldo < km) return fail(TRI_EINVAL, "ldo=%d < max k=%d", ldo, km);
  TRY(check_queries(q, (long long)B * s->d));
  if (km > TRI_MAX_K) {
    DeviceGuard g(s->device);
    cudaStream_t st = pick(stream, s->own);
    {
      std::lock_guard<std::mutex> lk(s->mu);
      Workspace* wp = nullptr;
      TRY(s->lanes.get(st, &wp));
      TRY(ensure(wp->q64, (size_t)B * s->d * sizeof(double)));
      TRY(ensure(wp->out_ids, (size_t)B * ldo * sizeof(long long)));
      TRY(ensure(wp->out_d, (size_t)B * ldo * sizeof(double)));
      wp->pad_real = -1;
      CU(cudaMemcpyAsync(wp->q64.p, q, (size_t)B * s->d * sizeof(double), cudaMemcpyHostToDevice, st));
      TRY(bruteforce_exhaustive(s, *wp, wp->q64.as<double>(), B, k, ldo, wp->out_ids.as<int64_t>(),
                                wp->out_d.as<double>(), st));
      CU(cudaMemcpyAsync(ids, wp->out_ids.p, (size_t)B * ldo * sizeof(long long), cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(dists, wp->out_d.p, (size_t)B * ldo * sizeof(double), cudaMemcpyDeviceToHost, st));
      TRY(lane_done(*wp, st));
    }
    CU(cudaStreamSynchronize(st));
    return TRI_OK;
  }
  DeviceGuard g(s->device);
  cudaStream_t st = pick(stream, s->own);
  const size_t qb = (size_t)B * s->d * sizeof(double), ob = (size_t)B * ldo * sizeof(double);
  void* dst_ids = ids;
  void* dst_d = dists;
  bool staged = false;
  Workspace* wp = nullptr;
  {  // the store's lock covers the enqueue, not the wait (other lanes' threads overlap)
  std::lock_guard<std::mutex> lk(s->mu);
  TRY(s->lanes.get(st, &wp));
  Workspace& w = *wp;
  if (pad_bf(B, k)) {
    staged = !(host_pinned(ids) && host_pinned(dists));
    if (staged) {
      TRY(ensure_host(w.h_bids, ob));
      TRY(ensure_host(w.h_bd, ob));
      dst_ids = w.h_bids.p;
      dst_d = w.h_bd.p;
    }
    TRY(padded_in(w, q, B, bucket_of(B), s->d, ldo, st));
    TRY(bf_padded(s, w, st, B, k, ldo));
    TRY(padded_out(w, B, ldo, static_cast<int64_t*>(dst_ids), static_cast<double*>(dst_d), st));
    TRY(lane_done(w, st));
  } else {
  w.pad_real = -1;
  TRY(ensure_query_bufs(w, B, s->d, s->qld));
  TRY(ensure(w.out_ids, (size_t)B * ldo * sizeof(long long)));
  TRY(ensure(w.out_d, (size_t)B * ldo * sizeof(double)));
  // With graphs on, the caller's (pageable) buffers are copied through the
  // lane's pinned ones, so a repeated shape replays as one graph launch.
  staged = g_graphs != 0;
  const void* qsrc = q;
  if (staged) {
    TRY(ensure_host(w.h_bq, qb));
    TRY(ensure_host(w.h_bids, ob));
    TRY(ensure_host(w.h_bd, ob));
    std::memcpy(w.h_bq.p, q, qb);
    qsrc = w.h_bq.p;
    dst_ids = w.h_bids.p;
    dst_d = w.h_bd.p;
  }
  auto body = [&]() -> int {
    CU(cudaMemcpyAsync(w.q64.p, qsrc, qb, cudaMemcpyHostToDevice, st));
    TRY(bruteforce_core(s, w, w, w.q64.as<double>(), B, k, ldo, w.out_ids.as<long long>(), w.out_d.as<double>(), st,
                        true));
    CU(cudaMemcpyAsync(dst_ids, w.out_ids.p, ob, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(dst_d, w.out_d.p, ob, cudaMemcpyDeviceToHost, st));
    return TRI_OK;
  };
  if (staged)
    TRY(graph_run(nullptr, w, nullptr, st, 2, B, k, k, ldo, qsrc, dst_ids, dst_d, body));
  else
    TRY(body());
  TRY(lane_done(w, st));
  }
  }
  CU(cudaStreamSynchronize(st));
  if (staged) {
    std::memcpy(ids, dst_ids, ob);
    std::memcpy(dists, dst_d, ob);
  }
  return TRI_OK;
}

int tri_store_last_fixups(tri_store* s, int32_t* n) {
  if (!s || !n) return fail(TRI_EINVAL, "NULL argument");
  DeviceGuard g(s->device);
  int v = 0;
  Workspace& w = s->lanes.recent();
  if (w.flags.p) {
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(&v, w.flags.p, sizeof(int), cudaMemcpyDeviceToHost));
  }
  *n = w.pad_real >= 0 ? std::min(v, w.pad_real) : v;  // padded: dummies copy query 0
  return TRI_OK;
}

int tri_rowwise_sq_dists(tri_store* s, const double* q, const int64_t* rows, int64_t n, double* out, void* stream) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (n < 0 || n > (1LL << 30)) return fail(TRI_EINVAL, "bad row count %lld", (long long)n);
  if (n == 0) return TRI_OK;
  std::vector<int32_t> owner(n, 0);
  return tri_distance_tasks(s, owner.data(), rows, (int32_t)n, q, 1, out, stream);
}

int tri_rowwise_sq_dists_f64(const double* q, int32_t q_rows, const double* rows, int64_t n, int32_t d, int32_t device,
                             double* out) {
  if (n < 0 || d < 1) return fail(TRI_EINVAL, "bad shape (%lld, %d)", (long long)n, d);
  if (q_rows != 1 && q_rows != n) return fail(TRI_EINVAL, "query rows must be 1 or %lld, got %d", (long long)n, q_rows);
  if (n == 0) return TRI_OK;
  if (!q || !rows || !out) return fail(TRI_EINVAL, "NULL argument");
  DeviceGuard g(device);
  cudaStream_t st = nullptr;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const size_t qb = (size_t)q_rows * d * sizeof(double), xb = (size_t)n * d * sizeof(double);
  void* buf = nullptr;
  cudaError_t e = cudaMallocAsync(&buf, qb + xb + (size_t)n * sizeof(double), st);
  double* dq = static_cast<double*>(buf);
  double* dx = dq + (size_t)q_rows * d;
  double* dout = dx + (size_t)n * d;
  if (e == cudaSuccess) e = cudaMemcpyAsync(dq, q, qb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dx, rows, xb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = launch_rowwise_f64(dq, q_rows == 1 ? 0 : d, dx, n, d, dout, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (buf) cudaFreeAsync(buf, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return fail(TRI_ECUDA, "rowwise_sq_dists: %s", cudaGetErrorString(e));
  return TRI_OK;
}

int tri_distance_tasks(tri_store* s, const int32_t* owner, const int64_t* cand, int32_t n_tasks,
                       const double* queries, int32_t n_queries, double* out, void* stream) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (n_tasks < 0 || n_queries < 0) return fail(TRI_EINVAL, "negative size");
  if (n_tasks == 0) return TRI_OK;
  for (int i = 0; i < n_tasks; ++i)
    if (owner[i] < 0 || owner[i] >= n_queries) return fail(TRI_EINVAL, "task %d owner %d out of range", i, owner[i]);
  std::lock_guard<std::mutex> lk(s->mu);
  DeviceGuard g(s->device);
  cudaStream_t st = pick(stream, s->own);
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t qb = (size_t)n_queries * s->d * sizeof(double);
  const size_t o_c = al(qb), o_o = o_c + al((size_t)n_tasks * sizeof(long long));
  const size_t o_out = o_o + al((size_t)n_tasks * sizeof(int));
  const size_t total = o_out + al((size_t)n_tasks * sizeof(double));
  Workspace* w = nullptr;
  TRY(s->lanes.get(st, &w));
  DevBuf& buf = w->merged;  // reuse a scratch buffer
  TRY(ensure(buf, total));
  unsigned char* base = buf.as<unsigned char>();
  double* dq = reinterpret_cast<double*>(base);
  long long* dc = reinterpret_cast<long long*>(base + o_c);
  int* dow = reinterpret_cast<int*>(base + o_o);
  double* dout = reinterpret_cast<double*>(base + o_out);
  TRY(ensure(w->flags, 64 * sizeof(int)));
  int* derr = w->flags.as<int>() + 1;
  CU(cudaMemcpyAsync(dq, queries, qb, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dc, cand, (size_t)n_tasks * sizeof(long long), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dow, owner, (size_t)n_tasks * sizeof(int), cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(derr, 0, sizeof(int), st));
  CU(launch_distance_tasks(dow, dc, n_tasks, dq, s->d, s->X, s->dp, s->n, dout, derr, st));
  int herr = 0;
  CU(cudaMemcpyAsync(out, dout, (size_t)n_tasks * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (herr) {
    for (int i = 0; i < n_tasks; ++i)
      if (cand[i] < 0 || cand[i] >= s->n)
        return fail(TRI_EINTERNAL, "candidate id %lld out of range [0, %lld)", (long long)cand[i], s->n);
    return fail(TRI_EINTERNAL, "candidate out of range");
  }
  return TRI_OK;
}

// ---------------------------------------------------------------------------
// IVF

// fp16 copy of the list-major rows for the tensor-core scan, scaled by
// sx = 2^(14 - ilogb(max|x|)).  Skipped (TF32 scan) when the data's largest
// magnitude is outside [2^-30, 2^30] or the rows are too wide for the TC scan.
static int ivf_half_copy(tri_ivf* v, cudaStream_t st) {
  if (v->n < 1 || v->qld > kTcMaxQld) return TRI_OK;
  unsigned int* mb = nullptr;
  CU(cudaMalloc(&mb, sizeof(unsigned int)));
  CU(cudaMemsetAsync(mb, 0, sizeof(unsigned int), st));
  CU(launch_absmax(v->Xl, v->n, v->d, v->dp, mb, st));
  unsigned int bits = 0;
  CU(cudaMemcpyAsync(&bits, mb, sizeof(bits), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(mb);
  float m;
  std::memcpy(&m, &bits, sizeof(m));
  if (!(m >= std::ldexp(1.0f, -30) && m <= std::ldexp(1.0f, 30))) return TRI_OK;
  v->sx = std::ldexp(1.0f, 14 - std::ilogb(m));
  v->dph = (v->d + 63) & ~63;
  CU(cudaMalloc(&v->Xh, (size_t)v->n * v->dph * 2));
  CU(launch_to_half(v->Xl, v->n, v->d, v->dp, v->sx, v->Xh, v->dph, st));
  TRY(make_tmap(&v->tmap_h, v->Xh, v->n, v->dph, true, true, v->box_rows));
  TRY(make_tmap(&v->tmap_h_tail, v->Xh, v->n, v->dph, true, true, 32));
  return TRI_OK;
}

static int ivf_layout(tri_ivf* v, const float* X, long long ldx, const long long* perm_dev, cudaStream_t st) {
  const long long n = v->n;
  CU(cudaMalloc(&v->Xl, (size_t)n * v->dp * sizeof(float)));
  CU(cudaMalloc(&v->xnl, (size_t)n * sizeof(float)));
  CU(cudaMalloc(&v->ids, (size_t)n * sizeof(long long)));
  CU(launch_gather_rows(X, ldx, perm_dev, n, v->dp, v->Xl, st));
  TRY(make_tmap(&v->tmap, v->Xl, n, v->dp, false));
  TRY(make_tmap(&v->tmap_tc, v->Xl, n, v->dp, true, false, (int)g_box_rows));
  TRY(make_tmap(&v->tmap_tc_tail, v->Xl, n, v->dp, true, false, 32));
  v->box_rows = (int)g_box_rows;
  unsigned long long* xm = nullptr;
  CU(cudaMalloc(&xm, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(xm, 0, sizeof(unsigned long long), st));
  CU(launch_norms(v->Xl, n, v->d, v->dp, v->xnl, xm, st));
  CU(cudaMemcpyAsync(v->ids, perm_dev, (size_t)n * sizeof(long long), cudaMemcpyDeviceToDevice, st));
  unsigned long long bits = 0;
  CU(cudaMemcpyAsync(&bits, xm, sizeof(bits), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  cudaFree(xm);
  std::memcpy(&v->xmax, &bits, sizeof(double));
  TRY(ivf_half_copy(v, st));
  // list order by descending size (ties: smaller list id first)
  std::vector<int> order(v->nlist);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return (v->h_off[a + 1] - v->h_off[a]) > (v->h_off[b + 1] - v->h_off[b]);
  });
  CU(cudaMalloc(&v->list_by_size, (size_t)v->nlist * sizeof(int)));
  CU(cudaMemcpyAsync(v->list_by_size, order.data(), (size_t)v->nlist * sizeof(int), cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));
  return TRI_OK;
}

static tri_ivf* ivf_new(tri_store* s, int nlist) {
  tri_ivf* v = new tri_ivf();
  v->device = s->device;
  v->n = s->n;
  v->d = s->d;
  v->dp = s->dp;
  v->qld = s->qld;
  v->nlist = nlist;
  v->id_offset = s->id_offset;
  return v;
}

// IVF centroid store: split copies sharing the lists' fp16 row width, so the
// queries' split comes from the fine scan's prep pass (scale ratio s_list / sc).
static int coarse_split_copy(tri_ivf* v, cudaStream_t st) {
  if (!v->Xh || v->dph > 1024 || v->nlist > kDenseMaxN) return TRI_OK;
  TRY(store_split_copy(v->cstore, v->dph, st));
  if (v->cstore->Ch) v->cstore->split_ratio = v->sx / v->cstore->sc;  // both powers of two: exact
  return TRI_OK;
}

static int ivf_finish(tri_ivf* v, tri_store* s, const float* Cdev, const int* assign_dev, cudaStream_t st) {
  // counts -> offsets (host) -> ordered members -> layout
  DevBuf cnt;
  TRY(ensure(cnt, (size_t)v->nlist * sizeof(int)));
  CU(launch_counts(assign_dev, v->n, v->nlist, cnt.as<int>(), st));
  std::vector<int> hc(v->nlist);
  CU(cudaMemcpyAsync(hc.data(), cnt.p, (size_t)v->nlist * sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  release(cnt);
  v->h_off.assign(v->nlist + 1, 0);
  for (int l = 0; l < v->nlist; ++l) v->h_off[l + 1] = v->h_off[l] + hc[l];
  CU(cudaMalloc(&v->list_off, (size_t)(v->nlist + 1) * sizeof(long long)));
  // on st, not the legacy stream: list_members_kernel (on the non-blocking st)
  // must see the offsets, and a pageable H2D cudaMemcpy may return before its DMA lands
  CU(cudaMemcpyAsync(v->list_off, v->h_off.data(), (size_t)(v->nlist + 1) * sizeof(long long),
                     cudaMemcpyHostToDevice, st));
  DevBuf perm;
  TRY(ensure(perm, (size_t)v->n * sizeof(long long)));
  CU(launch_list_members(assign_dev, v->n, v->nlist, v->list_off, perm.as<long long>(), st));
  TRY(ivf_layout(v, s->X, s->dp, perm.as<long long>(), st));
  release(perm);
  if (v->id_offset) {
    // ids are global: add the shard offset on the host-free path
    std::vector<long long> h(v->n);
    CU(cudaMemcpyAsync(h.data(), v->ids, (size_t)v->n * sizeof(long long), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (auto& x : h) x += v->id_offset;
    CU(cudaMemcpyAsync(v->ids, h.data(), (size_t)v->n * sizeof(long long), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
  }
  CU(cudaMalloc(&v->assign, (size_t)v->n * sizeof(int)));
  CU(cudaMemcpyAsync(v->assign, assign_dev, (size_t)v->n * sizeof(int), cudaMemcpyDeviceToDevice, st));
  TRY(store_from_device(Cdev, v->dp, v->nlist, v->d, v->device, &v->cstore));
  // Coarse step on the fp32 SIMT scan: centroid distances sit close together and
  // singleton lists give centroids data-point norms, so the TF32 bound would
  // rarely certify (measured: 251/256 fix-ups); fp32 certifies every query.
  v->cstore->prefer_simt = 1;
  TRY(coarse_split_copy(v, st));
  CU(cudaStreamCreateWithFlags(&v->own, cudaStreamNonBlocking));
  CU(cudaStreamSynchronize(st));
  return TRI_OK;
}

// Exact k-means assignment: every row of s goes to its nearest centroid by
// the exact float64 distance in the reference's operation order, ties to the
// smaller centroid id -- i.e. brute_force_knn(VectorStore(C), row, 1)
// (ann_graph.py:124-137) for each row, run as the certified batched brute
// force.  Deterministic, so the CPU oracle reproduces it bit-for-bit
// (oracle.kmeans).  C: nlist x ldc device rows (ldc = s->dp).
static int exact_assign(tri_store* s, const float* C, int nlist, int* asg, cudaStream_t st) {
  tri_store* cs = nullptr;
  TRY(store_from_device(C, s->dp, nlist, s->d, s->device, &cs));
  cs->prefer_simt = 1;  // centroid distances sit close together: the tight fp32 bound
  constexpr int kChunk = 4096;
  DevBuf q64, ids, dd;
  int rc = TRI_OK;
  do {
    Workspace* w = nullptr;
    if ((rc = cs->lanes.get(st, &w))) break;
    const long long n = s->n;
    if ((rc = ensure(q64, (size_t)kChunk * s->d * sizeof(double)))) break;
    if ((rc = ensure(ids, (size_t)n * sizeof(long long)))) break;
    if ((rc = ensure(dd, (size_t)kChunk * sizeof(double)))) break;
    std::vector<int> ones(kChunk, 1);
    for (long long r0 = 0; r0 < n && rc == TRI_OK; r0 += kChunk) {
      const int B = (int)std::min<long long>(kChunk, n - r0);
      cudaError_t e = launch_rows_to_f64(s->X + r0 * s->dp, s->dp, B, s->d, q64.as<double>(), st);
      if (e != cudaSuccess) {
        rc = fail(TRI_ECUDA, "k-means assignment: %s", cudaGetErrorString(e));
        break;
      }
      if ((rc = ensure_query_bufs(*w, B, s->d, cs->qld))) break;
      rc = bruteforce_core(cs, *w, *w, q64.as<double>(), B, ones.data(), 1, ids.as<long long>() + r0, dd.as<double>(),
                           st, true);
    }
    if (rc) break;
    cudaError_t e = launch_narrow_ids(ids.as<long long>(), n, asg, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(TRI_ECUDA, "k-means assignment: %s", cudaGetErrorString(e));
  } while (0);
  cudaStreamSynchronize(st);
  release(q64);
  release(ids);
  release(dd);
  tri_store_destroy(cs);
  return rc;
}

int tri_kmeans_assign(tri_store* s, const float* centroids, int32_t nlist, int32_t* assign) {
  if (!s || !centroids || !assign) return fail(TRI_EINVAL, "NULL argument");
  if (nlist < 1) return fail(TRI_EINVAL, "nlist must be >= 1");
  for (long long i = 0; i < (long long)nlist * s->d; ++i)
    if (!std::isfinite(centroids[i])) return fail(TRI_EINVAL, "centroids must be finite");
  DeviceGuard g(s->device);
  cudaStream_t st = s->own;
  DevBuf C, asg;
  int rc = ensure(C, (size_t)nlist * s->dp * sizeof(float));
  if (!rc) rc = ensure(asg, (size_t)s->n * sizeof(int));
  if (!rc) {
    cudaError_t e = cudaMemset2DAsync(C.p, s->dp * sizeof(float), 0, s->dp * sizeof(float), nlist, st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(C.p, s->dp * sizeof(float), centroids, s->d * sizeof(float), s->d * sizeof(float), nlist,
                            cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = fail(TRI_ECUDA, "upload: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = exact_assign(s, C.as<float>(), nlist, asg.as<int>(), st);
  if (!rc) {
    cudaError_t e = cudaMemcpy(assign, asg.p, (size_t)s->n * sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(TRI_ECUDA, "download: %s", cudaGetErrorString(e));
  }
  release(C);
  release(asg);
  return rc;
}

int tri_ivf_train(tri_store* s, int32_t nlist, int32_t iters, const int64_t* init_rows, tri_ivf** out) {
  if (!s || !out || !init_rows) return fail(TRI_EINVAL, "NULL argument");
  if (nlist < 1 || nlist > s->n) return fail(TRI_EINVAL, "nlist must be in [1, %lld], got %d", s->n, nlist);
  if (iters < 0) return fail(TRI_EINVAL, "iters must be >= 0");
  for (int i = 0; i < nlist; ++i)
    if (init_rows[i] < 0 || init_rows[i] >= s->n) return fail(TRI_EINVAL, "init row %lld out of range", (long long)init_rows[i]);
  DeviceGuard g(s->device);
  cudaStream_t st = s->own;
  tri_ivf* v = ivf_new(s, nlist);
  DevBuf C, cn, asg, cnt, perm, off, xm, initd;
  auto cleanup = [&]() {
    for (DevBuf* b : {&C, &cn, &asg, &cnt, &perm, &off, &xm, &initd}) release(*b);
  };
  int rc = TRI_OK;
  do {
    if ((rc = ensure(C, (size_t)nlist * s->dp * sizeof(float)))) break;
    if ((rc = ensure(cn, (size_t)nlist * sizeof(float)))) break;
    if ((rc = ensure(asg, (size_t)s->n * sizeof(int)))) break;
    if ((rc = ensure(cnt, (size_t)nlist * sizeof(int)))) break;
    if ((rc = ensure(perm, (size_t)s->n * sizeof(long long)))) break;
    if ((rc = ensure(off, (size_t)(nlist + 1) * sizeof(long long)))) break;
    if ((rc = ensure(xm, sizeof(unsigned long long)))) break;
    if ((rc = ensure(initd, (size_t)nlist * sizeof(long long)))) break;
    cudaError_t e = cudaMemcpyAsync(initd.p, init_rows, (size_t)nlist * sizeof(long long), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = launch_gather_rows(s->X, s->dp, initd.as<long long>(), nlist, s->dp, C.as<float>(), st);
    std::vector<int> hc(nlist);
    std::vector<long long> ho(nlist + 1);
    for (int it = 0; it <= iters && e == cudaSuccess; ++it) {
      if ((rc = exact_assign(s, C.as<float>(), nlist, asg.as<int>(), st))) break;
      if (it == iters) break;
      if (e == cudaSuccess) e = launch_counts(asg.as<int>(), s->n, nlist, cnt.as<int>(), st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), cnt.p, (size_t)nlist * sizeof(int), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) break;
      ho[0] = 0;
      for (int l = 0; l < nlist; ++l) ho[l + 1] = ho[l] + hc[l];
      e = cudaMemcpyAsync(off.p, ho.data(), (size_t)(nlist + 1) * sizeof(long long), cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = launch_list_members(asg.as<int>(), s->n, nlist, off.as<long long>(), perm.as<long long>(), st);
      if (e == cudaSuccess)
        e = launch_centroid_update(s->X, s->dp, s->d, perm.as<long long>(), off.as<long long>(), nlist, C.as<float>(), s->dp, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // ho is reused
    }
    if (rc) break;
    if (e != cudaSuccess) {
      rc = fail(TRI_ECUDA, "k-means: %s", cudaGetErrorString(e));
      break;
    }
    rc = ivf_finish(v, s, C.as<float>(), asg.as<int>(), st);
  } while (0);
  cleanup();
  if (rc != TRI_OK) {
    tri_ivf_destroy(v);
    return rc;
  }
  *out = v;
  return TRI_OK;
}

int tri_ivf_create(tri_store* s, const float* centroids, int32_t nlist, const int32_t* assign, int64_t id_offset,
                   tri_ivf** out) {
  if (!s || !out || !centroids || !assign) return fail(TRI_EINVAL, "NULL argument");
  if (nlist < 1) return fail(TRI_EINVAL, "nlist must be >= 1");
  for (long long i = 0; i < s->n; ++i)
    if (assign[i] < 0 || assign[i] >= nlist) return fail(TRI_EINVAL, "assign[%lld]=%d out of range", i, assign[i]);
  for (long long i = 0; i < (long long)nlist * s->d; ++i)
    if (!std::isfinite(centroids[i])) return fail(TRI_EINVAL, "centroids must be finite");
  DeviceGuard g(s->device);
  cudaStream_t st = s->own;
  tri_ivf* v = ivf_new(s, nlist);
  v->id_offset = id_offset;
  DevBuf C, asg;
  int rc = ensure(C, (size_t)nlist * s->dp * sizeof(float));
  if (!rc) rc = ensure(asg, (size_t)s->n * sizeof(int));
  if (!rc) {
    cudaError_t e = cudaMemset2DAsync(C.p, s->dp * sizeof(float), 0, s->dp * sizeof(float), nlist, st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(C.p, s->dp * sizeof(float), centroids, s->d * sizeof(float), s->d * sizeof(float), nlist,
                            cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(asg.p, assign, (size_t)s->n * sizeof(int), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = fail(TRI_ECUDA, "upload: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = ivf_finish(v, s, C.as<float>(), asg.as<int>(), st);
  release(C);
  release(asg);
  if (rc) {
    tri_ivf_destroy(v);
    return rc;
  }
  *out = v;
  return TRI_OK;
}

int tri_ivf_destroy(tri_ivf* v) {
  if (!v) return TRI_OK;
  DeviceGuard g(v->device);
  if (v->own) cudaStreamSynchronize(v->own);
  for (void* p : {(void*)v->Xl, (void*)v->xnl, (void*)v->ids, (void*)v->list_off, (void*)v->list_by_size,
                  (void*)v->assign, v->Xh})
    if (p) cudaFree(p);
  v->lanes.free_all();
  if (v->cstore) tri_store_destroy(v->cstore);
  for (cudaEvent_t e : v->ev) cudaEventDestroy(e);
  if (v->own) cudaStreamDestroy(v->own);
  delete v;
  return TRI_OK;
}

int tri_ivf_info(const tri_ivf* v, int32_t* nlist, int64_t* n, int32_t* d) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  if (nlist) *nlist = v->nlist;
  if (n) *n = v->n;
  if (d) *d = v->d;
  return TRI_OK;
}

int tri_ivf_export(tri_ivf* v, float* centroids, int32_t* assign) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  DeviceGuard g(v->device);
  if (centroids)
    CU(cudaMemcpy2D(centroids, v->d * sizeof(float), v->cstore->X, v->dp * sizeof(float), v->d * sizeof(float),
                    v->nlist, cudaMemcpyDeviceToHost));
  if (assign) CU(cudaMemcpy(assign, v->assign, (size_t)v->n * sizeof(int), cudaMemcpyDeviceToHost));
  return TRI_OK;
}

int tri_ivf_list_sizes(tri_ivf* v, int64_t* sizes) {
  if (!v || !sizes) return fail(TRI_EINVAL, "NULL argument");
  for (int l = 0; l < v->nlist; ++l) sizes[l] = v->h_off[l + 1] - v->h_off[l];
  return TRI_OK;
}

static int ivf_validate(tri_ivf* v, int32_t B, const int32_t* k, const int32_t* nprobe, int32_t ldo) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  if (B < 0) return fail(TRI_EINVAL, "batch size must be >= 0");
  if (B == 0) return TRI_OK;
  TRY(validate_k(k, B, (long long)1 << 40, "k"));
  TRY(validate_k(nprobe, B, v->nlist, "nprobe"));
  int km = *std::max_element(k, k + B);
  if (ldo < km) return fail(TRI_EINVAL, "ldo=%d < max k=%d", ldo, km);
  return TRI_OK;
}

// Enqueue one whole search on `st` (lane workspaces w / cw already chosen).
// dplan != nullptr: a padded fixed-shape batch (see launch_ragged_plan): k and
// nprobe are then the batch profile (max k, max nprobe for every row) that
// sizes every buffer, and the per-query plan is built on the device.
static int ivf_search_body(tri_ivf* v, Workspace& w, Workspace* cw, const double* q, int32_t B, const int32_t* k,
                           const int32_t* nprobe, int32_t ldo, int64_t* ids, double* dists, cudaStream_t st,
                           const int* dplan = nullptr) {
  const int npmax = *std::max_element(nprobe, nprobe + B);
  TRY(ensure_query_bufs(w, B, v->d, v->qld));
  const bool rec = v->prof && v->ev_used < kProfSearches;
  // NVTX ranges per pipeline stage (host enqueue; the device work of an eager
  // search follows them, a replayed graph shows as one tri.graph.replay range)
  static const char* kStageNames[6] = {"tri.ivf.coarse", "tri.ivf.plan_pack", "tri.ivf.scan", "tri.ivf.merge",
                                       "tri.ivf.rerank", "tri.ivf.fixup"};
  nvtxRangePushA("tri.ivf.prep");
  auto mark = [&](int j) -> int {
    nvtxRangePop();
    if (j < 6) nvtxRangePushA(kStageNames[j]);
    if (!rec) return TRI_OK;
    if (w.capturing) {  // event node; the launch points it at the profiling ring
      CU(cudaEventRecordWithFlags(w.cap_ph[j], st, cudaEventRecordExternal));
      return TRI_OK;
    }
    while ((int)v->ev.size() < 7 * (v->ev_used + 1)) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      v->ev.push_back(e);
    }
    CU(cudaEventRecord(v->ev[7 * v->ev_used + j], st));
    return TRI_OK;
  };
  // per-query plan (k, kp) and scan arithmetic: fp16 tensor-core scan when the
  // index holds the fp16 copy (scan_kernel 2 forces TF32)
  std::vector<int> kp;
  ScanChoice ch;
  TRY(choose_scan(v->qld, v->d, B, k, kp, ch, false));
  const bool f16 = ch.tc && v->Xh && g_scan_kernel != 2;
  if (f16) {
    ch.kp_max = kMinKp;
    for (int i = 0; i < B; ++i) {
      kp[i] = kp_for_f16(k[i]);
      ch.kp_max = std::max(ch.kp_max, kp[i]);
    }
    ch.cap = sel_cap(ch.kp_max);
  }
  const int kp_max = ch.kp_max, k_max = ch.k_max;
  // 0. queries: fp32 rows + norms (+ the fp16 scan copy) in one kernel
  if (f16) {
    TRY(ensure(w.Qh, (size_t)B * v->dph * 2));
    TRY(ensure(w.qinv, (size_t)B * sizeof(float)));
    w.split_q = g_coarse_tc && v->cstore->Ch && v->cstore->dph == v->dph;
    if (w.split_q) TRY(ensure(w.Ql, (size_t)B * v->dph * 2));
    CU(launch_prep(q, B, v->d, w.Q32.as<float>(), v->qld, w.qn32.as<float>(), w.qn64.as<double>(), nullptr, st,
                   v->sx, w.Qh.p, v->dph, w.qinv.as<float>(), w.split_q ? w.Ql.p : nullptr));
  } else {
    w.split_q = false;
    TRY(prep_queries(w, q, B, v->d, v->qld, st));
  }
  TRY(mark(0));

  // 1. coarse step: exact top-nprobe centroids per query
  TRY(ensure(w.probes, (size_t)B * npmax * sizeof(long long)));
  TRY(ensure(w.probe_d, (size_t)B * npmax * sizeof(double)));
  TRY(bruteforce_core(v->cstore, *cw, w, q, B, nprobe, npmax, w.probes.as<long long>(), w.probe_d.as<double>(),
                      st, false, /*set_only=*/true));

  // 2. per-query plan -> device
  long long part_keys = 0, members = 0;
  const size_t meta_bytes = (size_t)B * (sizeof(QueryMeta) + sizeof(int));
  for (int i = 0; i < B; ++i) {  // (padded batch: the worst case the device plan can reach)
    part_keys += (long long)nprobe[i] * kp[i];
    members += nprobe[i];
  }
  const int cap = ch.cap, gmax = ch.gmax;
  TRY(ensure(w.meta, meta_bytes + 64));
  QueryMeta* dmeta = w.meta.as<QueryMeta>();
  int* dnp = reinterpret_cast<int*>(dmeta + B);
  int cls_mask = 0;
  if (dplan) {
    cls_mask = (1 << (cls_of(kp_max) + 1)) - 1;  // any class up to the profile's
    TRY(ensure(w.rtot, 64));
    RaggedPlan rp;
    rp.in = dplan;
    rp.Bc = B;
    rp.f16 = f16 ? 1 : 0;
    rp.tc = ch.tc ? 1 : 0;
    rp.f16_div = (int)std::max<long long>(1, g_f16_div);
    rp.kp_extra = (int)g_kp_extra;
    rp.meta = dmeta;
    rp.nprobe = dnp;
    rp.total_keys = w.rtot.as<long long>();
    CU(launch_ragged_plan(rp, st));
  } else {
    int slot = 0;
    void* hbuf = nullptr;
    TRY(stage_host(w, meta_bytes + 64, &slot, &hbuf));
    QueryMeta* hm = static_cast<QueryMeta*>(hbuf);
    int* hnp = reinterpret_cast<int*>(hm + B);
    long long off = 0;
    for (int i = 0; i < B; ++i) {
      hm[i].k = k[i];
      hm[i].kp = kp[i];
      hm[i].n_slots = nprobe[i];
      hm[i].cls = cls_of(kp[i]);
      hm[i].part_off = off;
      hm[i].n_total = 0;
      hnp[i] = nprobe[i];
      off += (long long)nprobe[i] * kp[i];
      cls_mask |= 1 << hm[i].cls;
    }
    TRY(staged_upload(w, slot, w.meta.p, meta_bytes, st));
  }
  TRY(ensure(w.part, (size_t)part_keys * sizeof(unsigned long long)));
  TRY(ensure(w.merged, (size_t)B * kp_max * sizeof(unsigned long long)));
  TRY(ensure(w.exact, (size_t)B * kp_max * 16));
  if (dplan)
    CU(launch_fill_keys(w.part.as<unsigned long long>(), w.rtot.as<long long>(), 2 * sm_count(v->device), st));
  else
    CU(cudaMemsetAsync(w.part.p, 0xff, (size_t)part_keys * sizeof(unsigned long long), st));
  size_t cbytes = (size_t)v->nlist * kNumCls * sizeof(int);
  TRY(ensure(w.counts, cbytes));
  TRY(ensure(w.fill, cbytes));
  TRY(ensure(w.mbase, cbytes));
  TRY(ensure(w.items, (size_t)members * sizeof(WorkItem)));
  TRY(ensure(w.members, (size_t)members * sizeof(Member)));
  TRY(ensure(w.counters, 64 * sizeof(int)));
  int* ctr = w.counters.as<int>();
  CU(cudaMemsetAsync(ctr, 0, 4 * sizeof(int), st));

  TRY(mark(1));
  // 3. device packer
  PackLaunch pk;
  pk.probes = w.probes.as<long long>();
  pk.ld_probes = npmax;
  pk.nprobe = dnp;
  pk.meta = dmeta;
  pk.B = B;
  pk.list_off = v->list_off;
  pk.list_by_size = v->list_by_size;
  pk.nlist = v->nlist;
  pk.counts = w.counts.as<int>();
  pk.fill = w.fill.as<int>();
  pk.member_base = w.mbase.as<int>();
  pk.items = w.items.as<WorkItem>();
  pk.n_items = ctr;
  pk.members = w.members.as<Member>();
  pk.gmax = gmax;
  pk.cls_mask = cls_mask;
  pk.mixed = (ch.tc && g_pack_mixed) ? 1 : 0;  // the SIMT scan keeps per-class groups
  CU(launch_pack(pk, st));

  // 4. list scan (persistent, one CTA per SM)
  ScanLaunch sl{};
  sl.tmap = &v->tmap;
  sl.tmap_tc = f16 ? &v->tmap_h : &v->tmap_tc;
  sl.tmap_tc_tail = f16 ? &v->tmap_h_tail : &v->tmap_tc_tail;
  sl.f16 = f16 ? 1 : 0;
  sl.Qh = f16 ? w.Qh.p : nullptr;
  sl.qldh = v->dph;
  sl.qinv = f16 ? w.qinv.as<float>() : nullptr;
  if (g_gthr && ch.tc) {
    TRY(ensure(w.gthr, (size_t)B * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(w.gthr.p, 0xff, (size_t)B * sizeof(unsigned long long), st));
    sl.gthr = w.gthr.as<unsigned long long>();
    if (g_scan_pool > 0 && kp_max >= g_scan_pool_minkp) {  // wide members: the pooled cross-item bound
      const int cap = (int)std::min<long long>(1024, (g_scan_pool + 31) / 32 * 32);
      TRY(ensure(w.pool, (size_t)B * cap * sizeof(unsigned long long) + (size_t)B * sizeof(int)));
      CU(cudaMemsetAsync(w.pool.p, 0xff, (size_t)B * cap * sizeof(unsigned long long), st));
      sl.pool = w.pool.as<unsigned long long>();
      sl.pool_cnt = reinterpret_cast<int*>(sl.pool + (size_t)B * cap);
      CU(cudaMemsetAsync(sl.pool_cnt, 0, (size_t)B * sizeof(int), st));
      sl.pool_cap = cap;
      sl.pool_pub = (int)g_scan_pool_pub;
      sl.pool_minkp = (int)g_scan_pool_minkp;
    }
  }
  sl.X = v->Xl;
  sl.ldx = v->dp;
  sl.xnorm = v->xnl;
  sl.Q = w.Q32.as<float>();
  sl.qld = v->qld;
  sl.qnorm = w.qn32.as<float>();
  sl.items = w.items.as<WorkItem>();
  sl.n_items = ctr;
  sl.counter = ctr + 1;
  sl.members = w.members.as<Member>();
  sl.part = w.part.as<unsigned long long>();
  sl.dp = v->dp;
  sl.gmax = gmax;
  sl.cap = cap;
  // persistent scan: one CTA per SM, minus `scan_reserve` SMs left free for
  // batches in flight on other streams (the scan is HBM-bound, they are not)
  sl.grid = (int)std::max<long long>(1, std::min<long long>(sm_count(v->device) - scan_reserve_for(v), members));
  sl.dbg = (int)g_scan_debug;
  sl.l2hint = (int)g_scan_l2hint;  // lists stream once per batch: evict_first keeps centroids / queries in L2
  sl.qbufs = (int)g_scan_qbufs;
  // one append buffer: the list scan is stream-bound, and the 16 KB buy a ring stage
  sl.abufs = (int)g_scan_abufs;
  sl.nq = kTcGroup;
  sl.stages = tc_scan_stages(f16 ? v->dph * 2 : v->qld * 4, kSmemLimit, (int)g_tc_stages, sl.qbufs, sl.abufs, sl.nq);
  sl.box_rows = v->box_rows;
  TRY(mark(2));
  CU(ch.tc ? launch_scan_tc(sl, st) : launch_scan(sl, st));
  TRY(mark(3));

  // 5. merge, exact re-rank, certified fix-up
  CU(launch_merge(w.part.as<unsigned long long>(), dmeta, w.merged.as<unsigned long long>(), kp_max, B, kp_max, st));
  TRY(mark(4));
  int* n_flag = w.flags.as<int>();
  int* flag_list = n_flag + 64;
  CU(cudaMemsetAsync(n_flag, 0, 2 * sizeof(int), st));  // flag count + fix-up completion counter
  RerankLaunch rr{};
  rr.merged = w.merged.as<unsigned long long>();
  rr.exact = reinterpret_cast<Exact*>(w.exact.p);
  rr.ld_merged = kp_max;
  rr.meta = dmeta;
  rr.q64 = q;
  rr.d = v->d;
  rr.qn64 = w.qn64.as<double>();
  rr.X = v->Xl;
  rr.ldx = v->dp;
  rr.idmap = v->ids;
  rr.id_offset = 0;
  rr.xmax = v->xmax;
  const Bound bd = bound_for(v->d, f16 ? kF16 : ch.tc ? kTf32 : kSimt);
  rr.qinv = f16 ? w.qinv.as<float>() : nullptr;
  rr.cdot = g_force_fixup ? 1e30 : bd.cdot;
  rr.csum = bd.csum;
  rr.out_ids = reinterpret_cast<long long*>(ids);
  rr.out_d = dists;
  rr.ldo = ldo;
  TRY(ensure(w.fxs, fixup_scratch_bytes(B, k_max)));  // fix-up bounds + partial lists
  rr.fx_thr = static_cast<unsigned long long*>(w.fxs.p);
  rr.skip_far = (int)tri::g_rerank_skip;
  rr.n_flag = n_flag;
  rr.flag_list = flag_list;
  rr.B = B;
  rr.kp_max = kp_max;
  CU(launch_rerank(rr, st));
  TRY(mark(5));
  FixupLaunch fx;
  fx.n_flag = n_flag;
  fx.flag_list = flag_list;
  fx.meta = dmeta;
  fx.q64 = q;
  fx.d = v->d;
  fx.X = v->Xl;
  fx.ldx = v->dp;
  fx.n_rows = v->n;
  fx.probes = w.probes.as<long long>();
  fx.ld_probes = npmax;
  fx.nprobe = dnp;
  fx.list_off = v->list_off;
  fx.idmap = v->ids;
  fx.id_offset = 0;
  fx.out_ids = reinterpret_cast<long long*>(ids);
  fx.out_d = dists;
  fx.ldo = ldo;
  fx.B = B;
  fx.k_max = k_max;
  fx.fx_thr = static_cast<unsigned long long*>(w.fxs.p);
  fx.fx_cnt = reinterpret_cast<int*>(static_cast<unsigned char*>(w.fxs.p) + fixup_thr_bytes(B));
  fx.scratch = reinterpret_cast<Exact*>(static_cast<unsigned char*>(w.fxs.p) + fixup_thr_bytes(B) +
                                        fixup_cnt_bytes(B, k_max));
  fx.max_units = fixup_max_units(B, k_max);
  fx.slice_rows = (int)tri::g_fx_slice_rows;
  {
    const Bound bs = bound_for(v->d, kSimt);
    fx.Q32 = w.Q32.as<float>();
    fx.qld = v->qld;
    fx.qn32 = w.qn32.as<float>();
    fx.qn64 = w.qn64.as<double>();
    fx.xnorm = v->xnl;
    fx.xmax = v->xmax;
    fx.cdot = bs.cdot;
    fx.csum = bs.csum;
  }
  CU(launch_fixup(fx, st));
  TRY(mark(6));
  if (rec && !w.capturing) v->ev_used++;
  w.last_B = B;
  w.last_npmax = npmax;
  w.last_f16 = f16 ? 1 : 0;
  w.last_np.assign(nprobe, nprobe + B);
  return TRI_OK;
}


long long graph_opts() {
  return ((plan_opts() * 7 + g_tc_stages) * 1009 + g_scan_reserve) * 31 + g_force_fixup * 3 + g_gthr * 7 + g_scan_qbufs * 37 + g_coarse_tc * 13 + tri::g_coarse_split * 29 + g_f16_div * 131 + g_bound_margin * 523 + tri::g_dense_slices * 17 + tri::g_rerank_smem_cap * 3 + tri::g_rerank_f2f * 5 + tri::g_rerank_skip * 11 + tri::g_dense_fold * 3001 + tri::g_rerank_wide_slab * 577 + tri::g_rerank_lpt * 1931 + g_scan_pool * 37 + g_scan_early * 67 + g_scan_pool_pub * 41 + g_scan_pool_minkp * 47 + tri::g_fx_slice_rows * 7919 +
         g_scan_debug * 100003 + tri::g_pdl * 7907 + g_coarse_set * 7919 * 13 + g_pack_mixed * 104729 + g_scan_l2hint * 1000003 + g_scan_abufs * 10000019 + tri::g_rerank_split * 7 + tri::g_merge_split * 100019;
}


// Runs `body` (which enqueues one whole search on st) through the lane's CUDA
// graph cache.  A shape (mode, B, k[], nprobe[], ldo, buffers, options) seen
// once runs eagerly; the second time it is captured, instantiated and from
// then on replayed with one cudaGraphLaunch -- no host planning, no per-kernel
// launch latency.  Graph-owned pinned staging holds the uploaded plan, so
// replays never read a buffer another shape may overwrite; any scratch
// reallocation or plan rewrite (g_epoch) retires the graph.
}  // extern "C"

template <class Body>
static int graph_run(tri_ivf* v, Workspace& w, Workspace* cw, cudaStream_t st, int mode, int B, const int* k,
                     const int* np, int ldo, const void* q, const void* ids, const void* dists, Body&& body,
                     int nk) {
  if (nk < 0) nk = B;  // key entries of k[] / np[]: every query, or 1 (a padded batch's profile)
  // validity stamp of a captured graph: the global epoch (store-level changes)
  // plus the epochs of the workspaces it reads; all only grow, so the sum
  // changes exactly when one of them does
  auto stamp = [&]() { return g_epoch + w.epoch + (cw ? cw->epoch : 0); };
  if (v) set_reserve_now(v, st);
  if (!g_graphs) {
    ++g_gr_eager;
    return body();
  }
  const bool prof = v && v->prof && v->ev_used < kProfSearches;
  const long long opts = graph_opts() * 2 + (v && scan_reserve_for(v) > 0);
  Workspace::Graph* e = nullptr;
  for (auto& gr : w.graphs)
    if (gr.mode == mode && gr.B == B && gr.ldo == ldo && gr.q == q && gr.ids == ids && gr.dists == dists &&
        gr.prof == prof && gr.opts == opts && (int)gr.k.size() == nk && std::equal(gr.k.begin(), gr.k.end(), k) &&
        std::equal(gr.np.begin(), gr.np.end(), np)) {
      e = &gr;
      break;
    }
  if (!e) {
    if (w.graphs.size() >= 32) {  // evict the least recently used shape
      auto lru = std::min_element(w.graphs.begin(), w.graphs.end(),
                                  [](const Workspace::Graph& a, const Workspace::Graph& b) { return a.used < b.used; });
      lru->destroy();
      w.graphs.erase(lru);
    }
    w.graphs.emplace_back();
    e = &w.graphs.back();
    e->mode = mode;
    e->B = B;
    e->ldo = ldo;
    e->k.assign(k, k + nk);
    e->np.assign(np, np + nk);
    e->q = q;
    e->ids = ids;
    e->dists = dists;
    e->prof = prof;
    e->opts = opts;
  }
  e->used = ++w.graph_clock;
  if (e->state == 2 && e->epoch != stamp()) {  // scratch moved or plan rewritten since capture
    e->destroy();
    e->state = 0;
  }
  if (e->state == 0 || e->state == 3 || (e->state == 1 && e->epoch != stamp())) {
    ++g_gr_eager;
    const int rc = body();
    if (e->state != 3) {
      e->state = 1;
      e->epoch = stamp();
    }
    return rc;
  }
  if (e->state == 1) {
    // capture the second sighting of this shape
    nvtxRangePushA("tri.graph.capture");
    struct PopOnExit {
      ~PopOnExit() { nvtxRangePop(); }
    } pop_capture;
    TRY(ensure_host(e->host, (size_t)B * (sizeof(QueryMeta) + sizeof(int)) + 64));
    if (prof)
      for (auto& ev : e->ph)
        if (!ev) CU(cudaEventCreate(&ev));
    const long long ep0 = stamp();
    w.capturing = true;
    if (cw) cw->capturing = true;
    w.cap_host = &e->host;
    w.cap_ph = e->ph;
    cudaGraph_t gr = nullptr;
    cudaError_t ce = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    int rc = ce == cudaSuccess ? body() : TRI_ECUDA;
    if (ce == cudaSuccess) ce = cudaStreamEndCapture(st, &gr);
    if (ce == cudaSuccess && gr && std::getenv("TRI_GRAPH_DOT")) {  // debugging: the captured graph's nodes
      static int n_dot = 0;
      const std::string path = std::string(std::getenv("TRI_GRAPH_DOT")) + "." + std::to_string(n_dot++) + ".dot";
      cudaGraphDebugDotPrint(gr, path.c_str(), 0);
    }
    w.capturing = false;
    if (cw) cw->capturing = false;
    w.cap_host = nullptr;
    w.cap_ph = nullptr;
    cudaGraphExec_t ex = nullptr;
    if (rc == TRI_OK && ce == cudaSuccess && stamp() == ep0) ce = cudaGraphInstantiate(&ex, gr, 0);
    if (rc != TRI_OK || ce != cudaSuccess || stamp() != ep0 || !ex) {
      cudaGetLastError();
      if (gr) cudaGraphDestroy(gr);
      if (ex) cudaGraphExecDestroy(ex);
      e->state = (stamp() != ep0 && rc == TRI_OK && ce == cudaSuccess) ? 1 : 3;
      e->epoch = stamp();
      ++g_gr_eager;
      return body();  // not capturable: stay eager
    }
    if (prof) {
      size_t nn = 0;
      cudaGraphGetNodes(gr, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(gr, nodes.data(), &nn);
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t evx = nullptr;
        cudaGraphEventRecordNodeGetEvent(nd, &evx);
        for (int j = 0; j < 7; ++j)
          if (evx == e->ph[j]) e->evnode[j] = nd;
      }
    }
    // node handles stay valid for exec updates only while the graph lives; keep it
    // alive by instantiating from it and destroying it with the entry
    e->exec = ex;
    e->state = 2;
    e->epoch = stamp();
    e->last_B = w.last_B;
    e->last_npmax = w.last_npmax;
    e->last_f16 = w.last_f16;
    e->last_np = w.last_np;
    e->graph = gr;
    ++g_gr_captured;
  }
  // replay
  w.last_B = e->last_B;
  w.last_npmax = e->last_npmax;
  w.last_f16 = e->last_f16;
  w.last_np = e->last_np;
  if (prof) {
    while ((int)v->ev.size() < 7 * (v->ev_used + 1)) {
      cudaEvent_t ev;
      CU(cudaEventCreate(&ev));
      v->ev.push_back(ev);
    }
    for (int j = 0; j < 7; ++j)
      CU(cudaGraphExecEventRecordNodeSetEvent(e->exec, e->evnode[j], v->ev[7 * v->ev_used + j]));
  }
  nvtxRangePushA("tri.graph.replay");
  const cudaError_t le = cudaGraphLaunch(e->exec, st);
  nvtxRangePop();
  CU(le);
  ++g_gr_replayed;
  if (prof) v->ev_used++;
  return TRI_OK;
}


// ---------------------------------------------------------------------------
// Fixed-shape padded batches.  A batch whose shape would not repeat (ragged
// per-query k / nprobe, or a size that is not a power of two) runs as Bc =
// bucket(B) queries: dummies copy query 0 with k = nprobe = 1, the per-query
// plan is built on the device from an uploaded input, and the graph key is
// (Bc, max k, max nprobe) -- so a serving loop's ever-changing prefill /
// decode mixes replay a handful of captured graphs instead of planning every
// batch on the host ("round up with masked dummies").
static int bucket_of(int B) {
  int b = 16;
  while (b < B) b <<= 1;
  return b;
}

static bool uniform_shape(int B, const int* k, const int* np) {
  for (int i = 1; i < B; ++i)
    if (k[i] != k[0] || (np && np[i] != np[0])) return false;
  return true;
}

// plan input [B, 0, (k, nprobe) x Bc] for the next padded search on st
static int upload_ragged(Workspace& w, int B, int Bc, const int* k, const int* np, cudaStream_t st) {
  const size_t bytes = (size_t)(2 + 2 * Bc) * sizeof(int);
  int slot = 0;
  void* hp = nullptr;
  TRY(stage_host(w, bytes, &slot, &hp));
  int* h = static_cast<int*>(hp);
  h[0] = B;
  h[1] = 0;
  for (int i = 0; i < Bc; ++i) {
    h[2 + 2 * i] = i < B ? k[i] : 1;
    h[3 + 2 * i] = i < B ? (np ? np[i] : 1) : 1;
  }
  TRY(ensure(w.rplan, bytes));
  return staged_upload(w, slot, w.rplan.p, bytes, st);
}

static int ensure_padded(Workspace& w, int Bc, int d, int ldo) {
  TRY(ensure(w.qpad, (size_t)Bc * d * sizeof(double)));
  TRY(ensure(w.pad_ids, (size_t)Bc * ldo * sizeof(long long)));
  TRY(ensure(w.pad_d, (size_t)Bc * ldo * sizeof(double)));
  return TRI_OK;
}

// One padded IVF search on st: the B real query rows are already in w.qpad
// (copied there on the stream, outside the graph), results land in the first B
// rows of w.pad_ids / w.pad_d.  The graph touches only workspace buffers, so
// its key is (bucket, max k, max nprobe) whatever the caller's pointers are.
static int ivf_padded(tri_ivf* v, Workspace& w, Workspace* cw, cudaStream_t st, int B, const int* k, const int* np,
                      int ldo) {
  const int Bc = bucket_of(B);
  const int kmax = *std::max_element(k, k + B), npmax = *std::max_element(np, np + B);
  TRY(upload_ragged(w, B, Bc, k, np, st));
  TRY(ensure_query_bufs(w, Bc, v->d, v->qld));
  std::vector<int> kprof(Bc, kmax), npprof(Bc, npmax);
  TRY(graph_run(v, w, cw, st, 3, Bc, &kmax, &npmax, ldo, nullptr, nullptr, nullptr, [&]() -> int {
    const int* nB = w.rplan.as<int>();
    CU(launch_pad_rows(w.qpad.as<double>(), w.qpad.as<double>(), nB, Bc, v->d, st));
    return ivf_search_body(v, w, cw, w.qpad.as<double>(), Bc, kprof.data(), npprof.data(), ldo,
                           w.pad_ids.as<int64_t>(), w.pad_d.as<double>(), st, nB);
  }, 1));
  w.last_B = B;  // introspection (probes, scan bytes, fix-ups) sees the real batch
  w.last_np.assign(np, np + B);
  w.pad_real = B;
  if (cw) cw->pad_real = B;
  return TRI_OK;
}

// Padded brute force (uniform k): as ivf_padded.
static int bf_padded(tri_store* s, Workspace& w, cudaStream_t st, int B, const int* k, int ldo) {
  const int Bc = bucket_of(B);
  TRY(upload_ragged(w, B, Bc, k, nullptr, st));
  TRY(ensure_query_bufs(w, Bc, s->d, s->qld));
  std::vector<int> kk(Bc, k[0]);
  TRY(graph_run(nullptr, w, nullptr, st, 5, Bc, k, k, ldo, nullptr, nullptr, nullptr, [&]() -> int {
    const int* nB = w.rplan.as<int>();
    CU(launch_pad_rows(w.qpad.as<double>(), w.qpad.as<double>(), nB, Bc, s->d, st));
    return bruteforce_core(s, w, w, w.qpad.as<double>(), Bc, kk.data(), ldo, w.pad_ids.as<long long>(),
                           w.pad_d.as<double>(), st, true);
  }, 1));
  w.pad_real = B;
  return TRI_OK;
}

// Around a padded search: the B query rows in (any memory kind), the B result rows out.
static int padded_in(Workspace& w, const double* q, int B, int Bc, int d, int ldo, cudaStream_t st) {
  TRY(ensure_padded(w, Bc, d, ldo));
  CU(cudaMemcpyAsync(w.qpad.p, q, (size_t)B * d * sizeof(double), cudaMemcpyDefault, st));
  return TRI_OK;
}

static int padded_out(Workspace& w, int B, int ldo, int64_t* ids, double* dists, cudaStream_t st) {
  CU(cudaMemcpyAsync(ids, w.pad_ids.p, (size_t)B * ldo * sizeof(long long), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(dists, w.pad_d.p, (size_t)B * ldo * sizeof(double), cudaMemcpyDefault, st));
  return TRI_OK;
}

static bool pad_ivf(int B, const int* k, const int* np, bool pinned) {
  return g_graphs && g_ragged_graphs && !(pinned && uniform_shape(B, k, np) && B == bucket_of(B));
}

static bool pad_bf(int B, const int* k) {
  return g_graphs && g_ragged_graphs && uniform_shape(B, k, nullptr) && B != bucket_of(B);
}

extern "C" {

int tri_knn_bruteforce_dev(tri_store* s, const double* q, int32_t B, const int32_t* k, int32_t ldo, int64_t* ids,
                           double* dists, void* stream) {
  if (!s) return fail(TRI_EINVAL, "store is NULL");
  if (B < 0) return fail(TRI_EINVAL, "batch size must be >= 0");
  if (B == 0) return TRI_OK;
  TRY(validate_k(k, B, s->n, "k", false));
  int km = *std::max_element(k, k + B);
  if (ldo < km) return fail(TRI_EINVAL, "ldo=%d < max k=%d", ldo, km);
  std::lock_guard<std::mutex> lk(s->mu);
  DeviceGuard g(s->device);
  cudaStream_t st = pick(stream, s->own);
  Workspace* w = nullptr;
  TRY(s->lanes.get(st, &w));
  if (*std::max_element(k, k + B) > TRI_MAX_K) {
    w->pad_real = -1;
    TRY(bruteforce_exhaustive(s, *w, q, B, k, ldo, ids, dists, st));
    return lane_done(*w, st);
  }
  if (pad_bf(B, k)) {
    TRY(padded_in(*w, q, B, bucket_of(B), s->d, ldo, st));
    TRY(bf_padded(s, *w, st, B, k, ldo));
    TRY(padded_out(*w, B, ldo, ids, dists, st));
    return lane_done(*w, st);
  }
  TRY(ensure_query_bufs(*w, B, s->d, s->qld));
  w->pad_real = -1;
  TRY(graph_run(nullptr, *w, nullptr, st, 2, B, k, k, ldo, q, ids, dists, [&]() -> int {
    return bruteforce_core(s, *w, *w, q, B, k, ldo, reinterpret_cast<long long*>(ids), dists, st, true);
  }));
  return lane_done(*w, st);
}

int tri_ivf_search_dev(tri_ivf* v, const double* q, int32_t B, const int32_t* k, const int32_t* nprobe,
                       int32_t ldo, int64_t* ids, double* dists, void* stream) {
  TRY(ivf_validate(v, B, k, nprobe, ldo));
  if (B == 0) return TRI_OK;
  std::lock_guard<std::mutex> lk(v->mu);
  DeviceGuard g(v->device);
  cudaStream_t st = pick(stream, v->own);
  Workspace* wp = nullptr;
  Workspace* cw = nullptr;
  TRY(v->lanes.get(st, &wp));
  TRY(v->cstore->lanes.get(st, &cw));
  if (pad_ivf(B, k, nprobe, true)) {
    TRY(padded_in(*wp, q, B, bucket_of(B), v->d, ldo, st));
    TRY(ivf_padded(v, *wp, cw, st, B, k, nprobe, ldo));
    TRY(padded_out(*wp, B, ldo, ids, dists, st));
  } else {
    wp->pad_real = cw->pad_real = -1;
    TRY(graph_run(v, *wp, cw, st, 0, B, k, nprobe, ldo, q, ids, dists,
                  [&] { return ivf_search_body(v, *wp, cw, q, B, k, nprobe, ldo, ids, dists, st); }));
  }
  TRY(lane_done(*cw, st));
  return lane_done(*wp, st);
}

int tri_ivf_search(tri_ivf* v, const double* q, int32_t B, const int32_t* k, const int32_t* nprobe, int32_t ldo,
                   int64_t* ids, double* dists, void* stream) {
  TRY(ivf_validate(v, B, k, nprobe, ldo));
  if (B == 0) return TRI_OK;
  TRY(check_queries(q, (long long)B * v->d));
  DeviceGuard g(v->device);
  cudaStream_t st = pick(stream, v->own);
  const size_t ob = (size_t)B * ldo * sizeof(double);
  void* stage_ids = nullptr;
  void* stage_d = nullptr;
  {
    std::lock_guard<std::mutex> lk(v->mu);
    Workspace* wp = nullptr;
    Workspace* cw = nullptr;
    TRY(v->lanes.get(st, &wp));
    TRY(v->cstore->lanes.get(st, &cw));
    Workspace& w = *wp;
    const bool pinned = host_pinned(q) && host_pinned(ids) && host_pinned(dists);
    if (pad_ivf(B, k, nprobe, pinned)) {
      // queries straight into the padded buffer, one graph launch, results back
      // (through the lane's pinned buffers when the caller's are pageable, so
      // the index lock is never held across a wait)
      int64_t* oi = ids;
      double* od = dists;
      if (!(host_pinned(ids) && host_pinned(dists))) {
        TRY(ensure_host(w.h_bids, ob));
        TRY(ensure_host(w.h_bd, ob));
        oi = static_cast<int64_t*>(stage_ids = w.h_bids.p);
        od = static_cast<double*>(stage_d = w.h_bd.p);
      }
      TRY(padded_in(w, q, B, bucket_of(B), v->d, ldo, st));
      TRY(ivf_padded(v, w, cw, st, B, k, nprobe, ldo));
      TRY(padded_out(w, B, ldo, oi, od, st));
      TRY(lane_done(*cw, st));
      TRY(lane_done(w, st));
    } else {
    w.pad_real = cw->pad_real = -1;
    TRY(ensure(w.q64, (size_t)B * v->d * sizeof(double)));
    TRY(ensure(w.out_ids, (size_t)B * ldo * sizeof(long long)));
    TRY(ensure(w.out_d, (size_t)B * ldo * sizeof(double)));
    auto body = [&]() -> int {
      CU(cudaMemcpyAsync(w.q64.p, q, (size_t)B * v->d * sizeof(double), cudaMemcpyHostToDevice, st));
      TRY(ivf_search_body(v, w, cw, w.q64.as<double>(), B, k, nprobe, ldo, reinterpret_cast<int64_t*>(w.out_ids.p),
                          w.out_d.as<double>(), st));
      CU(cudaMemcpyAsync(ids, w.out_ids.p, (size_t)B * ldo * sizeof(long long), cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(dists, w.out_d.p, (size_t)B * ldo * sizeof(double), cudaMemcpyDeviceToHost, st));
      return TRI_OK;
    };
    // graph replay needs pinned host buffers (pageable copies cannot be captured)
    if (pinned) {
      TRY(graph_run(v, w, cw, st, 1, B, k, nprobe, ldo, q, ids, dists, body));
    } else {
      set_reserve_now(v, st);
      TRY(body());
    }
    TRY(lane_done(*cw, st));
    TRY(lane_done(w, st));
    }
  }
  CU(cudaStreamSynchronize(st));
  if (stage_ids) {
    std::memcpy(ids, stage_ids, ob);
    std::memcpy(dists, stage_d, ob);
  }
  return TRI_OK;
}

int tri_ivf_last_probes(tri_ivf* v, int64_t* probes, int32_t ld) {
  if (!v || !probes) return fail(TRI_EINVAL, "NULL argument");
  const Workspace& w = v->lanes.recent();
  if (ld < w.last_npmax) return fail(TRI_EINVAL, "ld=%d < nprobe max %d", ld, w.last_npmax);
  DeviceGuard g(v->device);
  CU(cudaDeviceSynchronize());
  std::vector<long long> h((size_t)w.last_B * w.last_npmax);
  if (!h.empty())
    CU(cudaMemcpy(h.data(), w.probes.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  for (int i = 0; i < w.last_B; ++i)
    for (int j = 0; j < ld; ++j)
      probes[(long long)i * ld + j] = j < w.last_np[i] ? h[(size_t)i * w.last_npmax + j] : -1;
  return TRI_OK;
}

int tri_ivf_last_fixups(tri_ivf* v, int32_t* n) {
  if (!v || !n) return fail(TRI_EINVAL, "NULL argument");
  DeviceGuard g(v->device);
  CU(cudaDeviceSynchronize());
  int a = 0, b = 0;
  const Workspace& w = v->lanes.recent();
  if (w.flags.p) CU(cudaMemcpy(&a, w.flags.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (v->cstore) {
    const Workspace& c = v->cstore->lanes.recent();
    if (c.flags.p) CU(cudaMemcpy(&b, c.flags.p, sizeof(int), cudaMemcpyDeviceToHost));
  }
  if (w.pad_real >= 0) {  // padded batch: dummies copy query 0
    a = std::min(a, w.pad_real);
    b = std::min(b, w.pad_real);
  }
  *n = a + b;
  return TRI_OK;
}

int tri_ivf_set_profiling(tri_ivf* v, int32_t on) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  v->prof = on != 0;
  for (double& x : v->stage_ms) x = 0.0;
  v->prof_n = 0;
  v->ev_used = 0;
  return TRI_OK;
}

static int ivf_collect(tri_ivf* v) {
  DeviceGuard g(v->device);
  for (int i = 0; i < v->ev_used; ++i) {
    CU(cudaEventSynchronize(v->ev[7 * i + 6]));
    for (int j = 0; j < kStagesProf; ++j) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, v->ev[7 * i + j], v->ev[7 * i + j + 1]));
      v->stage_ms[j] += ms;
    }
    v->prof_n += 1;
  }
  v->ev_used = 0;
  return TRI_OK;
}

int tri_ivf_scan_time(tri_ivf* v, double* total_ms, int32_t* launches) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  TRY(ivf_collect(v));
  if (total_ms) *total_ms = v->stage_ms[2];
  if (launches) *launches = v->prof_n;
  return TRI_OK;
}

int tri_ivf_stage_times(tri_ivf* v, double* ms, int32_t* searches) {
  if (!v || !ms) return fail(TRI_EINVAL, "NULL argument");
  TRY(ivf_collect(v));
  for (int j = 0; j < kStagesProf; ++j) ms[j] = v->stage_ms[j];
  if (searches) *searches = v->prof_n;
  return TRI_OK;
}

int tri_ivf_last_scan_bytes(tri_ivf* v, int64_t* bytes, int64_t* pairs) {
  if (!v) return fail(TRI_EINVAL, "index is NULL");
  const Workspace& w = v->lanes.recent();
  std::vector<int64_t> pr((size_t)w.last_B * std::max(1, w.last_npmax));
  TRY(tri_ivf_last_probes(v, pr.data(), std::max(1, w.last_npmax)));
  std::vector<char> hit(v->nlist, 0);
  long long pp = 0;
  for (int i = 0; i < w.last_B; ++i)
    for (int j = 0; j < w.last_np[i]; ++j) {
      long long l = pr[(size_t)i * w.last_npmax + j];
      hit[l] = 1;
      pp += v->h_off[l + 1] - v->h_off[l];
    }
  long long vec = 0;
  for (int l = 0; l < v->nlist; ++l)
    if (hit[l]) vec += v->h_off[l + 1] - v->h_off[l];
  if (bytes) *bytes = vec * ((long long)v->d * (w.last_f16 ? 2 : 4) + 4);  // row (fp16 / fp32) + its norm
  if (pairs) *pairs = pp;
  return TRI_OK;
}

int tri_ivf_last_scan_kind(tri_ivf* v, int32_t* kind) {
  if (!v || !kind) return fail(TRI_EINVAL, "null handle");
  const Workspace& w = v->lanes.recent();
  *kind = w.last_f16 ? 2 : (v->lanes.used ? 1 : 0);
  return TRI_OK;
}

int tri_debug_scan_ts(uint64_t* out, int32_t n) {
  CU(cudaDeviceSynchronize());
  CU(read_scan_ts(reinterpret_cast<unsigned long long*>(out), n));
  return TRI_OK;
}

int tri_debug_bound(int32_t d, int32_t mode, double* cdot, double* csum) {
  if (d < 1 || mode < 0 || mode > 3 || !cdot || !csum) return fail(TRI_EINVAL, "bad arguments");
  const Bound b = bound_for(d, mode);
  *cdot = b.cdot;
  *csum = b.csum;
  return TRI_OK;
}

int tri_ivf_debug_keys(tri_ivf* v, int32_t which, uint64_t* keys, int64_t cap, int64_t* n, int64_t* layout) {
  if (!v || !n) return fail(TRI_EINVAL, "NULL argument");
  if (which != 0 && which != 1) return fail(TRI_EINVAL, "which must be 0 (fine partial lists) or 1 (coarse lists)");
  DeviceGuard g(v->device);
  CU(cudaDeviceSynchronize());
  const Workspace& w = v->lanes.recent();
  const int B = w.last_B;
  if (which == 0) {
    std::vector<QueryMeta> m(B);
    if (B) CU(cudaMemcpy(m.data(), w.meta.p, (size_t)B * sizeof(QueryMeta), cudaMemcpyDeviceToHost));
    long long total = 0;
    for (int i = 0; i < B; ++i) {
      if (layout) {
        layout[3 * i] = m[i].part_off;
        layout[3 * i + 1] = m[i].kp;
        layout[3 * i + 2] = m[i].n_slots;
      }
      total = std::max(total, m[i].part_off + (long long)m[i].n_slots * m[i].kp);
    }
    *n = total;
    if (keys && total) {
      if (cap < total) return fail(TRI_EINVAL, "cap %lld < %lld keys", (long long)cap, total);
      CU(cudaMemcpy(keys, w.part.p, (size_t)total * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    }
    return TRI_OK;
  }
  const Workspace& c = v->cstore->lanes.recent();
  const long long total = (long long)B * c.kp_max;
  *n = total;
  if (layout) layout[0] = c.kp_max;
  if (keys && total) {
    if (cap < total) return fail(TRI_EINVAL, "cap %lld < %lld keys", (long long)cap, total);
    CU(cudaMemcpy(keys, c.merged.p, (size_t)total * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  }
  return TRI_OK;
}

int tri_merge_topk(const double* dists, const int64_t* ids, int32_t G, int32_t B, int32_t k_in, int32_t k_out,
                   double* out_dists, int64_t* out_ids, void* stream) {
  return tri_merge_topk_ld(dists, ids, G, B, k_in, k_in, (int64_t)B * k_in, k_out, out_dists, out_ids, k_out, stream);
}

int tri_merge_topk_ld(const double* dists, const int64_t* ids, int32_t G, int32_t B, int32_t k_in, int32_t ld_in,
                      int64_t g_stride, int32_t k_out, double* out_dists, int64_t* out_ids, int32_t ld_out,
                      void* stream) {
  if (G < 1 || B < 0 || k_in < 1 || k_out < 1) return fail(TRI_EINVAL, "bad merge shape");
  if (ld_in < k_in || ld_out < k_out) return fail(TRI_EINVAL, "ld_in=%d / ld_out=%d below k_in=%d / k_out=%d", ld_in,
                                                 ld_out, k_in, k_out);
  if (G > 1 && g_stride < (int64_t)B * ld_in) return fail(TRI_EINVAL, "g_stride=%lld below B*ld_in", (long long)g_stride);
  if ((long long)G * k_in > 8192) return fail(TRI_EINVAL, "G*k_in=%lld exceeds 8192", (long long)G * k_in);
  CU(launch_merge_exact(dists, reinterpret_cast<const long long*>(ids), G, B, k_in, k_out, out_dists,
                        reinterpret_cast<long long*>(out_ids), static_cast<cudaStream_t>(stream), ld_in, ld_out,
                        (long long)g_stride));
  return TRI_OK;
}

}  // extern "C"
