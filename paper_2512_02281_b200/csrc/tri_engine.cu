// Device-resident continuous-batching graph search (the reference's
// engine.ContinuousBatchEngine, pkg/src/trinity/engine.py:312-422).
//
// Every request lives in a device SLOT: its float64 query, its top-M list
// (fp64 distance, id, expanded flag) sorted by (dist, id), its visited bitmap
// over the store, and its counters (extends, no-change streak).  One launch of
// `engine_step_kernel` advances EVERY active request through exactly one
// extend -- one CTA per slot:
//
//   seed (admitted this step; engine.py:146-173)  ->  select parents
//   (engine.py:176-184)  ->  expand with test-and-set on the visited bitmap
//   (engine.py:187-205)  ->  exact distances of the emitted candidates in the
//   reference's float64 operation order (rowwise_sq_dists, ann_graph.py:97-105;
//   bit-identical)  ->  merge into top-M by (dist, id) (engine.py:259-275)  ->
//   early stop / finalize (engine.py:278-302).
//
// The reference's fixed-shape task array (build_task_array, engine.py:208-226)
// exists only to give its simulated GPU a static launch shape; its observable
// effect is the batch accounting, which depends only on the step's total
// emission count E: ceil(E / C) batches, the last one padded.  The kernel
// counts E per step and the host derives the identical EngineStats.  Results
// do not depend on how tasks are packed (a distance is independent of its
// batch, ann_graph.py:98-103).
//
// Steps run back to back on the device without host synchronisation; the host
// reads per-step counters (emissions, retirements, active count) once per
// chunk of steps, so run_to_completion costs one launch per extend.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/trinity_b200.h"
#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {
namespace {

constexpr int kEngMaxM = 4096;     // top-M capacity per request
constexpr int kEngMaxEmit = 8192;  // p * degree per extend
constexpr size_t kEngSmemCap = 200 * 1024;  // per CTA: slots per CTA shrink (4 -> 2 -> 1) for big m, p * degree
constexpr int kStats = 4;         // per-step counters: emissions, retired, active after, error
constexpr int kMaxChunk = 64;     // steps launched between host read-backs

enum SlotStatus : int { kFree = 0, kSeed = 1, kActive = 2 };
enum EngErr : int { kErrNone = 0, kErrRange = 1, kErrK = 2 };

struct EngineLaunch {
  const float* X;
  long long ldx;
  long long n;
  int d;
  const unsigned* adj;
  int D;
  int m, p, E, stop_streak, max_extends;
  int wpc;  // request slots (warps) per CTA
  int* status;
  const double* q64;
  const int* kq;
  const long long* rid;
  int* ext;
  int* streak;
  int* cnt;
  double* topd;
  int* topi;
  unsigned char* tope;
  unsigned* vis;
  long long vw;
  int* stats;  // this step's kStats counters
  int step;
  int n_slots;  // slots [0, n_slots) are launched
  // retirements (host drains after each chunk)
  int* res_n;
  long long* res_rid;
  int* res_ext;
  int* res_k;
  int* res_step;
  int* res_slot;
  int* res_ids;
  double* res_d;
};

__device__ __forceinline__ bool lt(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

// One WARP per request slot (kEngWarps slots per CTA): no block barriers, the
// request's lists live in the warp's slice of shared memory.
//   seed      strided entries floor(i*n/E) deduplicated, exact distances,
//             visited bits, sorted by rank counting
//   parents   ballot over the expanded flags, first p unexpanded in order
//   expand    one neighbour slot per lane: atomicOr test-and-set on the
//             visited bitmap, ballot compaction of the new ids
//   distances one candidate per lane, exact fp64 in the reference order
//   merge     old entry i -> rank i + #(new before it); new entry -> binary
//             search in the old list + #(new before it); entries past M drop
//   stop      ballots for "order changed" / "all expanded"
constexpr int kEngWarps = 4;

__global__ void __launch_bounds__(32 * kEngWarps) engine_step_kernel(EngineLaunch L) {
  extern __shared__ __align__(16) unsigned char eng_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * L.wpc + warp;
  if (s >= L.n_slots) return;
  const int st = L.status[s];
  if (st != kSeed && st != kActive) return;
  const int m = L.m, cap = m + L.p * L.D;
  // per-warp region: combined list (cap), merged list (m), parents (p)
  const size_t per_warp = (size_t)cap * 13 + (size_t)m * 13 + (size_t)L.p * 4 + 64;
  unsigned char* base = eng_smem + warp * ((per_warp + 15) & ~(size_t)15);
  double* cd = reinterpret_cast<double*>(base);
  double* od = cd + cap;
  int* ci = reinterpret_cast<int*>(od + m);
  int* oi = ci + cap;
  int* par = oi + m;
  unsigned char* ce = reinterpret_cast<unsigned char*>(par + L.p);
  unsigned char* oe = ce + cap;
  const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
  const double* q = L.q64 + (long long)s * L.d;
  unsigned* vis = L.vis + (long long)s * L.vw;
  const bool vec = (L.d & 1) == 0;  // double2 query loads need an even row stride
  auto dist_of = [&](int id) -> double {
    const float* x = L.X + (long long)id * L.ldx;
    return vec ? exact_sq_dist_v4(q, x, L.d) : exact_sq_dist(q, x, L.d);
  };
  auto less = [](double da, int ia, double db, int ib) { return da < db || (da == db && ia < ib); };

  int cnt;
  if (st == kSeed) {
    // entries floor(i*n/E), non-decreasing in i: keep the first of equal runs
    int c = 0;
    for (int b0 = 0; b0 < L.E; b0 += 32) {
      const int i = b0 + lane;
      bool keep = false;
      long long v = 0;
      if (i < L.E) {
        v = (long long)i * L.n / L.E;
        keep = i == 0 || v != (long long)(i - 1) * L.n / L.E;
      }
      const unsigned mk = __ballot_sync(FULL, keep);
      if (keep) ci[c + __popc(mk & lt)] = (int)v;
      c += __popc(mk);
    }
    __syncwarp();
    for (int i = lane; i < c; i += 32) {
      const int v = ci[i];
      cd[i] = dist_of(v);
      atomicOr(&vis[v >> 5], 1u << (v & 31));
    }
    __syncwarp();
    for (int i = lane; i < c; i += 32) {  // rank counting (ids unique)
      const double di = cd[i];
      const int ii = ci[i];
      int r = 0;
      for (int j = 0; j < c; ++j) r += less(cd[j], ci[j], di, ii);
      od[r] = di;
      oi[r] = ii;
    }
    __syncwarp();
    for (int i = lane; i < c; i += 32) {
      cd[i] = od[i];
      ci[i] = oi[i];
      ce[i] = 0;
    }
    cnt = c;
  } else {
    cnt = L.cnt[s];
    const long long b = (long long)s * m;
    for (int i = lane; i < cnt; i += 32) {
      cd[i] = L.topd[b + i];
      ci[i] = L.topi[b + i];
      ce[i] = L.tope[b + i];
    }
  }
  __syncwarp();

  // parents: the first <= p unexpanded entries in (dist, id) order
  int np = 0;
  for (int b0 = 0; b0 < cnt && np < L.p; b0 += 32) {
    unsigned mk = __ballot_sync(FULL, b0 + lane < cnt && !ce[b0 + lane]);
    while (mk && np < L.p) {
      const int bit = __ffs(mk) - 1;
      if (lane == 0) par[np] = b0 + bit;
      ++np;
      mk &= mk - 1;
    }
  }
  __syncwarp();

  // expand: test-and-set on the visited bitmap, ballot-compacted emissions
  int ne = 0, err = 0;
  const int slots = np * L.D;
  for (int t0 = 0; t0 < slots; t0 += 32) {
    const int t = t0 + lane;
    bool fresh = false;
    unsigned nid = 0;
    if (t < slots) {
      const int pi = t / L.D;
      nid = L.adj[(long long)ci[par[pi]] * L.D + (t - pi * L.D)];
      if ((long long)nid >= L.n) {
        err = 1;
      } else {
        const unsigned bit = 1u << (nid & 31);
        fresh = !(atomicOr(&vis[nid >> 5], bit) & bit);
      }
    }
    const unsigned mk = __ballot_sync(FULL, fresh);
    if (fresh) {
      ci[cnt + ne + __popc(mk & lt)] = (int)nid;
      ce[cnt + ne + __popc(mk & lt)] = 0;
    }
    ne += __popc(mk);
  }
  err = __any_sync(FULL, err);
  __syncwarp();
  for (int i = lane; i < np; i += 32) ce[par[i]] = 1;  // every parent, p may exceed 32

  // exact distances of the emissions, one candidate per lane
  for (int e = lane; e < ne; e += 32) cd[cnt + e] = dist_of(ci[cnt + e]);
  __syncwarp();

  // merge: ranks in the combined order; old list sorted, new ones unsorted
  const int newcnt = min(cnt + ne, m);
  for (int i = lane; i < cnt; i += 32) {
    const double di = cd[i];
    const int ii = ci[i];
    int r = i;
    for (int j = 0; j < ne; ++j) r += less(cd[cnt + j], ci[cnt + j], di, ii);
    if (r < m) {
      od[r] = di;
      oi[r] = ii;
      oe[r] = ce[i];
    }
  }
  for (int j = lane; j < ne; j += 32) {
    const double dj = cd[cnt + j];
    const int ij = ci[cnt + j];
    int lo = 0, hi = cnt;  // # old entries before it
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (less(cd[mid], ci[mid], dj, ij)) lo = mid + 1;
      else hi = mid;
    }
    int r = lo;
    for (int l = 0; l < ne; ++l) r += less(cd[cnt + l], ci[cnt + l], dj, ij);
    if (r < m) {
      od[r] = dj;
      oi[r] = ij;
      oe[r] = 0;
    }
  }
  __syncwarp();
  int diff = 0, unexp = 0;
  for (int r = lane; r < newcnt; r += 32) {
    diff |= (r >= cnt) || (oi[r] != ci[r]);
    unexp |= !oe[r];
  }
  const bool changed = ne > 0 && (__any_sync(FULL, diff) || newcnt != cnt);
  const bool all_expanded = !__any_sync(FULL, unexp);

  if (lane == 0) {
    if (ne) atomicAdd(&L.stats[0], ne);
    if (err) atomicMax(&L.stats[3], kErrRange);
  }
  const int extends = (st == kSeed ? 0 : L.ext[s]) + 1;
  const int streak = changed ? 0 : (st == kSeed ? 0 : L.streak[s]) + 1;
  const bool converged = streak >= L.stop_streak || all_expanded || extends >= L.max_extends;
  const int k = L.kq[s];
  if (converged) {  // finalize (engine.py:293-302): the first k entries
    int slot = -1;
    if (lane == 0) {
      if (k > newcnt) {
        atomicMax(&L.stats[3], kErrK);
      } else {
        slot = atomicAdd(L.res_n, 1);
        L.res_rid[slot] = L.rid[s];
        L.res_ext[slot] = extends;
        L.res_k[slot] = k;
        L.res_step[slot] = L.step;
        L.res_slot[slot] = s;
        atomicAdd(&L.stats[1], 1);
      }
      // free on the device; the host reuses it only after reading the record
      L.status[s] = kFree;
    }
    slot = __shfl_sync(FULL, slot, 0);
    if (slot >= 0)
      for (int r = lane; r < k; r += 32) {
        L.res_ids[(long long)slot * m + r] = oi[r];
        L.res_d[(long long)slot * m + r] = od[r];
      }
    return;
  }
  const long long b = (long long)s * m;
  for (int r = lane; r < newcnt; r += 32) {
    L.topd[b + r] = od[r];
    L.topi[b + r] = oi[r];
    L.tope[b + r] = oe[r];
  }
  if (lane == 0) {
    L.cnt[s] = newcnt;
    L.ext[s] = extends;
    L.streak[s] = streak;
    L.status[s] = kActive;
    atomicAdd(&L.stats[2], 1);
  }
}

size_t engine_warp_smem(int m, int p, int D) {
  const size_t cap = (size_t)m + (size_t)p * D;
  const size_t per_warp = cap * 13 + (size_t)m * 13 + (size_t)p * 4 + 64;
  return (per_warp + 15) & ~(size_t)15;
}

// slots per CTA: kEngWarps unless the per-warp lists are too big for that
int engine_wpc(int m, int p, int D) {
  int w = kEngWarps;
  while (w > 1 && (size_t)w * engine_warp_smem(m, p, D) > kEngSmemCap) w >>= 1;
  return w;
}

// Admission: copy the staged queries into their slots, reset counters and the
// visited bitmap (the reference's seed happens at submit; here it is the first
// thing the slot's next step does -- same values, engine.py:146-173).
__global__ void engine_admit_kernel(const int* __restrict__ slots, const long long* __restrict__ rids,
                                    const int* __restrict__ ks, const double* __restrict__ q, int d, int* status,
                                    double* q64, int* kq, long long* rid, unsigned* vis, long long vw) {
  const int a = blockIdx.x;
  const int s = slots[a];
  for (int i = threadIdx.x; i < d; i += blockDim.x) q64[(long long)s * d + i] = q[(long long)a * d + i];
  unsigned* v = vis + (long long)s * vw;
  for (long long i = threadIdx.x; i < vw; i += blockDim.x) v[i] = 0u;
  if (threadIdx.x == 0) {
    kq[s] = ks[a];
    rid[s] = rids[a];
    status[s] = kSeed;
  }
}

template <typename T>
cudaError_t grow(T*& p, size_t old_elems, size_t new_elems, cudaStream_t st) {
  T* np = nullptr;
  cudaError_t e = cudaMalloc(&np, new_elems * sizeof(T));
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(np, 0, new_elems * sizeof(T), st);
  if (e == cudaSuccess && p && old_elems) e = cudaMemcpyAsync(np, p, old_elems * sizeof(T), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    cudaFree(np);
    return e;
  }
  if (p) {
    cudaStreamSynchronize(st);
    cudaFree(p);
  }
  p = np;
  return cudaSuccess;
}

}  // namespace
}  // namespace tri

using namespace tri;

struct tri_engine {
  StoreView sv{};
  int D = 0, m = 0, p = 0, E = 0, C = 0, S = 0, maxext = 0;
  int wpc = 4;  // request slots per CTA of the step kernel
  unsigned* adj = nullptr;
  long long vw = 0;
  cudaStream_t st = nullptr;
  // slots
  int cap = 0, hw = 0;
  int *status = nullptr, *kq = nullptr, *ext = nullptr, *streak = nullptr, *cnt = nullptr;
  long long* rid = nullptr;
  double *q64 = nullptr, *topd = nullptr;
  int* topi = nullptr;
  unsigned char* tope = nullptr;
  unsigned* vis = nullptr;
  // retirements
  int* res_n = nullptr;
  long long* res_rid = nullptr;
  int *res_ext = nullptr, *res_k = nullptr, *res_step = nullptr, *res_slot = nullptr, *res_ids = nullptr;
  double* res_d = nullptr;
  int* stats = nullptr;  // kMaxChunk x kStats
  // admission staging
  int* a_slot = nullptr;
  long long* a_rid = nullptr;
  int* a_k = nullptr;
  double* a_q = nullptr;
  int a_cap = 0;
  // host state
  std::vector<int> free_slots;
  std::vector<long long> p_rid;
  std::vector<int> p_k;
  std::vector<double> p_q;
  long long next_rid = 0;
  int n_active = 0;
  // retired results not yet drained (flat, row stride m; drained from r_head)
  std::vector<long long> r_rid;
  std::vector<int> r_ext, r_k, r_step, r_ids;
  std::vector<double> r_d;
  size_t r_head = 0;
  // pinned staging: admission queries and retirement read-back
  double* h_q = nullptr;
  size_t h_q_cap = 0;
  void* h_res = nullptr;
  size_t h_res_cap = 0;
  // pinned read-back
  int* h_stats = nullptr;
  // device time of the step launches (CUDA events around each chunk)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double dev_ms = 0.0;
  long long dev_steps = 0;
  size_t smem = 0;  // dynamic shared memory of the step kernel
};

namespace {

#define ECU(expr)                                                                                     \
  do {                                                                                                \
    cudaError_t _e = (expr);                                                                          \
    if (_e != cudaSuccess) return set_error(TRI_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int ensure_pinned(void** p, size_t* cap, size_t bytes) {
  if (bytes <= *cap && *p) return TRI_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  const size_t want = std::max<size_t>(bytes + bytes / 2, 4096);
  ECU(cudaMallocHost(p, want));
  *cap = want;
  return TRI_OK;
}

int grow_slots(tri_engine* e, int need) {
  if (need <= e->cap) return TRI_OK;
  int nc = std::max(need, std::max(64, 2 * e->cap));
  const size_t oc = e->cap, ncz = nc, m = e->m, d = e->sv.d;
  cudaStream_t st = e->st;
  ECU(grow(e->status, oc, ncz, st));
  ECU(grow(e->kq, oc, ncz, st));
  ECU(grow(e->ext, oc, ncz, st));
  ECU(grow(e->streak, oc, ncz, st));
  ECU(grow(e->cnt, oc, ncz, st));
  ECU(grow(e->rid, oc, ncz, st));
  ECU(grow(e->q64, oc * d, ncz * d, st));
  ECU(grow(e->topd, oc * m, ncz * m, st));
  ECU(grow(e->topi, oc * m, ncz * m, st));
  ECU(grow(e->tope, oc * m, ncz * m, st));
  ECU(grow(e->vis, oc * e->vw, ncz * e->vw, st));
  // retirement buffers: at most one retirement per slot between read-backs
  ECU(grow(e->res_rid, 0, ncz, st));
  ECU(grow(e->res_ext, 0, ncz, st));
  ECU(grow(e->res_k, 0, ncz, st));
  ECU(grow(e->res_step, 0, ncz, st));
  ECU(grow(e->res_slot, 0, ncz, st));
  ECU(grow(e->res_ids, 0, ncz * m, st));
  ECU(grow(e->res_d, 0, ncz * m, st));
  for (int s = nc - 1; s >= e->cap; --s) e->free_slots.push_back(s);
  e->cap = nc;
  return TRI_OK;
}

// Admit every pending request into a free slot (engine.py:371-375).
int admit(tri_engine* e, int* admitted) {
  const int na = (int)e->p_rid.size();
  *admitted = na;
  if (!na) return TRI_OK;
  if ((int)e->free_slots.size() < na) {
    int rc = grow_slots(e, e->cap + na - (int)e->free_slots.size());
    if (rc) return rc;
  }
  if (na > e->a_cap) {
    int c = std::max(na, 2 * e->a_cap);
    ECU(grow(e->a_slot, 0, c, e->st));
    ECU(grow(e->a_rid, 0, c, e->st));
    ECU(grow(e->a_k, 0, c, e->st));
    ECU(grow(e->a_q, 0, (size_t)c * e->sv.d, e->st));
    e->a_cap = c;
  }
  std::vector<int> slots(na);
  for (int i = 0; i < na; ++i) {
    slots[i] = e->free_slots.back();
    e->free_slots.pop_back();
    e->hw = std::max(e->hw, slots[i] + 1);
  }
  ECU(cudaMemcpyAsync(e->a_slot, slots.data(), na * sizeof(int), cudaMemcpyHostToDevice, e->st));
  ECU(cudaMemcpyAsync(e->a_rid, e->p_rid.data(), na * sizeof(long long), cudaMemcpyHostToDevice, e->st));
  ECU(cudaMemcpyAsync(e->a_k, e->p_k.data(), na * sizeof(int), cudaMemcpyHostToDevice, e->st));
  {
    void* hp = e->h_q;
    int rc = ensure_pinned(&hp, &e->h_q_cap, e->p_q.size() * sizeof(double));
    if (rc) return rc;
    e->h_q = static_cast<double*>(hp);
    std::memcpy(e->h_q, e->p_q.data(), e->p_q.size() * sizeof(double));
    ECU(cudaMemcpyAsync(e->a_q, e->h_q, e->p_q.size() * sizeof(double), cudaMemcpyHostToDevice, e->st));
  }
  engine_admit_kernel<<<na, 256, 0, e->st>>>(e->a_slot, e->a_rid, e->a_k, e->a_q, e->sv.d, e->status, e->q64,
                                             e->kq, e->rid, e->vis, e->vw);
  ECU(cudaGetLastError());
  // the host vectors must outlive the async copies
  ECU(cudaStreamSynchronize(e->st));
  e->p_rid.clear();
  e->p_k.clear();
  e->p_q.clear();
  e->n_active += na;
  return TRI_OK;
}

EngineLaunch launch_of(tri_engine* e) {
  EngineLaunch L;
  L.X = e->sv.X;
  L.ldx = e->sv.ldx;
  L.n = e->sv.n;
  L.d = e->sv.d;
  L.adj = e->adj;
  L.D = e->D;
  L.m = e->m;
  L.p = e->p;
  L.E = e->E;
  L.stop_streak = e->S;
  L.max_extends = e->maxext;
  L.wpc = e->wpc;
  L.status = e->status;
  L.q64 = e->q64;
  L.kq = e->kq;
  L.rid = e->rid;
  L.ext = e->ext;
  L.streak = e->streak;
  L.cnt = e->cnt;
  L.topd = e->topd;
  L.topi = e->topi;
  L.tope = e->tope;
  L.vis = e->vis;
  L.vw = e->vw;
  L.res_n = e->res_n;
  L.res_rid = e->res_rid;
  L.res_ext = e->res_ext;
  L.res_k = e->res_k;
  L.res_step = e->res_step;
  L.res_slot = e->res_slot;
  L.res_ids = e->res_ids;
  L.res_d = e->res_d;
  return L;
}

// Read back this chunk's retirements (one pinned copy per field) and return
// their slots to the free list.
int collect(tri_engine* e) {
  int n = 0;
  ECU(cudaMemcpyAsync(&n, e->res_n, sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaStreamSynchronize(e->st));
  if (!n) return TRI_OK;
  const int m = e->m;
  const size_t scal = (size_t)n * (sizeof(long long) + 4 * sizeof(int));
  const size_t rows = (size_t)n * m * (sizeof(int) + sizeof(double));
  int rc = ensure_pinned(&e->h_res, &e->h_res_cap, scal + rows + 64);
  if (rc) return rc;
  char* h = static_cast<char*>(e->h_res);
  long long* rid = reinterpret_cast<long long*>(h);
  double* d = reinterpret_cast<double*>(rid + n);
  int* ext = reinterpret_cast<int*>(d + (size_t)n * m);
  int* k = ext + n;
  int* step = k + n;
  int* slot = step + n;
  int* ids = slot + n;
  ECU(cudaMemcpyAsync(rid, e->res_rid, n * sizeof(long long), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(d, e->res_d, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(ext, e->res_ext, n * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(k, e->res_k, n * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(step, e->res_step, n * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(slot, e->res_slot, n * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemcpyAsync(ids, e->res_ids, (size_t)n * m * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  ECU(cudaMemsetAsync(e->res_n, 0, sizeof(int), e->st));
  ECU(cudaStreamSynchronize(e->st));
  for (int i = 0; i < n; ++i) e->free_slots.push_back(slot[i]);
  e->n_active -= n;
  // reuse the lowest slots first so the step grid stays compact
  std::sort(e->free_slots.begin(), e->free_slots.end(), std::greater<int>());
  if (e->n_active == 0) e->hw = 0;
  // retirements in step order, ascending request id within a step (engine.py:398-411)
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return step[a] != step[b] ? step[a] < step[b] : rid[a] < rid[b]; });
  if (e->r_head > 0 && e->r_head == e->r_rid.size()) {  // everything drained: restart the buffers
    e->r_rid.clear();
    e->r_ext.clear();
    e->r_k.clear();
    e->r_step.clear();
    e->r_ids.clear();
    e->r_d.clear();
    e->r_head = 0;
  }
  for (int i : order) {
    e->r_rid.push_back(rid[i]);
    e->r_ext.push_back(ext[i]);
    e->r_k.push_back(k[i]);
    e->r_step.push_back(step[i]);
    e->r_ids.insert(e->r_ids.end(), ids + (size_t)i * m, ids + (size_t)(i + 1) * m);
    e->r_d.insert(e->r_d.end(), d + (size_t)i * m, d + (size_t)(i + 1) * m);
  }
  return TRI_OK;
}

}  // namespace

extern "C" {

int tri_engine_create(tri_store* s, const uint32_t* adjacency, int32_t degree, int32_t m, int32_t p,
                      int32_t entry_count, int32_t batch_capacity, int32_t stop_streak, int32_t max_extends,
                      tri_engine** out) {
  if (!out) return set_error(TRI_EINVAL, "out is NULL");
  StoreView sv;
  int rc = store_view(s, &sv);
  if (rc) return rc;
  if (degree < 1) return set_error(TRI_EINVAL, "degree must be >= 1, got %d", degree);
  if (!(1 <= p && p <= m)) return set_error(TRI_EINVAL, "p must be in [1, m=%d], got %d", m, p);
  if (!(1 <= entry_count && entry_count <= m))
    return set_error(TRI_EINVAL, "entry_count must be in [1, m=%d], got %d", m, entry_count);
  if (batch_capacity < 1) return set_error(TRI_EINVAL, "batch_capacity must be >= 1, got %d", batch_capacity);
  if (stop_streak < 1) return set_error(TRI_EINVAL, "stop_streak must be >= 1, got %d", stop_streak);
  if (max_extends < 1) return set_error(TRI_EINVAL, "max_extends must be >= 1, got %d", max_extends);
  if (m > kEngMaxM) return set_error(TRI_EINVAL, "the device engine supports m <= %d, got %d", kEngMaxM, m);
  if ((long long)p * degree > kEngMaxEmit)
    return set_error(TRI_EINVAL, "the device engine supports p * degree <= %d, got %lld", kEngMaxEmit,
                     (long long)p * degree);
  Guard g(sv.device);
  tri_engine* e = new tri_engine();
  e->sv = sv;
  e->D = degree;
  e->m = m;
  e->p = p;
  e->E = entry_count;
  e->C = batch_capacity;
  e->S = stop_streak;
  e->maxext = max_extends;
  e->vw = (sv.n + 31) / 32;
  auto bail = [&](int code) {
    tri_engine_destroy(e);
    return code;
  };
  if (cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking) != cudaSuccess)
    return bail(set_error(TRI_ECUDA, "stream creation failed"));
  const size_t adj_bytes = (size_t)sv.n * degree * sizeof(unsigned);
  if (cudaMalloc(&e->adj, adj_bytes) != cudaSuccess ||
      cudaMemcpyAsync(e->adj, adjacency, adj_bytes, cudaMemcpyHostToDevice, e->st) != cudaSuccess ||
      cudaStreamSynchronize(e->st) != cudaSuccess ||
      cudaMalloc(&e->res_n, sizeof(int)) != cudaSuccess || cudaMemsetAsync(e->res_n, 0, sizeof(int), e->st) != cudaSuccess ||
      cudaMalloc(&e->stats, kMaxChunk * kStats * sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&e->h_stats, kMaxChunk * kStats * sizeof(int)) != cudaSuccess ||
      cudaEventCreate(&e->ev0) != cudaSuccess || cudaEventCreate(&e->ev1) != cudaSuccess)
    return bail(set_error(TRI_ECUDA, "engine allocation failed"));
  e->wpc = engine_wpc(m, p, degree);
  e->smem = (size_t)e->wpc * engine_warp_smem(m, p, degree);
  if (e->smem > kEngSmemCap)
    return bail(set_error(TRI_EINVAL, "m=%d, p*degree=%lld need %zu bytes of shared memory per request (max %zu)", m,
                          (long long)p * degree, e->smem, kEngSmemCap));
  if (e->smem > 48 * 1024 &&
      cudaFuncSetAttribute(engine_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e->smem) != cudaSuccess)
    return bail(set_error(TRI_ECUDA, "engine shared memory %zu bytes not available", e->smem));
  rc = grow_slots(e, 64);
  if (rc) return bail(rc);
  *out = e;
  return TRI_OK;
}

int tri_engine_destroy(tri_engine* e) {
  if (!e) return TRI_OK;
  Guard g(e->sv.device);
  if (e->st) cudaStreamSynchronize(e->st);
  void* bufs[] = {e->adj, e->status, e->kq, e->ext, e->streak, e->cnt, e->rid, e->q64, e->topd, e->topi,
                  e->tope, e->vis, e->res_n, e->res_rid, e->res_ext, e->res_k, e->res_step, e->res_slot, e->res_ids,
                  e->res_d, e->stats, e->a_slot, e->a_rid, e->a_k, e->a_q};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (e->h_stats) cudaFreeHost(e->h_stats);
  if (e->h_q) cudaFreeHost(e->h_q);
  if (e->h_res) cudaFreeHost(e->h_res);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->st) cudaStreamDestroy(e->st);
  delete e;
  return TRI_OK;
}

int tri_engine_submit(tri_engine* e, const double* q, int32_t k, int64_t* rid) {
  if (!e || !q) return set_error(TRI_EINVAL, "null argument");
  for (int i = 0; i < e->sv.d; ++i)
    if (!std::isfinite(q[i])) return set_error(TRI_EINVAL, "query must be finite");
  if (!(1 <= k && k <= e->m)) return set_error(TRI_EINVAL, "k must be in [1, m=%d], got %d", e->m, k);
  const long long r = e->next_rid++;
  e->p_rid.push_back(r);
  e->p_k.push_back(k);
  e->p_q.insert(e->p_q.end(), q, q + e->sv.d);
  if (rid) *rid = r;
  return TRI_OK;
}

int tri_engine_submit_batch(tri_engine* e, const double* q, int32_t B, const int32_t* k, int64_t* rids) {
  if (!e || (B > 0 && (!q || !k))) return set_error(TRI_EINVAL, "null argument");
  const long long n = (long long)B * e->sv.d;
  for (long long i = 0; i < n; ++i)
    if (!std::isfinite(q[i])) return set_error(TRI_EINVAL, "query must be finite");
  for (int i = 0; i < B; ++i)
    if (!(1 <= k[i] && k[i] <= e->m)) return set_error(TRI_EINVAL, "k must be in [1, m=%d], got %d", e->m, k[i]);
  for (int i = 0; i < B; ++i) {
    const long long r = e->next_rid++;
    e->p_rid.push_back(r);
    e->p_k.push_back(k[i]);
    if (rids) rids[i] = r;
  }
  e->p_q.insert(e->p_q.end(), q, q + n);
  return TRI_OK;
}

int tri_engine_device_time(tri_engine* e, double* ms, int64_t* steps) {
  if (!e) return set_error(TRI_EINVAL, "engine is NULL");
  if (ms) *ms = e->dev_ms;
  if (steps) *steps = e->dev_steps;
  return TRI_OK;
}

// White-box read of one active request's state (the reference's
// SearchRequestState, engine.py:70-83): top-M (dist, id, expanded) in list
// order, the visited bitmap, extends and no-change streak.  Synchronises the
// engine stream; introspection only (the reference's tests read
// ContinuousBatchEngine._active, test_engine.py:304-332).
int tri_engine_request_state(tri_engine* e, int64_t rid, int32_t* found, int32_t* n_top, double* top_d,
                             int32_t* top_i, uint8_t* top_e, uint32_t* visited, int32_t* extends, int32_t* streak) {
  if (!e || !found) return set_error(TRI_EINVAL, "NULL argument");
  *found = 0;
  Guard g(e->sv.device);
  ECU(cudaStreamSynchronize(e->st));
  if (e->hw <= 0) return TRI_OK;
  std::vector<int> st(e->hw);
  std::vector<long long> rids(e->hw);
  ECU(cudaMemcpy(st.data(), e->status, e->hw * sizeof(int), cudaMemcpyDeviceToHost));
  ECU(cudaMemcpy(rids.data(), e->rid, e->hw * sizeof(long long), cudaMemcpyDeviceToHost));
  int s = -1;
  for (int i = 0; i < e->hw; ++i)
    if (st[i] == kActive && rids[i] == rid) s = i;
  if (s < 0) return TRI_OK;
  int n = 0;
  ECU(cudaMemcpy(&n, e->cnt + s, sizeof(int), cudaMemcpyDeviceToHost));
  const long long b = (long long)s * e->m;
  if (top_d) ECU(cudaMemcpy(top_d, e->topd + b, n * sizeof(double), cudaMemcpyDeviceToHost));
  if (top_i) ECU(cudaMemcpy(top_i, e->topi + b, n * sizeof(int), cudaMemcpyDeviceToHost));
  if (top_e) ECU(cudaMemcpy(top_e, e->tope + b, n * sizeof(unsigned char), cudaMemcpyDeviceToHost));
  if (visited) ECU(cudaMemcpy(visited, e->vis + (long long)s * e->vw, e->vw * sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (extends) ECU(cudaMemcpy(extends, e->ext + s, sizeof(int), cudaMemcpyDeviceToHost));
  if (streak) ECU(cudaMemcpy(streak, e->streak + s, sizeof(int), cudaMemcpyDeviceToHost));
  if (n_top) *n_top = n;
  *found = 1;
  return TRI_OK;
}

int tri_engine_counts(tri_engine* e, int32_t* active, int32_t* pending) {
  if (!e) return set_error(TRI_EINVAL, "engine is NULL");
  if (active) *active = e->n_active;
  if (pending) *pending = (int32_t)e->p_rid.size();
  return TRI_OK;
}

int tri_engine_run(tri_engine* e, int32_t max_steps, int32_t until_idle, int32_t* steps_done,
                   int64_t* emissions, int32_t* admitted, int32_t* retired) {
  if (!e) return set_error(TRI_EINVAL, "engine is NULL");
  if (max_steps < 0) return set_error(TRI_EINVAL, "max_steps must be >= 0");
  Guard g(e->sv.device);
  int done = 0;
  if (steps_done) *steps_done = 0;
  if (until_idle && e->n_active == 0 && e->p_rid.empty()) return TRI_OK;
  int chunk = 4;
  while (done < max_steps) {
    int adm = 0;
    if (done == 0) {
      int rc = admit(e, &adm);
      if (rc) return rc;
    }
    const int n = std::min({chunk, kMaxChunk, max_steps - done});
    ECU(cudaMemsetAsync(e->stats, 0, n * kStats * sizeof(int), e->st));
    EngineLaunch L = launch_of(e);
    L.n_slots = e->hw;
    ECU(cudaEventRecord(e->ev0, e->st));
    for (int i = 0; i < n; ++i) {
      L.stats = e->stats + i * kStats;
      L.step = done + i;
      if (e->hw > 0)
        engine_step_kernel<<<(e->hw + e->wpc - 1) / e->wpc, 32 * e->wpc, e->smem, e->st>>>(L);
    }
    ECU(cudaGetLastError());
    ECU(cudaEventRecord(e->ev1, e->st));
    ECU(cudaMemcpyAsync(e->h_stats, e->stats, n * kStats * sizeof(int), cudaMemcpyDeviceToHost, e->st));
    int rc = collect(e);  // synchronises
    if (rc) return rc;
    float ms = 0.f;
    ECU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    int used = n;
    for (int i = 0; i < n; ++i) {
      const int* sti = e->h_stats + i * kStats;
      if (sti[3] == kErrRange)
        return set_error(TRI_EINTERNAL, "candidate id out of range [0, %lld) (engine.py:249-250)", e->sv.n);
      if (sti[3] == kErrK) return set_error(TRI_EINVAL, "k exceeds top-M length (engine.py:299-300)");
      if (emissions) emissions[done + i] = sti[0];
      if (retired) retired[done + i] = sti[1];
      if (admitted) admitted[done + i] = (done + i == 0) ? adm : 0;
      if (until_idle && sti[2] == 0) {
        used = i + 1;
        break;
      }
    }
    done += used;
    e->dev_ms += ms * used / n;  // steps past idle are empty launches
    e->dev_steps += used;
    if (until_idle && e->h_stats[(used - 1) * kStats + 2] == 0) break;
    chunk = std::min(kMaxChunk, chunk * 2);
  }
  if (steps_done) *steps_done = done;
  return TRI_OK;
}

int tri_engine_retired(tri_engine* e, int32_t cap, int32_t ld, int32_t* n, int64_t* rids, int32_t* extends,
                       int32_t* ks, int32_t* steps, int64_t* ids, double* dists) {
  if (!e || !n) return set_error(TRI_EINVAL, "null argument");
  const int m = e->m;
  const int cnt = std::min<int>(cap, (int)(e->r_rid.size() - e->r_head));
  for (int i = 0; i < cnt; ++i) {
    const size_t r = e->r_head + i;
    const int k = e->r_k[r];
    if (rids) rids[i] = e->r_rid[r];
    if (extends) extends[i] = e->r_ext[r];
    if (ks) ks[i] = k;
    if (steps) steps[i] = e->r_step[r];
    const int w = std::min(k, (int)ld);
    for (int j = 0; j < w; ++j) {
      if (ids) ids[(size_t)i * ld + j] = e->r_ids[r * m + j];
      if (dists) dists[(size_t)i * ld + j] = e->r_d[r * m + j];
    }
  }
  e->r_head += cnt;
  *n = cnt;
  return TRI_OK;
}

int tri_engine_retired_by_id(tri_engine* e, int64_t capacity, int32_t ld, int32_t* n, int64_t* rids, int32_t* ids,
                             double* dists, int32_t* extends, int32_t* ks) {
  if (!e || !n) return set_error(TRI_EINVAL, "null argument");
  const int m = e->m;
  const size_t avail = e->r_rid.size() - e->r_head;
  for (size_t i = 0; i < avail; ++i)
    if (e->r_rid[e->r_head + i] >= capacity)
      return set_error(TRI_EINVAL, "request id %lld >= capacity %lld", e->r_rid[e->r_head + i], (long long)capacity);
  for (size_t i = 0; i < avail; ++i) {
    const size_t r = e->r_head + i;
    const long long id = e->r_rid[r];
    const int k = e->r_k[r], w = std::min(k, (int)ld);
    if (rids) rids[i] = id;
    if (ids) std::memcpy(ids + id * ld, e->r_ids.data() + r * m, w * sizeof(int32_t));
    if (dists) std::memcpy(dists + id * ld, e->r_d.data() + r * m, w * sizeof(double));
    if (extends) extends[id] = e->r_ext[r];
    if (ks) ks[id] = k;
  }
  e->r_head += avail;
  *n = (int32_t)avail;
  return TRI_OK;
}

int tri_engine_pending_retired(tri_engine* e, int32_t* n) {
  if (!e || !n) return set_error(TRI_EINVAL, "null argument");
  *n = (int32_t)(e->r_rid.size() - e->r_head);
  return TRI_OK;
}

}  // extern "C"
