// IVF-Flat device pieces: the continuous-batch packer (ragged per-query k and
// nprobe -> list-major work items in one launch) and the k-means / inverted
// list layout used at index build.
#include "tri_common.cuh"
#include "tri_internal.h"

#include <algorithm>

namespace tri {

// ---------------------------------------------------------------------------
// Packer.  Given each query's probed lists (from the exact coarse step) build
//   * per (list, capacity-class) member counts,
//   * work items in descending list-size order (longest-processing-time first
//     for the persistent scan), one per group of <= gmax queries,
//   * the members: (query, partial-list slot) pairs.
// Member order inside a group is atomic-order dependent, which never changes
// results: a (query, row) distance is computed by the same instruction chain in
// whichever group position the query lands.

__global__ void pack_hist_kernel(PackLaunch p) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int q = blockIdx.x;
  const int np = p.nprobe[q];
  const int cls = p.mixed ? 0 : p.meta[q].cls;
  long long tot = 0;
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    long long l = p.probes[(long long)q * p.ld_probes + j];
    if (l < 0) continue;  // non-finite query: its coarse step returned no lists
    atomicAdd(&p.counts[l * kNumCls + cls], 1);
    tot += p.list_off[l + 1] - p.list_off[l];
  }
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  __shared__ long long part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    p.meta[q].n_total = s;
  }
}

__global__ void __launch_bounds__(1024) pack_items_kernel(PackLaunch p) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  __shared__ int s_mem[32], s_grp[32];
  __shared__ int carry_mem, carry_grp;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    carry_mem = 0;
    carry_grp = 0;
  }
  __syncthreads();
  int pc[kNumCls], npc = 0;  // capacity classes present in this batch (one slot when mixed)
  for (int c = 0; c < kNumCls; ++c)
    if (p.mixed ? c == 0 : (p.cls_mask & (1 << c))) pc[npc++] = c;
  const int E = p.nlist * npc;
  for (int base = 0; base < E; base += 1024) {
    const int e = base + tid;
    int cnt = 0, ngrp = 0, l = 0, cls = 0;
    long long lsize = 0;
    if (e < E) {
      l = p.list_by_size[e / npc];
      cls = pc[e % npc];
      cnt = p.counts[l * kNumCls + cls];
      lsize = p.list_off[l + 1] - p.list_off[l];
      ngrp = (cnt > 0 && lsize > 0) ? (cnt + p.gmax - 1) / p.gmax : 0;
    }
    // block exclusive scan of (cnt, ngrp)
    int im = cnt, ig = ngrp;
    for (int o = 1; o < 32; o <<= 1) {
      int a = __shfl_up_sync(0xffffffffu, im, o), b = __shfl_up_sync(0xffffffffu, ig, o);
      if (lane >= o) {
        im += a;
        ig += b;
      }
    }
    if (lane == 31) {
      s_mem[warp] = im;
      s_grp[warp] = ig;
    }
    __syncthreads();
    if (warp == 0) {
      int vm = s_mem[lane], vg = s_grp[lane];
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(0xffffffffu, vm, o), b = __shfl_up_sync(0xffffffffu, vg, o);
        if (lane >= o) {
          vm += a;
          vg += b;
        }
      }
      s_mem[lane] = vm;
      s_grp[lane] = vg;
    }
    __syncthreads();
    const int mem_before = carry_mem + (warp ? s_mem[warp - 1] : 0) + im - cnt;
    const int grp_before = carry_grp + (warp ? s_grp[warp - 1] : 0) + ig - ngrp;
    if (e < E) {
      p.member_base[l * kNumCls + cls] = mem_before;
      if (p.mixed) p.counts[l * kNumCls + 1] = grp_before;  // class slot 1 is unused when mixed
      for (int g = 0; g < ngrp; ++g) {
        WorkItem w;
        w.row_begin = p.list_off[l];
        w.row_count = (int)lsize;
        w.member_begin = mem_before + g * p.gmax;
        w.member_count = min(p.gmax, cnt - g * p.gmax);
        w.kp = p.mixed ? kMinKp : kMinKp << cls;  // mixed: raised to the members' max by pack_fill
        w.pad0 = l;
        w.pad1 = 0;
        p.items[grp_before + g] = w;
      }
    }
    __syncthreads();
    if (tid == 0) {
      carry_mem += s_mem[31];
      carry_grp += s_grp[31];
    }
    __syncthreads();
  }
  if (tid == 0) *p.n_items = carry_grp;
}

__global__ void pack_fill_kernel(PackLaunch p) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int q = blockIdx.x;
  const int np = p.nprobe[q];
  const QueryMeta m = p.meta[q];
  const int cls = p.mixed ? 0 : m.cls;
  for (int j = threadIdx.x; j < np; j += blockDim.x) {
    long long l = p.probes[(long long)q * p.ld_probes + j];
    if (l < 0) continue;
    int slot = atomicAdd(&p.fill[l * kNumCls + cls], 1);
    Member mb;
    mb.q = q;
    mb.pad = m.kp;
    mb.slot = m.part_off + (long long)j * m.kp;
    p.members[p.member_base[l * kNumCls + cls] + slot] = mb;
    if (p.mixed) atomicMax(&p.items[p.counts[l * kNumCls + 1] + slot / p.gmax].kp, m.kp);
  }
}

cudaError_t launch_pack(const PackLaunch& p, cudaStream_t st) {
  if (p.B <= 0) return cudaSuccess;
  size_t cbytes = (size_t)p.nlist * kNumCls * sizeof(int);
  cudaError_t e = cudaMemsetAsync(p.counts, 0, cbytes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.fill, 0, cbytes, st);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(pack_hist_kernel, p.B, 64, 0, st, p);
  (void)launch_pdl(pack_items_kernel, 1, 1024, 0, st, p);
  (void)launch_pdl(pack_fill_kernel, p.B, 64, 0, st, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fixed-shape ragged batches (CUDA graphs for any prefill / decode mix).  A
// batch of B queries runs as a padded batch of Bc = bucket(B) queries whose
// plan is built HERE from an uploaded input, so one captured graph per
// (Bc, max k, max nprobe) replays for every mix -- the paper's fixed-shape
// step (engine.py:208-226: round up with masked dummies).
//   in[0] = B (real queries), in[1] unused, in[2 + 2 i] = k_i, in[3 + 2 i] = nprobe_i
// Dummies (i >= B) carry k = 1, nprobe = 1 and a copy of query 0, and their
// outputs stay in the padded workspace rows.

__device__ __forceinline__ int ragged_kp(int k, const RaggedPlan& r) {
  long long want;
  if (r.f16) want = (long long)k + max(16LL, (long long)k / max(1, r.f16_div)) + r.kp_extra;
  else want = (long long)k + (r.tc ? max(16LL, (long long)k) : max(16LL, (long long)k / 4)) + r.kp_extra;
  int kp = kMinKp;
  while (kp < want) kp <<= 1;
  return kp;
}

__global__ void __launch_bounds__(1024) ragged_plan_kernel(RaggedPlan r) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  __shared__ long long s_warp[32];
  __shared__ long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < r.Bc; base += 1024) {
    const int i = base + tid;
    int k = 0, np = 0, kp = 0;
    if (i < r.Bc) {
      k = r.in[2 + 2 * i];
      np = r.in[3 + 2 * i];
      kp = ragged_kp(k, r);
    }
    const long long keys = (long long)np * kp;
    long long x = keys;
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long v = s_warp[lane];
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      s_warp[lane] = v;
    }
    __syncthreads();
    const long long before = s_carry + (warp ? s_warp[warp - 1] : 0) + x - keys;
    if (i < r.Bc) {
      QueryMeta m;
      m.k = k;
      m.kp = kp;
      m.n_slots = np;
      int c = 0;
      while ((kMinKp << c) < kp) ++c;
      m.cls = c;
      m.part_off = before;
      m.n_total = 0;
      r.meta[i] = m;
      r.nprobe[i] = np;
    }
    __syncthreads();
    if (tid == 0) s_carry += s_warp[31];
    __syncthreads();
  }
  if (tid == 0) *r.total_keys = s_carry;
}

cudaError_t launch_ragged_plan(const RaggedPlan& r, cudaStream_t st) {
  (void)launch_pdl(ragged_plan_kernel, 1, 1024, 0, st, r);
  return cudaGetLastError();
}

// Every partial-list key starts as "empty" (all ones); the count comes from the plan.
__global__ void fill_keys_kernel(unsigned long long* __restrict__ p, const long long* __restrict__ count) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const long long n = *count;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = ~0ull;
}

cudaError_t launch_fill_keys(unsigned long long* p, const long long* count, int grid, cudaStream_t st) {
  (void)launch_pdl(fill_keys_kernel, grid, 512, 0, st, p, count);
  return cudaGetLastError();
}

// dst row i = src row i for i < B, src row 0 otherwise (B read on the device);
// src == dst pads in place.
__global__ void pad_rows_kernel(const double* __restrict__ src, double* __restrict__ dst, const int* __restrict__ nB,
                                int Bc, int d) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int B = *nB;
  const long long total = (long long)Bc * d;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / d, c = e - r * d;
    if (r < B) {
      if (src != dst) dst[e] = src[e];
    } else {
      dst[e] = src[c];
    }
  }
}

cudaError_t launch_pad_rows(const double* src, double* dst, const int* nB, int Bc, int d, cudaStream_t st) {
  const long long total = (long long)Bc * d;
  const int grid = (int)std::min<long long>((total + 255) / 256, 1184);
  (void)launch_pdl(pad_rows_kernel, grid, 256, 0, st, src, dst, nB, Bc, d);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------

__global__ void counts_kernel(const int* __restrict__ assign, long long n, int* counts) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&counts[assign[i]], 1);
}

// Exact k-means assignment helpers: rows widened to the float64 queries the
// exact brute force takes, and its int64 top-1 ids narrowed to list ids.
__global__ void rows_to_f64_kernel(const float* __restrict__ X, long long ldx, long long n, int d,
                                   double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * d) return;
  const long long r = i / d;
  out[i] = (double)X[r * ldx + (i - r * d)];
}

cudaError_t launch_rows_to_f64(const float* X, long long ldx, long long n, int d, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  rows_to_f64_kernel<<<(unsigned)((n * d + 255) / 256), 256, 0, st>>>(X, ldx, n, d, out);
  return cudaGetLastError();
}

__global__ void narrow_ids_kernel(const long long* __restrict__ ids, long long n, int* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)ids[i];
}

cudaError_t launch_narrow_ids(const long long* ids, long long n, int* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  narrow_ids_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ids, n, out);
  return cudaGetLastError();
}

cudaError_t launch_counts(const int* assign, long long n, int nlist, int* counts, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)nlist * sizeof(int), st);
  if (e != cudaSuccess || n <= 0) return e;
  counts_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(assign, n, counts);
  return cudaGetLastError();
}

// One CTA per list: ballot-compact the ids assigned to it, in ascending order.
__global__ void __launch_bounds__(1024) list_members_kernel(const int* __restrict__ assign, long long n,
                                                            const long long* __restrict__ offsets,
                                                            long long* __restrict__ perm) {
  __shared__ int wsum[32];
  __shared__ long long s_run;
  const int l = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_run = offsets[l];
  __syncthreads();
  for (long long base = 0; base < n; base += 1024) {
    long long i = base + threadIdx.x;
    bool hit = i < n && assign[i] == l;
    unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < 32; ++w) {
      int v = wsum[w];
      if (w < warp) before += v;
      total += v;
    }
    if (hit) perm[s_run + before + __popc(m & ((1u << lane) - 1))] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_run += total;
    __syncthreads();
  }
}

cudaError_t launch_list_members(const int* assign, long long n, int nlist, const long long* offsets,
                                long long* perm, cudaStream_t st) {
  if (nlist <= 0) return cudaSuccess;
  list_members_kernel<<<nlist, 1024, 0, st>>>(assign, n, offsets, perm);
  return cudaGetLastError();
}

// Deterministic mean: members summed in ascending id order in float64.
__global__ void __launch_bounds__(256) centroid_update_kernel(const float* __restrict__ X, long long ldx, int d,
                                                              const long long* __restrict__ perm,
                                                              const long long* __restrict__ offsets,
                                                              float* __restrict__ C, long long ldc) {
  const int l = blockIdx.x;
  const long long lo = offsets[l], hi = offsets[l + 1];
  if (hi <= lo) return;  // empty list keeps its previous centroid
  const double inv = 1.0 / (double)(hi - lo);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    long long m = lo;
    for (; m + 4 <= hi; m += 4) {
      float a = X[perm[m] * ldx + j], b = X[perm[m + 1] * ldx + j];
      float c = X[perm[m + 2] * ldx + j], e = X[perm[m + 3] * ldx + j];
      s += (double)a;
      s += (double)b;
      s += (double)c;
      s += (double)e;
    }
    for (; m < hi; ++m) s += (double)X[perm[m] * ldx + j];
    C[(long long)l * ldc + j] = __double2float_rn(s * inv);
  }
}

cudaError_t launch_centroid_update(const float* X, long long ldx, int d, const long long* perm,
                                   const long long* offsets, int nlist, float* C, long long ldc, cudaStream_t st) {
  if (nlist <= 0) return cudaSuccess;
  centroid_update_kernel<<<nlist, 256, 0, st>>>(X, ldx, d, perm, offsets, C, ldc);
  return cudaGetLastError();
}

__global__ void gather_rows_kernel(const float* __restrict__ X, long long ldx, const long long* __restrict__ perm,
                                   long long n, int dp, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const float4* src = reinterpret_cast<const float4*>(X + perm[r] * ldx);
  float4* dst = reinterpret_cast<float4*>(out + r * (long long)dp);
  for (int j = lane; j < dp / 4; j += 32) dst[j] = src[j];
}

cudaError_t launch_gather_rows(const float* X, long long ldx, const long long* perm, long long n, int dp,
                               float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  gather_rows_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(X, ldx, perm, n, dp, out);
  return cudaGetLastError();
}

}  // namespace tri
