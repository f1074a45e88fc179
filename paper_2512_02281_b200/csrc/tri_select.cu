// Per-query kernels around the list scan (tri_listscan.cu):
//   prep      fp64 queries -> fp32 rows (zero padded) + norms
//   merge     per query: top-kp over its partial lists
//   exact     one thread pair per (query, candidate): fp64 distance in the
//             reference's exact summation order (the two numpy lanes are two
//             threads), then per query: sort by (dist, id) and certify
//   fixup     per uncertified query: exact fp64 scan of its whole candidate set
//
// Certification: every dropped candidate has approx distance >= T (the kp-th
// kept one) and |approx - exact| <= E = cdot*2|q|max|x| + csum*(|q|+max|x|)^2, so if the k-th
// exact distance + E < T no dropped vector can enter the exact top-k.
#include <cuda_fp16.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

// Forked stream per (caller stream, device) for the split merge /
// re-rank: the narrow
// launch runs on it between an event fork and join, so inside a captured
// graph the two launches are sibling nodes.  Created on first use, kept.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static std::mutex g_side_mu;
static std::map<std::pair<cudaStream_t, int>, SideStream> g_side;

static cudaError_t side_stream(cudaStream_t st, SideStream** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_side_mu);
  SideStream& sd = g_side[{st, dev}];
  if (!sd.s) {
    if ((e = cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  *out = &sd;
  return cudaSuccess;
}


constexpr int kThreads = 256;
long long g_rerank_smem_cap = 0;
long long g_rerank_f2f = 1;
long long g_rerank_skip = 1;
long long g_rerank_lpt = 1;  // fused re-rank in LPT query order when capacities mix (option "rerank_lpt")
// mixed-capacity batches: the kp-32 queries re-rank in a second, narrow
// launch (64-thread CTAs, several per SM) on a forked stream beside the wide
// one, instead of each holding a 512-thread CTA (option "rerank_split")
long long g_rerank_split = 1;
// the same split for the partial-list merge (option "merge_split")
long long g_merge_split = 1;
long long g_rerank_wide_slab = 80;  // slab width for kp >= 128 (option "rerank_wide_slab"; 0 = the 8192/kp rule)
long long g_pdl = 0;  // programmatic dependent launch of the hot kernels (option "pdl")
long long g_fx_slice_rows = 256;

// ---------------------------------------------------------------------------
// Query preparation and row norms.

// One CTA (128 threads) per query; every element load is issued before any
// store (<= 16 per thread, qld <= 2048), then: fp32 row + |q32|^2 (fp32 of an
// fp64 sum), |q64| (fp64), and -- when Qh != nullptr -- the fp16 scan copy
// (see prep_half_kernel) in the same pass.
constexpr int kPrepThreads = 128, kPrepMaxU = 16;

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const double* __restrict__ q64, int d,
                                                            float* __restrict__ Q32, int qld, float* __restrict__ qn32,
                                                            double* __restrict__ qn64, int* bad, float sx,
                                                            __half* __restrict__ Qh, int ldh,
                                                            float* __restrict__ qinv, __half* __restrict__ Ql,
                                                            ClearList cl) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int q = blockIdx.x, tid = threadIdx.x;
  // per-search counters / buffers the later kernels expect filled (instead of
  // one cudaMemsetAsync each)
  for (int r = 0; r < cl.n; ++r)
    for (long long i = (long long)q * kPrepThreads + tid; i < cl.words[r]; i += (long long)gridDim.x * kPrepThreads)
      static_cast<uint32_t*>(cl.p[r])[i] = cl.val[r];
  double v[kPrepMaxU];
#pragma unroll
  for (int u = 0; u < kPrepMaxU; ++u) {
    const int j = tid + u * kPrepThreads;
    v[u] = j < d ? q64[(long long)q * d + j] : 0.0;
  }
  double s32 = 0.0, s64 = 0.0;
  float m = 0.f;
  bool finite = true;
  float f[kPrepMaxU];
#pragma unroll
  for (int u = 0; u < kPrepMaxU; ++u) {
    const int j = tid + u * kPrepThreads;
    finite = finite && isfinite(v[u]);
    f[u] = __double2float_rn(v[u]);
    if (j < qld) Q32[(long long)q * qld + j] = f[u];
    s32 += (double)f[u] * (double)f[u];
    s64 += v[u] * v[u];
    m = fmaxf(m, fabsf(f[u]));
  }
  __shared__ double r32[kPrepThreads / 32], r64[kPrepThreads / 32];
  __shared__ float rm[kPrepThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    s32 += __shfl_xor_sync(0xffffffffu, s32, o);
    s64 += __shfl_xor_sync(0xffffffffu, s64, o);
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  const int nf = __syncthreads_or(!finite);
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) {
    r32[warp] = s32;
    r64[warp] = s64;
    rm[warp] = m;
  }
  __syncthreads();
  double a = 0.0, b = 0.0;
  m = 0.f;
#pragma unroll
  for (int w = 0; w < kPrepThreads / 32; ++w) {
    a += r32[w];
    b += r64[w];
    m = fmaxf(m, rm[w]);
  }
  if (tid == 0) {
    qn32[q] = __double2float_rn(a);
    qn64[q] = nf ? __longlong_as_double(0x7ff8000000000000ll) : sqrt(b);  // NaN marks a non-finite query
    if (nf && bad) atomicExch(bad, 1);
  }
  if (Qh) {
    bool badh = false;
    float sq = 1.f;
    if (m > 0.f) {
      const int e = ilogbf(m);
      badh = e < -60 || e > 60;
      sq = badh ? 0.f : ldexpf(1.f, 14 - e);
    }
#pragma unroll
    for (int u = 0; u < kPrepMaxU; ++u) {
      const int j = tid + u * kPrepThreads;
      if (j < ldh) {
        const float v = j < d ? f[u] * sq : 0.f;  // exact (power-of-two scale)
        const __half h = __float2half_rn(v);
        Qh[(long long)q * ldh + j] = h;
        if (Ql) Ql[(long long)q * ldh + j] = __float2half_rn(v - __half2float(h));  // exact difference
      }
    }
    if (tid == 0) qinv[q] = badh ? -1.f : 1.f / (sq * sx);
  }
}

cudaError_t launch_prep(const double* q64, int B, int d, float* Q32, int qld, float* qn32, double* qn64,
                        int* bad, cudaStream_t st, float sx, void* Qh, int ldh, float* qinv, void* Ql,
                        const ClearList* clears) {
  if (B <= 0) return cudaSuccess;
  if (qld > kPrepThreads * kPrepMaxU || (Qh && ldh > kPrepThreads * kPrepMaxU)) return cudaErrorInvalidValue;
  ClearList cl{};
  if (clears) cl = *clears;
  (void)launch_pdl(prep_kernel, B, kPrepThreads, 0, st, q64, d, Q32, qld, qn32, qn64, bad, sx, static_cast<__half*>(Qh), ldh,
                                          qinv, static_cast<__half*>(Ql), cl);
  return cudaGetLastError();
}

__global__ void norms_kernel(const float* __restrict__ X, long long n, int d, long long ldx,
                             float* __restrict__ xnorm, unsigned long long* xmax_bits) {
  const int lane = threadIdx.x & 31;
  long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n) return;
  const float* x = X + row * ldx;
  double s = 0.0;
  for (int j = lane; j < d; j += 32) s += (double)x[j] * (double)x[j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    xnorm[row] = __double2float_rn(s);
    double r = sqrt(s);
    atomicMax(xmax_bits, (unsigned long long)__double_as_longlong(r));
  }
}

cudaError_t launch_norms(const float* X, long long n, int d, long long ldx, float* xnorm,
                         unsigned long long* xmax_bits, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 7) / 8;
  norms_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, n, d, ldx, xnorm, xmax_bits);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// fp16 candidate-generation copies.  Both sides are
// scaled by powers of two so the largest magnitude lands in [2^14, 2^15):
// scaling is exact, fp16 cannot overflow, and the subnormal floor is 2^-38 of
// the largest element.  The scan multiplies the accumulator by
// qinv = 1 / (s_q * s_x), also exact.

__global__ void absmax_kernel(const float* __restrict__ X, long long n, int d, long long ldx,
                              unsigned int* __restrict__ bits) {
  float m = 0.f;
  const long long total = n * (long long)d;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / d;
    m = fmaxf(m, fabsf(X[r * ldx + (i - r * d)]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(bits, __float_as_uint(m));  // m >= 0: bit order = value order
}

cudaError_t launch_absmax(const float* X, long long n, int d, long long ldx, unsigned int* bits, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  absmax_kernel<<<4 * 148, 256, 0, st>>>(X, n, d, ldx, bits);
  return cudaGetLastError();
}

// Xh[r, j] = fp16(X[r, j] * sx) for j < d, 0 for d <= j < ldh.
__global__ void to_half_kernel(const float* __restrict__ X, long long n, int d, long long ldx, float sx,
                               __half* __restrict__ Xh, int ldh) {
  const long long total = n * (long long)ldh;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ldh;
    const int j = (int)(i - r * ldh);
    Xh[i] = __float2half_rn(j < d ? X[r * ldx + j] * sx : 0.f);
  }
}

cudaError_t launch_to_half(const float* X, long long n, int d, long long ldx, float sx, void* Xh, int ldh,
                           cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  to_half_kernel<<<8 * 148, 256, 0, st>>>(X, n, d, ldx, sx, static_cast<__half*>(Xh), ldh);
  return cudaGetLastError();
}

// Per query: s_q = 2^(14 - ilogb(max|Q32|)), Qh = fp16(Q32 * s_q) (zero padded
// to ldh), qinv = 1 / (s_q * sx).  Queries whose largest element is outside
// [2^-60, 2^60] get qinv = -1 and a zero row: the re-rank never certifies
// them, so the exact fix-up answers them.  All-zero queries are exact (s_q = 1).
__global__ void prep_half_kernel(const float* __restrict__ Q32, int qld, int d, float sx, __half* __restrict__ Qh,
                                 int ldh, float* __restrict__ qinv) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int q = blockIdx.x;
  const float* row = Q32 + (long long)q * qld;
  float m = 0.f;
  for (int j = threadIdx.x; j < d; j += blockDim.x) m = fmaxf(m, fabsf(row[j]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
  bool bad = false;
  float sq = 1.f;
  if (m > 0.f) {
    const int e = ilogbf(m);
    bad = e < -60 || e > 60;
    sq = bad ? 0.f : ldexpf(1.f, 14 - e);
  }
  for (int j = threadIdx.x; j < ldh; j += blockDim.x)
    Qh[(long long)q * ldh + j] = __float2half_rn(j < d ? row[j] * sq : 0.f);
  if (threadIdx.x == 0) qinv[q] = bad ? -1.f : 1.f / (sq * sx);
}

cudaError_t launch_prep_half(const float* Q32, int B, int qld, int d, float sx, void* Qh, int ldh, float* qinv,
                             cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  (void)launch_pdl(prep_half_kernel, B, 128, 0, st, Q32, qld, d, sx, static_cast<__half*>(Qh), ldh, qinv);
  return cudaGetLastError();
}

// Queue an uncertified query for the exact fix-up.  Its fix-up bound starts
// at dk, the k-th exact distance among the re-ranked candidates: k real rows
// lie at or below it, so the exact top-k does too (+inf when dk is not finite).
__device__ __forceinline__ void flag_query(const RerankLaunch& r, int q, double dk) {
  const int fi = atomicAdd(r.n_flag, 1);
  r.flag_list[fi] = q;
  r.fx_thr[fi] = (dk >= 0.0 && dk < INFINITY) ? (unsigned long long)__double_as_longlong(dk) : 0x7ff0000000000000ull;
}

// Certification test (k-th exact distance dk, kp-th kept approx distance T).
// A non-finite T (overflowed approx distances) or an unscalable fp16 query
// is never certified.
__device__ __forceinline__ bool certified(const RerankLaunch& r, int q, double dk, double T) {
  if (!(T < INFINITY)) return false;
  if (r.qinv && r.qinv[q] < 0.f) return false;
  const double s = r.qn64[q] + r.xmax;
  const double E = (r.cdot * 2.0 * r.qn64[q] * r.xmax + r.csum * s * s) * 1.001 + 1e-30;
  return dk + E < T;
}

// ---------------------------------------------------------------------------
// Per-query merge of partial top-kp lists.

__global__ void __launch_bounds__(kThreads) merge_kernel(const unsigned long long* __restrict__ part,
                                                         const QueryMeta* __restrict__ meta,
                                                         unsigned long long* __restrict__ merged, int ld_merged,
                                                         int buf_n) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ unsigned long long buf[];
  __shared__ int s_cnt;
  __shared__ unsigned long long s_thr;
  const int q = blockIdx.x;
  const QueryMeta m = meta[q];
  const int kp = m.kp;
  const long long total = (long long)m.n_slots * kp;
  const unsigned long long* src = part + m.part_off;
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_thr = TRI_KEY_MAX;
  }
  __syncthreads();
  const int round = kThreads * 4;
  for (long long start = 0; start < total; start += round) {
    const unsigned long long thr = s_thr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      long long idx = start + j * kThreads + threadIdx.x;
      if (idx < total) {
        unsigned long long key = src[idx];
        if (key < thr) buf[atomicAdd(&s_cnt, 1)] = key;
      }
    }
    __syncthreads();
    const int n = s_cnt;
    if (n > buf_n - round) {
      const int p2 = next_pow2(n);
      for (int i = n + threadIdx.x; i < p2; i += kThreads) buf[i] = TRI_KEY_MAX;
      __syncthreads();
      block_sort(buf, p2, KeyLess());
      if (threadIdx.x == 0) {
        if (n >= kp) {
          s_cnt = kp;
          s_thr = buf[kp - 1];
        }
      }
    }
    __syncthreads();
  }
  const int n = s_cnt;
  const int p2 = next_pow2(n > 0 ? n : 1);
  for (int i = n + threadIdx.x; i < p2; i += kThreads) buf[i] = TRI_KEY_MAX;
  __syncthreads();
  block_sort(buf, p2, KeyLess());
  for (int i = threadIdx.x; i < kp; i += kThreads) merged[(long long)q * ld_merged + i] = i < n ? buf[i] : TRI_KEY_MAX;
}

// Warp-tree merge (kp <= 256): 8 warps per query; warp w folds slots
// w, w+8, ... into a register list (each partial list is sorted, so one bitonic
// split + merge per slot; a slot whose best key cannot beat the list is
// skipped), then the 8 lists are merged pairwise through shared memory.
constexpr int kMergeWarps = 8;

template <int KL, int W = kMergeWarps>
__device__ __forceinline__ void merge_tree(const unsigned long long* __restrict__ src, int n_slots,
                                           unsigned long long* __restrict__ dst, unsigned long long* sm) {
  constexpr int KP = 32 * KL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long L[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) L[j] = TRI_KEY_MAX;
  unsigned long long thr = TRI_KEY_MAX;
  for (int s0 = warp; s0 < n_slots; s0 += 2 * W) {
    // two slots in flight per warp: both loads issue before either merge
    unsigned long long P0[KL], P1[KL];
    const int s1 = s0 + W;
    const unsigned long long* a0 = src + (long long)s0 * KP;
    const unsigned long long* a1 = src + (long long)s1 * KP;
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      P0[j] = a0[(KL - 1 - j) * 32 + (31 - lane)];
      P1[j] = s1 < n_slots ? a1[(KL - 1 - j) * 32 + (31 - lane)] : TRI_KEY_MAX;
    }
    if (__shfl_sync(0xffffffffu, P0[KL - 1], 31) < thr) {  // P0[KL-1] on lane 31 = the slot's best key
      list_merge_rev<KL>(L, P0, lane);
      thr = __shfl_sync(0xffffffffu, L[KL - 1], 31);
    }
    if (__shfl_sync(0xffffffffu, P1[KL - 1], 31) < thr) {
      list_merge_rev<KL>(L, P1, lane);
      thr = __shfl_sync(0xffffffffu, L[KL - 1], 31);
    }
  }
  for (int stride = 1; stride < W; stride <<= 1) {
    if ((warp & (2 * stride - 1)) == stride) {
#pragma unroll
      for (int j = 0; j < KL; ++j) sm[warp * KP + j * 32 + lane] = L[j];
    }
    __syncthreads();
    if ((warp & (2 * stride - 1)) == 0) {
      unsigned long long R[KL];
#pragma unroll
      for (int j = 0; j < KL; ++j) R[j] = sm[(warp + stride) * KP + (KL - 1 - j) * 32 + (31 - lane)];
      list_merge_rev<KL>(L, R, lane);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KL; ++j) dst[j * 32 + lane] = L[j];
  }
}

__global__ void __launch_bounds__(32 * kMergeWarps) merge_tree_kernel(const unsigned long long* __restrict__ part,
                                                                      const QueryMeta* __restrict__ meta,
                                                                      unsigned long long* __restrict__ merged,
                                                                      int ld_merged) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ unsigned long long msm[];
  const int q = blockIdx.x;
  const QueryMeta m = meta[q];
  const unsigned long long* src = part + m.part_off;
  unsigned long long* dst = merged + (long long)q * ld_merged;
  switch (m.kp) {
    case 32: merge_tree<1>(src, m.n_slots, dst, msm); break;
    case 64: merge_tree<2>(src, m.n_slots, dst, msm); break;
    case 128: merge_tree<4>(src, m.n_slots, dst, msm); break;
    default: merge_tree<8>(src, m.n_slots, dst, msm); break;
  }
}

// Split merge of a mixed-capacity batch (option "merge_split"): W warps per
// query over the classes lo..hi only, CTA b taking the b-th query of those
// classes in descending class order (lpt_query; CTAs past their count exit).
// The kp-32 class runs 8-warp CTAs on a forked stream, the wide classes
// 16-warp CTAs (half the slots folded per warp) beside it.
__device__ __forceinline__ int lpt_query(const QueryMeta* __restrict__ meta, int B, int b, int lo, int hi);
template <int W>
__global__ void __launch_bounds__(32 * W) merge_tree_split_kernel(const unsigned long long* __restrict__ part,
                                                                  const QueryMeta* __restrict__ meta,
                                                                  unsigned long long* __restrict__ merged,
                                                                  int ld_merged, int B, int lo, int hi) {
  pdl_wait();
  extern __shared__ unsigned long long msm[];
  const int q = lpt_query(meta, B, blockIdx.x, lo, hi);
  if (q < 0) return;
  const QueryMeta m = meta[q];
  const unsigned long long* src = part + m.part_off;
  unsigned long long* dst = merged + (long long)q * ld_merged;
  switch (m.kp) {
    case 32: merge_tree<1, W>(src, m.n_slots, dst, msm); break;
    case 64: merge_tree<2, W>(src, m.n_slots, dst, msm); break;
    case 128: merge_tree<4, W>(src, m.n_slots, dst, msm); break;
    default: merge_tree<8, W>(src, m.n_slots, dst, msm); break;
  }
}

// Compact merge (wide brute force with a cross-item seed): query q's
// candidates are cnt[q] UNSORTED keys at the front of its partial region
// (every scan CTA appended at most kp of its survivors there).  Warp w folds
// keys w*32, w*32 + 256, ... 32 at a time, then the 8 lists merge pairwise.
template <int KL>
__device__ __forceinline__ void merge_compact(const unsigned long long* __restrict__ src, int n,
                                              unsigned long long* __restrict__ dst, unsigned long long* sm) {
  constexpr int KP = 32 * KL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long L[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) L[j] = TRI_KEY_MAX;
  for (int b = warp * 32; b < n; b += 32 * kMergeWarps) list_fold32<KL>(L, b + lane < n ? __ldcg(src + b + lane) : TRI_KEY_MAX, lane);
  for (int stride = 1; stride < kMergeWarps; stride <<= 1) {
    if ((warp & (2 * stride - 1)) == stride) {
#pragma unroll
      for (int j = 0; j < KL; ++j) sm[warp * KP + j * 32 + lane] = L[j];
    }
    __syncthreads();
    if ((warp & (2 * stride - 1)) == 0 && warp + stride < kMergeWarps && stride * 32 < n) {
      unsigned long long R[KL];
#pragma unroll
      for (int j = 0; j < KL; ++j) R[j] = sm[(warp + stride) * KP + (KL - 1 - j) * 32 + (31 - lane)];
      list_merge_rev<KL>(L, R, lane);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KL; ++j) dst[j * 32 + lane] = L[j];
  }
}

// The same merge by the first `nw` warps of a CTA (nw a power of two, every
// thread of the CTA calls it): the fused re-rank's prologue.
template <int KL>
__device__ __forceinline__ void merge_compact_nw(const unsigned long long* __restrict__ src, int n,
                                                 unsigned long long* __restrict__ dst, unsigned long long* sm, int nw) {
  constexpr int KP = 32 * KL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long L[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) L[j] = TRI_KEY_MAX;
  if (warp < nw) {
    // every load of a round of 8 folds in flight before the first fold (the
    // keys come from L2: one latency per round instead of one per fold)
    constexpr int kPf = 8;
    for (int b0 = warp * 32; b0 < n; b0 += kPf * 32 * nw) {
      unsigned long long kb[kPf];
#pragma unroll
      for (int j = 0; j < kPf; ++j) {
        const int b = b0 + j * 32 * nw + lane;
        kb[j] = b < n ? __ldcg(src + b) : TRI_KEY_MAX;
      }
#pragma unroll
      for (int j = 0; j < kPf; ++j)
        if (b0 + j * 32 * nw < n) list_fold32<KL>(L, kb[j], lane);
    }
  }
  for (int stride = 1; stride < nw; stride <<= 1) {
    if (warp < nw && (warp & (2 * stride - 1)) == stride) {
#pragma unroll
      for (int j = 0; j < KL; ++j) sm[warp * KP + j * 32 + lane] = L[j];
    }
    __syncthreads();
    if (warp < nw && (warp & (2 * stride - 1)) == 0 && warp + stride < nw && stride * 32 < n) {
      unsigned long long R[KL];
#pragma unroll
      for (int j = 0; j < KL; ++j) R[j] = sm[(warp + stride) * KP + (KL - 1 - j) * 32 + (31 - lane)];
      list_merge_rev<KL>(L, R, lane);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KL; ++j) dst[j * 32 + lane] = L[j];
  }
}

__global__ void __launch_bounds__(32 * kMergeWarps) merge_compact_kernel(const unsigned long long* __restrict__ part,
                                                                         const int* __restrict__ cnt,
                                                                         const QueryMeta* __restrict__ meta,
                                                                         unsigned long long* __restrict__ merged,
                                                                         int ld_merged) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ unsigned long long msm[];
  const int q = blockIdx.x;
  const QueryMeta m = meta[q];
  const unsigned long long* src = part + m.part_off;
  unsigned long long* dst = merged + (long long)q * ld_merged;
  const int n = min(cnt[q], m.n_slots * m.kp);
  switch (m.kp) {
    case 32: merge_compact<1>(src, n, dst, msm); break;
    case 64: merge_compact<2>(src, n, dst, msm); break;
    case 128: merge_compact<4>(src, n, dst, msm); break;
    default: merge_compact<8>(src, n, dst, msm); break;
  }
}

cudaError_t launch_merge_compact(const unsigned long long* part, const int* cnt, const QueryMeta* meta,
                                 unsigned long long* merged, int ld_merged, int B, int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (kp_max > 256) return cudaErrorInvalidValue;
  const size_t smem = (size_t)kMergeWarps * kp_max * sizeof(unsigned long long);
  cudaError_t e = cudaFuncSetAttribute(merge_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(merge_compact_kernel, B, 32 * kMergeWarps, smem, st, part, cnt, meta, merged, ld_merged);
  return cudaGetLastError();
}

cudaError_t launch_merge(const unsigned long long* part, const QueryMeta* meta, unsigned long long* merged,
                         int ld_merged, int B, int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (kp_max <= 256 && kp_max > kMinKp && g_merge_split && !g_pdl) {
    // mixed capacities: kp-32 queries (8 warps) on a forked stream, wider ones
    // (16 warps) here; each grid has B CTAs, those past its class count exit
    SideStream* sd = nullptr;
    cudaError_t e = side_stream(st, &sd);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(sd->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(sd->s, sd->fork, 0)) != cudaSuccess) return e;
    const size_t sn = (size_t)8 * kMinKp * sizeof(unsigned long long);
    (void)launch_pdl(merge_tree_split_kernel<8>, B, 256, sn, sd->s, part, meta, merged, ld_merged, B, 0, 0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaEventRecord(sd->join, sd->s)) != cudaSuccess) return e;
    const size_t sw = (size_t)16 * kp_max * sizeof(unsigned long long);
    e = cudaFuncSetAttribute(merge_tree_split_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sw);
    if (e != cudaSuccess) return e;
    (void)launch_pdl(merge_tree_split_kernel<16>, B, 512, sw, st, part, meta, merged, ld_merged, B, 1, kNumCls - 1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaStreamWaitEvent(st, sd->join, 0);
  }
  if (kp_max <= 256) {
    const size_t smem = (size_t)kMergeWarps * kp_max * sizeof(unsigned long long);
    cudaError_t e = cudaFuncSetAttribute(merge_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    (void)launch_pdl(merge_tree_kernel, B, 32 * kMergeWarps, smem, st, part, meta, merged, ld_merged);
    return cudaGetLastError();
  }
  int buf_n = next_pow2(kp_max + kThreads * 4);
  size_t smem = (size_t)buf_n * sizeof(unsigned long long);
  cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(merge_kernel, B, kThreads, smem, st, part, meta, merged, ld_merged, buf_n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact fp64 re-rank + certification.
//
// exact_pairs_kernel: one warp-sized CTA per (query, 16 candidates); thread
// pair (2c, 2c+1) computes candidate c, thread 2c+l running numpy lane l
// (elements 8b + 2*sub + l, sub = 3..0, then the 2-lane tail), so the value is
// bit-identical to exact_sq_dist / the reference.  The candidate rows arrive
// in shared memory by 1-D bulk copies (one per row per <= 1024-float slab,
// one mbarrier); slabs are 8-aligned so numpy's 8-element blocks never
// straddle one.

constexpr int kPairCands = 16;
constexpr int kPairSlab = 1024;  // floats

__device__ __forceinline__ uint32_t sel_su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(2 * kPairCands) exact_pairs_kernel(RerankLaunch r, int row_stride) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char pair_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ long long pos_s[kPairCands];
  double* qs = reinterpret_cast<double*>(pair_smem);
  const int slab_max = min(kPairSlab, (r.d + 15) & ~15);
  float* xs = reinterpret_cast<float*>(qs + slab_max);
  const int groups = r.ld_merged / kPairCands;
  const int q = blockIdx.x / groups;
  const int c = (blockIdx.x - q * groups) * kPairCands + (threadIdx.x >> 1);
  const int ln = threadIdx.x & 1, lane = threadIdx.x;
  const int kp = r.meta[q].kp;
  if ((c & ~(kPairCands - 1)) >= kp) return;  // whole CTA beyond this query's capacity
  const long long p = (long long)q * r.ld_merged + c;
  const unsigned long long key = r.merged[p];
  const bool active = key != TRI_KEY_MAX;
  const long long pos = active ? (long long)key_pos(key) : -1;
  if (ln == 0) pos_s[lane >> 1] = pos;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sel_su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int d = r.d;
  const double* qg = r.q64 + (long long)q * d;
  double acc = 0.0;
  uint32_t phase = 0;
  for (int s0 = 0; s0 < d; s0 += kPairSlab) {
    const int w = min(kPairSlab, d - s0);
    const int w16 = (w + 15) & ~15;  // stored rows are zero padded to a multiple of 16
    if (lane == 0) {
      int nrow = 0;
      for (int i = 0; i < kPairCands; ++i) nrow += pos_s[i] >= 0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sel_su32(&bar)),
                   "r"((uint32_t)(nrow * w16 * 4))
                   : "memory");
      for (int i = 0; i < kPairCands; ++i)
        if (pos_s[i] >= 0)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                           sel_su32(xs + i * row_stride)),
                       "l"(r.X + pos_s[i] * r.ldx + s0), "r"((uint32_t)(w16 * 4)), "r"(sel_su32(&bar))
                       : "memory");
    }
    for (int j = lane; j < w; j += 32) qs[j] = qg[s0 + j];
    __syncwarp();
    asm volatile(
        "{\n .reg .pred P;\n PWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra PWAIT_%=;\n}\n" ::"r"(
            sel_su32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    if (active) {
      const float* xr = xs + (lane >> 1) * row_stride;
      int i = 0;
      for (; i < w && s0 + i + 8 <= d; i += 8) {
#pragma unroll
        for (int sub = 3; sub >= 0; --sub) {
          const int e = i + 2 * sub + ln;
          const double df = __dsub_rn(qs[e], (double)xr[e]);
          acc = __dadd_rn(__dmul_rn(df, df), acc);
        }
      }
      for (; i < w; i += 2) {  // numpy's 2-lane tail (last slab only)
        const int e = i + ln;
        if (s0 + e < d) {
          const double df = __dsub_rn(qs[e], (double)xr[e]);
          acc = __dadd_rn(__dmul_rn(df, df), acc);
        }
      }
    }
    __syncwarp();
  }
  const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
  if (ln == 0 && c < kp) {
    Exact e = exact_max();
    if (active) {
      e.d = __dadd_rn(acc, other);
      e.id = (r.idmap ? r.idmap[pos] : pos) + r.id_offset;
    }
    r.exact[p] = e;
  }
}

// Columns [k, ldo) of an output row: id -1, distance +inf (a defined result
// row whatever the caller's buffer held).
__device__ __forceinline__ void pad_row(long long* ids, double* d, int k, int ldo, int t, int nt) {
  for (int j = k + t; j < ldo; j += nt) {
    ids[j] = -1;
    d[j] = __longlong_as_double(0x7ff0000000000000ll);
  }
}

// finalize: one warp per query sorts its kp exact (dist, id) entries in
// registers (bitonic network over element j*32 + lane), certifies, writes k.
__device__ __forceinline__ bool ex_less(double ad, long long ai, double bd, long long bi) {
  return ad < bd || (ad == bd && ai < bi);
}

template <int KL>
__device__ __forceinline__ void finalize_query(const RerankLaunch& r, int q, int lane) {
  constexpr int KP = 32 * KL;
  const QueryMeta m = r.meta[q];
  double d[KL];
  long long id[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) {
    const Exact e = r.exact[(long long)q * r.ld_merged + j * 32 + lane];
    d[j] = e.d;
    id[j] = e.id;
  }
#pragma unroll
  for (int k = 2; k <= KP; k <<= 1)
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= 32) {
        const int dj = jj >> 5;
#pragma unroll
        for (int j = 0; j < KL; ++j)
          if ((j & dj) == 0) {
            const int e = j * 32 + lane;
            const bool up = (e & k) == 0;
            const bool sw = up ? ex_less(d[j + dj], id[j + dj], d[j], id[j]) : ex_less(d[j], id[j], d[j + dj], id[j + dj]);
            if (sw) {
              const double td = d[j];
              const long long ti = id[j];
              d[j] = d[j + dj];
              id[j] = id[j + dj];
              d[j + dj] = td;
              id[j + dj] = ti;
            }
          }
      } else {
#pragma unroll
        for (int j = 0; j < KL; ++j) {
          const double od = __shfl_xor_sync(0xffffffffu, d[j], jj);
          const long long oi = __shfl_xor_sync(0xffffffffu, id[j], jj);
          const int e = j * 32 + lane;
          const bool keep_min = ((e & k) == 0) == ((lane & jj) == 0);
          const bool other_less = ex_less(od, oi, d[j], id[j]);
          if (keep_min == other_less) {
            d[j] = od;
            id[j] = oi;
          }
        }
      }
    }
  // certification: every dropped candidate has approx distance >= T
  bool cert = true;
  double dk = INFINITY;
  if (m.n_total > m.kp) {
    const int kk = m.k - 1;
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      const double t = __shfl_sync(0xffffffffu, d[j], kk & 31);
      if (j == (kk >> 5)) dk = t;
    }
    cert = certified(r, q, dk, (double)key_dist(r.merged[(long long)q * r.ld_merged + m.kp - 1]));
  }
  if ((!cert || isnan(r.qn64[q])) && lane == 0) flag_query(r, q, dk);
#pragma unroll
  for (int j = 0; j < KL; ++j) {
    const int e = j * 32 + lane;
    if (e < m.k) {
      const bool ok = id[j] != 0x7fffffffffffffffll;
      r.out_ids[(long long)q * r.ldo + e] = ok ? id[j] : -1;
      r.out_d[(long long)q * r.ldo + e] = d[j];
    }
  }
  pad_row(r.out_ids + (long long)q * r.ldo, r.out_d + (long long)q * r.ldo, m.k, r.ldo, lane, 32);
}

__global__ void __launch_bounds__(128) finalize_warp_kernel(RerankLaunch r) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  const int q = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (q >= r.B) return;
  const int lane = threadIdx.x & 31;
  switch (r.meta[q].kp) {
    case 32: finalize_query<1>(r, q, lane); break;
    case 64: finalize_query<2>(r, q, lane); break;
    case 128: finalize_query<4>(r, q, lane); break;
    default: finalize_query<8>(r, q, lane); break;
  }
}

__global__ void __launch_bounds__(128) finalize_kernel(RerankLaunch r) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ Exact ebuf[];
  const int q = blockIdx.x;
  const QueryMeta m = r.meta[q];
  const int kp = m.kp;
  for (int i = threadIdx.x; i < kp; i += blockDim.x) ebuf[i] = r.exact[(long long)q * r.ld_merged + i];
  __syncthreads();
  block_sort(ebuf, kp, ExactLess());
  if (threadIdx.x == 0) {
    bool cert = true;
    if (m.n_total > kp) {
      cert = certified(r, q, ebuf[m.k - 1].d, (double)key_dist(r.merged[(long long)q * r.ld_merged + kp - 1]));
    }
    if (!cert || isnan(r.qn64[q])) flag_query(r, q, ebuf[m.k - 1].d);
  }
  for (int j = threadIdx.x; j < m.k; j += blockDim.x) {
    const Exact e = ebuf[j];
    const bool ok = e.id != 0x7fffffffffffffffll;
    r.out_ids[(long long)q * r.ldo + j] = ok ? e.id : -1;
    r.out_d[(long long)q * r.ldo + j] = e.d;
  }
  pad_row(r.out_ids + (long long)q * r.ldo, r.out_d + (long long)q * r.ldo, m.k, r.ldo, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------------------
// Fused exact re-rank (kp <= 256): one CTA per query, 2*kp_max threads.
// The fp64 query is staged in shared memory once; thread pair (2c, 2c+1) runs
// numpy's two lanes for candidate c reading the row straight from L2/HBM in
// 4-block (32-float) groups, double-buffered in registers; warp 0 then sorts
// the kp (dist, id) pairs in registers, certifies and writes the top k.

// Fused exact re-rank (kp <= 256): one CTA per query, 2*kp_max threads.
// The fp64 query is staged in shared memory once; thread pair (2c, 2c+1) runs
// numpy's two lanes for candidate c, reading the row straight from L2/HBM in
// 4-block (32-float) groups with the next group's 8 float4 loads in flight.
// fp32 -> fp64 is done with integer bit moves for normal numbers (F2F sits on
// a slow conversion pipe; the value is identical since the conversion is
// exact).  The (dist, id) order comes from parallel rank counting (O(kp^2)
// compares, no serial sorting network); rank k-1 feeds the certification.

// One 1-D bulk copy per candidate row per slab, issued by the candidate's own
// pair-leader thread (all rows in flight at once, no per-16B address math).
// Stage an fp64 query row (zero-padded to dpad) in shared memory with every
// global load issued before the first store: a strided load/store loop would
// pay one memory latency per iteration.
constexpr int kStageMaxU = 32;
__device__ __forceinline__ void stage_query(const double* __restrict__ qg, int d, int dpad, double* qs, int tid, int nthr) {
  for (int base = 0; base < dpad; base += kStageMaxU * nthr) {
    double v[kStageMaxU];
#pragma unroll
    for (int u = 0; u < kStageMaxU; ++u) {
      const int j = base + tid + u * nthr;
      v[u] = j < d ? qg[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kStageMaxU; ++u) {
      const int j = base + tid + u * nthr;
      if (j < dpad) qs[j] = v[u];
    }
  }
}
__device__ __forceinline__ void rf_issue(float* buf, uint64_t* bar, int S, int c, long long pos, const float* X,
                                         long long ldx, int s0, int dpad, int nvalid, bool leader) {
  const int w = min(S, dpad - s0);
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"((uint32_t)(nvalid * w * 4))
                 : "memory");
  if (leader && pos >= 0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(buf + c * (S + 4)))),
                 "l"(X + pos * ldx + s0), "r"((uint32_t)(w * 4)),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

// Exact fp32 -> fp64 without the F2F pipe for normal numbers and zeros
// (branch-free); *sub is set when x is subnormal (caller falls back to F2F).
__device__ __forceinline__ double f2d_bits(float x, bool& sub) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t e = (u >> 23) & 0xffu;
  const uint32_t nz = e ? 0xffffffffu : 0u;
  sub = sub || (e == 0 && (u & 0x7fffffu));
  return __hiloint2double((int)((u & 0x80000000u) | ((((e + 896u) << 20) | ((u >> 3) & 0xfffffu)) & nz)),
                          (int)((u << 29) & nz));
}

// Longest-processing-time order for a mixed-capacity batch: CTA b takes the
// b-th query in (capacity class descending, query ascending) order, so the
// wide prefill lists start in the first wave and the short decode lists fill
// in behind them.  Two block-wide passes over the classes in meta (L2-resident).
// Only classes lo..hi are taken (a split launch); a CTA past their count gets -1.
__device__ __forceinline__ int lpt_query(const QueryMeta* __restrict__ meta, int B, int b, int lo, int hi) {
  __shared__ int s_cnt[kNumCls];
  __shared__ int s_w[16];
  __shared__ int s_q;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kNumCls) s_cnt[tid] = 0;
  if (tid == 0) s_q = b;
  __syncthreads();
  for (int i = tid; i < B; i += nthr) atomicAdd(&s_cnt[meta[i].cls], 1);
  __syncthreads();
  int acc = 0, c = hi;
  for (; c >= lo; --c) {
    if (b < acc + s_cnt[c]) break;
    acc += s_cnt[c];
  }
  if (c < lo) return -1;  // block-uniform (s_cnt, b)
  int j = b - acc;  // rank of the wanted query inside class c
  for (int base = 0; base < B; base += nthr) {
    const int i = base + tid;
    const bool m = i < B && meta[i].cls == c;
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (nthr >> 5); ++w) {
      before += w < warp ? s_w[w] : 0;
      total += s_w[w];
    }
    if (j < total) {
      if (m && before + __popc(bal & ((1u << lane) - 1u)) == j) s_q = i;
      __syncthreads();
      break;
    }
    j -= total;
    __syncthreads();
  }
  return s_q;
}

template <bool F2F>
__global__ void __launch_bounds__(512) rerank_fused_kernel(RerankLaunch r, int S) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char rf_smem[];
  __shared__ double s_dk;
  __shared__ __align__(8) uint64_t bars[3];
  int qb = blockIdx.x;
  if (r.lpt) {
    qb = lpt_query(r.meta, r.B, blockIdx.x, r.lpt_cls == 2 ? 1 : 0, r.lpt_cls == 1 ? 0 : kNumCls - 1);
    if (qb < 0) return;  // split launch: this CTA's class range has fewer queries
  }
  const int q = qb;
  const QueryMeta m = r.meta[q];
  const int d = r.d, kpm = r.kp_max, kp = m.kp;
  const int dpad = (d + 15) & ~15;
  double* qs = reinterpret_cast<double*>(rf_smem);       // dpad
  double* exd = qs + dpad;                               // kp_max
  long long* exi = reinterpret_cast<long long*>(exd + kpm);
  unsigned long long* mk = reinterpret_cast<unsigned long long*>(exi + kpm);  // kp_max (fused merge)
  float* ring = reinterpret_cast<float*>(mk + kpm);      // 2 x kp_max x (S + 4)
  const int tid = threadIdx.x, nthr = blockDim.x, c = tid >> 1, ln = tid & 1;
  // the query row streams into shared memory (one bulk copy on bars[2]) while
  // the candidate list is merged; an odd d (row not 16-byte aligned) is staged
  // by the threads after the merge
  const double* qg = r.q64 + (long long)q * d;
  const bool qbulk = (d & 1) == 0 && (reinterpret_cast<uintptr_t>(qg) & 15) == 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bars[0]))));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bars[1]))));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&bars[2]))));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (qbulk) {
      const uint32_t b2 = static_cast<uint32_t>(__cvta_generic_to_shared(&bars[2]));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b2), "r"((uint32_t)(d * 8)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(qs))),
                   "l"(qg), "r"((uint32_t)(d * 8)), "r"(b2)
                   : "memory");
    }
  }
  const double qn64 = r.qn64[q];
  // the query's sorted candidate list: the merge kernel's output, or (brute
  // force with a cross-item seed) merged right here from the scan's compact
  // region -- one launch and one global round trip less
  const unsigned long long* mrow = r.merged + (long long)q * r.ld_merged;
  if (r.compact_cnt) {
    const int n = min(r.compact_cnt[q], m.n_slots * kp);
    const unsigned long long* src = r.part + m.part_off;
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(ring);  // free until the first slab
    const int nw = min(nthr >> 5, 8);
    switch (kp) {
      case 32: merge_compact_nw<1>(src, n, mk, scratch, nw); break;
      case 64: merge_compact_nw<2>(src, n, mk, scratch, nw); break;
      case 128: merge_compact_nw<4>(src, n, mk, scratch, nw); break;
      default: merge_compact_nw<8>(src, n, mk, scratch, nw); break;
    }
    __syncthreads();
    for (int i = tid; i < kp; i += nthr) const_cast<unsigned long long*>(r.merged)[(long long)q * r.ld_merged + i] = mk[i];
    mrow = mk;
  }
  unsigned long long key = TRI_KEY_MAX;
  if (c < kp) key = mrow[c];
  bool active = key != TRI_KEY_MAX;
  // A candidate whose approx key exceeds the k-th approx key by more than 2E
  // cannot enter the exact top-k.  Its exact distance is > approx(k) + E >= D_k,
  // since the k smallest-key candidates have exact <= approx + E.  So its fp64
  // row is neither loaded nor computed.  (merged is sorted; unscalable fp16
  // queries keep every candidate.)
  if (active && r.skip_far && m.k < kp && !(r.qinv && r.qinv[q] < 0.f)) {
    const unsigned long long kk = mrow[m.k - 1];
    const double sn = qn64 + r.xmax;
    const double E = (r.cdot * 2.0 * qn64 * r.xmax + r.csum * sn * sn) * 1.001 + 1e-30;
    if (kk != TRI_KEY_MAX && (double)key_dist(key) > (double)key_dist(kk) + 2.0 * E) active = false;
  }
  const long long pos = active ? (long long)key_pos(key) : -1;
  const bool leader = ln == 0 && c < kp;
  if (qbulk) {
    for (int j = d + tid; j < dpad; j += nthr) qs[j] = 0.0;
  } else {
    stage_query(qg, d, dpad, qs, tid, nthr);
  }
  const int nvalid = __syncthreads_count(leader && active);
  if (qbulk)
    asm volatile(
        "{\n .reg .pred P;\n RFQ_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra RFQ_%=;\n}\n" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&bars[2])))
        : "memory");
  const int nslab = (dpad + S - 1) / S;
  const int buf_floats = kpm * (S + 4);
  rf_issue(ring, &bars[0], S, c, pos, r.X, r.ldx, 0, dpad, nvalid, leader);
  double acc = 0.0;
  const int nfull = d >> 3;  // numpy's full 8-element blocks (global count)
  for (int s = 0; s < nslab; ++s) {
    if (s + 1 < nslab)
      rf_issue(ring + ((s + 1) & 1) * buf_floats, &bars[(s + 1) & 1], S, c, pos, r.X, r.ldx, (s + 1) * S, dpad, nvalid,
               leader);
    asm volatile(
        "{\n .reg .pred P;\n RFW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra RFW_%=;\n}\n" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&bars[s & 1]))),
        "r"((uint32_t)((s >> 1) & 1))
        : "memory");
    const int s0 = s * S;
    if (active) {
      const float* xr = ring + (s & 1) * buf_floats + c * (S + 4);
      const double* qb = qs + s0;
      const int bend = min(S >> 3, nfull - (s0 >> 3));  // full blocks inside this slab
      int b = 0;
      for (; b + 4 <= bend; b += 4) {
        // 16 independent squared differences first, then the 16-step chain
        double t2[16];
        bool sub = false;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const float4 lo = *reinterpret_cast<const float4*>(xr + 8 * (b + bb));
          const float4 hi = *reinterpret_cast<const float4*>(xr + 8 * (b + bb) + 4);
          const float xs[4] = {ln ? hi.w : hi.z, ln ? hi.y : hi.x, ln ? lo.w : lo.z, ln ? lo.y : lo.x};
#pragma unroll
          for (int t = 0; t < 4; ++t) {  // sub = 3 - t -> element 2*(3-t) + ln
            const double df = __dsub_rn(qb[8 * (b + bb) + 2 * (3 - t) + ln], F2F ? (double)xs[t] : f2d_bits(xs[t], sub));
            t2[bb * 4 + t] = __dmul_rn(df, df);
          }
        }
        if (__builtin_expect(__any_sync(__activemask(), sub), 0)) {
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int e = 8 * (b + bb) + 2 * (3 - t) + ln;
              const double df = __dsub_rn(qb[e], (double)xr[e]);
              t2[bb * 4 + t] = __dmul_rn(df, df);
            }
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) acc = __dadd_rn(t2[t], acc);
      }
      for (; b < bend; ++b) {
#pragma unroll
        for (int sub = 3; sub >= 0; --sub) {
          const int e = 8 * b + 2 * sub + ln;
          const double df = __dsub_rn(qb[e], (double)xr[e]);
          acc = __dadd_rn(__dmul_rn(df, df), acc);
        }
      }
      if (s0 + 8 * bend >= 8 * nfull) {  // numpy's 2-lane tail lives in this slab
        for (int i = 8 * nfull - s0; i < min(S, d - s0); i += 2) {
          const int e = i + ln;
          if (s0 + e < d) {
            const double df = __dsub_rn(qb[e], (double)xr[e]);
            acc = __dadd_rn(__dmul_rn(df, df), acc);
          }
        }
      }
    }
    __syncthreads();  // buffer (s & 1) is refilled by the next iteration's stage
  }
  const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
  if (ln == 0 && c < kpm) {
    exd[c] = active ? __dadd_rn(acc, other) : __longlong_as_double(0x7ff0000000000000ll);
    exi[c] = active ? (r.idmap ? r.idmap[pos] : pos) + r.id_offset : 0x7fffffffffffffffll;
  }
  __syncthreads();
  if (tid < kp) {
    const double md = exd[tid];
    const long long mi = exi[tid];
    int rank = 0;
    for (int j = 0; j < kp; ++j) {  // (dist, id) order; slot index breaks ties between empty slots
      const double dj = exd[j];
      const long long ij = exi[j];
      rank += ex_less(dj, ij, md, mi) || (dj == md && ij == mi && j < tid);
    }
    if (rank < m.k) {
      const bool ok = mi != 0x7fffffffffffffffll;
      r.out_ids[(long long)q * r.ldo + rank] = ok ? mi : -1;
      r.out_d[(long long)q * r.ldo + rank] = md;
    }
    if (rank == m.k - 1) s_dk = md;
  }
  pad_row(r.out_ids + (long long)q * r.ldo, r.out_d + (long long)q * r.ldo, m.k, r.ldo, tid, nthr);
  __syncthreads();
  if (tid == 0) {
    bool cert = true;
    if (m.n_total > kp) {
      cert = certified(r, q, s_dk, (double)key_dist(mrow[kp - 1]));
    }
    if (!cert || isnan(r.qn64[q])) flag_query(r, q, s_dk);
  }
}

// IVF coarse step with set semantics.  The fine step scans the UNION of a
// query's probed lists, so only WHICH nprobe centroids are the exact top-nprobe
// by (dist, id) matters, not their order.  With the certificate's error bound
// E (|D~ - D| <= E) and the merged candidates sorted by approximate distance
// a_0 <= a_1 <= ...:
//   * certified (no dropped centroid can enter): a_{kp-1} - E > a_{k-1} + E;
//   * IN  (certainly in the top-k): #{j : a_j <= a_i + 2E} <= k -- fewer than
//     k others can have an exact distance at or below i's;
//   * OUT (certainly not): #{j : a_j < a_i - 2E} >= k -- k others are
//     strictly closer;
//   * the top-k = IN + the (k - |IN|) smallest of the rest by exact (dist, id).
// Exact fp64 distances (reference order) are computed only for the uncertain
// rest -- usually none or a few per query instead of every candidate.  Probes
// come out in approximate order (IN exact-or-approx distances are not needed
// downstream); an uncertified query goes to the fix-up, which writes the exact
// ordered top-k.
constexpr int kSetMax = 256;   // candidates per query (kp_max)
constexpr int kSetMaxD = 1024; // dimensions (the query and the uncertain rows are staged in shared memory)
constexpr int kSetRows = 16;   // uncertain rows computed at once (one lane pair each)
constexpr int kSetWarps = 1;   // one query (warp) per CTA: its staged rows take up to 64 KB
__global__ void __launch_bounds__(32 * kSetWarps) coarse_set_kernel(RerankLaunch r) {
  pdl_wait();
  __shared__ double sa[kSetWarps][kSetMax];
  __shared__ double sx[kSetWarps][kSetMax];
  __shared__ int su[kSetWarps][kSetMax];
  extern __shared__ __align__(16) unsigned char cs_smem[];  // query (d doubles) + kSetRows rows (dpad floats)
  __shared__ __align__(8) uint64_t cs_bar;
  const int wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * kSetWarps + wq;
  if (q >= r.B) return;
  const QueryMeta m = r.meta[q];
  const int kp = m.kp, k = m.k, d = r.d;
  const unsigned long long* mrow = r.merged + (long long)q * r.ld_merged;
  double* a = sa[wq];
  double* ex = sx[wq];
  int* ul = su[wq];
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int i = lane; i < kp; i += 32) {
    const unsigned long long key = mrow[i];
    a[i] = key != TRI_KEY_MAX ? (double)key_dist(key) : inf;
    ex[i] = inf;
  }
  __syncwarp();
  // per-candidate error bound E_i = E(|q|, |c_i|) from the candidate's own
  // norm (singleton lists make a few centroids data-point sized, so the
  // store-wide E_max is ~25x too wide for typical centroids); rows NOT among
  // the candidates are bounded with E_max (their norm is unknown)
  const double qn = r.qn64[q];
  auto bound = [&](double xn) {
    const double s = qn + xn;
    return (r.cdot * 2.0 * qn * xn + r.csum * s * s) * 1.001 + 1e-30;
  };
  const double Emax = bound(r.xmax);
  // [a_i - E_i, a_i + E_i] as fp32 rounded outward (a_i is an fp32 value):
  // the counts below only get more conservative, and run on the fp32 pipe
  float* lo = reinterpret_cast<float*>(ex);  // ex is free until the exact pass
  float* hi = lo + kSetMax;
  const float finf = __int_as_float(0x7f800000);
  for (int i = lane; i < kp; i += 32) {
    const unsigned long long key = mrow[i];
    if (key != TRI_KEY_MAX) {
      // |c|^2 is stored rounded to fp32: widen by 1e-6 relative to stay an upper bound
      const float e = __double2float_ru(bound(sqrt((double)r.xnorm[key_pos(key)]) * (1.0 + 1e-6)));
      const float af = key_dist(key);
      const bool fin = af < finf && e < finf;  // else: could be anywhere
      lo[i] = fin ? __fsub_rd(af, e) : -finf;
      hi[i] = fin ? __fadd_ru(af, e) : finf;
    } else {
      lo[i] = finf;
      hi[i] = finf;
    }
  }
  __syncwarp();
  const double ak = a[k - 1], akp = a[kp - 1];
  bool cert = !isnan(qn) && ak < inf;
  // U = an upper bound of the exact k-th distance: the k-th smallest a_j + E_j
  float U = finf;
  if (cert) {
    for (int b = 0; b < kp; b += 32) {
      const int i = b + lane;
      float ui = finf;
      if (i < kp && hi[i] < finf) {
        ui = hi[i];
        int below = 0;  // #{j : hi_j < ui} (ties: index order)
        for (int j = 0; j < kp; ++j) {
          const float uj = hi[j];
          below += uj < ui || (uj == ui && j < i);
        }
        if (below != k - 1) ui = finf;
      }
      for (int o = 16; o > 0; o >>= 1) ui = fminf(ui, __shfl_xor_sync(0xffffffffu, ui, o));
      U = fminf(U, ui);
    }
    if (m.n_total > kp) cert = akp < inf && !(r.qinv && r.qinv[q] < 0.f) && (double)U < akp - Emax;
  }
  long long* oid = r.out_ids + (long long)q * r.ldo;
  double* od = r.out_d + (long long)q * r.ldo;
  if (!cert) {  // the fix-up rewrites this query's exact ordered top-k; until then the
    // approximate top-k (valid ids), or no lists at all for a non-finite query
    const bool nq = isnan(qn);
    for (int j = lane; j < k; j += 32) {
      const unsigned long long key = mrow[j];
      const bool ok = !nq && key != TRI_KEY_MAX;
      oid[j] = ok ? (r.idmap ? r.idmap[key_pos(key)] : (long long)key_pos(key)) + r.id_offset : -1;
      od[j] = ok ? a[j] : __longlong_as_double(0x7ff8000000000000ll);
    }
    pad_row(oid, od, k, r.ldo, lane, 32);
    if (lane == 0) flag_query(r, q, U < finf ? (double)U : ak + Emax);
    return;
  }
  // classify: IN if fewer than k others can be at or below it, OUT if k others
  // are certainly strictly below it
  int nin = 0, nun = 0;
  unsigned injm = 0;  // bit b: this lane's entry of round b is IN
  for (int b = 0, bi = 0; b < kp; b += 32, ++bi) {
    const int i = b + lane;
    bool in = false, out = true;
    if (i < kp && mrow[i] != TRI_KEY_MAX) {  // (an infinite bound leaves the entry uncertain)
      const float lo_i = lo[i], hi_i = hi[i];
      int maybe = 0, sure = 0;
      for (int j = 0; j < kp; ++j) {
        const float lj = lo[j], hj = hi[j];
        maybe += lj <= hi_i;  // j could be at or below i (i itself included)
        sure += hj < lo_i;    // j is strictly below i
      }
      in = maybe <= k;  // fewer than k others
      out = sure >= k;
    }
    injm |= (unsigned)in << bi;
    const bool un = !in && !out;
    const unsigned bin = __ballot_sync(0xffffffffu, in), bun = __ballot_sync(0xffffffffu, un);
    const unsigned lt = (1u << lane) - 1u;
    if (un) ul[nun + __popc(bun & lt)] = i;
    nin += __popc(bin);
    nun += __popc(bun);
  }
  __syncwarp();
  for (int b = 0, bi = 0; b < kp; b += 32, ++bi) {
    const int i = b + lane;
    if (i < kp) ex[i] = ((injm >> bi) & 1u) ? -1.0 : inf;  // marker: -1 = IN
  }
  __syncwarp();
  // exact distances of the uncertain candidates: the warp stages the query
  // and one row at a time in shared memory (coalesced, one L2 latency per
  // row), lanes 0 / 1 run numpy's two lanes in the reference order
  if (nun > 0) {
    // the query (fp64) and up to 16 uncertain rows at a time in shared memory
    // (rows by 1-D bulk copies, one mbarrier: one L2 latency per 16 rows),
    // then lane pair (2c, 2c+1) runs numpy's two lanes of candidate c
    const int dpad = (d + 15) & ~15;
    double* qs = reinterpret_cast<double*>(cs_smem);
    float* rows = reinterpret_cast<float*>(qs + dpad);
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&cs_bar));
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    const double* qg = r.q64 + (long long)q * d;
    {
      constexpr int U = kSetMaxD / 32;
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = u * 32 + lane;
        v[u] = jj < d ? qg[jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int jj = u * 32 + lane;
        if (jj < dpad) qs[jj] = v[u];
      }
    }
    __syncwarp();
    uint32_t phase = 0;
    for (int t0 = 0; t0 < nun; t0 += kSetRows) {
      const int nb = min(kSetRows, nun - t0);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                     "r"((uint32_t)(nb * dpad * 4))
                     : "memory");
        for (int c = 0; c < nb; ++c) {
          const long long pos = key_pos(mrow[ul[t0 + c]]);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  static_cast<uint32_t>(__cvta_generic_to_shared(rows + c * dpad))),
              "l"(r.X + pos * r.ldx), "r"((uint32_t)(dpad * 4)), "r"(bar)
              : "memory");
        }
      }
      asm volatile(
          "{\n .reg .pred P;\n CSW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra CSW_%=;\n}\n" ::"r"(
              bar),
          "r"(phase)
          : "memory");
      phase ^= 1;
      const int c = lane >> 1, ln = lane & 1;
      double acc = 0.0;
      if (c < nb) {
        const float* xs = rows + c * dpad;
        int jj = 0;
        for (; jj + 32 <= d; jj += 32) {  // 16 independent squared differences, then the 16-step chain
          double t2[16];
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
#pragma unroll
            for (int sub = 3; sub >= 0; --sub) {
              const int e = jj + 8 * bb + 2 * sub + ln;
              const double df = __dsub_rn(qs[e], (double)xs[e]);
              t2[bb * 4 + (3 - sub)] = __dmul_rn(df, df);
            }
#pragma unroll
          for (int t = 0; t < 16; ++t) acc = __dadd_rn(t2[t], acc);
        }
        for (; jj + 8 <= d; jj += 8)
#pragma unroll
          for (int sub = 3; sub >= 0; --sub) {
            const int e = jj + 2 * sub + ln;
            const double df = __dsub_rn(qs[e], (double)xs[e]);
            acc = __dadd_rn(__dmul_rn(df, df), acc);
          }
        for (; jj < d; jj += 2) {
          const int e = jj + ln;
          if (e < d) {
            const double df = __dsub_rn(qs[e], (double)xs[e]);
            acc = __dadd_rn(__dmul_rn(df, df), acc);
          }
        }
      }
      const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
      if (ln == 0 && c < nb) ex[ul[t0 + c]] = __dadd_rn(acc, other);
      __syncwarp();  // the row buffers are refilled by the next round
    }
  }
  // the (k - nin) smallest uncertain by (exact, id) join the IN set
  const int need = k - nin;
  for (int t = lane; t < nun; t += 32) {
    const int i = ul[t];
    const double di = ex[i];
    const long long ii = (long long)key_pos(mrow[i]);
    int rank = 0;
    for (int u = 0; u < nun; ++u) {
      const int j = ul[u];
      const double dj = ex[j];
      const long long ij = (long long)key_pos(mrow[j]);
      rank += dj < di || (dj == di && ij < ii);
    }
    if (rank < need) a[i] = -a[i] - 1.0;  // selected (approx distances are >= 0): mark by negation
  }
  __syncwarp();
  // emit in approximate order: IN entries and the selected uncertain ones
  int outn = 0;
  for (int b = 0; b < kp; b += 32) {
    const int i = b + lane;
    const bool sel = i < kp && (ex[i] == -1.0 || a[i] < 0.0);
    const unsigned bs = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int o = outn + __popc(bs & ((1u << lane) - 1u));
      const long long pos = key_pos(mrow[i]);
      oid[o] = (r.idmap ? r.idmap[pos] : pos) + r.id_offset;
      od[o] = ex[i] == -1.0 ? (double)key_dist(mrow[i]) : ex[i];
    }
    outn += __popc(bs);
  }
  pad_row(oid, od, k, r.ldo, lane, 32);
}

cudaError_t launch_coarse_set(const RerankLaunch& r, cudaStream_t st) {
  if (r.B <= 0) return cudaSuccess;
  if (r.kp_max > kSetMax || r.d > kSetMaxD) return cudaErrorInvalidValue;
  const int dpad = (r.d + 15) & ~15;
  const size_t smem = (size_t)dpad * 8 + (size_t)kSetRows * dpad * 4;
  cudaError_t e = cudaFuncSetAttribute(coarse_set_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(coarse_set_kernel, (r.B + kSetWarps - 1) / kSetWarps, 32 * kSetWarps, smem, st, r);
  return cudaGetLastError();
}

cudaError_t launch_rerank(const RerankLaunch& r, cudaStream_t st) {
  if (r.B <= 0) return cudaSuccess;
  // fused re-rank geometry for a capacity kpm: slab width S, threads, smem
  struct Geom {
    int S, threads;
    size_t smem;
  };
  auto geom = [&](int kpm) {
    // slab width: 2 buffers x kp x (S+4) floats <= ~72 KB (several CTAs per SM)
    int S = std::max(32, std::min(256, 8192 / kpm)) / 16 * 16;  // slabs hold whole 8-element blocks, 16B rows
    // wide candidate lists run 256-512 threads at ~100 registers: 1-2 CTAs per
    // SM whatever the ring size, so the ring may grow to the SM's shared memory
    // (fewer, larger bulk-copy rounds; option "rerank_wide_slab", 0 = off)
    if (g_rerank_wide_slab > 0 && kpm >= 128 && !g_rerank_smem_cap) {
      const long long fixed = (long long)((r.d + 15) & ~15) * 8 + (long long)kpm * 24;
      const long long fit = (200 * 1024 - fixed) / (2LL * kpm * 4) - 4;
      S = (int)std::max<long long>(S, std::min<long long>({(long long)g_rerank_wide_slab, fit, 256LL}) / 16 * 16);
    }
    if (g_rerank_smem_cap > 0) {  // leave room for co-resident CTAs (option "rerank_smem_cap")
      const long long fixed = (long long)((r.d + 15) & ~15) * 8 + (long long)kpm * 16;
      const long long fit = (g_rerank_smem_cap - fixed) / (2LL * kpm * 4) - 4;
      S = (int)std::max<long long>(32, std::min<long long>(S, fit / 16 * 16));
    }
    // a fused compact merge gets 8 warps (the distance phase uses 2 threads per candidate)
    const int threads = r.compact_cnt ? std::max(2 * kpm, 256) : 2 * kpm;
    const size_t smem = (size_t)((r.d + 15) & ~15) * sizeof(double) + (size_t)kpm * 24 +
                        std::max((size_t)2 * kpm * (S + 4) * sizeof(float),
                                 (size_t)std::min(8, threads / 32) * kpm * 8);
    return Geom{S, threads, smem};
  };
  auto fused = [&](const RerankLaunch& rl, const Geom& g, cudaStream_t s) -> cudaError_t {
    auto* kern = g_rerank_f2f ? rerank_fused_kernel<true> : rerank_fused_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) return e;
    (void)launch_pdl(kern, r.B, g.threads, g.smem, s, rl, g.S);
    return cudaGetLastError();
  };
  const Geom gw = geom(r.kp_max);
  if (r.kp_max <= 256 && gw.smem <= 200 * 1024) {
    RerankLaunch rl = r;
    rl.lpt = g_rerank_lpt && r.kp_max > kMinKp;  // one class only: the order is the identity anyway
    rl.lpt_cls = 0;
    if (!(rl.lpt && g_rerank_split && !g_pdl && !r.compact_cnt)) return fused(rl, gw, st);
    // mixed capacities: the kp-32 class on the forked stream, the wider
    // classes here; each grid has B CTAs, those past its class count exit
    SideStream* sd = nullptr;
    cudaError_t e = side_stream(st, &sd);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(sd->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(sd->s, sd->fork, 0)) != cudaSuccess) return e;
    RerankLaunch rn = rl;
    rn.kp_max = kMinKp;
    rn.lpt_cls = 1;
    if ((e = fused(rn, geom(kMinKp), sd->s)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(sd->join, sd->s)) != cudaSuccess) return e;
    rl.lpt_cls = 2;
    if ((e = fused(rl, gw, st)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(st, sd->join, 0);
  }
  if (r.compact_cnt) {  // the pair kernels read merged lists: merge first
    cudaError_t me = launch_merge_compact(r.part, r.compact_cnt, r.meta, const_cast<unsigned long long*>(r.merged),
                                          r.ld_merged, r.B, r.kp_max, st);
    if (me != cudaSuccess) return me;
  }
  const int slab = std::min(kPairSlab, (r.d + 15) & ~15);
  const int row_stride = slab + 4;  // floats; 16B-aligned rows, 2-way worst bank conflict
  const size_t smem = (size_t)slab * sizeof(double) + (size_t)kPairCands * row_stride * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(exact_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(exact_pairs_kernel, (unsigned)(r.B * (r.ld_merged / kPairCands)), 2 * kPairCands, smem, st, r, row_stride);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (r.kp_max <= 256) {
    (void)launch_pdl(finalize_warp_kernel, (r.B + 3) / 4, 128, 0, st, r);
    return cudaGetLastError();
  }
  const size_t fsm = (size_t)r.kp_max * sizeof(Exact);
  e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(finalize_kernel, r.B, 128, fsm, st, r);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact fix-up for uncertified queries: fp64 scan of the full candidate set.

// Split fix-up.  Each uncertified query's candidate set (the concatenation of
// its probed lists, or all rows) is cut into slices of >= kThreads rows, at
// most S per query, S chosen on the device from the flagged count so that the
// units fill about kFxWaves x the grid (one flagged query alone spreads over
// every SM).  The query's bound fx_thr starts at the re-rank's k-th exact
// distance (flag_query), so only rows at or below it can enter the top-k.
// A unit screens its rows with the fp32 distance of the SIMT scan: only rows
// within 4x the SIMT error bound of the bound get the exact float64 distance
// (the reference order), because fp64 runs at a small fraction of the fp32
// rate.  Survivors are kept as the slice's top-k (threshold + compaction +
// smem sort), and a full slice publishes its k-th distance to fx_thr
// (atomicMin on the double's bits, d >= 0).  The last CTA merges each
// query's slice lists, keeping only entries at or below the final bound.
// With no flagged query the kernel exits at once.
constexpr int kFxWaves = 3;
constexpr int kFxSurv = 1024;  // screened rows per slice awaiting their exact distance

// Block-wide sum over the block of a 64-bit value (every thread gets it).
__device__ __forceinline__ long long fx_block_sum(long long v, long long* s_w) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) t += s_w[w];
  __syncthreads();
  return t;
}

// Candidate-set size of query q: its probed lists' lengths summed by the block
// (one parallel round of loads instead of a chain of nprobe dependent ones).
__device__ __forceinline__ long long fx_total(const FixupLaunch& f, int q, long long* s_w) {
  if (!f.probes) return f.n_rows;
  long long t = 0;
  for (int j = threadIdx.x; j < f.nprobe[q]; j += kThreads) {
    const long long l = f.probes[(long long)q * f.ld_probes + j];
    if (l >= 0) t += f.list_off[l + 1] - f.list_off[l];
  }
  return fx_block_sum(t, s_w);
}

// Slices of a query's candidate set: >= rows_min rows each, at most S.
__device__ __forceinline__ int fx_slices_of(long long total, int S, int rows_min) {
  return (int)max(1LL, min((long long)S, total / rows_min));
}

// The query's current fix-up bound as an Exact (ties at the bound distance pass).
__device__ __forceinline__ Exact fx_bound(const FixupLaunch& f, int fi) {
  Exact e;
  e.d = __longlong_as_double((long long)__ldcg(f.fx_thr + fi));
  e.id = 0x7fffffffffffffffll;
  return e;
}

// Stream-compacted candidates in fbuf (count s_cnt, capacity cap): sort and keep
// the k best once fewer than kThreads free slots remain (or when forced).
// Returns the count, negative when fbuf was left unsorted.
__device__ __forceinline__ int fx_compact(Exact* fbuf, int* s_cnt, int cap, int k, bool force) {
  const int n = *s_cnt;
  if (force || n > cap - kThreads) {
    const int p2 = next_pow2(n > 0 ? n : 1);
    for (int i = n + threadIdx.x; i < p2; i += kThreads) fbuf[i] = exact_max();
    __syncthreads();
    block_sort(fbuf, p2, ExactLess());
    __syncthreads();
    if (threadIdx.x == 0 && n > k) *s_cnt = k;
    __syncthreads();
    return min(n, k);
  }
  return -1 - n;
}

// After a round of appends (and a barrier): compact if needed, publish a full
// list's k-th distance to the query's bound, pick up a tighter bound.  Ends
// with a barrier.
__device__ __forceinline__ void fx_update(const FixupLaunch& f, int fi, int k, Exact* fbuf, int* s_cnt, int cap,
                                          Exact* s_thr) {
  const int n = fx_compact(fbuf, s_cnt, cap, k, false);  // < 0: not sorted this round
  if (threadIdx.x == 0) {
    if (n >= k && exact_less(fbuf[k - 1], *s_thr)) {
      *s_thr = fbuf[k - 1];
      atomicMin(f.fx_thr + fi, (unsigned long long)__double_as_longlong(fbuf[k - 1].d));
    }
    const Exact g = fx_bound(f, fi);  // tighter bound from another slice
    if (exact_less(g, *s_thr)) *s_thr = g;
  }
  __syncthreads();
}

__device__ void fixup_merge_all(const FixupLaunch& f, int S, const Exact* part, int ldp, Exact* fbuf, int cap,
                                int* s_cnt, long long* s_w);

__global__ void __launch_bounds__(kThreads) fixup_part_kernel(FixupLaunch f, int cap, Exact* part, int ldp) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ Exact fbuf[];
  __shared__ int s_cnt;
  __shared__ Exact s_thr;
  __shared__ int s_last;
  __shared__ long long s_w[kThreads / 32];
  __shared__ long long s_rlo[kThreads], s_rlen[kThreads], s_rpre[kThreads];
  __shared__ long long s_surv[kFxSurv];
  __shared__ int s_ns, s_ovf;
  const int nf = *f.n_flag;
  if (nf == 0) return;  // every query certified: nothing to do (the common case)
  const int S = max(1, min((kFxWaves * (int)gridDim.x + nf - 1) / nf, f.max_units / nf));
  const int units = nf * S;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int fi = u / S, sl = u - fi * S;
    const int q = f.flag_list[fi];
    if (isnan(f.qn64[q])) continue;  // non-finite query: no rescan, the merge writes an empty row
    const int k = f.meta[q].k;
    const double* qv = f.q64 + (long long)q * f.d;
    const long long total = fx_total(f, q, s_w);
    const int Sq = fx_slices_of(total, S, f.slice_rows);
    if (sl >= Sq) continue;  // uniform per CTA
    const long long c0 = total * sl / Sq, c1 = total * (sl + 1) / Sq;
    const float4* q4 = reinterpret_cast<const float4*>(f.Q32 + (size_t)q * f.qld);
    const float qn = f.qn32[q];
    const double sn = f.qn64[q] + f.xmax;
    const double Epre = 4.0 * (f.cdot * 2.0 * f.qn64[q] * f.xmax + f.csum * sn * sn) + 1e-30;
    if (threadIdx.x == 0) {
      s_cnt = 0;
      s_thr = fx_bound(f, fi);
    }
    __syncthreads();
    // Pass 0 screens every row of the slice with its fp32 distance, one warp
    // per 4 rows (coalesced row loads), and records survivors in s_surv; pass
    // 1 (only if s_surv overflowed) computes the exact distance of every row.
    if (threadIdx.x == 0) {
      s_ns = 0;
      s_ovf = 0;
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1 && !s_ovf) break;  // uniform: read after a barrier
      // walk the ranges overlapping [c0, c1) of the concatenated candidate
      // order, kThreads probes at a time: lengths loaded in parallel, block prefix sum
      const int nranges = f.probes ? f.nprobe[q] : 1;
      long long before = 0;
      for (int cs = 0; cs < nranges && before < c1; cs += kThreads) {
        const int j = cs + threadIdx.x;
        long long lo = 0, len = 0;
        if (j < nranges) {
          if (f.probes) {
            const long long l = f.probes[(long long)q * f.ld_probes + j];
            if (l >= 0) {
              lo = f.list_off[l];
              len = f.list_off[l + 1] - lo;
            }
          } else {
            len = f.n_rows;
          }
        }
        long long inc = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, inc, o);
          if ((threadIdx.x & 31) >= o) inc += y;
        }
        if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = inc;
        __syncthreads();
        long long off = 0, chunk = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
          if (w < (threadIdx.x >> 5)) off += s_w[w];
          chunk += s_w[w];
        }
        s_rlo[threadIdx.x] = lo;
        s_rlen[threadIdx.x] = len;
        s_rpre[threadIdx.x] = before + off + inc - len;
        __syncthreads();
        const int nr = min(kThreads, nranges - cs);
        for (int rg = 0; rg < nr; ++rg) {
          const long long pre = s_rpre[rg], rlen = s_rlen[rg], rlo = s_rlo[rg];
          const long long a = max(c0, pre), b = min(c1, pre + rlen);
          if (a >= b) continue;  // uniform: shared-memory values
          const long long r0 = rlo + (a - pre), r1 = rlo + (b - pre);
          if (pass == 0) {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const double lim = fx_bound(f, fi).d + Epre;
            for (long long row0 = r0 + warp * 4; row0 < r1; row0 += kThreads / 32 * 4) {
              // the 4 rows' loads issue together (rows past r1 re-read row r1 - 1)
              float acc[4] = {0.f, 0.f, 0.f, 0.f};
              const float4* x4[4];
#pragma unroll
              for (int i = 0; i < 4; ++i)
                x4[i] = reinterpret_cast<const float4*>(f.X + min(row0 + i, r1 - 1) * f.ldx);
#pragma unroll 2
              for (int c = lane; c < (f.qld >> 2); c += 32) {
                const float4 y = __ldg(q4 + c);
                float4 x[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = __ldg(x4[i] + c);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  acc[i] = __fmaf_rn(x[i].x, y.x, acc[i]);
                  acc[i] = __fmaf_rn(x[i].y, y.y, acc[i]);
                  acc[i] = __fmaf_rn(x[i].z, y.z, acc[i]);
                  acc[i] = __fmaf_rn(x[i].w, y.w, acc[i]);
                }
              }
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int o = 16; o; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
              if (lane < 4 && row0 + lane < r1) {
                const long long row = row0 + lane;
                const float dot = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
                const float d32 = __fmaf_rn(-2.f, dot, __fadd_rn(qn, f.xnorm[row]));
                if (!isfinite(d32) || (double)d32 <= lim) {
                  const int idx = atomicAdd(&s_ns, 1);
                  if (idx < kFxSurv) s_surv[idx] = row;
                  else s_ovf = 1;
                }
              }
            }
          } else {
            for (long long base = r0; base < r1; base += kThreads) {
              const long long row = base + threadIdx.x;
              const Exact thr = s_thr;
              if (row < r1) {
                Exact e;
                e.d = exact_sq_dist_any(qv, f.X + row * f.ldx, f.d);
                e.id = (f.idmap ? f.idmap[row] : row) + f.id_offset;
                if (exact_less(e, thr)) fbuf[atomicAdd(&s_cnt, 1)] = e;
              }
              __syncthreads();
              fx_update(f, fi, k, fbuf, &s_cnt, cap, &s_thr);
            }
          }
        }
        before += chunk;
        __syncthreads();  // s_w / s_r* are rewritten by the next chunk
      }
      if (pass == 0 && !s_ovf) {
        // exact distances of the survivors, kThreads at a time
        const int ns = s_ns;
        for (int b0 = 0; b0 < ns; b0 += kThreads) {
          const Exact thr = s_thr;
          if (b0 + (int)threadIdx.x < ns) {
            const long long row = s_surv[b0 + threadIdx.x];
            Exact e;
            e.d = exact_sq_dist_any(qv, f.X + row * f.ldx, f.d);
            e.id = (f.idmap ? f.idmap[row] : row) + f.id_offset;
            if (exact_less(e, thr)) fbuf[atomicAdd(&s_cnt, 1)] = e;
          }
          __syncthreads();
          fx_update(f, fi, k, fbuf, &s_cnt, cap, &s_thr);
        }
      }
      __syncthreads();
    }
    const int n = fx_compact(fbuf, &s_cnt, cap, k, true);
    if (threadIdx.x == 0 && n >= k)
      atomicMin(f.fx_thr + fi, (unsigned long long)__double_as_longlong(fbuf[k - 1].d));
    Exact* dst = part + ((long long)fi * S + sl) * ldp;
    for (int j = threadIdx.x; j < n; j += kThreads) dst[j] = fbuf[j];
    if (threadIdx.x == 0) f.fx_cnt[fi * S + sl] = n;
    __syncthreads();
  }
  // the last CTA to finish merges every flagged query's slices (partials and
  // bounds published with a fence before the completion ticket)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(const_cast<int*>(f.n_flag) + 1, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  fixup_merge_all(f, S, part, ldp, fbuf, cap, &s_cnt, s_w);
}

__device__ void fixup_merge_all(const FixupLaunch& f, int S, const Exact* part, int ldp, Exact* fbuf, int cap,
                                int* s_cnt, long long* s_w) {
  for (int fi = 0; fi < *f.n_flag; ++fi) {
    const int q = f.flag_list[fi];
    const int k = f.meta[q].k;
    if (isnan(f.qn64[q])) {  // non-finite query (device-buffer entry points): id -1, distance NaN
      for (int j = threadIdx.x; j < k; j += kThreads) {
        f.out_ids[(long long)q * f.ldo + j] = -1;
        f.out_d[(long long)q * f.ldo + j] = __longlong_as_double(0x7ff8000000000000ll);
      }
      continue;
    }
    const Exact bound = fx_bound(f, fi);
    if (threadIdx.x == 0) *s_cnt = 0;
    __syncthreads();
    // slice lists are sorted: thread t walks slices t, t + kThreads, ... one
    // entry per round (at most kThreads appends between compactions) and
    // stops at the first entry above the bound
    const int Sq = fx_slices_of(fx_total(f, q, s_w), S, f.slice_rows);
    for (int s0 = 0; s0 < Sq; s0 += kThreads) {
      const int sl = s0 + threadIdx.x;
      const int cnt = sl < Sq ? f.fx_cnt[fi * S + sl] : 0;
      const Exact* src = part + ((long long)fi * S + sl) * ldp;
      int j = 0;
      for (;;) {
        bool more = false;
        if (j < cnt) {
          const Exact e = src[j];
          if (!exact_less(bound, e)) {
            fbuf[atomicAdd(s_cnt, 1)] = e;
            more = ++j < cnt;
          } else {
            j = cnt;
          }
        }
        if (!__syncthreads_or(more)) break;
        fx_compact(fbuf, s_cnt, cap, k, false);
        __syncthreads();  // the count is read before anyone appends again
      }
      fx_compact(fbuf, s_cnt, cap, k, false);
      __syncthreads();
    }
    const int n = fx_compact(fbuf, s_cnt, cap, k, true);
    for (int j = threadIdx.x; j < k; j += kThreads) {
      const Exact e = j < n ? fbuf[j] : exact_max();
      const bool ok = e.id != 0x7fffffffffffffffll;
      f.out_ids[(long long)q * f.ldo + j] = ok ? e.id : -1;
      f.out_d[(long long)q * f.ldo + j] = e.d;
    }
    __syncthreads();
  }
}

int fixup_slices(int k_max) { return std::max(1, std::min(32, 4096 / std::max(1, k_max))); }

size_t fixup_thr_bytes(int B) { return ((size_t)B * sizeof(unsigned long long) + 255) & ~(size_t)255; }

int fixup_max_units(int B, int k_max) { return B * fixup_slices(k_max); }

size_t fixup_cnt_bytes(int B, int k_max) {
  return ((size_t)fixup_max_units(B, k_max) * sizeof(int) + 255) & ~(size_t)255;
}

size_t fixup_scratch_bytes(int B, int k_max) {
  return fixup_thr_bytes(B) + fixup_cnt_bytes(B, k_max) + (size_t)fixup_max_units(B, k_max) * k_max * sizeof(Exact);
}

cudaError_t launch_fixup(const FixupLaunch& f, cudaStream_t st) {
  if (f.B <= 0) return cudaSuccess;
  const int cap = next_pow2(f.k_max + kThreads);
  const size_t smem = (size_t)cap * sizeof(Exact);
  cudaError_t e = cudaFuncSetAttribute(fixup_part_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  (void)launch_pdl(fixup_part_kernel, 4 * nsm, kThreads, smem, st, f, cap, f.scratch, f.k_max);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fixed-shape distance batch (engine.execute_distance_batch, engine.py:229-256).

__global__ void distance_tasks_kernel(const int* __restrict__ owner, const long long* __restrict__ cand,
                                      int n_tasks, const double* __restrict__ q64, int d,
                                      const float* __restrict__ X, long long ldx, long long n_rows,
                                      double* __restrict__ out, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_tasks) return;
  long long c = cand[i];
  if (c < 0 || c >= n_rows) {
    atomicExch(err, 1);
    out[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  out[i] = exact_sq_dist_any(q64 + (long long)owner[i] * d, X + c * ldx, d);
}

cudaError_t launch_distance_tasks(const int* owner, const long long* cand, int n_tasks, const double* q64, int d,
                                  const float* X, long long ldx, long long n_rows, double* out, int* err,
                                  cudaStream_t st) {
  if (n_tasks <= 0) return cudaSuccess;
  distance_tasks_kernel<<<(n_tasks + 127) / 128, 128, 0, st>>>(owner, cand, n_tasks, q64, d, X, ldx, n_rows, out,
                                                                 err);
  return cudaGetLastError();
}

// rowwise_sq_dists on float64 rows (ann_graph.py:97-105) for rows that are not
// in a float32 store: same einsum operation order as exact_sq_dist, both
// operands float64.  q_stride = 0 broadcasts one query; d pairs row i with
// query row i (numpy broadcasting of a (n, d) query).
__global__ void rowwise_f64_kernel(const double* __restrict__ q, long long q_stride, const double* __restrict__ X,
                                   long long n, int d, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* qq = q + i * q_stride;
  const double* x = X + i * d;
  double l0 = 0.0, l1 = 0.0;
  int j = 0;
  for (; j + 8 <= d; j += 8) {
#pragma unroll
    for (int sub = 3; sub >= 0; --sub) {
      const double t0 = __dsub_rn(qq[j + 2 * sub], x[j + 2 * sub]);
      const double t1 = __dsub_rn(qq[j + 2 * sub + 1], x[j + 2 * sub + 1]);
      l0 = __dadd_rn(__dmul_rn(t0, t0), l0);
      l1 = __dadd_rn(__dmul_rn(t1, t1), l1);
    }
  }
  for (; j < d; j += 2) {
    const double t0 = __dsub_rn(qq[j], x[j]);
    l0 = __dadd_rn(__dmul_rn(t0, t0), l0);
    if (j + 1 < d) {
      const double t1 = __dsub_rn(qq[j + 1], x[j + 1]);
      l1 = __dadd_rn(__dmul_rn(t1, t1), l1);
    }
  }
  out[i] = __dadd_rn(l0, l1);
}

cudaError_t launch_rowwise_f64(const double* q, long long q_stride, const double* X, long long n, int d, double* out,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  rowwise_f64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(q, q_stride, X, n, d, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact merge of G per-shard top-k lists (dist, id) -> global top-k.

__global__ void __launch_bounds__(kThreads) merge_exact_kernel(const double* __restrict__ dists,
                                                               const long long* __restrict__ ids, int G, int B,
                                                               int k_in, int k_out, double* __restrict__ out_d,
                                                               long long* __restrict__ out_ids, int n2, int ld_in,
                                                               int ld_out, long long g_stride) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ Exact mbuf[];
  const int q = blockIdx.x;
  const int n = G * k_in;
  for (int i = threadIdx.x; i < n2; i += kThreads) {
    Exact e = exact_max();
    if (i < n) {
      int g = i / k_in, j = i - g * k_in;
      long long off = (long long)g * g_stride + (long long)q * ld_in + j;
      long long id = ids[off];
      if (id >= 0) {
        e.d = dists[off];
        e.id = id;
      }
    }
    mbuf[i] = e;
  }
  __syncthreads();
  block_sort(mbuf, n2, ExactLess());
  for (int j = threadIdx.x; j < ld_out; j += kThreads) {  // columns past k_out: id -1, distance +inf
    const Exact e = j < k_out ? mbuf[j] : exact_max();
    const bool ok = e.id != 0x7fffffffffffffffll;
    out_ids[(long long)q * ld_out + j] = ok ? e.id : -1;
    out_d[(long long)q * ld_out + j] = ok ? e.d : __longlong_as_double(0x7ff0000000000000ll);
  }
}

cudaError_t launch_merge_exact(const double* dists, const long long* ids, int G, int B, int k_in, int k_out,
                               double* out_d, long long* out_ids, cudaStream_t st, int ld_in, int ld_out,
                               long long g_stride) {
  if (B <= 0) return cudaSuccess;
  int n2 = next_pow2(G * k_in);
  size_t smem = (size_t)n2 * sizeof(Exact);
  cudaError_t e =
      cudaFuncSetAttribute(merge_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(merge_exact_kernel, B, kThreads, smem, st, dists, ids, G, B, k_in, k_out, out_d, out_ids, n2, ld_in, ld_out,
                                                   g_stride);
  return cudaGetLastError();
}

}  // namespace tri
