// Dense brute force for small stores (the IVF coarse step over the centroids,
// small brute-force stores): the full B x n approximate distance matrix is
// cheap to materialise in L2, so instead of the streaming list scan:
//   dense_gemm_kernel   fp32 SIMT GEMM tile (64 queries x 128 rows per CTA,
//                       8x8 outputs per thread, split-K, K staged through smem)
//                       with the same error model as the SIMT scan (sequential
//                       fp32 FMA chains over K: cdot = gamma_d);
//   dense_select_kernel one CTA per query: slice sum + dot-form distance keys,
//                       shared-memory bitonic sort, first kp keys -> the
//                       `merged` candidate list consumed by the exact re-rank.
#include <algorithm>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

// ---------------------------------------------------------------------------
// dense_gemm_kernel: CTA tile 64 queries x 128 rows, 128 threads, 8 x 8
// outputs per thread (queries tq*4+{0..3} and 32+tq*4+{0..3}, rows tr*4+{0..3}
// and 64+tr*4+{0..3}), K in 16-wide steps double-buffered through shared
// memory with the next step's global loads in flight during the FMAs.
// Split-K over blockIdx.z fills the GPU (the problem is only ~B*n/64 threads
// wide); each slice is a sequential fp32 FMA chain over its K range, so the
// summed dot stays within gamma_d (the select kernel adds the slices in a
// fixed order).
constexpr int kGq = 64, kGr = 128, kGk = 16, kGThreads = 128;
int g_dense_slices = 8;

struct GemmRegs {
  float4 q[2], x[4];
};

__device__ __forceinline__ void gemm_load(GemmRegs& r, const float* __restrict__ Q, int qld, int B, int q0,
                                          const float* __restrict__ X, long long ldx, long long n, long long r0,
                                          int k0, int ke, int tid) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * kGThreads, qq = i >> 2, kk = (i & 3) * 4;
    r.q[u] = (q0 + qq < B && k0 + kk < ke) ? *reinterpret_cast<const float4*>(Q + (long long)(q0 + qq) * qld + k0 + kk)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = tid + u * kGThreads, rr = i >> 2, kk = (i & 3) * 4;
    r.x[u] = (r0 + rr < n && k0 + kk < ke) ? *reinterpret_cast<const float4*>(X + (r0 + rr) * ldx + k0 + kk)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__device__ __forceinline__ void gemm_store(const GemmRegs& r, float (*Qs)[kGq], float (*Xs)[kGr], int tid) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * kGThreads, qq = i >> 2, kk = (i & 3) * 4;
    Qs[kk + 0][qq] = r.q[u].x;
    Qs[kk + 1][qq] = r.q[u].y;
    Qs[kk + 2][qq] = r.q[u].z;
    Qs[kk + 3][qq] = r.q[u].w;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = tid + u * kGThreads, rr = i >> 2, kk = (i & 3) * 4;
    Xs[kk + 0][rr] = r.x[u].x;
    Xs[kk + 1][rr] = r.x[u].y;
    Xs[kk + 2][rr] = r.x[u].z;
    Xs[kk + 3][rr] = r.x[u].w;
  }
}

__global__ void __launch_bounds__(kGThreads) dense_gemm_kernel(const float* __restrict__ Q, int qld, int B,
                                                               const float* __restrict__ X, long long ldx, long long n,
                                                               int dp, int kslice, float* __restrict__ P,
                                                               long long ldd) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  __shared__ __align__(16) float Qs[2][kGk][kGq];
  __shared__ __align__(16) float Xs[2][kGk][kGr];
  const int tid = threadIdx.x;
  const int tq = tid >> 4, tr = tid & 15;
  const int q0 = blockIdx.x * kGq;
  const long long r0 = (long long)blockIdx.y * kGr;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  const int kb = blockIdx.z * kslice, ke = min(dp, kb + kslice);
  GemmRegs reg;
  gemm_load(reg, Q, qld, B, q0, X, ldx, n, r0, kb, ke, tid);
  gemm_store(reg, Qs[0], Xs[0], tid);
  __syncthreads();
  int buf = 0;
  for (int k0 = kb; k0 < ke; k0 += kGk) {
    const bool more = k0 + kGk < ke;
    if (more) gemm_load(reg, Q, qld, B, q0, X, ldx, n, r0, k0 + kGk, ke, tid);
#pragma unroll
    for (int kk = 0; kk < kGk; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&Qs[buf][kk][tq * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&Qs[buf][kk][32 + tq * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Xs[buf][kk][tr * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Xs[buf][kk][64 + tr * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) gemm_store(reg, Qs[buf ^ 1], Xs[buf ^ 1], tid);
    __syncthreads();
    buf ^= 1;
  }
  float* Pz = P + (long long)blockIdx.z * B * ldd;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int q = q0 + (i < 4 ? tq * 4 + i : 32 + tq * 4 + i - 4);
    if (q >= B) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long r = r0 + h * 64 + tr * 4;
      float* dst = Pz + (long long)q * ldd + r;
      if (r + 3 < n) {
        *reinterpret_cast<float4*>(dst) = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (r + j < n) dst[j] = acc[i][4 * h + j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// dense_select_kernel: one CTA (256 threads) per query, up to 16 rows per
// thread in registers.  Sums the split-K slices in a fixed order and forms the
// dot-form distance fl(fl(|q|^2 + |x|^2) - 2 q.x) exactly as the scans do;
// then a bisection on the order-preserving distance bits finds a threshold T
// with kp <= #{dist <= T} <= 2 kp (one block count per step), the survivors are
// compacted and bitonic-sorted in shared memory, and the first kp keys are the
// query's candidate list.  If ties make the window unreachable (> cap equal
// distances) the list is left empty: the re-rank cannot certify it and the
// exact fix-up answers the query.
constexpr int kSelThreads = 256, kSelPer = 16, kSelCap = 512;
long long g_dense_fold = 1;  // warp-list selection instead of bisection (option "dense_fold")

__global__ void __launch_bounds__(kSelThreads) dense_select_kernel(const float* __restrict__ P, int nsl,
                                                                   long long ldd, int B,
                                                                   const float* __restrict__ qn,
                                                                   const float* __restrict__ xn, long long n,
                                                                   const QueryMeta* __restrict__ meta,
                                                                   unsigned long long* __restrict__ merged,
                                                                   int ld_merged) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  __shared__ unsigned long long cand[kSelCap];
  __shared__ int red[2][kSelThreads / 32];
  __shared__ int s_cnt;
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* row = P + (long long)q * ldd;
  const long long slice_ld = (long long)B * ldd;
  const float qv = qn[q];
  const int kp = meta[q].kp;
  // thread t owns rows 4t..4t+3 of every 1024-row block (float4 loads; ldd and
  // the slices are 4-aligned), slices summed in order as before
  uint32_t ord[kSelPer];
  uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
  for (int g = 0; g < kSelPer / 4; ++g) {
    const long long i0 = (long long)g * 4 * kSelThreads + 4 * tid;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i0 < n) {
      for (int z = 0; z < nsl; ++z) {
        const float4 v = *reinterpret_cast<const float4*>(row + z * slice_ld + i0);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
    }
    const float av[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long i = i0 + j;
      ord[4 * g + j] = 0xffffffffu;
      if (i < n) {
        ord[4 * g + j] = f2ord(__fmaf_rn(-2.f, av[j], __fadd_rn(qv, xn[i])));
        lo = min(lo, ord[4 * g + j]);
        hi = max(hi, ord[4 * g + j]);
      }
    }
  }
  // block min / max of the keys' distance bits
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) {
    red[0][warp] = (int)(lo ^ 0x80000000u);
    red[1][warp] = (int)(hi ^ 0x80000000u);
  }
  __syncthreads();
  lo = 0xffffffffu;
  hi = 0u;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) {
    lo = min(lo, (uint32_t)red[0][w] ^ 0x80000000u);
    hi = max(hi, (uint32_t)red[1][w] ^ 0x80000000u);
  }
  // bisection: smallest-found T with kp <= count(ord <= T) <= cap (count(hi) = n >= kp when n >= kp)
  uint32_t T = hi;
  if (n > kSelCap) {
    uint32_t a = lo, b = hi;  // invariant: count(b) >= kp
    for (int it = 0; it < 40 && a < b; ++it) {
      const uint32_t mid = a + ((b - a) >> 1);
      int c = 0;
#pragma unroll
      for (int u = 0; u < kSelPer; ++u) c += ord[u] <= mid;
      c = __reduce_add_sync(0xffffffffu, c);
      __syncthreads();  // red reused
      if (lane == 0) red[0][warp] = c;
      __syncthreads();
      c = 0;
#pragma unroll
      for (int w = 0; w < kSelThreads / 32; ++w) c += red[0][w];
      if (c >= kp) {
        b = mid;
        if (c <= max(2 * kp, 64)) break;  // small sort window; the cap only guards ties
      } else {
        a = mid + 1;
      }
    }
    T = b;
  }
  if (tid == 0) s_cnt = 0;
  for (int i = tid; i < kSelCap; i += kSelThreads) cand[i] = TRI_KEY_MAX;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSelPer; ++u) {
    const long long i = (long long)(u >> 2) * 4 * kSelThreads + 4 * tid + (u & 3);
    if (i < n && ord[u] <= T) {
      const int p = atomicAdd(&s_cnt, 1);
      if (p < kSelCap) cand[p] = ((unsigned long long)ord[u] << 32) | (unsigned long long)i;
    }
  }
  __syncthreads();
  const int c = min(s_cnt, kSelCap);
  block_sort(cand, next_pow2(max(c, 2)), KeyLess());
  // more than kSelCap equal-distance survivors: an empty list is never
  // certified, so the query goes to the exact fix-up scan
  const bool over = s_cnt > kSelCap;
  for (int j = tid; j < kp; j += kSelThreads)
    merged[(long long)q * ld_merged + j] = (j < c && !over) ? cand[j] : TRI_KEY_MAX;
}

cudaError_t launch_dense(const float* Q, int qld, const float* qn, int B, const float* X, long long ldx,
                         const float* xn, long long n, int dp, float* D, long long ldd, const QueryMeta* meta,
                         unsigned long long* merged, int ld_merged, int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const int nsl = std::max(1, std::min(kDenseSlices, g_dense_slices));
  const int kslice = ((dp + nsl - 1) / nsl + kGk - 1) / kGk * kGk;
  const int used = (dp + kslice - 1) / kslice;
  dim3 grid((B + kGq - 1) / kGq, (unsigned)((n + kGr - 1) / kGr), used);
  (void)launch_pdl(dense_gemm_kernel, grid, kGThreads, 0, st, Q, qld, B, X, ldx, n, dp, kslice, D, ldd);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_dense_select(D, used, ldd, B, qn, xn, n, meta, merged, ld_merged, kp_max, st);
}

// The same selection by warp-resident sorted lists: every warp folds its rows'
// keys 32 at a time into a KL x 32 list (list_fold32: insertion when few beat
// the list's last key), then the 8 warp lists merge pairwise through shared
// memory.  Keys (fp32 order bits << 32 | row) are unique, so the kp smallest
// come out exactly as the bisection path produces them (option "dense_fold").
template <int KL>
__global__ void __launch_bounds__(kSelThreads) dense_select_fold_kernel(const float* __restrict__ P, int nsl,
                                                                        long long ldd, int B,
                                                                        const float* __restrict__ qn,
                                                                        const float* __restrict__ xn, long long n,
                                                                        const QueryMeta* __restrict__ meta,
                                                                        unsigned long long* __restrict__ merged,
                                                                        int ld_merged) {
  pdl_wait();
  constexpr int KP = 32 * KL, NW = kSelThreads / 32;
  __shared__ unsigned long long sm[NW / 2][KP];
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* row = P + (long long)q * ldd;
  const long long slice_ld = (long long)B * ldd;
  const float qv = qn[q];
  const int kp = meta[q].kp;
  unsigned long long L[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) L[j] = TRI_KEY_MAX;
  // thread t owns rows 4t..4t+3 of every 1024-row block (float4 loads), slices summed in order
#pragma unroll
  for (int g = 0; g < kSelPer / 4; ++g) {
    const long long i0 = (long long)g * 4 * kSelThreads + 4 * tid;
    if ((long long)g * 4 * kSelThreads >= n) break;  // block-uniform
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i0 < n) {
      for (int z = 0; z < nsl; ++z) {
        const float4 v = *reinterpret_cast<const float4*>(row + z * slice_ld + i0);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
    }
    const float av[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long i = i0 + j;
      const unsigned long long key =
          i < n ? ((unsigned long long)f2ord(__fmaf_rn(-2.f, av[j], __fadd_rn(qv, xn[i]))) << 32) | (unsigned long long)i
                : TRI_KEY_MAX;
      list_fold32<KL>(L, key, lane);
    }
  }
  // pairwise merge of the warp lists: warp w + stride hands its list (reversed) to warp w
  for (int stride = 1; stride < NW; stride <<= 1) {
    if ((warp & (2 * stride - 1)) == stride) {
#pragma unroll
      for (int j = 0; j < KL; ++j) sm[warp >> 1][j * 32 + lane] = L[j];
    }
    __syncthreads();
    if ((warp & (2 * stride - 1)) == 0) {
      unsigned long long R[KL];
#pragma unroll
      for (int j = 0; j < KL; ++j) R[j] = sm[(warp + stride) >> 1][(KL - 1 - j) * 32 + (31 - lane)];
      list_merge_rev<KL>(L, R, lane);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      const int e = j * 32 + lane;
      if (e < kp) merged[(long long)q * ld_merged + e] = L[j];
    }
  }
}

cudaError_t launch_dense_select(const float* D, int nsl, long long ldd, int B, const float* qn, const float* xn,
                                long long n, const QueryMeta* meta, unsigned long long* merged, int ld_merged,
                                int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (n > (long long)kSelThreads * kSelPer || kp_max > kSelCap / 2) return cudaErrorInvalidValue;
  if (g_dense_fold) {
    const int kl = next_pow2((kp_max + 31) / 32);
    switch (kl) {
      case 1: (void)launch_pdl(dense_select_fold_kernel<1>, B, kSelThreads, 0, st, D, nsl, ldd, B, qn, xn, n, meta,
                               merged, ld_merged); break;
      case 2: (void)launch_pdl(dense_select_fold_kernel<2>, B, kSelThreads, 0, st, D, nsl, ldd, B, qn, xn, n, meta,
                               merged, ld_merged); break;
      case 4: (void)launch_pdl(dense_select_fold_kernel<4>, B, kSelThreads, 0, st, D, nsl, ldd, B, qn, xn, n, meta,
                               merged, ld_merged); break;
      default: (void)launch_pdl(dense_select_fold_kernel<8>, B, kSelThreads, 0, st, D, nsl, ldd, B, qn, xn, n, meta,
                                merged, ld_merged); break;
    }
    return cudaGetLastError();
  }
  (void)launch_pdl(dense_select_kernel, B, kSelThreads, 0, st, D, nsl, ldd, B, qn, xn, n, meta, merged, ld_merged);
  return cudaGetLastError();
}

}  // namespace tri
