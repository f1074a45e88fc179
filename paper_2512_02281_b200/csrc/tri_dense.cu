// Dense brute force for small stores (the IVF coarse step over the centroids,
// small brute-force stores): the full B x n approximate distance matrix is
// cheap to materialise in L2, so instead of the streaming list scan:
//   dense_dist_kernel  fp32 SIMT GEMM tile (64 queries x 64 rows per CTA,
//                      4x4 outputs per thread, split-K, K staged through smem) with the
//                      same dot-form distance and error model as the SIMT scan
//                      (sequential fp32 FMA chain over K: cdot = gamma_d);
//   dense_select_kernel one warp per query: ballot-compacted appends of the
//                      keys beating the running threshold into a per-warp smem
//                      batch, folded 32 at a time into a register top-kp list
//                      (tri_common.cuh networks) -> the `merged` candidate list
//                      consumed by the exact re-rank.
#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

constexpr int kDq = 64, kDr = 64, kDk = 32;

// Global -> register prefetch of one K slab (2 float4 of Q, 4 float4 of X per
// thread), stored transposed into shared memory after the current slab's FMAs.
struct DenseRegs {
  float4 q[2], x[2];
};

__device__ __forceinline__ void dense_load(DenseRegs& r, const float* __restrict__ Q, int qld, int B, int q0,
                                           const float* __restrict__ X, long long ldx, long long n, long long r0,
                                           int k0, int dp, int tid) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * 256, qq = i >> 3, kk = (i & 7) * 4;
    r.q[u] = (q0 + qq < B && k0 + kk < dp) ? *reinterpret_cast<const float4*>(Q + (long long)(q0 + qq) * qld + k0 + kk)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * 256, rr = i >> 3, kk = (i & 7) * 4;
    r.x[u] = (r0 + rr < n && k0 + kk < dp) ? *reinterpret_cast<const float4*>(X + (r0 + rr) * ldx + k0 + kk)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__device__ __forceinline__ void dense_store(const DenseRegs& r, float (*Qs)[kDq], float (*Xs)[kDr + 4], int tid) {
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * 256, qq = i >> 3, kk = (i & 7) * 4;
    Qs[kk + 0][qq] = r.q[u].x;
    Qs[kk + 1][qq] = r.q[u].y;
    Qs[kk + 2][qq] = r.q[u].z;
    Qs[kk + 3][qq] = r.q[u].w;
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int i = tid + u * 256, rr = i >> 3, kk = (i & 7) * 4;
    Xs[kk + 0][rr] = r.x[u].x;
    Xs[kk + 1][rr] = r.x[u].y;
    Xs[kk + 2][rr] = r.x[u].z;
    Xs[kk + 3][rr] = r.x[u].w;
  }
}

// Partial dot products over one K slice (split-K: blockIdx.z); the select
// kernel sums the slices in a fixed order (any order stays within gamma_d).
__global__ void __launch_bounds__(256) dense_dist_kernel(const float* __restrict__ Q, int qld,
                                                         int B, const float* __restrict__ X, long long ldx,
                                                         long long n, int dp, int kslice,
                                                         float* __restrict__ P, long long ldd) {
  __shared__ __align__(16) float Qs[2][kDk][kDq];
  __shared__ __align__(16) float Xs[2][kDk][kDr + 4];
  const int tid = threadIdx.x;
  const int tq = tid >> 4, tr = tid & 15;  // 16 x 16 threads: queries tq*4+{0..3}, rows tr*4+{0..3}
  const int q0 = blockIdx.x * kDq;
  const long long r0 = (long long)blockIdx.y * kDr;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int kb = blockIdx.z * kslice, ke = min(dp, kb + kslice);
  DenseRegs reg;
  dense_load(reg, Q, qld, B, q0, X, ldx, n, r0, kb, ke, tid);
  dense_store(reg, Qs[0], Xs[0], tid);
  __syncthreads();
  int buf = 0;
  for (int k0 = kb; k0 < ke; k0 += kDk) {
    const bool more = k0 + kDk < ke;
    if (more) dense_load(reg, Q, qld, B, q0, X, ldx, n, r0, k0 + kDk, ke, tid);  // in flight during the FMAs
#pragma unroll 8
    for (int kk = 0; kk < kDk; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&Qs[buf][kk][tq * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Xs[buf][kk][tr * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) dense_store(reg, Qs[buf ^ 1], Xs[buf ^ 1], tid);
    __syncthreads();
    buf ^= 1;
  }
  float* Pz = P + (long long)blockIdx.z * B * ldd;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = q0 + tq * 4 + i;
    if (q >= B) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long r = r0 + tr * 4 + j;
      if (r < n) Pz[(long long)q * ldd + r] = acc[i][j];
    }
  }
}

constexpr int kSelWarps = 8;

// Warp w folds elements [w*n/8, (w+1)*n/8) of the query's row into a register
// top-kp list (ballot-compacted 32-key batches), then the 8 lists merge
// pairwise through shared memory.
template <int KL>
__device__ __forceinline__ void dense_select_query(const float* __restrict__ P, int nsl, long long slice_ld, float qv,
                                                   const float* __restrict__ xn, long long n,
                                                   unsigned long long* __restrict__ dst, unsigned long long* buf,
                                                   unsigned long long* tree) {
  constexpr int KP = 32 * KL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long L[KL];
#pragma unroll
  for (int j = 0; j < KL; ++j) L[j] = TRI_KEY_MAX;
  unsigned long long thr = TRI_KEY_MAX;
  int cnt = 0;
  const unsigned lt = (1u << lane) - 1u;
  const long long per = (n + kSelWarps - 1) / kSelWarps;
  const long long lo = warp * per, hi = min(n, lo + per);
  for (long long blk = lo; blk < hi; blk += 128) {
    float dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // 4 independent rows in flight per lane
      const long long i = blk + u * 32 + lane;
      float acc = 0.f;
      if (i < hi) {
        for (int z = 0; z < nsl; ++z) acc = __fadd_rn(acc, P[z * slice_ld + i]);
        acc = __fmaf_rn(-2.f, acc, __fadd_rn(qv, xn[i]));
      }
      dv[u] = acc;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = blk + u * 32 + lane;
      const unsigned long long key = i < hi ? make_key(dv[u], (uint32_t)i) : TRI_KEY_MAX;
      const bool pass = key < thr;
      const unsigned m = __ballot_sync(0xffffffffu, pass);
      if (pass) buf[cnt + __popc(m & lt)] = key;
      cnt += __popc(m);
      if (cnt >= 32) {
        __syncwarp();
        unsigned long long x = buf[lane];
        const int rem = cnt - 32;
        const unsigned long long tail = lane < rem ? buf[32 + lane] : 0ull;
        __syncwarp();
        if (lane < rem) buf[lane] = tail;
        cnt = rem;
        x = warp_sort32(x, lane);
        list_merge32<KL>(L, x, lane);
        thr = __shfl_sync(0xffffffffu, L[KL - 1], 31);
        __syncwarp();
      }
    }
  }
  if (cnt > 0) {
    __syncwarp();
    unsigned long long x = lane < cnt ? buf[lane] : TRI_KEY_MAX;
    x = warp_sort32(x, lane);
    list_merge32<KL>(L, x, lane);
  }
  for (int stride = 1; stride < kSelWarps; stride <<= 1) {
    if ((warp & (2 * stride - 1)) == stride) {
#pragma unroll
      for (int j = 0; j < KL; ++j) tree[warp * KP + j * 32 + lane] = L[j];
    }
    __syncthreads();
    if ((warp & (2 * stride - 1)) == 0) {
      unsigned long long R[KL];
#pragma unroll
      for (int j = 0; j < KL; ++j) R[j] = tree[(warp + stride) * KP + (KL - 1 - j) * 32 + (31 - lane)];
      list_merge_rev<KL>(L, R, lane);
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int j = 0; j < KL; ++j) dst[j * 32 + lane] = L[j];
  }
}

__global__ void __launch_bounds__(32 * kSelWarps) dense_select_kernel(const float* __restrict__ P, int nsl, long long ldd,
                                                                      int B, const float* __restrict__ qn,
                                                                      const float* __restrict__ xn, long long n,
                                                                      const QueryMeta* __restrict__ meta,
                                                                      unsigned long long* __restrict__ merged,
                                                                      int ld_merged) {
  extern __shared__ unsigned long long dsm[];
  __shared__ unsigned long long buf[kSelWarps][64];
  const int q = blockIdx.x;
  const float* row = P + (long long)q * ldd;
  const long long slice_ld = (long long)B * ldd;
  unsigned long long* dst = merged + (long long)q * ld_merged;
  unsigned long long* wb = buf[threadIdx.x >> 5];
  switch (meta[q].kp) {
    case 32: dense_select_query<1>(row, nsl, slice_ld, qn[q], xn, n, dst, wb, dsm); break;
    case 64: dense_select_query<2>(row, nsl, slice_ld, qn[q], xn, n, dst, wb, dsm); break;
    case 128: dense_select_query<4>(row, nsl, slice_ld, qn[q], xn, n, dst, wb, dsm); break;
    default: dense_select_query<8>(row, nsl, slice_ld, qn[q], xn, n, dst, wb, dsm); break;
  }
}

cudaError_t launch_dense(const float* Q, int qld, const float* qn, int B, const float* X, long long ldx,
                         const float* xn, long long n, int dp, float* D, long long ldd, const QueryMeta* meta,
                         unsigned long long* merged, int ld_merged, int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const int nsl = kDenseSlices;
  const int kslice = ((dp + nsl - 1) / nsl + kDk - 1) / kDk * kDk;
  const int used = (dp + kslice - 1) / kslice;
  dim3 grid((B + kDq - 1) / kDq, (unsigned)((n + kDr - 1) / kDr), used);
  dense_dist_kernel<<<grid, 256, 0, st>>>(Q, qld, B, X, ldx, n, dp, kslice, D, ldd);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t)kSelWarps * kp_max * sizeof(unsigned long long);
  e = cudaFuncSetAttribute(dense_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dense_select_kernel<<<B, 32 * kSelWarps, smem, st>>>(D, used, ldd, B, qn, xn, n, meta, merged, ld_merged);
  return cudaGetLastError();
}

}  // namespace tri
