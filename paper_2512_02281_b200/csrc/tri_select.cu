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
#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Query preparation and row norms.

__global__ void prep_kernel(const double* __restrict__ q64, int d, float* __restrict__ Q32, int qld,
                            float* __restrict__ qn32, double* __restrict__ qn64, int* bad) {
  const int q = blockIdx.x;
  double s32 = 0.0, s64 = 0.0;
  bool finite = true;
  for (int j = threadIdx.x; j < qld; j += blockDim.x) {
    double v = j < d ? q64[(long long)q * d + j] : 0.0;
    finite = finite && isfinite(v);
    float f = __double2float_rn(v);
    Q32[(long long)q * qld + j] = f;
    s32 += (double)f * (double)f;
    s64 += v * v;
  }
  __shared__ double r32[32], r64[32];
  for (int o = 16; o > 0; o >>= 1) {
    s32 += __shfl_xor_sync(0xffffffffu, s32, o);
    s64 += __shfl_xor_sync(0xffffffffu, s64, o);
  }
  int nf = __syncthreads_or(!finite);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    r32[warp] = s32;
    r64[warp] = s64;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += r32[w];
      b += r64[w];
    }
    qn32[q] = __double2float_rn(a);
    qn64[q] = sqrt(b);
    if (nf && bad) atomicExch(bad, 1);
  }
}

cudaError_t launch_prep(const double* q64, int B, int d, float* Q32, int qld, float* qn32, double* qn64,
                        int* bad, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  prep_kernel<<<B, 128, 0, st>>>(q64, d, Q32, qld, qn32, qn64, bad);
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
// Per-query merge of partial top-kp lists.

__global__ void __launch_bounds__(kThreads) merge_kernel(const unsigned long long* __restrict__ part,
                                                         const QueryMeta* __restrict__ meta,
                                                         unsigned long long* __restrict__ merged, int ld_merged,
                                                         int buf_n) {
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

cudaError_t launch_merge(const unsigned long long* part, const QueryMeta* meta, unsigned long long* merged,
                         int ld_merged, int B, int kp_max, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  int buf_n = next_pow2(kp_max + kThreads * 4);
  size_t smem = (size_t)buf_n * sizeof(unsigned long long);
  cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  merge_kernel<<<B, kThreads, smem, st>>>(part, meta, merged, ld_merged, buf_n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact fp64 re-rank + certification.
//
// exact_pairs_kernel: one CTA per (query, 32 candidates); thread pair
// (2c, 2c+1) computes candidate c, thread 2c+l running numpy lane l (elements
// 8b + 2*sub + l, sub = 3..0, then the 2-lane tail), so the value is
// bit-identical to exact_sq_dist / the reference.  Candidate rows and the
// fp64 query are staged through shared memory in 256-float slabs with
// cp.async (all loads in flight at once); slabs are 8-aligned so numpy's
// 8-element blocks never straddle one.

constexpr int kPairCands = 32;
constexpr int kPairSlab = 256;
constexpr int kPairStride = kPairSlab + 4;  // 2-way worst bank conflict, 16B aligned rows

__global__ void __launch_bounds__(2 * kPairCands) exact_pairs_kernel(RerankLaunch r) {
  __shared__ __align__(16) float xs[kPairCands * kPairStride];
  __shared__ __align__(16) double qs[kPairSlab];
  __shared__ long long pos_s[kPairCands];
  const int groups = r.ld_merged / kPairCands;
  const int q = blockIdx.x / groups;
  const int c = (blockIdx.x - q * groups) * kPairCands + (threadIdx.x >> 1);
  const int ln = threadIdx.x & 1;
  const int kp = r.meta[q].kp;
  if ((c & ~(kPairCands - 1)) >= kp) return;  // whole CTA beyond this query's capacity
  const long long p = (long long)q * r.ld_merged + c;
  const unsigned long long key = r.merged[p];
  const bool active = key != TRI_KEY_MAX;
  const long long pos = active ? (long long)key_pos(key) : -1;
  if (ln == 0) pos_s[threadIdx.x >> 1] = pos;
  __syncthreads();
  const int d = r.d;
  const double* qg = r.q64 + (long long)q * d;
  double acc = 0.0;
  for (int s0 = 0; s0 < d; s0 += kPairSlab) {
    const int w = min(kPairSlab, d - s0);
    const int w4 = (w + 3) >> 2;  // stored rows are zero padded to a multiple of 16
    const uint32_t xbase = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
    for (int i = threadIdx.x; i < kPairCands * w4; i += blockDim.x) {
      const int row = i / w4, ch = i - row * w4;
      const long long rp = pos_s[row];
      const float* src = rp >= 0 ? r.X + rp * r.ldx + s0 + ch * 4 : r.X;
      const uint32_t dst = xbase + (uint32_t)((row * kPairStride + ch * 4) * 4);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(rp >= 0 ? 16 : 0));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    for (int j = threadIdx.x; j < w; j += blockDim.x) qs[j] = qg[s0 + j];
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (active) {
      const float* xr = xs + (threadIdx.x >> 1) * kPairStride;
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
    __syncthreads();
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

__global__ void __launch_bounds__(128) finalize_kernel(RerankLaunch r) {
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
      const double T = (double)key_dist(r.merged[(long long)q * r.ld_merged + kp - 1]);
      const double s = r.qn64[q] + r.xmax;
      const double E = (r.cdot * 2.0 * r.qn64[q] * r.xmax + r.csum * s * s) * 1.001 + 1e-30;
      cert = ebuf[m.k - 1].d + E < T;
    }
    if (!cert) r.flag_list[atomicAdd(r.n_flag, 1)] = q;
  }
  for (int j = threadIdx.x; j < m.k; j += blockDim.x) {
    const Exact e = ebuf[j];
    const bool ok = e.id != 0x7fffffffffffffffll;
    r.out_ids[(long long)q * r.ldo + j] = ok ? e.id : -1;
    r.out_d[(long long)q * r.ldo + j] = e.d;
  }
}

cudaError_t launch_rerank(const RerankLaunch& r, cudaStream_t st) {
  if (r.B <= 0) return cudaSuccess;
  exact_pairs_kernel<<<(unsigned)(r.B * (r.ld_merged / kPairCands)), 2 * kPairCands, 0, st>>>(r);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  size_t smem = (size_t)r.kp_max * sizeof(Exact);
  e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  finalize_kernel<<<r.B, 128, smem, st>>>(r);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact fix-up for uncertified queries: fp64 scan of the full candidate set.

__global__ void __launch_bounds__(kThreads) fixup_kernel(FixupLaunch f, int cap) {
  extern __shared__ Exact fbuf[];
  __shared__ int s_cnt;
  __shared__ Exact s_thr;
  if ((int)blockIdx.x >= *f.n_flag) return;
  const int q = f.flag_list[blockIdx.x];
  const int k = f.meta[q].k;
  const double* qv = f.q64 + (long long)q * f.d;
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_thr = exact_max();
  }
  __syncthreads();
  const int nranges = f.probes ? f.nprobe[q] : 1;
  for (int rg = 0; rg < nranges; ++rg) {
    long long lo = 0, hi = f.n_rows;
    if (f.probes) {
      long long l = f.probes[(long long)q * f.ld_probes + rg];
      lo = f.list_off[l];
      hi = f.list_off[l + 1];
    }
    for (long long base = lo; base < hi; base += kThreads) {
      const long long row = base + threadIdx.x;
      const Exact thr = s_thr;
      if (row < hi) {
        Exact e;
        e.d = exact_sq_dist(qv, f.X + row * f.ldx, f.d);
        e.id = (f.idmap ? f.idmap[row] : row) + f.id_offset;
        if (exact_less(e, thr)) fbuf[atomicAdd(&s_cnt, 1)] = e;
      }
      __syncthreads();
      const int n = s_cnt;
      if (n > cap - kThreads) {
        const int p2 = next_pow2(n);
        for (int i = n + threadIdx.x; i < p2; i += kThreads) fbuf[i] = exact_max();
        __syncthreads();
        block_sort(fbuf, p2, ExactLess());
        if (threadIdx.x == 0 && n >= k) {
          s_cnt = k;
          s_thr = fbuf[k - 1];
        }
      }
      __syncthreads();
    }
  }
  const int n = s_cnt;
  const int p2 = next_pow2(n > 0 ? n : 1);
  for (int i = n + threadIdx.x; i < p2; i += kThreads) fbuf[i] = exact_max();
  __syncthreads();
  block_sort(fbuf, p2, ExactLess());
  for (int j = threadIdx.x; j < k; j += kThreads) {
    const Exact e = j < n ? fbuf[j] : exact_max();
    const bool ok = j < n;
    f.out_ids[(long long)q * f.ldo + j] = ok ? e.id : -1;
    f.out_d[(long long)q * f.ldo + j] = e.d;
  }
}

cudaError_t launch_fixup(const FixupLaunch& f, cudaStream_t st) {
  if (f.B <= 0) return cudaSuccess;
  int cap = next_pow2(f.k_max + kThreads);
  size_t smem = (size_t)cap * sizeof(Exact);
  cudaError_t e = cudaFuncSetAttribute(fixup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fixup_kernel<<<f.B, kThreads, smem, st>>>(f, cap);
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
  out[i] = exact_sq_dist(q64 + (long long)owner[i] * d, X + c * ldx, d);
}

cudaError_t launch_distance_tasks(const int* owner, const long long* cand, int n_tasks, const double* q64, int d,
                                  const float* X, long long ldx, long long n_rows, double* out, int* err,
                                  cudaStream_t st) {
  if (n_tasks <= 0) return cudaSuccess;
  distance_tasks_kernel<<<(n_tasks + 127) / 128, 128, 0, st>>>(owner, cand, n_tasks, q64, d, X, ldx, n_rows, out,
                                                                 err);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact merge of G per-shard top-k lists (dist, id) -> global top-k.

__global__ void __launch_bounds__(kThreads) merge_exact_kernel(const double* __restrict__ dists,
                                                               const long long* __restrict__ ids, int G, int B,
                                                               int k_in, int k_out, double* __restrict__ out_d,
                                                               long long* __restrict__ out_ids, int n2) {
  extern __shared__ Exact mbuf[];
  const int q = blockIdx.x;
  const int n = G * k_in;
  for (int i = threadIdx.x; i < n2; i += kThreads) {
    Exact e = exact_max();
    if (i < n) {
      int g = i / k_in, j = i - g * k_in;
      long long off = ((long long)g * B + q) * k_in + j;
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
  for (int j = threadIdx.x; j < k_out; j += kThreads) {
    const Exact e = mbuf[j];
    const bool ok = e.id != 0x7fffffffffffffffll;
    out_ids[(long long)q * k_out + j] = ok ? e.id : -1;
    out_d[(long long)q * k_out + j] = e.d;
  }
}

cudaError_t launch_merge_exact(const double* dists, const long long* ids, int G, int B, int k_in, int k_out,
                               double* out_d, long long* out_ids, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  int n2 = next_pow2(G * k_in);
  size_t smem = (size_t)n2 * sizeof(Exact);
  cudaError_t e =
      cudaFuncSetAttribute(merge_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  merge_exact_kernel<<<B, kThreads, smem, st>>>(dists, ids, G, B, k_in, k_out, out_d, out_ids, n2);
  return cudaGetLastError();
}

}  // namespace tri
