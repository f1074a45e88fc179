// Candidate generation, merge, exact re-rank and certified fix-up kernels.
//
// Pipeline for one batch of queries (brute force, IVF coarse step and IVF
// list scan all share it):
//   prep      fp64 queries -> fp32 rows + norms
//   scan      persistent CTAs take WorkItems (row range x query group); each
//             thread owns 2 rows per 512-row pass, rows stream HBM -> smem via
//             a 3-stage cp.async pipeline (16-float slabs, XOR swizzle), queries
//             sit in smem and are read as broadcasts; fp32 dot-form distances
//             feed a per-query threshold-filtered selection buffer in smem
//             (warp bitonic compaction).  The distance matrix never reaches HBM:
//             only a top-kp list per (query, work item) is written.
//   merge     per query: top-kp over its partial lists
//   rerank    per query: fp64 distances in the reference's exact summation
//             order, sort by (dist, id), certify (see below)
//   fixup     per uncertified query: exact fp64 scan of its whole candidate set
//
// Certification: every dropped candidate has approx distance >= T (the kp-th
// kept one) and |approx - exact| <= E = cbound*(|q|+max|x|)^2, so if the k-th
// exact distance + E < T no dropped vector can enter the exact top-k.
#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

constexpr int kThreads = 256;
constexpr int kRowsPerThread = 2;
constexpr int kChunk = kThreads * kRowsPerThread;  // rows per pass
constexpr int kSlabW = 16;                          // floats per slab row
constexpr int kStages = 3;
constexpr int kSlabFloats = kChunk * kSlabW;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

size_t scan_smem_bytes(int gmax, int qld, int cap) {
  return (size_t)gmax * qld * sizeof(float) + (size_t)kStages * kSlabFloats * sizeof(float) +
         (size_t)gmax * cap * sizeof(unsigned long long);
}

int scan_gmax(int qld, int cap, int smem_limit) {
  for (int g = 16; g >= 1; g >>= 1)
    if (scan_smem_bytes(g, qld, cap) <= (size_t)smem_limit) return g;
  return 0;
}

// Stage one 512-row x 16-float slab of X into shared memory (zero-filled
// outside the valid rows / columns).  Row r, 16-byte chunk c lands at float4
// index r*4 + (c ^ ((r >> 1) & 3)), which makes the row-per-thread LDS.128
// reads below bank-conflict free.
__device__ __forceinline__ void load_slab(float* slab, const float* __restrict__ X, long long ldx,
                                          long long row0, int rows, int col0, int dp) {
  const uint32_t base = smem_u32(slab);
#pragma unroll
  for (int j = 0; j < (kChunk * 4) / kThreads; ++j) {
    int i = threadIdx.x + j * kThreads;
    int r = i >> 2, c = i & 3;
    int col = col0 + c * 4;
    bool ok = (r < rows) && (col < dp);
    const float* src = ok ? X + (row0 + r) * ldx + col : X;
    uint32_t dst = base + (uint32_t)((r * 4 + (c ^ ((r >> 1) & 3))) * 16);
    cp_async16(dst, src, ok ? 16 : 0);
  }
}

struct ScanShared {
  int cnt[16];
  unsigned long long thr[16];
  float qn[16];
  int item;
};

template <int GT>
__device__ void scan_item(const ScanLaunch& a, const WorkItem& w, float* Qs, float* slabs,
                          unsigned long long* sel, ScanShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gc = w.member_count;
  const int kp = w.kp;
  const int cap = a.cap;
  const int qld = a.qld;

  // Stage the group's queries (zero rows past gc) and reset selection state.
  {
    const float4* Q4 = reinterpret_cast<const float4*>(a.Q);
    float4* Qs4 = reinterpret_cast<float4*>(Qs);
    const int q4 = qld >> 2;
    for (int i = tid; i < GT * q4; i += kThreads) {
      int g = i / q4, c = i - g * q4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g < gc) v = Q4[(long long)a.members[w.member_begin + g].q * q4 + c];
      Qs4[i] = v;
    }
    if (tid < GT) {
      sh.cnt[tid] = 0;
      sh.thr[tid] = TRI_KEY_MAX;
      sh.qn[tid] = tid < gc ? a.qnorm[a.members[w.member_begin + tid].q] : 0.f;
    }
  }
  __syncthreads();

  const int nslab = qld / kSlabW;
  const float4* Qs4 = reinterpret_cast<const float4*>(Qs);
  const int q4 = qld >> 2;
  const int r0 = tid, r1 = tid + kThreads;
  const int sw = (tid >> 1) & 3;  // same for r0 and r1

  for (int c0 = 0; c0 < w.row_count; c0 += kChunk) {
    const int rows = min(kChunk, w.row_count - c0);
    const long long row0 = w.row_begin + c0;
    float acc0[GT], acc1[GT];
#pragma unroll
    for (int g = 0; g < GT; ++g) acc0[g] = acc1[g] = 0.f;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nslab) load_slab(slabs + s * kSlabFloats, a.X, a.ldx, row0, rows, s * kSlabW, a.dp);
      cp_async_commit();
    }
    for (int s = 0; s < nslab; ++s) {
      int sn = s + kStages - 1;
      if (sn < nslab) load_slab(slabs + (sn % kStages) * kSlabFloats, a.X, a.ldx, row0, rows, sn * kSlabW, a.dp);
      cp_async_commit();
      cp_async_wait<kStages - 1>();
      __syncthreads();
      const float4* sl = reinterpret_cast<const float4*>(slabs + (s % kStages) * kSlabFloats);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float4 x0 = sl[r0 * 4 + (c ^ sw)];
        float4 x1 = sl[r1 * 4 + (c ^ sw)];
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          float4 qv = Qs4[g * q4 + s * 4 + c];
          acc0[g] = fmaf(x0.x, qv.x, acc0[g]);
          acc0[g] = fmaf(x0.y, qv.y, acc0[g]);
          acc0[g] = fmaf(x0.z, qv.z, acc0[g]);
          acc0[g] = fmaf(x0.w, qv.w, acc0[g]);
          acc1[g] = fmaf(x1.x, qv.x, acc1[g]);
          acc1[g] = fmaf(x1.y, qv.y, acc1[g]);
          acc1[g] = fmaf(x1.z, qv.z, acc1[g]);
          acc1[g] = fmaf(x1.w, qv.w, acc1[g]);
        }
      }
      __syncthreads();
    }

    // Approximate distances -> threshold-filtered append.
    const bool v0 = r0 < rows, v1 = r1 < rows;
    const float xn0 = v0 ? a.xnorm[row0 + r0] : 0.f;
    const float xn1 = v1 ? a.xnorm[row0 + r1] : 0.f;
    const uint32_t p0 = (uint32_t)(row0 + r0), p1 = (uint32_t)(row0 + r1);
    uint32_t pend = 0;
#pragma unroll
    for (int g = 0; g < GT; ++g) {
      if (g < gc) {
        const float qn = sh.qn[g];
        const unsigned long long thr = sh.thr[g];
        if (v0) {
          unsigned long long key = make_key(__fmaf_rn(-2.f, acc0[g], __fadd_rn(qn, xn0)), p0);
          if (key < thr) {
            int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else pend |= 1u << (2 * g);
          }
        }
        if (v1) {
          unsigned long long key = make_key(__fmaf_rn(-2.f, acc1[g], __fadd_rn(qn, xn1)), p1);
          if (key < thr) {
            int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else pend |= 1u << (2 * g + 1);
          }
        }
      }
    }
    while (true) {
      __syncthreads();
      for (int g = warp; g < gc; g += kThreads / 32) {
        int n = sh.cnt[g];
        if (n > kp) {
          int m = min(n, cap);
          int p2 = next_pow2(m);
          unsigned long long* s = sel + g * cap;
          for (int i = m + lane; i < p2; i += 32) s[i] = TRI_KEY_MAX;
          __syncwarp();
          warp_sort(s, p2, lane, KeyLess());
          if (lane == 0) {
            sh.cnt[g] = kp;
            sh.thr[g] = s[kp - 1];
          }
          __syncwarp();
        }
      }
      if (!__syncthreads_or(pend != 0)) break;
      uint32_t still = 0;
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        if (pend & (1u << (2 * g))) {
          unsigned long long key = make_key(__fmaf_rn(-2.f, acc0[g], __fadd_rn(sh.qn[g], xn0)), p0);
          if (key < sh.thr[g]) {
            int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else still |= 1u << (2 * g);
          }
        }
        if (pend & (1u << (2 * g + 1))) {
          unsigned long long key = make_key(__fmaf_rn(-2.f, acc1[g], __fadd_rn(sh.qn[g], xn1)), p1);
          if (key < sh.thr[g]) {
            int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else still |= 1u << (2 * g + 1);
          }
        }
      }
      pend = still;
    }
  }

  // Final per-query sort and write-out of the top-kp partial list.
  for (int g = warp; g < gc; g += kThreads / 32) {
    int n = sh.cnt[g];
    int p2 = next_pow2(n > 0 ? n : 1);
    unsigned long long* s = sel + g * cap;
    for (int i = n + lane; i < p2; i += 32) s[i] = TRI_KEY_MAX;
    __syncwarp();
    warp_sort(s, p2, lane, KeyLess());
    unsigned long long* out = a.part + a.members[w.member_begin + g].slot;
    for (int i = lane; i < kp; i += 32) out[i] = i < n ? s[i] : TRI_KEY_MAX;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) scan_kernel(ScanLaunch a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ ScanShared sh;
  float* Qs = reinterpret_cast<float*>(smem_raw);
  float* slabs = Qs + (size_t)a.gmax * a.qld;
  unsigned long long* sel = reinterpret_cast<unsigned long long*>(slabs + (size_t)kStages * kSlabFloats);
  const int n_items = *a.n_items;
  while (true) {
    if (threadIdx.x == 0) sh.item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int it = sh.item;
    __syncthreads();
    if (it >= n_items) break;
    const WorkItem w = a.items[it];
    if (w.row_count <= 0) continue;
    const int gc = w.member_count;
    if (gc <= 1) scan_item<1>(a, w, Qs, slabs, sel, sh);
    else if (gc <= 2) scan_item<2>(a, w, Qs, slabs, sel, sh);
    else if (gc <= 4) scan_item<4>(a, w, Qs, slabs, sel, sh);
    else if (gc <= 8) scan_item<8>(a, w, Qs, slabs, sel, sh);
    else scan_item<16>(a, w, Qs, slabs, sel, sh);
  }
}

cudaError_t launch_scan(const ScanLaunch& s, cudaStream_t st) {
  size_t smem = scan_smem_bytes(s.gmax, s.qld, s.cap);
  cudaError_t e = cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  scan_kernel<<<s.grid, kThreads, smem, st>>>(s);
  return cudaGetLastError();
}

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

__global__ void __launch_bounds__(kThreads) rerank_kernel(RerankLaunch r) {
  extern __shared__ Exact ebuf[];
  const int q = blockIdx.x;
  const QueryMeta m = r.meta[q];
  const int kp = m.kp;
  const unsigned long long* mk = r.merged + (long long)q * r.ld_merged;
  const double* qv = r.q64 + (long long)q * r.d;
  for (int i = threadIdx.x; i < kp; i += kThreads) {
    unsigned long long key = mk[i];
    Exact e = exact_max();
    if (key != TRI_KEY_MAX) {
      long long pos = key_pos(key);
      e.d = exact_sq_dist(qv, r.X + pos * r.ldx, r.d);
      e.id = (r.idmap ? r.idmap[pos] : pos) + r.id_offset;
    }
    ebuf[i] = e;
  }
  __syncthreads();
  block_sort(ebuf, kp, ExactLess());
  if (threadIdx.x == 0) {
    bool cert = true;
    if (m.n_total > kp) {
      const double T = (double)key_dist(mk[kp - 1]);
      const double s = r.qn64[q] + r.xmax;
      const double E = r.cbound * s * s * 1.001 + 1e-30;
      cert = ebuf[m.k - 1].d + E < T;
    }
    if (!cert) r.flag_list[atomicAdd(r.n_flag, 1)] = q;
  }
  for (int j = threadIdx.x; j < m.k; j += kThreads) {
    const Exact e = ebuf[j];
    const bool ok = e.id != 0x7fffffffffffffffll;
    r.out_ids[(long long)q * r.ldo + j] = ok ? e.id : -1;
    r.out_d[(long long)q * r.ldo + j] = e.d;
  }
}

cudaError_t launch_rerank(const RerankLaunch& r, cudaStream_t st) {
  if (r.B <= 0) return cudaSuccess;
  size_t smem = (size_t)r.kp_max * sizeof(Exact);
  cudaError_t e = cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  rerank_kernel<<<r.B, kThreads, smem, st>>>(r);
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
