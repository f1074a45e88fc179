// Tensor-core coarse GEMM for the IVF coarse step (queries x centroids):
// tcgen05.mma kind::f16 on SPLIT fp16 operands, K-split TMEM accumulators.
//
// Both sides are scaled by powers of two (exact) and split into fp16 hi + lo:
//   c sc = ch + cl + ec,  q sq = qh + ql + eq     (|e| <= 2^-22 |.| + subnormal floor)
// and the dot is formed from three exact fp16 x fp16 products per element,
//   q.c ~ (qh.ch + qh.cl + ql.ch) / (sq sc)       (ql.cl ~ 2^-22 relative dropped),
// accumulated in fp32 by the tensor core in 32-wide K slices -- one TMEM
// accumulator per slice (96 products) -- and the slices summed in order in
// fp32 by the epilogue.  The error bound (bound_for(kSplit), tri_api.cu) is
// below the fp32 SIMT GEMM's gamma_d, so the coarse certificate behaves as
// before while the contraction runs on tensor cores.
//
// CTA: 128 centroid rows (MMA M) x 16 queries (MMA N), 192 threads:
//   warp 0    TMA producer: per 64-wide K slab, the hi and lo 128 x 64 tiles
//             (128B swizzle) of the centroid copies into a ring of slab pairs;
//   warp 1    MMA issuer: per slab, 2 K-slices x 2 k16 steps x 3 products;
//   warps 2-5 stage the 16 queries' hi/lo rows (SW128 K-major) into shared
//             memory, then read the accumulators (thread = row) and write the
//             fp32 dot to P (B x ldd), consumed by dense_select_kernel.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

int g_coarse_split = 4;  // split-K slices of the tensor-core coarse GEMM (option "coarse_split")

namespace {

constexpr int kCoRows = 128, kCoN = 16, kCoThreads = 192, kCoStages = 3;
constexpr int kCoSlab = 128 * 128;        // bytes of one 128-row x 64-half tile
constexpr int kCoQTile = kCoN * 128;      // bytes of 16 queries x 64 halves
constexpr uint32_t kCoIdesc = (1u << 4) | ((uint32_t)(kCoN >> 3) << 17) | ((uint32_t)(kCoRows >> 4) << 24);

__device__ __forceinline__ uint32_t csu32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cmb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(csu32(b)), "r"(c));
}
__device__ __forceinline__ void cmb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(csu32(b)) : "memory");
}
__device__ __forceinline__ void cmb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(csu32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cmb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n CWAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CWAIT_%=;\n}\n" ::"r"(csu32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ctma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(csu32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(csu32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t csw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void cumma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kCoIdesc), "r"(accumulate));
}
__device__ __forceinline__ void ccommit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(csu32(bar))
               : "memory");
}

struct CoSmem {
  uint64_t full[kCoStages], empty[kCoStages];
  uint64_t qready, done;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kCoThreads, 1) coarse_tc_kernel(const __grid_constant__ CUtensorMap map_h,
                                                                   const __grid_constant__ CUtensorMap map_l,
                                                                   CoarseLaunch a) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(1024) unsigned char co_raw[];
  __shared__ CoSmem sh;
  unsigned char* base = co_raw + ((1024u - (csu32(co_raw) & 1023u)) & 1023u);
  unsigned char* ring = base;                                    // kCoStages x (hi, lo) tiles
  unsigned char* qh_t = ring + (size_t)kCoStages * 2 * kCoSlab;  // nslab x 2 KB
  unsigned char* ql_t = qh_t + (size_t)a.slab_cap * kCoQTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * kCoRows, q0 = blockIdx.y * kCoN;
  // split-K: CTA z owns slabs [sb, se) and writes slice z of P (summed in order by the select)
  const int sb = (int)((long long)a.nslab * blockIdx.z / gridDim.z);
  const int se = (int)((long long)a.nslab * (blockIdx.z + 1) / gridDim.z);
  const int ns = se - sb;
  const int nacc = 2 * ns;  // one accumulator per 32-wide K slice
  if (threadIdx.x == 0) {
    for (int s = 0; s < kCoStages; ++s) {
      cmb_init(&sh.full[s], 1);
      cmb_init(&sh.empty[s], 1);
    }
    cmb_init(&sh.qready, 4 * 32);
    cmb_init(&sh.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(csu32(&sh.tmem_base)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = sh.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0, ph = 0;
      for (int s = 0; s < ns; ++s) {
        cmb_wait(&sh.empty[stage], ph ^ 1);
        unsigned char* dst = ring + (size_t)stage * 2 * kCoSlab;
        cmb_expect(&sh.full[stage], 2 * kCoSlab);
        ctma_2d(dst, &map_h, (sb + s) * 64, row0, &sh.full[stage]);
        ctma_2d(dst + kCoSlab, &map_l, (sb + s) * 64, row0, &sh.full[stage]);
        if (++stage == kCoStages) {
          stage = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    cmb_wait(&sh.qready, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    int stage = 0, ph = 0;
    for (int s = 0; s < ns; ++s) {
      cmb_wait(&sh.full[stage], ph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
        const uint32_t ah = csu32(ring + (size_t)stage * 2 * kCoSlab), al = ah + kCoSlab;
        const uint32_t bh = csu32(qh_t + (size_t)s * kCoQTile), bl = csu32(ql_t + (size_t)s * kCoQTile);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t d = tmem + (uint32_t)((2 * s + half) * kCoN);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint32_t off = (uint32_t)((2 * half + kk) * 32);  // 16 halves = 32 B of K per MMA
            cumma(d, csw128(ah + off), csw128(bh + off), kk != 0);
            cumma(d, csw128(ah + off), csw128(bl + off), 1);
            cumma(d, csw128(al + off), csw128(bh + off), 1);
          }
        }
        ccommit(&sh.empty[stage]);
        if (s == ns - 1) ccommit(&sh.done);
      }
      __syncwarp();
      if (++stage == kCoStages) {
        stage = 0;
        ph ^= 1;
      }
    }
  } else {
    // warps 2-5: stage the 16 queries (hi / lo) in the UMMA SW128 K-major layout:
    // slab s, query g, 16-byte chunk c at s*2KB + g*128 + ((c ^ (g & 7)) << 4)
    const int t = threadIdx.x - 64;  // 0..127
    const int q4 = a.ldq >> 3;       // 16-byte chunks per query row
    const int total = ns * kCoN * 8;
    // hi and lo loads of a round are all in flight before any store
    const uint4* srch = reinterpret_cast<const uint4*>(a.Qh);
    const uint4* srcl = reinterpret_cast<const uint4*>(a.Ql);
    for (int i0 = 0; i0 < total; i0 += 128 * 4) {
      uint4 vh[4], vl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 128 + t;
        const int c = i & 7, g = (i >> 3) & (kCoN - 1), sl = i >> 7;
        const int q = q0 + g;
        vh[u] = make_uint4(0u, 0u, 0u, 0u);
        vl[u] = vh[u];
        if (i < total && q < a.B) {
          const long long o = (long long)q * q4 + (sb + sl) * 8 + c;
          vh[u] = srch[o];
          vl[u] = srcl[o];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 128 + t;
        const int c = i & 7, g = (i >> 3) & (kCoN - 1), sl = i >> 7;
        if (i < total) {
          const int off = sl * kCoQTile + g * 128 + ((c ^ (g & 7)) << 4);
          *reinterpret_cast<uint4*>(qh_t + off) = vh[u];
          *reinterpret_cast<uint4*>(ql_t + off) = vl[u];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core reads
    cmb_arrive(&sh.qready);
    // epilogue: thread = TMEM lane = centroid row of this tile; sum the K slices in order
    cmb_wait(&sh.done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int quad = warp & 3;  // warps 2..5 -> TMEM lane quadrants 2,3,0,1
    const int row = row0 + quad * 32 + lane;
    float acc[kCoN];
#pragma unroll
    for (int g = 0; g < kCoN; ++g) acc[g] = 0.f;
    for (int s = 0; s < nacc; ++s) {
      uint32_t v[kCoN];
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(s * kCoN);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int g = 0; g < kCoN; ++g) acc[g] = __fadd_rn(acc[g], __uint_as_float(v[g]));
    }
    if (row < a.n) {
#pragma unroll
      for (int g = 0; g < kCoN; ++g) {
        const int q = q0 + g;
        if (q < a.B) {
          const float qi = a.qinv[q];
          // qinv < 0: the query could not be scaled; its list is never certified
          a.P[((long long)blockIdx.z * a.B + q) * a.ldd + row] =
              qi > 0.f ? acc[g] * (qi * a.ratio) : __int_as_float(0x7fc00000);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(a.tmem_cols));
  }
}

}  // namespace

int coarse_tc_slices(int nslab) { return std::max(1, std::min(g_coarse_split, nslab)); }

size_t coarse_tc_smem(int slab_cap) { return 1024 + (size_t)kCoStages * 2 * kCoSlab + (size_t)2 * slab_cap * kCoQTile; }

cudaError_t launch_coarse_tc(const CoarseLaunch& a0, cudaStream_t st) {
  if (a0.B <= 0) return cudaSuccess;
  CoarseLaunch a = a0;
  const int S = coarse_tc_slices(a.nslab);
  a.slab_cap = (a.nslab + S - 1) / S;
  int cols = 32;
  while (cols < 2 * a.slab_cap * kCoN) cols <<= 1;  // TMEM allocations are powers of two >= 32
  if (cols > 512) return cudaErrorInvalidValue;
  a.tmem_cols = cols;
  const size_t smem = coarse_tc_smem(a.slab_cap);
  cudaError_t e = cudaFuncSetAttribute(coarse_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.n + kCoRows - 1) / kCoRows), (unsigned)((a.B + kCoN - 1) / kCoN), (unsigned)S);
  (void)launch_pdl(coarse_tc_kernel, grid, kCoThreads, smem, st, *reinterpret_cast<const CUtensorMap*>(a.map_h),
                                                   *reinterpret_cast<const CUtensorMap*>(a.map_l), a);
  return cudaGetLastError();
}

// lo part of the split copy: Xl[r, j] = fp16(X[r, j] * sx - fp16(X[r, j] * sx)) (the difference is exact in fp32)
__global__ void to_half_lo_kernel(const float* __restrict__ X, long long n, int d, long long ldx, float sx,
                                  __half* __restrict__ Xl, int ldh) {
  const long long total = n * (long long)ldh;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ldh;
    const int j = (int)(i - r * ldh);
    float lo = 0.f;
    if (j < d) {
      const float v = X[r * ldx + j] * sx;
      lo = v - __half2float(__float2half_rn(v));
    }
    Xl[i] = __float2half_rn(lo);
  }
}

cudaError_t launch_to_half_lo(const float* X, long long n, int d, long long ldx, float sx, void* Xl, int ldh,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  to_half_lo_kernel<<<4 * 148, 256, 0, st>>>(X, n, d, ldx, sx, static_cast<__half*>(Xl), ldh);
  return cudaGetLastError();
}

}  // namespace tri
