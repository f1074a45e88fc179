// The list-scan kernel: candidate generation for brute force, the IVF coarse
// step and the IVF inverted-list scan.
//
// Warp-specialised, persistent (one CTA per SM):
//   warp 8 (producer, one lane): claims work items with an atomic counter,
//     publishes them through a 2-slot descriptor ring, streams the item's rows
//     HBM -> shared memory with 2-D TMA (64-row x 16-float boxes, 64B swizzle)
//     into a STAGES-deep ring of 512-row slabs, and stages the group's queries
//     with 1-D bulk copies.  All hand-offs are mbarriers; the producer never
//     waits on a CTA barrier, so HBM keeps streaming while consumers select.
//   warps 0-7 (consumers): thread t owns rows t and t+256 of each 512-row
//     chunk; fp32 dot products against <= 16 queries read as shared-memory
//     broadcasts; then the fp32 dot-form distance qn + xn - 2 q.x feeds a
//     per-query threshold-filtered selection buffer (warp bitonic compaction,
//     named barrier 1 among the 256 consumer threads).  Only the top-kp list of
//     each (query, work item) is written to HBM.
#include <cuda.h>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

constexpr int kConsumers = 256;
constexpr int kThreadsScan = kConsumers + 32;
constexpr int kChunkRows = 2 * kConsumers;  // 512
constexpr int kSlab = 16;                   // floats per row per stage (64 B)
constexpr int kBoxRows = 64;
constexpr int kStageBytes = kChunkRows * kSlab * 4;  // 32 KB
constexpr int kStagesScan = 3;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(su32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
__device__ __forceinline__ int consumer_any(int v) {
  int r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 q, %1, 0;\n bar.red.or.pred p, 1, 256, q;\n selp.s32 %0, 1, 0, p;\n}\n"
      : "=r"(r)
      : "r"(v)
      : "memory");
  return r;
}

struct ScanSmem {
  uint64_t full[kStagesScan];
  uint64_t empty[kStagesScan];
  uint64_t wfull[2], wempty[2];
  uint64_t qfull, qempty;
  WorkItem witem[2];
  int wend[2];
  int cnt[16];
  unsigned long long thr[16];
  float qn[16];
};

size_t scan_smem_bytes(int gmax, int qld, int cap) {
  return 1024 + (size_t)kStagesScan * kStageBytes + (size_t)gmax * qld * sizeof(float) +
         (size_t)gmax * cap * sizeof(unsigned long long);
}

int scan_gmax(int qld, int cap, int smem_limit) {
  for (int g = 16; g >= 1; g >>= 1)
    if (scan_smem_bytes(g, qld, cap) <= (size_t)smem_limit) return g;
  return 0;
}

// --------------------------------------------------------------------------
// producer

__device__ void scan_producer(const ScanLaunch& a, const CUtensorMap* map, ScanSmem& sh, float* stages, float* Qs) {
  const int n_items = *a.n_items;
  int wslot = 0, wphase = 0, stage = 0, sphase = 0, qphase = 0;
  const int nslab = a.qld / kSlab;
  for (;;) {
    const int it = atomicAdd(a.counter, 1);
    mb_wait(&sh.wempty[wslot], wphase ^ 1);
    if (it >= n_items) {
      sh.wend[wslot] = 1;
      mb_arrive(&sh.wfull[wslot]);
      return;
    }
    const WorkItem w = a.items[it];
    sh.witem[wslot] = w;
    sh.wend[wslot] = 0;
    mb_arrive(&sh.wfull[wslot]);
    if (++wslot == 2) {
      wslot = 0;
      wphase ^= 1;
    }
    const int nchunk = (w.row_count + kChunkRows - 1) / kChunkRows;
    const long long total = (long long)nchunk * nslab;
    const long long q_at = total < kStagesScan ? total : kStagesScan;  // stage queries once the ring is primed
    const uint32_t qbytes = (uint32_t)a.qld * 4u;
    long long j = 0;
    // j == q_at: stage the group's queries (after priming the ring, so HBM
    // keeps streaming while the previous item's consumers finish)
    for (int c = 0; c <= nchunk; ++c) {
      const int rows = c < nchunk ? min(kChunkRows, w.row_count - c * kChunkRows) : 0;
      const int nbox = (rows + kBoxRows - 1) / kBoxRows;
      const int row0 = (int)(w.row_begin + (long long)c * kChunkRows);
      const int ns = c < nchunk ? nslab : 1;
      for (int s = 0; s < ns; ++s, ++j) {
        if (j == q_at) {
          mb_wait(&sh.qempty, qphase ^ 1);
          mb_expect_tx(&sh.qfull, qbytes * (uint32_t)w.member_count);
          for (int g = 0; g < w.member_count; ++g) {
            const int q = a.members[w.member_begin + g].q;
            bulk_1d(Qs + (size_t)g * a.qld, a.Q + (size_t)q * a.qld, qbytes, &sh.qfull);
          }
          qphase ^= 1;
        }
        if (c == nchunk) break;
        mb_wait(&sh.empty[stage], sphase ^ 1);
        float* dst = stages + (size_t)stage * (kStageBytes / 4);
        mb_expect_tx(&sh.full[stage], (uint32_t)nbox * kBoxRows * kSlab * 4u);
        for (int b = 0; b < nbox; ++b)
          tma_2d(dst + b * kBoxRows * kSlab, map, s * kSlab, row0 + b * kBoxRows, &sh.full[stage]);
        if (++stage == kStagesScan) {
          stage = 0;
          sphase ^= 1;
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// consumers

template <int GT>
__device__ __forceinline__ int scan_consume_item(const ScanLaunch& a, const WorkItem& w, ScanSmem& sh,
                                                  const float* stages, const float* Qs, unsigned long long* sel,
                                                  int ring) {
  int stage = ring & 0xffff, sphase = ring >> 16;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gc = w.member_count, kp = w.kp, cap = a.cap;
  const int nslab = a.qld / kSlab;
  const int q4 = a.qld >> 2;
  const float4* Qs4 = reinterpret_cast<const float4*>(Qs);
  const int sw = (tid >> 1) & 3;
  const int nchunk = (w.row_count + kChunkRows - 1) / kChunkRows;
  for (int c = 0; c < nchunk; ++c) {
    const int rows = min(kChunkRows, w.row_count - c * kChunkRows);
    const long long row0 = w.row_begin + (long long)c * kChunkRows;
    float acc0[GT], acc1[GT];
#pragma unroll
    for (int g = 0; g < GT; ++g) acc0[g] = acc1[g] = 0.f;
    for (int s = 0; s < nslab; ++s) {
      mb_wait(&sh.full[stage], sphase);
      const float4* sl = reinterpret_cast<const float4*>(stages + (size_t)stage * (kStageBytes / 4));
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const float4 x0 = sl[tid * 4 + (cc ^ sw)];
        const float4 x1 = sl[(tid + kConsumers) * 4 + (cc ^ sw)];
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          const float4 qv = Qs4[g * q4 + s * 4 + cc];
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
      __syncwarp();
      if (lane == 0) mb_arrive(&sh.empty[stage]);
      if (++stage == kStagesScan) {
        stage = 0;
        sphase ^= 1;
      }
    }
    if (c == nchunk - 1) {
      __syncwarp();
      if (lane == 0) mb_arrive(&sh.qempty);  // queries no longer needed
    }

    // approximate distances -> threshold-filtered append
    const int r0 = tid, r1 = tid + kConsumers;
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
          const unsigned long long key = make_key(__fmaf_rn(-2.f, acc0[g], __fadd_rn(qn, xn0)), p0);
          if (key < thr) {
            const int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else pend |= 1u << (2 * g);
          }
        }
        if (v1) {
          const unsigned long long key = make_key(__fmaf_rn(-2.f, acc1[g], __fadd_rn(qn, xn1)), p1);
          if (key < thr) {
            const int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else pend |= 1u << (2 * g + 1);
          }
        }
      }
    }
    for (;;) {
      consumer_sync();
      for (int g = warp; g < gc; g += kConsumers / 32) {
        const int n = sh.cnt[g];
        if (n > kp) {
          const int m = min(n, cap);
          const int p2 = next_pow2(m);
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
      if (!consumer_any(pend != 0)) break;
      uint32_t still = 0;
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        if (pend & (1u << (2 * g))) {
          const unsigned long long key = make_key(__fmaf_rn(-2.f, acc0[g], __fadd_rn(sh.qn[g], xn0)), p0);
          if (key < sh.thr[g]) {
            const int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else still |= 1u << (2 * g);
          }
        }
        if (pend & (1u << (2 * g + 1))) {
          const unsigned long long key = make_key(__fmaf_rn(-2.f, acc1[g], __fadd_rn(sh.qn[g], xn1)), p1);
          if (key < sh.thr[g]) {
            const int p = atomicAdd(&sh.cnt[g], 1);
            if (p < cap) sel[g * cap + p] = key; else still |= 1u << (2 * g + 1);
          }
        }
      }
      pend = still;
    }
  }
  if (nchunk == 0) {
    __syncwarp();
    if (lane == 0) mb_arrive(&sh.qempty);
  }
  // final per-query sort and write-out of the top-kp partial list
  for (int g = warp; g < gc; g += kConsumers / 32) {
    const int n = sh.cnt[g];
    const int p2 = next_pow2(n > 0 ? n : 1);
    unsigned long long* s = sel + g * cap;
    for (int i = n + lane; i < p2; i += 32) s[i] = TRI_KEY_MAX;
    __syncwarp();
    warp_sort(s, p2, lane, KeyLess());
    unsigned long long* out = a.part + a.members[w.member_begin + g].slot;
    for (int i = lane; i < kp; i += 32) out[i] = i < n ? s[i] : TRI_KEY_MAX;
  }
  return stage | (sphase << 16);
}

__device__ void scan_consumers(const ScanLaunch& a, ScanSmem& sh, const float* stages, const float* Qs,
                               unsigned long long* sel) {
  const int tid = threadIdx.x, lane = tid & 31;
  int wslot = 0, wphase = 0, ring = 0, qphase = 0;
  for (;;) {
    mb_wait(&sh.wfull[wslot], wphase);
    const int end = sh.wend[wslot];
    const WorkItem w = sh.witem[wslot];
    __syncwarp();
    if (lane == 0) mb_arrive(&sh.wempty[wslot]);
    if (++wslot == 2) {
      wslot = 0;
      wphase ^= 1;
    }
    if (end) return;
    consumer_sync();  // previous item's selection buffers are free
    if (tid < 16) {
      sh.cnt[tid] = 0;
      sh.thr[tid] = TRI_KEY_MAX;
      sh.qn[tid] = tid < w.member_count ? a.qnorm[a.members[w.member_begin + tid].q] : 0.f;
    }
    consumer_sync();
    mb_wait(&sh.qfull, qphase);
    qphase ^= 1;
    const int gc = w.member_count;
    if (gc <= 1) ring = scan_consume_item<1>(a, w, sh, stages, Qs, sel, ring);
    else if (gc <= 2) ring = scan_consume_item<2>(a, w, sh, stages, Qs, sel, ring);
    else if (gc <= 4) ring = scan_consume_item<4>(a, w, sh, stages, Qs, sel, ring);
    else if (gc <= 8) ring = scan_consume_item<8>(a, w, sh, stages, Qs, sel, ring);
    else if (gc <= 12) ring = scan_consume_item<12>(a, w, sh, stages, Qs, sel, ring);
    else ring = scan_consume_item<16>(a, w, sh, stages, Qs, sel, ring);
  }
}

__global__ void __launch_bounds__(kThreadsScan, 1) scan_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                                   ScanLaunch a) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ ScanSmem sh;
  // 1024-byte aligned stage ring (64B swizzle atoms), then queries, then selection buffers
  // (pointer arithmetic on smem_raw keeps the shared address space visible to
  // the compiler -> LDS/STS instead of generic LD/ST)
  unsigned char* base = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  float* stages = reinterpret_cast<float*>(base);
  float* Qs = stages + (size_t)kStagesScan * (kStageBytes / 4);
  unsigned long long* sel = reinterpret_cast<unsigned long long*>(Qs + (size_t)a.gmax * a.qld);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesScan; ++s) {
      mb_init(&sh.full[s], 1);
      mb_init(&sh.empty[s], kConsumers / 32);
    }
    for (int s = 0; s < 2; ++s) {
      mb_init(&sh.wfull[s], 1);
      mb_init(&sh.wempty[s], kConsumers / 32);
    }
    mb_init(&sh.qfull, 1);
    mb_init(&sh.qempty, kConsumers / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == kConsumers / 32) {
    if ((threadIdx.x & 31) == 0) scan_producer(a, &map, sh, stages, Qs);
  } else {
    scan_consumers(a, sh, stages, Qs, sel);
  }
}

cudaError_t launch_scan(const ScanLaunch& s, cudaStream_t st) {
  const size_t smem = scan_smem_bytes(s.gmax, s.qld, s.cap);
  cudaError_t e = cudaFuncSetAttribute(scan_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  (void)launch_pdl(scan_tma_kernel, s.grid, kThreadsScan, smem, st, *reinterpret_cast<const CUtensorMap*>(s.tmap), s);
  return cudaGetLastError();
}

}  // namespace tri
