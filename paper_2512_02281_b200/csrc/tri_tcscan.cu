// Tensor-core list scan (sm_100a): tcgen05.mma kind::f16 (fp16 copy of the
// lists) or kind::tf32 (fp32 lists), TMEM accumulators,
// TMA-fed shared-memory ring.  Same work items / partial-list contract as the
// SIMT scan in tri_listscan.cu, which remains the path for qld > kTcMaxQld.
//
// Roles (one persistent CTA per SM, 352 threads):
//   warp 0  producer : claims work items and publishes each one ahead of
//                      streaming it, then TMA-loads the item's rows (32-row x
//                      128-byte boxes, 128B swizzle = the UMMA K-major SW128
//                      canonical layout) into a ring of 128-row x 128-byte
//                      slabs (64 halves or 32 floats of every row).
//   warp 10 queries  : stages the next item's (<= 16) query rows into the
//                      free one of two query tiles (same SW128 layout).
//   warp 1  MMA      : allocates 64 TMEM columns (a ring of four 128x16
//                      fp32 accumulators); one elected lane issues 4 MMAs
//                      (M=128 rows, N=16 queries, K=16 f16 / K=8 tf32) per slab,
//                      tcgen05.commit frees the slab / the query tile and
//                      publishes a chunk.
//   warps 2-9 epilogue: per 128-row chunk, tcgen05.ld their TMEM lane quadrant
//                      (thread = row) x column half (8 queries), form the fp32
//                      dot-form distance qn + xn - 2 q.x and run the
//                      threshold-filtered per-query top-kp selection.
// Distances are approximate (fp16 / TF32 inputs); the certified fp64 re-rank
// (tri_select.cu) makes the final result exact.
#include <cuda.h>

#include <algorithm>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

constexpr int kTcThreads = 352;  // producer warp, MMA warp, 8 epilogue warps, query-staging warp
constexpr int kWSlots = 4;        // work-item ring (the producer publishes one item ahead)
constexpr int kTcRows = 128;                    // MMA M = rows per chunk
constexpr int kTcN = 16;                        // MMA N = queries per group
constexpr int kTcRowB = 128;                    // bytes per row per slab (one SW128 row)
constexpr int kTcSlabBytes = kTcRows * kTcRowB;  // 16 KB
constexpr int kTcMaxStages = 12;  // ring depth: as many 16 KB slabs as shared memory allows (ScanLaunch::stages)
constexpr int kTcAcc = 4;                       // TMEM accumulator ring (x16 columns)
constexpr int kTcQTile = kTcN * kTcRowB;        // 2 KB of queries per slab
// Instruction descriptors: F32 accumulator, K-major A/B, N=16, M=128; A/B
// format TF32 (2) for kind::tf32, F16 (0) for kind::f16.
constexpr uint32_t kTcIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                                  ((uint32_t)(kTcRows >> 4) << 24);
constexpr uint32_t kTcIdescF16 = (1u << 4) | ((uint32_t)(kTcN >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
template <bool H>
__host__ __device__ constexpr int slab_elems() { return H ? 64 : 32; }
__host__ __device__ inline int tc_nslab(int row_bytes) { return (row_bytes + kTcRowB - 1) / kTcRowB; }

__device__ __forceinline__ uint32_t tsu32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tmb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tsu32(b)), "r"(c));
}
__device__ __forceinline__ void tmb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tsu32(b)) : "memory");
}
__device__ __forceinline__ void tmb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tsu32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tmb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n TWAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TWAIT_%=;\n}\n" ::"r"(tsu32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ttma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(tsu32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(tsu32(bar))
      : "memory");
}
__device__ __forceinline__ void ttma_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(tsu32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(tsu32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 2, 256;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <bool H>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  if (H) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kTcIdescF16), "r"(accumulate));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kTcIdescTf32), "r"(accumulate));
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(tsu32(bar))
               : "memory");
}

struct TcSmem {
  uint64_t full[kTcMaxStages], empty[kTcMaxStages];
  uint64_t wfull[kWSlots], wempty[kWSlots];
  uint64_t qfull[2], qempty[2];
  uint64_t tfull[kTcAcc], tempty[kTcAcc];
  WorkItem witem[kWSlots];
  int wend[kWSlots];
  uint32_t tmem_base;
  int cnt[2][kTcN];
  unsigned long long thr[kTcN];
  int qid[kTcN];
  int kpq[kTcN];  // each member's kp (Member::pad): <= the item's kp in mixed-class groups
  float qn[kTcN];
  float qinv[kTcN];
};

// alignment pad + qbufs query tiles + abufs append-list buffers
static size_t tc_fixed_smem(int row_bytes, int qbufs, int abufs) {
  return 1024 + (size_t)qbufs * tc_nslab(row_bytes) * kTcQTile + (size_t)abufs * kTcN * kTcRows * 8;
}

size_t tc_scan_smem_bytes(int row_bytes) { return tc_fixed_smem(row_bytes, 2, 2) + (size_t)kTcMinStages * kTcSlabBytes; }

int tc_scan_stages(int row_bytes, int smem_limit, int want, int qbufs, int abufs) {
  int n = (int)(((long long)smem_limit - (long long)tc_fixed_smem(row_bytes, qbufs, abufs)) / kTcSlabBytes);
  if (want > 0) n = std::min(n, want);
  return std::max(std::min(n, kTcMaxStages), 0);
}

template <bool H>
__device__ __forceinline__ int row_bytes_of(const ScanLaunch& a) { return H ? a.qldh * 2 : a.qld * 4; }

// Consumer side of the work-item ring (every consumer warp sees every item, in order).
struct ItemRing {
  int slot = 0, phase = 0;
};
__device__ __forceinline__ bool next_item(TcSmem& sh, ItemRing& r, WorkItem& w, int lane) {
  tmb_wait(&sh.wfull[r.slot], r.phase);
  const int end = sh.wend[r.slot];
  w = sh.witem[r.slot];
  __syncwarp();
  if (lane == 0) tmb_arrive(&sh.wempty[r.slot]);
  if (++r.slot == kWSlots) {
    r.slot = 0;
    r.phase ^= 1;
  }
  return !end;
}

// ---------------------------------------------------------------------------

// Producer (one thread): claims work items, publishes each one ring slot
// AHEAD of streaming it (so the query-staging warp prepares item i+1 while
// item i streams), then TMA-loads the item's rows slab by slab.
template <bool H>
__device__ void tc_producer(const ScanLaunch& a, const CUtensorMap* map, const CUtensorMap* tail, TcSmem& sh,
                            unsigned char* ring) {
  const int n_items = *a.n_items;
  const int nslab = tc_nslab(row_bytes_of<H>(a));
  int wslot = 0, wphase = 0, stage = 0, sphase = 0;
  auto publish = [&](int it) -> bool {
    tmb_wait(&sh.wempty[wslot], wphase ^ 1);
    const bool ok = it < n_items;
    if (ok) sh.witem[wslot] = a.items[it];
    sh.wend[wslot] = ok ? 0 : 1;
    tmb_arrive(&sh.wfull[wslot]);
    if (++wslot == kWSlots) {
      wslot = 0;
      wphase ^= 1;
    }
    return ok;
  };
  uint64_t pol = 0;
  if (a.l2hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  if (a.l2hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  int cur = atomicAdd(a.counter, 1);
  if (!publish(cur)) return;
  for (;;) {
    const WorkItem w = a.items[cur];
    const int nxt = atomicAdd(a.counter, 1);
    const bool more = publish(nxt);
    const int nchunk = (w.row_count + kTcRows - 1) / kTcRows;
    for (int c = 0; c < nchunk; ++c) {
      const int rows = min(kTcRows, w.row_count - c * kTcRows);
      // full chunks: box_rows-row boxes (few TMA ops: the per-SM TMA issue rate
      // bounds the stream otherwise); a partial last chunk: 32-row boxes
      // (over-reads at most 31 rows of the next list)
      const bool full = rows == kTcRows;
      const CUtensorMap* m = full ? map : tail;
      const int br = full ? a.box_rows : 32;
      const int nbox = (rows + br - 1) / br;
      const int row0 = (int)(w.row_begin + (long long)c * kTcRows);
      for (int s = 0; s < nslab; ++s) {
        tmb_wait(&sh.empty[stage], sphase ^ 1);
        unsigned char* dst = ring + (size_t)stage * kTcSlabBytes;
        tmb_expect(&sh.full[stage], (uint32_t)(nbox * br * kTcRowB));
        for (int b = 0; b < nbox; ++b) {
          if (a.l2hint)
            ttma_2d_hint(dst + b * br * kTcRowB, m, s * slab_elems<H>(), row0 + b * br, &sh.full[stage], pol);
          else
            ttma_2d(dst + b * br * kTcRowB, m, s * slab_elems<H>(), row0 + b * br, &sh.full[stage]);
        }
        if (++stage == a.stages) {
          stage = 0;
          sphase ^= 1;
        }
      }
    }
    if (!more) return;
    cur = nxt;
  }
}

// Query-staging warp: copies the next item's (up to 16) query rows into the
// free query tile in the UMMA SW128 K-major layout -- slab s, query g, 16-byte
// chunk c at s*2KB + g*128 + ((c ^ (g&7)) << 4) -- then hands it to the MMA warp.
template <bool H>
__device__ void tc_qstage(const ScanLaunch& a, TcSmem& sh, unsigned char* qs, int qtile_bytes) {
  const int lane = threadIdx.x & 31;
  const int row_bytes = row_bytes_of<H>(a);
  const int nslab = tc_nslab(row_bytes);
  const uint4* Q4 = reinterpret_cast<const uint4*>(H ? a.Qh : static_cast<const void*>(a.Q));
  const int q4 = row_bytes >> 4;
  const int total = nslab * kTcN * 8;
  ItemRing r;
  WorkItem w;
  for (int j = 0; next_item(sh, r, w, lane); ++j) {
    const int qb = j % a.qbufs;
    tmb_wait(&sh.qempty[qb], ((j / a.qbufs) & 1) ^ 1);
    unsigned char* dst = qs + qb * qtile_bytes;
    const int gc = w.member_count;
    const int myq = lane < gc ? a.members[w.member_begin + lane].q : 0;
    for (int i0 = 0; i0 < total; i0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 32 + lane;
        const int c = i & 7, g = (i >> 3) & (kTcN - 1), sl = i >> 7;
        const int col4 = sl * 8 + c;
        const int qq = __shfl_sync(0xffffffffu, myq, g);
        v[u] = make_uint4(0u, 0u, 0u, 0u);
        if (i < total && g < gc && col4 < q4) v[u] = Q4[(long long)qq * q4 + col4];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 32 + lane;
        const int c = i & 7, g = (i >> 3) & (kTcN - 1), sl = i >> 7;
        if (i < total) *reinterpret_cast<uint4*>(dst + sl * kTcQTile + g * 128 + ((c ^ (g & 7)) << 4)) = v[u];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core reads
    __syncwarp();
    if (lane == 0) tmb_arrive(&sh.qfull[qb]);
  }
}

template <bool H>
__device__ void tc_mma(const ScanLaunch& a, TcSmem& sh, unsigned char* ring, unsigned char* qs, int qtile_bytes) {
  const int lane = threadIdx.x & 31;
  const int nslab = tc_nslab(row_bytes_of<H>(a));
  int stage = 0, sphase = 0, acc = 0, aphase = 0;
  const uint32_t tmem = sh.tmem_base;
  const uint32_t ring_s = tsu32(ring);
  ItemRing r;
  WorkItem w;
  for (int j = 0; next_item(sh, r, w, lane); ++j) {
    const int qb = j % a.qbufs;
    tmb_wait(&sh.qfull[qb], (j / a.qbufs) & 1);
    const uint32_t qs_s = tsu32(qs + qb * qtile_bytes);
    const int nchunk = (w.row_count + kTcRows - 1) / kTcRows;
    for (int c = 0; c < nchunk; ++c) {
      tmb_wait(&sh.tempty[acc], aphase ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t d_tmem = tmem + (uint32_t)(acc * kTcN);
      for (int s = 0; s < nslab; ++s) {
        tmb_wait(&sh.full[stage], sphase);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = ring_s + (uint32_t)stage * kTcSlabBytes;
          const uint32_t b0 = qs_s + (uint32_t)s * kTcQTile;
          if (!(a.dbg & 2)) {
#pragma unroll
            for (int k = 0; k < kTcRowB / 32; ++k)  // 32 B of K per MMA (16 halves / 8 floats)
              umma<H>(d_tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), (s | k) != 0);
          }
          umma_commit(&sh.empty[stage]);  // slab reusable once these MMAs retire
          if (s == nslab - 1) {
            umma_commit(&sh.tfull[acc]);
            if (c == nchunk - 1) umma_commit(&sh.qempty[qb]);  // query tile reusable
          }
        }
        __syncwarp();
        if (++stage == a.stages) {
          stage = 0;
          sphase ^= 1;
        }
      }
      if (++acc == kTcAcc) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Epilogue selection (8 warps).  Warp w reads TMEM lane quadrant w % 4 (=
// chunk rows 32*(w%4) ..) and column half h = ew / 4 (queries 8h .. 8h+7).
// Every query g of the group has one owner warp (ew = g % 8) that keeps its
// running top-kp list sorted in registers (element j*32 + lane in v[j],
// kp = 32*KL).  Per 128-row chunk, all 256 threads append the candidates that
// beat the query's threshold to its smem buffer (double-buffered by chunk
// parity); after ONE named barrier each owner folds its buffer in 32 at a
// time: by insertion when few of them beat the list's last key (list_insert),
// else register bitonic sort (shuffles), bitonic split against the list's
// last 32, bitonic merge.  Thresholds are published by the owner and read
// (possibly one chunk stale, which only admits more candidates) by appenders.
constexpr int kEpiWarps = 8;

template <bool H, int KL>
__device__ __forceinline__ int tc_epi_item(const ScanLaunch& a, const WorkItem& w, TcSmem& sh,
                                           unsigned long long* sel, int ring) {
  int acc = ring & 0xff, aphase = ring >> 8;
  const int e = threadIdx.x - 64, lane = threadIdx.x & 31, ew = e >> 5;
  const int quad = (threadIdx.x >> 5) & 3;
  const int half = ew >> 2;
  const int row_in_chunk = quad * 32 + lane;  // == TMEM lane
  const int gc = w.member_count;
  const uint32_t tmem = sh.tmem_base;
  unsigned long long L[2][KL];
#pragma unroll
  for (int qi = 0; qi < 2; ++qi)
#pragma unroll
    for (int j = 0; j < KL; ++j) L[qi][j] = TRI_KEY_MAX;
  const int nchunk = (w.row_count + kTcRows - 1) / kTcRows;
  float xn_next = row_in_chunk < w.row_count ? a.xnorm[w.row_begin + row_in_chunk] : 0.f;
  volatile unsigned long long* thr = sh.thr;
  unsigned long long gpre[2] = {TRI_KEY_MAX, TRI_KEY_MAX};  // owner lane 0: cross-item bound, loaded ahead
  for (int c = 0; c < nchunk; ++c) {
    const int buf = a.abufs == 2 ? (c & 1) : 0;
    const int rows = min(kTcRows, w.row_count - c * kTcRows);
    if (a.gthr && lane == 0) {  // issued before the TMEM wait: the L2 round trip overlaps it
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {
        const int g = ew + kEpiWarps * qi;
        if (g < gc) gpre[qi] = __ldcg(a.gthr + sh.qid[g]);
      }
    }
    const long long row = w.row_begin + (long long)c * kTcRows + row_in_chunk;
    const bool valid = row_in_chunk < rows;
    const float xn = xn_next;  // loaded one chunk ahead (HBM latency off the critical path)
    if ((c + 1) * kTcRows + row_in_chunk < w.row_count) xn_next = a.xnorm[row + kTcRows];
    tmb_wait(&sh.tfull[acc], aphase);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * kTcN + half * 8);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) tmb_arrive(&sh.tempty[acc]);
    if (++acc == kTcAcc) {
      acc = 0;
      aphase ^= 1;
    }
    if (a.dbg & 1) continue;
    if (valid) {
      const uint32_t pos = (uint32_t)row;
      unsigned long long* sb = sel + (size_t)buf * kTcN * kTcRows;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int g = half * 8 + j;
        if (g < gc) {
          const float dot = H ? __uint_as_float(v[j]) * sh.qinv[g] : __uint_as_float(v[j]);
          const unsigned long long key = make_key(__fmaf_rn(-2.f, dot, __fadd_rn(sh.qn[g], xn)), pos);
          if (key < thr[g]) sb[g * kTcRows + atomicAdd(&sh.cnt[buf][g], 1)] = key;  // <= 128 per chunk
        }
      }
    }
    epi_sync();
#pragma unroll
    for (int qi = 0; qi < 2; ++qi) {
      const int g = ew + kEpiWarps * qi;
      if (g < gc) {
        const int n = sh.cnt[buf][g];
        const unsigned long long* sb = sel + (size_t)buf * kTcN * kTcRows + g * kTcRows;
        for (int b = 0; b < n; b += 32) {
          list_fold32<KL>(L[qi], b + lane < n ? sb[b + lane] : TRI_KEY_MAX, lane);
        }
        if (n > 0) {
          // the member's own kp-th key (a mixed-class group runs at the largest kp)
          const int jq = (sh.kpq[g] >> 5) - 1;
          unsigned long long t = TRI_KEY_MAX;
#pragma unroll
          for (int j = 0; j < KL; ++j) {
            const unsigned long long y = __shfl_sync(0xffffffffu, L[qi][j], 31);
            if (j == jq) t = y;
          }
          if (lane == 0) {
            if (a.gthr) {
              // cross-item threshold: a full list's kp-th key bounds the query's
              // final kp-th key, so every CTA scanning this query may drop rows
              // at or above it (publish without waiting; pick up others' bounds)
              unsigned long long* gq = a.gthr + sh.qid[g];
              const unsigned long long gt = gpre[qi];
              if (t != TRI_KEY_MAX && t < gt) atomicMin(gq, t);
              t = t < gt ? t : gt;
            }
            thr[g] = t;
          }
        }
        __syncwarp();
        if (lane == 0) sh.cnt[buf][g] = 0;
      }
    }
    if (a.abufs == 1) epi_sync();  // single append buffer: drained before the next chunk appends
  }
#pragma unroll
  for (int qi = 0; qi < 2; ++qi) {
    const int g = ew + kEpiWarps * qi;
    if (g < gc) {
      unsigned long long* out = a.part + a.members[w.member_begin + g].slot;
#pragma unroll
      for (int j = 0; j < KL; ++j)
        if (j * 32 < sh.kpq[g]) out[j * 32 + lane] = L[qi][j];  // the member's kp entries
    }
  }
  return acc | (aphase << 8);
}

// Epilogue: 8 warps (256 threads); see tc_epi_item for the TMEM mapping.
template <bool H>
__device__ void tc_epilogue(const ScanLaunch& a, TcSmem& sh, unsigned long long* sel) {
  const int e = threadIdx.x - 64;  // 0..255
  const int lane = threadIdx.x & 31;
  int ring = 0;
  ItemRing r;
  WorkItem w;
  while (next_item(sh, r, w, lane)) {
    const int gc = w.member_count;
    if (e < kTcN) {
      const int q = e < gc ? a.members[w.member_begin + e].q : -1;
      sh.cnt[0][e] = 0;
      sh.cnt[1][e] = 0;
      sh.thr[e] = (a.gthr && q >= 0) ? __ldcg(a.gthr + q) : TRI_KEY_MAX;
      sh.qid[e] = q < 0 ? 0 : q;
      sh.kpq[e] = q >= 0 ? a.members[w.member_begin + e].pad : kMinKp;
      sh.qn[e] = q >= 0 ? a.qnorm[q] : 0.f;
      sh.qinv[e] = (H && q >= 0) ? a.qinv[q] : 0.f;
    }
    epi_sync();
    switch (w.kp) {
      case 32: ring = tc_epi_item<H, 1>(a, w, sh, sel, ring); break;
      case 64: ring = tc_epi_item<H, 2>(a, w, sh, sel, ring); break;
      case 128: ring = tc_epi_item<H, 4>(a, w, sh, sel, ring); break;
      default: ring = tc_epi_item<H, 8>(a, w, sh, sel, ring); break;  // 256 (host caps tc kp at kTcMaxKp)
    }
    epi_sync();  // counters and append buffers are free for the next item
  }
}

template <bool H>
__global__ void __launch_bounds__(kTcThreads, 1) scan_tc_kernel(const __grid_constant__ CUtensorMap map,
                                                                const __grid_constant__ CUtensorMap tail, ScanLaunch a) {
  extern __shared__ __align__(1024) unsigned char tsmem_raw[];
  __shared__ TcSmem sh;
  unsigned char* base = tsmem_raw + ((1024u - (tsu32(tsmem_raw) & 1023u)) & 1023u);
  unsigned char* ring = base;
  unsigned char* qs = ring + (size_t)a.stages * kTcSlabBytes;
  const int qtile_bytes = tc_nslab(row_bytes_of<H>(a)) * kTcQTile;
  unsigned long long* sel = reinterpret_cast<unsigned long long*>(qs + (size_t)a.qbufs * qtile_bytes);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      tmb_init(&sh.full[s], 1);
      tmb_init(&sh.empty[s], 1);
    }
    for (int s = 0; s < kWSlots; ++s) {
      tmb_init(&sh.wfull[s], 1);
      tmb_init(&sh.wempty[s], 10);  // MMA warp + 8 epilogue warps + query-staging warp
    }
    for (int s = 0; s < 2; ++s) {
      tmb_init(&sh.qfull[s], 1);
      tmb_init(&sh.qempty[s], 1);
    }
    for (int s = 0; s < kTcAcc; ++s) {
      tmb_init(&sh.tfull[s], 1);
      tmb_init(&sh.tempty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(tsu32(&sh.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) {
    if ((threadIdx.x & 31) == 0) tc_producer<H>(a, &map, &tail, sh, ring);
  } else if (warp == 1) {
    tc_mma<H>(a, sh, ring, qs, qtile_bytes);
  } else if (warp == 10) {
    tc_qstage<H>(a, sh, qs, qtile_bytes);
  } else {
    tc_epilogue<H>(a, sh, sel);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(sh.tmem_base));
  }
}

template <bool H>
cudaError_t launch_tc(const ScanLaunch& s, cudaStream_t st) {
  if (s.stages < kTcMinStages || s.stages > kTcMaxStages) return cudaErrorInvalidValue;
  if (s.qbufs < 1 || s.qbufs > 2 || s.abufs < 1 || s.abufs > 2) return cudaErrorInvalidValue;
  const size_t smem = tc_fixed_smem(H ? s.qldh * 2 : s.qld * 4, s.qbufs, s.abufs) + (size_t)s.stages * kTcSlabBytes;
  cudaError_t e = cudaFuncSetAttribute(scan_tc_kernel<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  scan_tc_kernel<H><<<s.grid, kTcThreads, smem, st>>>(*reinterpret_cast<const CUtensorMap*>(s.tmap_tc),
                                                      *reinterpret_cast<const CUtensorMap*>(s.tmap_tc_tail), s);
  return cudaGetLastError();
}

cudaError_t launch_scan_tc(const ScanLaunch& s, cudaStream_t st) {
  return s.f16 ? launch_tc<true>(s, st) : launch_tc<false>(s, st);
}

}  // namespace tri
