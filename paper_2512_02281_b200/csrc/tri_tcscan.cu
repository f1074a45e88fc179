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
constexpr int kTcRowB = 128;                    // bytes per row per slab (one SW128 row)
constexpr int kTcSlabBytes = kTcRows * kTcRowB;  // 16 KB
constexpr int kTcMaxStages = 12;  // ring depth: as many 16 KB slabs as shared memory allows (ScanLaunch::stages)
// TMEM accumulator ring (x N columns): 4 x 16 for list items; 8 x 64 (all 512
// columns) for brute-force items, which hold every chunk of an item (<= 8
// chunks, host-guaranteed) so the epilogue can read them twice (tc_seed_pass)
template <int N>
__host__ __device__ constexpr int tc_acc() { return N == 64 ? 8 : 4; }
constexpr int kTcAccMax = 8;
// Query-group width N (MMA N): 16 for IVF list items (few queries per list),
// 64 for brute force, where one item covers a row range for up to 64 queries
// so every row slab is read from L2 once per 64 queries (ScanLaunch::nq).
// Instruction descriptor: F32 accumulator, K-major A/B, N, M=128; A/B format
// TF32 (2) for kind::tf32, F16 (0) for kind::f16.
template <bool H, int N>
__host__ __device__ constexpr uint32_t tc_idesc() {
  return (1u << 4) | (H ? 0u : ((2u << 7) | (2u << 10))) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kTcRows >> 4) << 24);
}
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
// epilogue-wide OR (named barrier 3 over the 8 epilogue warps)
__device__ __forceinline__ bool __syncthreads_or_epi(bool p) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred ip, op;\n setp.ne.u32 ip, %1, 0;\n barrier.red.or.pred op, 3, 256, ip;\n selp.u32 %0, 1, 0, op;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)p)
      : "memory");
  return r != 0;
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <bool H, int N>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  constexpr uint32_t kIdesc = tc_idesc<H, N>();
  if (H) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(tsu32(bar))
               : "memory");
}

template <int N>
struct TcSmem {
  uint64_t full[kTcMaxStages], empty[kTcMaxStages];
  uint64_t wfull[kWSlots], wempty[kWSlots];
  uint64_t qfull[2], qempty[2];
  uint64_t tfull[kTcAccMax], tempty[kTcAccMax];
  WorkItem witem[kWSlots];
  int wend[kWSlots];
  uint32_t tmem_base;
  int cnt[2][N];
  unsigned long long thr[N];
  int qid[N];
  int kpq[N];  // each member's kp (Member::pad): <= the item's kp in mixed-class groups
  float qn[N];
  float qinv[N];
  uint32_t smin[N];  // cross-item seed: the item's smallest distance per query (fp32 order bits)
  int anyapp[2];     // single append buffer: some candidate was appended in chunk c (slot c & 1)
  float xns[N == 64 ? 8 * 128 : 1];  // wide items: every chunk's row norms (seed pass -> selection pass)
};

constexpr int kTcSmemMax = 227 * 1024;  // dynamic + static shared memory per CTA (opt-in maximum)

// alignment pad + qbufs query tiles + abufs append-list buffers
static size_t tc_fixed_smem(int row_bytes, int qbufs, int abufs, int nq) {
  return 1024 + (size_t)qbufs * tc_nslab(row_bytes) * nq * kTcRowB + (size_t)abufs * nq * kTcRows * 8;
}

size_t tc_scan_smem_bytes(int row_bytes, int nq) {
  return tc_fixed_smem(row_bytes, 2, 2, nq) + (size_t)kTcMinStages * kTcSlabBytes;
}

int tc_scan_stages(int row_bytes, int smem_limit, int want, int qbufs, int abufs, int nq) {
  const long long stat = nq == kTcGroupWide ? sizeof(TcSmem<kTcGroupWide>) : sizeof(TcSmem<kTcGroup>);
  const long long lim = std::min<long long>(smem_limit, kTcSmemMax - stat);
  int n = (int)((lim - (long long)tc_fixed_smem(row_bytes, qbufs, abufs, nq)) / kTcSlabBytes);
  if (want > 0) n = std::min(n, want);
  return std::max(std::min(n, kTcMaxStages), 0);
}

// Timeline probe (ScanLaunch::dbg & 8, experiments only): per CTA globaltimer
// stamps of the pipeline's milestones, read back by tri_debug_scan_ts.
constexpr int kTsCtas = 256, kTsSlots = 16;
__device__ unsigned long long g_scan_ts[kTsCtas * kTsSlots];
// dbg & 16: [0] candidates appended, [1] (chunk, query) folds with n > 0,
// [2] seeds left open, [3] seeds set (brute force) / [2] appended, [3] folds
// of kp >= 128 members (list scan)
__device__ unsigned long long g_scan_cnt[4];
__device__ __forceinline__ void ts_mark(const ScanLaunch& a, int slot) {
  if ((a.dbg & 8) && blockIdx.x < kTsCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_scan_ts[blockIdx.x * kTsSlots + slot] = t;
  }
}

template <bool H>
__device__ __forceinline__ int row_bytes_of(const ScanLaunch& a) { return H ? a.qldh * 2 : a.qld * 4; }

// Consumer side of the work-item ring (every consumer warp sees every item, in order).
struct ItemRing {
  int slot = 0, phase = 0;
};
template <int N>
__device__ __forceinline__ bool next_item(TcSmem<N>& sh, ItemRing& r, WorkItem& w, int lane) {
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
template <bool H, int N>
__device__ void tc_producer(const ScanLaunch& a, const CUtensorMap* map, const CUtensorMap* tail, TcSmem<N>& sh,
                            unsigned char* ring) {
  const int n_items = *a.n_items;
  const int nslab = tc_nslab(row_bytes_of<H>(a));
  int wslot = 0, wphase = 0, stage = 0, sphase = 0;
  auto publish = [&](int it) -> bool {
    tmb_wait(&sh.wempty[wslot], wphase ^ 1);
    const bool ok = it < n_items;
    if (ok) {
      sh.witem[wslot] = a.items[it];
      sh.witem[wslot].pad0 = it;  // the item's index (seed slot of the cross-CTA bound)
    }
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
  // cross-item seeding needs every item in flight at once: CTA i takes item i
  // (the host launches one CTA per item); otherwise items are claimed dynamically
  const bool fixed = a.seed == 2;
  int cur = fixed ? (int)blockIdx.x : atomicAdd(a.counter, 1);
  if (!publish(cur)) return;
  ts_mark(a, 2);
  for (;;) {
    const WorkItem w = a.items[cur];
    const int nxt = fixed ? n_items : atomicAdd(a.counter, 1);
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
    if (!more) {
      ts_mark(a, 6);
      return;
    }
    cur = nxt;
  }
}

// Query-staging warp: copies the next item's (up to N) query rows into the
// free query tile in the UMMA SW128 K-major layout -- slab s, query g, 16-byte
// chunk c at s*(N*128) + g*128 + ((c ^ (g&7)) << 4) -- then hands it to the MMA warp.
template <bool H, int N>
__device__ void tc_qstage(const ScanLaunch& a, const CUtensorMap* qmap, TcSmem<N>& sh, unsigned char* qs,
                          int qtile_bytes) {
  constexpr int kLogN = N == 64 ? 6 : 4;
  constexpr int kQTile = N * kTcRowB;
  const int lane = threadIdx.x & 31;
  const int row_bytes = row_bytes_of<H>(a);
  const int nslab = tc_nslab(row_bytes);
  const uint4* Q4 = reinterpret_cast<const uint4*>(H ? a.Qh : static_cast<const void*>(a.Q));
  const int q4 = row_bytes >> 4;
  const int total = nslab * N * 8;
  ItemRing r;
  WorkItem w;
  for (int j = 0; next_item(sh, r, w, lane); ++j) {
    const int qb = j % a.qbufs;
    tmb_wait(&sh.qempty[qb], ((j / a.qbufs) & 1) ^ 1);
    unsigned char* dst = qs + qb * qtile_bytes;
    const int gc = w.member_count;
    if (a.q_tma) {
      // the item's members are consecutive queries: one TMA box (32 floats x N
      // rows, SW128) per slab straight into the tile; rows past B read as zeros
      if (lane == 0) {
        const int q0 = a.members[w.member_begin].q;
        tmb_expect(&sh.qfull[qb], (uint32_t)(nslab * kQTile));
        for (int sl = 0; sl < nslab; ++sl) ttma_2d(dst + sl * kQTile, qmap, sl * slab_elems<H>(), q0, &sh.qfull[qb]);
        if (j == 0) ts_mark(a, 3);
      }
      __syncwarp();
      continue;
    }
    int myq[N / 32 > 0 ? N / 32 : 1];
#pragma unroll
    for (int h = 0; h < (N + 31) / 32; ++h) {
      const int m = h * 32 + lane;
      myq[h] = (m < gc && m < N) ? a.members[w.member_begin + m].q : 0;
    }
    for (int i0 = 0; i0 < total; i0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 32 + lane;
        const int c = i & 7, g = (i >> 3) & (N - 1), sl = i >> (3 + kLogN);
        const int col4 = sl * 8 + c;
        int qq = __shfl_sync(0xffffffffu, myq[0], g & 31);
        if (N > 32) {
          const int q1 = __shfl_sync(0xffffffffu, myq[N > 32 ? 1 : 0], g & 31);
          if (g >= 32) qq = q1;
        }
        v[u] = make_uint4(0u, 0u, 0u, 0u);
        if (i < total && g < gc && col4 < q4) v[u] = Q4[(long long)qq * q4 + col4];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 32 + lane;
        const int c = i & 7, g = (i >> 3) & (N - 1), sl = i >> (3 + kLogN);
        if (i < total) *reinterpret_cast<uint4*>(dst + sl * kQTile + g * 128 + ((c ^ (g & 7)) << 4)) = v[u];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core reads
    __syncwarp();
    if (lane == 0) {
      if (j == 0) ts_mark(a, 3);
      tmb_arrive(&sh.qfull[qb]);
    }
  }
}

template <bool H, int N>
__device__ void tc_mma(const ScanLaunch& a, TcSmem<N>& sh, unsigned char* ring, unsigned char* qs, int qtile_bytes) {
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
      const uint32_t d_tmem = tmem + (uint32_t)(acc * N);  // ring of tc_acc<N>() accumulators
      for (int s = 0; s < nslab; ++s) {
        tmb_wait(&sh.full[stage], sphase);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = ring_s + (uint32_t)stage * kTcSlabBytes;
          const uint32_t b0 = qs_s + (uint32_t)s * (N * kTcRowB);
          if (!(a.dbg & 2)) {
#pragma unroll
            for (int k = 0; k < kTcRowB / 32; ++k)  // 32 B of K per MMA (16 halves / 8 floats)
              umma<H, N>(d_tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), (s | k) != 0);
          }
          umma_commit(&sh.empty[stage]);  // slab reusable once these MMAs retire
          if (j == 0 && c == 0 && s == nslab - 1) ts_mark(a, 4);
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
      if (++acc == tc_acc<N>()) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Epilogue selection (8 warps).  Warp w reads TMEM lane quadrant w % 4 (=
// chunk rows 32*(w%4) ..) and column half h = ew / 4 (queries N/2*h ..
// N/2*h + N/2 - 1).  Every query g of the group has one owner warp (ew = g % 8)
// that keeps its running top-kp list sorted in registers (element j*32 + lane
// in v[j], kp = 32*KL).  Per 128-row chunk, all 256 threads append the
// candidates that beat the query's threshold to its smem buffer
// (double-buffered by chunk parity); after ONE named barrier each owner folds
// its buffer in 32 at a time: by insertion when few of them beat the list's
// last key (list_insert), else register bitonic sort (shuffles), bitonic split
// against the list's last 32, bitonic merge.  Thresholds are published by the
// owner and read (possibly one chunk stale, which only admits more candidates)
// by appenders.
constexpr int kEpiWarps = 8;
constexpr int kSeedPerLane = 5;  // cross-CTA seed: up to 160 items (one wave of 148 SMs)

template <int QPT>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&v)[QPT]) {
  if constexpr (QPT == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
  } else {
    static_assert(QPT == 32, "query columns per epilogue thread");
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  }
}


// Seed pass of a brute-force item (N = 64; every chunk of the item is resident
// in TMEM).  Each epilogue thread takes, per query of its column half, the
// minimum approximate distance over its rows (row_in_chunk of every chunk):
// 128 group minima per query, each an actual row's value.  The kp-th smallest
// group minimum is therefore >= the item's kp-th smallest distance (kp distinct
// rows lie at or below it), and it admits only ~kp/(rows per group) of the
// item's rows -- the selection pass then folds a few dozen candidates per
// query instead of a first chunk's 128 and its running-threshold stragglers.
// The owner warp finds that order statistic by bisection on the fp32 order bits
// (ballot counts), publishes it as the query's cross-item bound and seeds thr.
// The chunk ring is left untouched (no tempty arrivals): the selection pass
// re-reads the same accumulators.
template <bool H, int N>
__device__ __forceinline__ void tc_seed_pass(const ScanLaunch& a, const WorkItem& w, TcSmem<N>& sh,
                                             unsigned long long* sel, int acc, int aphase) {
  constexpr int QPT = N / 2, OWN = N / kEpiWarps;
  const int e = threadIdx.x - 64, lane = threadIdx.x & 31, ew = e >> 5;
  const int quad = (threadIdx.x >> 5) & 3;
  const int half = ew >> 2;
  const int row_in_chunk = quad * 32 + lane;
  const int gc = w.member_count;
  const int nchunk = (w.row_count + kTcRows - 1) / kTcRows;
  const float inf = __int_as_float(0x7f800000);
  float mn[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) mn[j] = inf;
  // rolled loop (one copy of the body stays in the instruction cache); the
  // next chunk's norm is loaded one chunk ahead and every norm is kept in
  // shared memory for the selection pass
  float xn_next = row_in_chunk < w.row_count ? a.xnorm[w.row_begin + row_in_chunk] : 0.f;
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    const bool valid = c * kTcRows + row_in_chunk < w.row_count;
    const float xn = xn_next;
    if ((c + 1) * kTcRows + row_in_chunk < w.row_count) xn_next = a.xnorm[w.row_begin + (long long)(c + 1) * kTcRows + row_in_chunk];
    if (half == 0) sh.xns[c * kTcRows + row_in_chunk] = xn;
    tmb_wait(&sh.tfull[acc], aphase);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t v[QPT];
    tmem_ld_cols<QPT>(sh.tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * N + half * QPT), v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (valid) {
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        const int g = half * QPT + j;
        const float dot = H ? __uint_as_float(v[j]) * sh.qinv[g] : __uint_as_float(v[j]);
        mn[j] = fminf(mn[j], __fmaf_rn(-2.f, dot, __fadd_rn(sh.qn[g], xn)));
      }
    }
    if (++acc == tc_acc<N>()) {
      acc = 0;
      aphase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 64) ts_mark(a, 8);
  volatile unsigned long long* thr = sh.thr;
  if (a.seed == 2) {
    // (1) the item's minimum per query: butterfly transpose-min over the warp's
    // 32 rows (lane j ends with query half*32 + j), then the 4 row quadrants
    // combine with shared atomicMin on the order bits
    static_assert(QPT == 32, "cross-item seed: 32 query columns per thread");
    // keep this thread's per-query minima (its rows of every chunk) for the
    // selection pass: it re-reads only the columns whose minimum passes the seed
    float* mnb = reinterpret_cast<float*>(sel);  // [QPT][256] (first 32 KB of the append buffer)
#pragma unroll
    for (int j = 0; j < QPT; ++j) mnb[j * 256 + e] = mn[j];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < off; ++i) {
        const float send = up ? mn[i] : mn[i + off];
        const float keep = up ? mn[i + off] : mn[i];
        mn[i] = fminf(keep, __shfl_xor_sync(0xffffffffu, send, off));
      }
    }
    atomicMin(&sh.smin[half * 32 + lane], f2ord(mn[0]));
    epi_sync();
    // (2) publish, arrive, wait briefly for the other items (any subset of
    // published minima yields a valid bound; unpublished slots read +inf)
    if (e < gc) a.seed_min[(long long)sh.qid[e] * a.seed_items + w.pad0] = sh.smin[e];
    __threadfence();
    epi_sync();
    if (threadIdx.x == 64) {
      ts_mark(a, 9);
      atomicAdd(a.seed_ctr, 1);
      unsigned long long t0, t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        int c;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(c) : "l"(a.seed_ctr) : "memory");
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (c >= a.seed_items || t1 - t0 > 20000ull) break;
        __nanosleep(32);
      }
      ts_mark(a, 10);
    }
    epi_sync();
    // (3) bound per query without sorting: lane l takes the r-th smallest
    // (r = kp / 32) of the minima in slots l, l + 32, ...; the warp maximum T
    // has, in each of the 32 lanes, r distinct items at or below it -- kp
    // distinct rows -- so T >= the query's global kp-th distance
    const uint32_t oinf = f2ord(inf);
    uint32_t x[OWN][kSeedPerLane];  // every owned query's published minima: all loads issued before any store
#pragma unroll
    for (int qi = 0; qi < OWN; ++qi) {
      const int g = ew + kEpiWarps * qi;
      const uint32_t* sm = a.seed_min + (long long)sh.qid[g < gc ? g : 0] * a.seed_items;
#pragma unroll
      for (int i = 0; i < kSeedPerLane; ++i) {
        const int it = i * 32 + lane;
        x[qi][i] = (g < gc && it < a.seed_items) ? __ldcg(sm + it) : 0xffffffffu;
      }
    }
    uint32_t tq[OWN];
#pragma unroll
    for (int qi = 0; qi < OWN; ++qi) {
      const int g = ew + kEpiWarps * qi;
      uint32_t m1 = 0xffffffffu, m2 = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < kSeedPerLane; ++i) {
        m2 = min(m2, max(m1, x[qi][i]));
        m1 = min(m1, x[qi][i]);
      }
      tq[qi] = (g < gc && sh.kpq[g] > 32) ? m2 : m1;
    }
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1)
#pragma unroll
      for (int qi = 0; qi < OWN; ++qi) tq[qi] = max(tq[qi], __shfl_xor_sync(0xffffffffu, tq[qi], sft));
    if (lane == 0) {
#pragma unroll
      for (int qi = 0; qi < OWN; ++qi) {
        const int g = ew + kEpiWarps * qi;
        if (g >= gc || tq[qi] >= oinf) continue;
        const unsigned long long seed = ((unsigned long long)tq[qi] << 32) | 0xffffffffull;
        if (a.dbg & 16) atomicAdd(&g_scan_cnt[3], 1ull);
        const unsigned long long cur = thr[g];
        thr[g] = seed < cur ? seed : cur;
      }
    }
    epi_sync();
    if (threadIdx.x == 64) ts_mark(a, 11);
    return;
  }
  float* grp = reinterpret_cast<float*>(sel);  // N x 128 group minima (query-major) in the append buffer
#pragma unroll
  for (int j = 0; j < QPT; ++j) grp[(half * QPT + j) * kTcRows + row_in_chunk] = mn[j];
  epi_sync();
#pragma unroll
  for (int qi = 0; qi < OWN; ++qi) {
    const int g = ew + kEpiWarps * qi;
    if (g >= gc) continue;
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = f2ord(grp[g * kTcRows + i * 32 + lane]);
    uint32_t mx = max(max(o[0], o[1]), max(o[2], o[3])), mi = min(min(o[0], o[1]), min(o[2], o[3]));
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, sft));
      mi = min(mi, __shfl_xor_sync(0xffffffffu, mi, sft));
    }
    // invariant: count(o <= hi) >= kp (all 128 at the start; kp <= 64);
    // count(o <= lo) < kp (lo = min - 1: none).  Stops at 2^-11 relative width.
    const int kp = sh.kpq[g];
    unsigned long long seed = TRI_KEY_MAX;
    if (a.seed == 1) {
      long long lo = (long long)mi - 1, hi = mx;
      for (int it = 0; it < 32 && hi - lo > (long long)(1u << 12); ++it) {
        const uint32_t mid = (uint32_t)(lo + ((hi - lo) >> 1));
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) cnt += __popc(__ballot_sync(0xffffffffu, o[i] <= mid));
        if (cnt >= kp) hi = mid;
        else lo = mid;
      }
      // rows past the item / non-finite distances hold +inf (or NaN) minima:
      // with fewer than kp finite groups the seed stays open
      if ((uint32_t)hi < f2ord(inf)) seed = ((unsigned long long)(uint32_t)hi << 32) | 0xffffffffull;
    }
    if (lane == 0) {
      if (a.dbg & 16) atomicAdd(&g_scan_cnt[seed == TRI_KEY_MAX ? 2 : 3], 1ull);
      unsigned long long t = seed;
      if (a.gthr) {
        unsigned long long* gq = a.gthr + sh.qid[g];
        if (seed != TRI_KEY_MAX) atomicMin(gq, seed);
        const unsigned long long gt = __ldcg(gq);  // others' bounds published so far
        t = gt < t ? gt : t;
      }
      thr[g] = t;
    }
  }
  epi_sync();  // thresholds seeded; the append buffer is free again
  if (threadIdx.x == 64) ts_mark(a, 11);
}

// Cross-item bound from a pool of per-item winners (list scan, kp >= 128).
// An item's local kp-th key bounds only its own list, and with lists of ~1000
// rows a kp = 256 member admits about a quarter of every list it scans.  The
// pool collects each finished item's 32 smallest keys for the query (distinct
// rows: a row belongs to one list, a (query, list) pair to one item); the
// kp-th smallest key in the pool is then a bound on the query's kp-th key (kp
// real rows lie at or below it) that tightens with every finished list.
// Unwritten slots read as all ones and are not counted.  Bisection on the
// distance bits (the bound keeps every row id: low word all ones).
constexpr int kPoolMax = 1024;
template <int KL>
__device__ __forceinline__ void pool_publish(const ScanLaunch& a, int q, int kp, const unsigned long long (&L)[KL],
                                             int lane, uint32_t rmin) {
  // the list's 32 smallest keys with row id >= rmin (a finished item skips its
  // first chunk's rows, which it published when that chunk was folded)
  unsigned m[KL];
  int avail = 0;
#pragma unroll
  for (int j = 0; j < KL; ++j) {
    m[j] = __ballot_sync(0xffffffffu, L[j] != TRI_KEY_MAX && (uint32_t)L[j] >= rmin);
    avail += __popc(m[j]);
  }
  if (avail == 0) return;
  int slot = 0;
  if (lane == 0) slot = atomicAdd(a.pool_cnt + q, 32);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  if (slot + 32 > a.pool_cap) return;  // full: later lists no longer tighten the bound
  unsigned long long* P = a.pool + (long long)q * a.pool_cap;
  int taken = 0;
#pragma unroll
  for (int j = 0; j < KL; ++j) {
    const int r = taken + __popc(m[j] & ((1u << lane) - 1u));
    if (((m[j] >> lane) & 1u) && r < 32) P[slot + r] = L[j];
    taken += __popc(m[j]);
  }
  const int n = slot + 32;
  if (n < kp) return;
  __syncwarp();
  constexpr int kPer = kPoolMax / 32;
  uint32_t h[kPer];
  uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = j * 32 + lane;
    h[j] = i < n ? (uint32_t)(__ldcg(P + i) >> 32) : 0xffffffffu;
    if (h[j] != 0xffffffffu) {
      mn = min(mn, h[j]);
      mx = max(mx, h[j]);
    }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  int c = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) c += h[j] <= mx && h[j] != 0xffffffffu;
  if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) < kp) return;  // fewer than kp written keys yet
  // invariant: count(<= hi) >= kp, count(<= lo) < kp
  long long lo = (long long)mn - 1, hi = mx;
  for (int it = 0; it < 32 && hi - lo > (long long)(1u << 12); ++it) {
    const uint32_t mid = (uint32_t)(lo + ((hi - lo) >> 1));
    c = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) c += h[j] <= mid;
    if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) >= kp) hi = mid;
    else lo = mid;
  }
  if (lane == 0) atomicMin(a.gthr + q, ((unsigned long long)(uint32_t)hi << 32) | 0xffffffffull);
}

template <bool H, int N, int KL>
__device__ __forceinline__ int tc_epi_item(const ScanLaunch& a, const WorkItem& w, TcSmem<N>& sh,
                                           unsigned long long* sel, int ring) {
  constexpr int QPT = N / 2;          // query columns per thread (one column half)
  constexpr int OWN = N / kEpiWarps;  // queries owned per warp
  int acc = ring & 0xff, aphase = ring >> 8;
  const int e = threadIdx.x - 64, lane = threadIdx.x & 31, ew = e >> 5;
  const int quad = (threadIdx.x >> 5) & 3;
  const int half = ew >> 2;
  const int row_in_chunk = quad * 32 + lane;  // == TMEM lane
  const int gc = w.member_count;
  const uint32_t tmem = sh.tmem_base;
  unsigned long long L[OWN][KL];
#pragma unroll
  for (int qi = 0; qi < OWN; ++qi)
#pragma unroll
    for (int j = 0; j < KL; ++j) L[qi][j] = TRI_KEY_MAX;
  const int nchunk = (w.row_count + kTcRows - 1) / kTcRows;
  float xn_next = row_in_chunk < w.row_count ? a.xnorm[w.row_begin + row_in_chunk] : 0.f;
  volatile unsigned long long* thr = sh.thr;
  unsigned long long gpre[OWN];  // owner lane 0: cross-item bound, loaded ahead
#pragma unroll
  for (int qi = 0; qi < OWN; ++qi) gpre[qi] = TRI_KEY_MAX;
  if constexpr (N == kTcGroupWide) {
    if (a.seed) tc_seed_pass<H, N>(a, w, sh, sel, acc, aphase);
    // With a cross-item seed the item's every chunk is still resident and only
    // a handful of rows per query survive: append across all chunks with no
    // per-chunk barrier, then fold once.  A query whose survivors overflow its
    // 128-key buffer (adversarial ties) sends the item down the per-chunk path
    // below, which re-reads the same accumulators.
    if (a.seed == 2 && !(a.dbg & 1)) {
      // sparse selection: a (thread, query) pair is revisited only when the
      // thread's minimum over its rows (kept by the seed pass) passes the
      // query's bound; its column is then read from every chunk (x1 TMEM
      // loads, one wait) and each row tested exactly
      constexpr int kApp = 64;  // append slots per query (second 32 KB of the buffer)
      const float* mnb = reinterpret_cast<const float*>(sel);
      unsigned long long* sb = sel + 4096;
      const unsigned long long* thr_nv = sh.thr;  // fixed during this pass: loads may be hoisted
      // four query columns at a time: one x4 TMEM load per resident chunk and
      // ONE wait per group (a warp almost always has some lane passing a
      // column's bound, so per-column loads serialised 32 waits per item)
#pragma unroll 1
      for (int j0 = 0; j0 < QPT; j0 += 4) {
        bool hit[4];
        unsigned long long tk[4];
        bool any = false;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int g = half * QPT + j0 + t;
          tk[t] = thr_nv[g];
          hit[t] = g < gc && !(mnb[(j0 + t) * 256 + e] > ord2f((uint32_t)(tk[t] >> 32)));
          any |= hit[t];
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        uint32_t col[kTcWideMaxChunks][4];
        const uint32_t cbase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * QPT + j0);
#pragma unroll
        for (int c = 0; c < kTcWideMaxChunks; ++c) {
          col[c][0] = col[c][1] = col[c][2] = col[c][3] = 0u;
          if (c < nchunk)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                         : "=r"(col[c][0]), "=r"(col[c][1]), "=r"(col[c][2]), "=r"(col[c][3])
                         : "r"(cbase + (uint32_t)(((acc + c) & (kTcWideMaxChunks - 1)) * N)));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (!any) continue;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (!hit[t]) continue;
          const int g = half * QPT + j0 + t;
          const float qng = sh.qn[g];
          const float qig = sh.qinv[g];
#pragma unroll
          for (int c = 0; c < kTcWideMaxChunks; ++c) {
            if (c < nchunk && c * kTcRows + row_in_chunk < w.row_count) {
              const float dot = H ? __uint_as_float(col[c][t]) * qig : __uint_as_float(col[c][t]);
              const float d = __fmaf_rn(-2.f, dot, __fadd_rn(qng, sh.xns[c * kTcRows + row_in_chunk]));
              const unsigned long long key =
                  make_key(d, (uint32_t)(w.row_begin + (long long)c * kTcRows + row_in_chunk));
              if (key < tk[t]) {
                const int slot = atomicAdd(&sh.cnt[0][g], 1);
                if (slot < kApp) sb[g * kApp + slot] = key;
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      if (threadIdx.x == 64) ts_mark(a, 12);
      epi_sync();
      if (threadIdx.x == 64) ts_mark(a, 13);
      bool over = false;
#pragma unroll
      for (int qi = 0; qi < OWN; ++qi) {
        const int g = ew + kEpiWarps * qi;
        over |= g < gc && sh.cnt[0][g] > kApp;
      }
      over = __syncthreads_or_epi(over);
      if (!over) {
        // one item per CTA under the cross-item seed: no later chunk needs the
        // accumulators, so they are not handed back to the MMA warp
        // each query's survivors (or, beyond kp of them, their top kp) go
        // unsorted to the front of its partial region: launch_merge_compact
        if (threadIdx.x == 64) ts_mark(a, 14);
        // one returning atomic per owned query, all in flight at once (lane qi)
        int base = 0;
        long long poff = 0;
        if (lane < OWN) {
          const int g = ew + kEpiWarps * lane;
          const int n = g < gc ? sh.cnt[0][g] : 0;
          if (n > 0) {
            base = atomicAdd(a.compact_cnt + sh.qid[g], min(n, sh.kpq[g]));
            poff = a.meta[sh.qid[g]].part_off;
          }
        }
#pragma unroll
        for (int qi = 0; qi < OWN; ++qi) {
          const int g = ew + kEpiWarps * qi;
          const int qbase = __shfl_sync(0xffffffffu, base, qi);
          const long long qoff = __shfl_sync(0xffffffffu, poff, qi);
          if (g < gc) {
            const int n = sh.cnt[0][g];
            if (n == 0) continue;
            const int kp = sh.kpq[g];
            unsigned long long* out = a.part + qoff + qbase;
            if ((a.dbg & 16) && lane == 0) {
              atomicAdd(&g_scan_cnt[0], (unsigned long long)n);
              atomicAdd(&g_scan_cnt[1], 1ull);
            }
            if (n <= kp) {
              for (int b = lane; b < n; b += 32) out[b] = sb[g * kApp + b];
            } else {
              for (int b = 0; b < n; b += 32) list_fold32<KL>(L[qi], b + lane < n ? sb[g * kApp + b + lane] : TRI_KEY_MAX, lane);
#pragma unroll
              for (int j = 0; j < KL; ++j)
                if (j * 32 < kp) out[j * 32 + lane] = L[qi][j];
            }
          }
        }
        if (threadIdx.x == 64) ts_mark(a, 15);
        return acc | (aphase << 8);
      }
      // overflow: start over with the per-chunk selection (counts cleared)
      if (e < N) sh.cnt[0][e] = 0;
      epi_sync();
    }
  }
  for (int c = 0; c < nchunk; ++c) {
    const int buf = a.abufs == 2 ? (c & 1) : 0;
    const int rows = min(kTcRows, w.row_count - c * kTcRows);
    if (a.gthr && lane == 0 && !(a.dbg & 32)) {  // issued before the TMEM wait: the L2 round trip overlaps it
#pragma unroll
      for (int qi = 0; qi < OWN; ++qi) {
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
    if (c == 0 && threadIdx.x == 64) ts_mark(a, 5);
    uint32_t v[QPT];
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * N + half * QPT);
    tmem_ld_cols<QPT>(taddr, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) tmb_arrive(&sh.tempty[acc]);
    if (++acc == tc_acc<N>()) {
      acc = 0;
      aphase ^= 1;
    }
    if (a.dbg & 1) continue;
    if (valid) {
      // distances and a survivor mask first (no side effects: the loop
      // pipelines), then the rare survivors' exact key test and append.  The
      // fp32 test !(d > ord2f(thr's high word)) admits a superset of
      // key < thr (ties on the distance bits, -0 vs +0, NaN, thr = MAX).
      const uint32_t pos = (uint32_t)row;
      unsigned long long* sb = sel + (size_t)buf * N * kTcRows;
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        const int g = half * QPT + j;
        const float dot = H ? __uint_as_float(v[j]) * sh.qinv[g] : __uint_as_float(v[j]);
        const float d = __fmaf_rn(-2.f, dot, __fadd_rn(sh.qn[g], xn));
        v[j] = __float_as_uint(d);
        const float tf = ord2f((uint32_t)(thr[g] >> 32));
        m |= (uint32_t)(!(d > tf) && g < gc) << j;
      }
      if (m) {
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
          if (m & (1u << j)) {
            const int g = half * QPT + j;
            const unsigned long long key = make_key(__uint_as_float(v[j]), pos);
            if (key < thr[g]) {
              sb[g * kTcRows + atomicAdd(&sh.cnt[buf][g], 1)] = key;  // <= 128 per chunk
              sh.anyapp[c & 1] = 1;
            }
          }
        }
      }
    }
    epi_sync();
    if (a.dbg & 64) continue;
    // single append buffer: skip the owners' pass over a chunk nobody appended
    // to (slot c & 1 is reset between the two barriers of chunk c + 1)
    if (a.abufs == 1) {
      const bool any = sh.anyapp[c & 1] != 0;
      if (threadIdx.x == 64) sh.anyapp[(c + 1) & 1] = 0;  // between this chunk's barriers: untouched
      if (!any) {
        epi_sync();
        continue;
      }
    }
#pragma unroll
    for (int qi = 0; qi < OWN; ++qi) {
      const int g = ew + kEpiWarps * qi;
      if (g < gc) {
        const int n = sh.cnt[buf][g];
        if ((a.dbg & 16) && lane == 0 && n > 0) {
          atomicAdd(&g_scan_cnt[0], (unsigned long long)n);
          atomicAdd(&g_scan_cnt[1], 1ull);
          if (N != kTcGroupWide && sh.kpq[g] >= 128) {  // list scan: the wide (prefill) members' share
            atomicAdd(&g_scan_cnt[2], (unsigned long long)n);
            atomicAdd(&g_scan_cnt[3], 1ull);
          }
        }
        const unsigned long long* sb = sel + (size_t)buf * N * kTcRows + g * kTcRows;
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
        // early pool entry: the first chunk's winners (published once; the
        // item's end adds its best rows beyond this chunk)
        if (N != kTcGroupWide && c == 0 && a.pool && a.pool_pub >= 2 && n > 0 && sh.kpq[g] >= a.pool_minkp)
          pool_publish<KL>(a, sh.qid[g], sh.kpq[g], L[qi], lane, 0u);
      }
    }
    if (a.abufs == 1) epi_sync();  // single append buffer: drained before the next chunk appends
  }
#pragma unroll
  for (int qi = 0; qi < OWN; ++qi) {
    const int g = ew + kEpiWarps * qi;
    if (g < gc) {
      unsigned long long* out = a.part + a.members[w.member_begin + g].slot;
      if (a.compact_cnt) {  // cross-item seed (overflow fallback): append to the compact region
        int base = 0;
        if (lane == 0) base = atomicAdd(a.compact_cnt + sh.qid[g], sh.kpq[g]);
        out = a.part + a.meta[sh.qid[g]].part_off + __shfl_sync(0xffffffffu, base, 0);
      }
#pragma unroll
      for (int j = 0; j < KL; ++j)
        if (j * 32 < sh.kpq[g]) out[j * 32 + lane] = L[qi][j];  // the member's kp entries
      if (N != kTcGroupWide && a.pool && sh.kpq[g] >= a.pool_minkp)
        pool_publish<KL>(a, sh.qid[g], sh.kpq[g], L[qi], lane,
                         a.pool_pub >= 2 ? (uint32_t)(w.row_begin + kTcRows) : 0u);
    }
  }
  return acc | (aphase << 8);
}

// Epilogue: 8 warps (256 threads); see tc_epi_item for the TMEM mapping.
template <bool H, int N>
__device__ void tc_epilogue(const ScanLaunch& a, TcSmem<N>& sh, unsigned long long* sel) {
  const int e = threadIdx.x - 64;  // 0..255
  const int lane = threadIdx.x & 31;
  int ring = 0;
  ItemRing r;
  WorkItem w;
  while (next_item(sh, r, w, lane)) {
    const int gc = w.member_count;
    if (e < N) {
      const int q = e < gc ? a.members[w.member_begin + e].q : -1;
      sh.cnt[0][e] = 0;
      sh.cnt[1][e] = 0;
      sh.thr[e] = (a.gthr && q >= 0) ? __ldcg(a.gthr + q) : TRI_KEY_MAX;
      sh.qid[e] = q < 0 ? 0 : q;
      sh.kpq[e] = q >= 0 ? a.members[w.member_begin + e].pad : kMinKp;
      sh.qn[e] = q >= 0 ? a.qnorm[q] : 0.f;
      sh.qinv[e] = (H && q >= 0) ? a.qinv[q] : 0.f;
      sh.smin[e] = 0xffffffffu;
      if (e < 2) sh.anyapp[e] = 0;
    }
    epi_sync();
    if constexpr (N == kTcGroupWide) {  // brute force: kp <= kTcWideMaxKp
      switch (w.kp) {
        case 32: ring = tc_epi_item<H, N, 1>(a, w, sh, sel, ring); break;
        default: ring = tc_epi_item<H, N, 2>(a, w, sh, sel, ring); break;  // 64
      }
    } else {
      switch (w.kp) {
        case 32: ring = tc_epi_item<H, N, 1>(a, w, sh, sel, ring); break;
        case 64: ring = tc_epi_item<H, N, 2>(a, w, sh, sel, ring); break;
        case 128: ring = tc_epi_item<H, N, 4>(a, w, sh, sel, ring); break;
        default: ring = tc_epi_item<H, N, 8>(a, w, sh, sel, ring); break;  // 256 (host caps tc kp at kTcMaxKp)
      }
    }
    epi_sync();  // counters and append buffers are free for the next item
  }
  if (threadIdx.x == 64) ts_mark(a, 7);
}

template <bool H, int N>
__global__ void __launch_bounds__(kTcThreads, 1) scan_tc_kernel(const __grid_constant__ CUtensorMap map,
                                                                const __grid_constant__ CUtensorMap tail,
                                                                const __grid_constant__ CUtensorMap qmap, ScanLaunch a) {
  // programmatic dependent launch: the previous kernel's results are visible
  // after griddepcontrol.wait.  An early launch (a.early) defers the wait to
  // the roles that read them, so the setup and the row stream overlap the prep.
  if (!a.early) pdl_wait();
  else asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  constexpr int kTmemCols = tc_acc<N>() * N;  // power of two >= 32
  extern __shared__ __align__(1024) unsigned char tsmem_raw[];
  __shared__ TcSmem<N> sh;
  unsigned char* base = tsmem_raw + ((1024u - (tsu32(tsmem_raw) & 1023u)) & 1023u);
  unsigned char* ring = base;
  unsigned char* qs = ring + (size_t)a.stages * kTcSlabBytes;
  const int qtile_bytes = tc_nslab(row_bytes_of<H>(a)) * N * kTcRowB;
  unsigned long long* sel = reinterpret_cast<unsigned long long*>(qs + (size_t)a.qbufs * qtile_bytes);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) ts_mark(a, 0);
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
    for (int s = 0; s < tc_acc<N>(); ++s) {
      tmb_init(&sh.tfull[s], 1);
      tmb_init(&sh.tempty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tsu32(&sh.tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) ts_mark(a, 1);
  if (warp == 0) {
    // rows and a fixed (host-uploaded) item assignment do not depend on the prep
    if (a.early && a.seed != 2) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if ((threadIdx.x & 31) == 0) tc_producer<H, N>(a, &map, &tail, sh, ring);
  } else if (warp == 1) {
    tc_mma<H, N>(a, sh, ring, qs, qtile_bytes);
  } else if (warp == 10) {
    if (a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the prepared query tile
    tc_qstage<H, N>(a, &qmap, sh, qs, qtile_bytes);
  } else {
    if (a.early) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // norms, bounds, counters
    tc_epilogue<H, N>(a, sh, sel);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(sh.tmem_base), "n"(kTmemCols));
  }
}

template <bool H, int N>
cudaError_t launch_tc(const ScanLaunch& s, cudaStream_t st) {
  if (s.stages < kTcMinStages || s.stages > kTcMaxStages) return cudaErrorInvalidValue;
  if (s.qbufs < 1 || s.qbufs > 2 || s.abufs < 1 || s.abufs > 2) return cudaErrorInvalidValue;
  const size_t smem =
      tc_fixed_smem(H ? s.qldh * 2 : s.qld * 4, s.qbufs, s.abufs, N) + (size_t)s.stages * kTcSlabBytes;
  cudaError_t e = cudaFuncSetAttribute(scan_tc_kernel<H, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const CUtensorMap* qm = reinterpret_cast<const CUtensorMap*>(s.q_tma ? s.tmap_q : s.tmap_tc);
  if (s.early) {
    const long long saved = g_pdl;
    g_pdl = 1;
    (void)launch_pdl(scan_tc_kernel<H, N>, s.grid, kTcThreads, smem, st, *reinterpret_cast<const CUtensorMap*>(s.tmap_tc),
                     *reinterpret_cast<const CUtensorMap*>(s.tmap_tc_tail), *qm, s);
    g_pdl = saved;
    return cudaGetLastError();
  }
  (void)launch_pdl(scan_tc_kernel<H, N>, s.grid, kTcThreads, smem, st, *reinterpret_cast<const CUtensorMap*>(s.tmap_tc),
                                                         *reinterpret_cast<const CUtensorMap*>(s.tmap_tc_tail), *qm, s);
  return cudaGetLastError();
}

cudaError_t read_scan_ts(unsigned long long* out, int n) {
  if (n == 4) {  // the dbg & 16 counters (read and reset)
    cudaError_t e = cudaMemcpyFromSymbol(out, g_scan_cnt, sizeof(g_scan_cnt));
    unsigned long long z[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_scan_cnt, z, sizeof(z));
    return e;
  }
  return cudaMemcpyFromSymbol(out, g_scan_ts, sizeof(unsigned long long) * std::min(n, kTsCtas * kTsSlots));
}

cudaError_t launch_scan_tc(const ScanLaunch& s, cudaStream_t st) {
  if (s.nq == kTcGroupWide) return s.f16 ? launch_tc<true, kTcGroupWide>(s, st) : launch_tc<false, kTcGroupWide>(s, st);
  return s.f16 ? launch_tc<true, kTcGroup>(s, st) : launch_tc<false, kTcGroup>(s, st);
}

}  // namespace tri
