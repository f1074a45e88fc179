// Shared device helpers for the Trinity B200 search library (sm_100a).
//
// Candidate keys.  Every approximate candidate is a 64-bit key
//   (order-preserving bits of the fp32 approximate distance) << 32 | position
// so "smaller key" == "smaller (approx distance, position)".  TRI_KEY_MAX is the
// empty slot.  Exact results use (fp64 distance, global id) pairs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define TRI_KEY_MAX 0xFFFFFFFFFFFFFFFFull
#define TRI_THREADS 256

namespace tri {

// Programmatic dependent launch (launch_pdl): a kernel's CTAs may start while
// the previous kernel on the stream is finishing; griddepcontrol.wait blocks
// until that kernel has completed and its writes are visible, and
// launch_dependents lets the NEXT kernel begin launching as soon as every CTA
// of this one is running.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float ord2f(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(b);
}

__device__ __forceinline__ unsigned long long make_key(float d, uint32_t pos) {
  return ((unsigned long long)f2ord(d) << 32) | (unsigned long long)pos;
}

__device__ __forceinline__ uint32_t key_pos(unsigned long long k) { return (uint32_t)(k & 0xffffffffull); }
__device__ __forceinline__ float key_dist(unsigned long long k) { return ord2f((uint32_t)(k >> 32)); }

// Squared L2 distance in float64 between an fp64 query and an fp32 row, in the
// exact operation order of numpy's einsum("ij,ij->i") on float64 (the
// reference's rowwise_sq_dists, ann_graph.py:97-105): two lanes, blocks of 8
// elements whose 2-lane sub-blocks run in reverse order, unfused mul then add,
// a 2-lane tail, lane0 + lane1.  Intrinsics keep nvcc from contracting to DFMA.
// Result is bit-identical to the reference.
__device__ __forceinline__ double exact_sq_dist(const double* __restrict__ q, const float* __restrict__ x, int d) {
  double l0 = 0.0, l1 = 0.0;
  int i = 0;
  for (; i + 8 <= d; i += 8) {
#pragma unroll
    for (int sub = 3; sub >= 0; --sub) {
      double t0 = __dsub_rn(q[i + 2 * sub], (double)x[i + 2 * sub]);
      double t1 = __dsub_rn(q[i + 2 * sub + 1], (double)x[i + 2 * sub + 1]);
      l0 = __dadd_rn(__dmul_rn(t0, t0), l0);
      l1 = __dadd_rn(__dmul_rn(t1, t1), l1);
    }
  }
  for (; i < d; i += 2) {
    double t0 = __dsub_rn(q[i], (double)x[i]);
    l0 = __dadd_rn(__dmul_rn(t0, t0), l0);
    if (i + 1 < d) {
      double t1 = __dsub_rn(q[i + 1], (double)x[i + 1]);
      l1 = __dadd_rn(__dmul_rn(t1, t1), l1);
    }
  }
  return __dadd_rn(l0, l1);
}

// Squared L2 in the reference's float64 order (exact_sq_dist) with 16-byte loads: per 8-element block two float4 of the
// row and four double2 of the query, then sub-blocks 3..0, unfused mul/add.
__device__ __forceinline__ double exact_sq_dist_v4(const double* __restrict__ q, const float* __restrict__ x, int d) {
  double l0 = 0.0, l1 = 0.0;
  int i = 0;
#pragma unroll 4
  for (; i + 8 <= d; i += 8) {
    const float4 lo = *reinterpret_cast<const float4*>(x + i);
    const float4 hi = *reinterpret_cast<const float4*>(x + i + 4);
    const double2 q0 = *reinterpret_cast<const double2*>(q + i);
    const double2 q1 = *reinterpret_cast<const double2*>(q + i + 2);
    const double2 q2 = *reinterpret_cast<const double2*>(q + i + 4);
    const double2 q3 = *reinterpret_cast<const double2*>(q + i + 6);
    const double a6 = __dsub_rn(q3.x, (double)hi.z), a7 = __dsub_rn(q3.y, (double)hi.w);
    const double a4 = __dsub_rn(q2.x, (double)hi.x), a5 = __dsub_rn(q2.y, (double)hi.y);
    const double a2 = __dsub_rn(q1.x, (double)lo.z), a3 = __dsub_rn(q1.y, (double)lo.w);
    const double a0 = __dsub_rn(q0.x, (double)lo.x), a1 = __dsub_rn(q0.y, (double)lo.y);
    l0 = __dadd_rn(__dmul_rn(a6, a6), l0);
    l1 = __dadd_rn(__dmul_rn(a7, a7), l1);
    l0 = __dadd_rn(__dmul_rn(a4, a4), l0);
    l1 = __dadd_rn(__dmul_rn(a5, a5), l1);
    l0 = __dadd_rn(__dmul_rn(a2, a2), l0);
    l1 = __dadd_rn(__dmul_rn(a3, a3), l1);
    l0 = __dadd_rn(__dmul_rn(a0, a0), l0);
    l1 = __dadd_rn(__dmul_rn(a1, a1), l1);
  }
  for (; i < d; i += 2) {
    const double t0 = __dsub_rn(q[i], (double)x[i]);
    l0 = __dadd_rn(__dmul_rn(t0, t0), l0);
    if (i + 1 < d) {
      const double t1 = __dsub_rn(q[i + 1], (double)x[i + 1]);
      l1 = __dadd_rn(__dmul_rn(t1, t1), l1);
    }
  }
  return __dadd_rn(l0, l1);
}

// Vectorised when the query row is 16-byte aligned and d even (double2 loads).
__device__ __forceinline__ double exact_sq_dist_any(const double* __restrict__ q, const float* __restrict__ x, int d) {
  return ((d & 1) == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(x)) & 15) == 0)
             ? exact_sq_dist_v4(q, x, d)
             : exact_sq_dist(q, x, d);
}

// Exact result entry ordered by (dist, id) -- the reference tie rule
// (ann_graph.py:8-9, lexsort at :136).
struct Exact {
  double d;
  long long id;
};

__device__ __forceinline__ bool exact_less(const Exact& a, const Exact& b) {
  return a.d < b.d || (a.d == b.d && a.id < b.id);
}

__device__ __forceinline__ Exact exact_max() {
  Exact e;
  e.d = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  e.id = 0x7fffffffffffffffll;
  return e;
}

// ---------------------------------------------------------------------------
// In-shared-memory bitonic sorts (ascending).  n must be a power of two.

template <typename T, typename Less>
__device__ __forceinline__ void bitonic_pass(T* a, int n, int k, int j, int t, int nt, Less less) {
  for (int i = t; i < (n >> 1); i += nt) {
    int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
    int hi = lo + j;
    bool up = (lo & k) == 0;
    T x = a[lo], y = a[hi];
    bool swap = up ? less(y, x) : less(x, y);
    if (swap) {
      a[lo] = y;
      a[hi] = x;
    }
  }
}

template <typename T, typename Less>
__device__ void warp_sort(T* a, int n, int lane, Less less) {
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      bitonic_pass(a, n, k, j, lane, 32, less);
      __syncwarp();
    }
}

template <typename T, typename Less>
__device__ void block_sort(T* a, int n, Less less) {
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      bitonic_pass(a, n, k, j, threadIdx.x, blockDim.x, less);
      __syncthreads();
    }
}

struct KeyLess {
  __device__ __forceinline__ bool operator()(unsigned long long a, unsigned long long b) const { return a < b; }
};
struct ExactLess {
  __device__ __forceinline__ bool operator()(const Exact& a, const Exact& b) const { return exact_less(a, b); }
};

// ---------------------------------------------------------------------------
// Warp-register bitonic networks.  A sorted list of 32*KL keys lives in a warp
// as v[j] on lane l = element j*32 + l.

__device__ __forceinline__ unsigned long long kmin(unsigned long long x, unsigned long long y) { return x < y ? x : y; }
__device__ __forceinline__ unsigned long long kmax(unsigned long long x, unsigned long long y) { return x < y ? y : x; }

// Sort 32 keys (one per lane) ascending.
__device__ __forceinline__ unsigned long long warp_sort32(unsigned long long x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, j);
      x = (((lane & k) == 0) == ((lane & j) == 0)) ? kmin(x, y) : kmax(x, y);
    }
  return x;
}

// Sort a bitonic register list ascending (all compare-exchanges ascending).
template <int KL>
__device__ __forceinline__ void bitonic_merge_regs(unsigned long long (&v)[KL], int lane) {
#pragma unroll
  for (int dj = KL / 2; dj >= 1; dj >>= 1)
#pragma unroll
    for (int j = 0; j < KL; ++j)
      if ((j & dj) == 0) {
        const unsigned long long lo = kmin(v[j], v[j + dj]), hi = kmax(v[j], v[j + dj]);
        v[j] = lo;
        v[j + dj] = hi;
      }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1)
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, v[j], d);
      v[j] = (lane & d) ? kmax(v[j], y) : kmin(v[j], y);
    }
}

// v (sorted, 32*KL keys) <- smallest 32*KL of v U {x (sorted, one per lane)}, sorted:
// bitonic split of v's last 32 against the reversed batch, then a bitonic merge.
template <int KL>
__device__ __forceinline__ void list_merge32(unsigned long long (&v)[KL], unsigned long long x, int lane) {
  v[KL - 1] = kmin(v[KL - 1], __shfl_sync(0xffffffffu, x, 31 - lane));
  bitonic_merge_regs<KL>(v, lane);
}

// v (sorted, 32*KL distinct keys) <- smallest 32*KL of v U {x}: x lands at
// pos = #{v < x}, the tail shifts up one (a no-op when pos == 32*KL).  A few
// shuffles per key instead of a 32-wide sort + merge: the fold for chunks that
// admit only a handful of candidates.
template <int KL>
__device__ __forceinline__ void list_insert(unsigned long long (&v)[KL], unsigned long long x, int lane) {
  int pos = 0;
#pragma unroll
  for (int j = 0; j < KL; ++j) pos += __popc(__ballot_sync(0xffffffffu, v[j] < x));
  unsigned long long carry = 0;
#pragma unroll
  for (int j = 0; j < KL; ++j) {
    unsigned long long up = __shfl_up_sync(0xffffffffu, v[j], 1);
    const unsigned long long last = __shfl_sync(0xffffffffu, v[j], 31);
    if (lane == 0) up = carry;
    const int i = j * 32 + lane;
    v[j] = i < pos ? v[j] : (i == pos ? x : up);
    carry = last;
  }
}

// Fold up to 32 candidates (one per lane, TRI_KEY_MAX = none) into the sorted
// list: by insertion when at most kInsMax of them beat the list's last key,
// else by sort + bitonic merge.
constexpr int kInsMax = 8;
template <int KL>
__device__ __forceinline__ void list_fold32(unsigned long long (&v)[KL], unsigned long long x, int lane) {
  const unsigned long long kth = __shfl_sync(0xffffffffu, v[KL - 1], 31);
  unsigned m = __ballot_sync(0xffffffffu, x < kth);
  if (__popc(m) <= kInsMax) {
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      list_insert<KL>(v, __shfl_sync(0xffffffffu, x, src), lane);
    }
  } else {
    list_merge32<KL>(v, warp_sort32(x, lane), lane);
  }
}

// v (sorted) <- smallest 32*KL of v U p where p is a sorted list of the same
// size given REVERSED (p_rev[j] on lane l = p[KP-1 - (j*32+l)]).
template <int KL>
__device__ __forceinline__ void list_merge_rev(unsigned long long (&v)[KL], const unsigned long long (&p_rev)[KL],
                                               int lane) {
#pragma unroll
  for (int j = 0; j < KL; ++j) v[j] = kmin(v[j], p_rev[j]);
  bitonic_merge_regs<KL>(v, lane);
}

__host__ __device__ __forceinline__ int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace tri
