// Exhaustive exact kNN for k beyond the candidate-scan capacity (k > TRI_MAX_K):
// brute_force_knn accepts any k <= N (ann_graph.py:131-133), including k = N
// (test_ann_graph.py:77-79 "full k is a permutation").  Every row's exact
// float64 distance in the reference's einsum order (exact_sq_dist_any), then a
// stable device radix sort of (distance bits, row) -- non-negative doubles
// order like their bit patterns and the rows enter in ascending order, so the
// result is the reference's lexsort((ids, dists)) order (ann_graph.py:136).
#include <cub/device/device_radix_sort.cuh>

#include "tri_common.cuh"
#include "tri_internal.h"

namespace tri {

__global__ void all_dists_kernel(const double* __restrict__ q, int d, const float* __restrict__ X, long long ldx,
                                 long long n, unsigned long long* __restrict__ keys, long long* __restrict__ rows) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double dd = exact_sq_dist_any(q, X + i * ldx, d);
    keys[i] = (unsigned long long)__double_as_longlong(dd);
    rows[i] = i;
  }
}

__global__ void take_k_kernel(const unsigned long long* __restrict__ keys, const long long* __restrict__ rows, int k,
                              int ldo, long long id_offset, long long* __restrict__ out_ids,
                              double* __restrict__ out_d) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ldo; j += gridDim.x * blockDim.x) {
    if (j < k) {
      out_ids[j] = rows[j] + id_offset;
      out_d[j] = __longlong_as_double((long long)keys[j]);
    } else {
      out_ids[j] = -1;
      out_d[j] = __longlong_as_double(0x7ff0000000000000ll);  // +inf past k
    }
  }
}

size_t exhaustive_scratch_bytes(long long n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const long long*)nullptr, (long long*)nullptr, (int)n);
  return 4 * (size_t)n * 8 + temp + 256;
}

cudaError_t launch_exhaustive_knn(const StoreView& sv, long long id_offset, const double* q64, int B, const int* k,
                                  int ldo, long long* ids, double* dists, void* scratch, cudaStream_t st) {
  const long long n = sv.n;
  unsigned long long* k0 = static_cast<unsigned long long*>(scratch);
  unsigned long long* k1 = k0 + n;
  long long* r0 = reinterpret_cast<long long*>(k1 + n);
  long long* r1 = r0 + n;
  void* temp = r1 + n;
  size_t temp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, k0, k1, r0, r1, (int)n, 0, 64, st);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<long long>((n + 255) / 256, 4 * 148);
  for (int b = 0; b < B; ++b) {
    all_dists_kernel<<<grid, 256, 0, st>>>(q64 + (long long)b * sv.d, sv.d, sv.X, sv.ldx, n, k0, r0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k0, k1, r0, r1, (int)n, 0, 64, st);
    if (e != cudaSuccess) return e;
    take_k_kernel<<<(ldo + 255) / 256, 256, 0, st>>>(k1, r1, k[b], ldo, id_offset, ids + (long long)b * ldo,
                                                     dists + (long long)b * ldo);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tri
