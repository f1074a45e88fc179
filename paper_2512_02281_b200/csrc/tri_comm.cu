// Native sharded search over NCCL (C-ABI: tri_comm_*, tri_ivf_search_sharded).
//
// One call runs a vector-sharded IVF batch end to end on the caller's stream
// (BASELINE config C4): the local search writes ids then
// float64 distances into one [2, B, k] block, ONE ncclAllGather moves every
// rank's block (B*k*16 bytes each) over NVLink, and the exact (dist, id) merge
// (tri_merge_topk_ld) reads the gathered [G, 2, B, k] in place.  Every kernel
// and the collective are stream-ordered, so the whole call is CUDA-graph
// capturable.  NCCL is resolved at run time (dlopen of libnccl.so.2, reusing
// the copy torch already loaded when there is one), so the library keeps
// loading on machines without NCCL; the caller owns the communicator's
// lifetime (tri_comm_init / tri_comm_destroy) like the reference's single
// owner of a stepper.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <deque>
#include <mutex>
#include <vector>

#include "tri_internal.h"
#include "../../include/trinity_b200.h"

namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, when loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather && n.error_string;
  });
  return n;
}

}  // namespace

struct tri_comm {
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0, device = 0;
  std::mutex mu;
  struct Bufs {
    cudaStream_t st;
    int B, k;
    int64_t* local;  // [2, B, k]: ids, then distance bits
    int64_t* all;    // [world, 2, B, k]
  };
  std::deque<Bufs> bufs;  // stable addresses: other streams' calls may append meanwhile
};

#define NCCL_TRY(x)                                                                                        \
  do {                                                                                                    \
    ncclResult_t r_ = (x);                                                                                \
    if (r_ != ncclSuccess) return tri::set_error(TRI_ECUDA, "%s failed: %s", #x, nccl().error_string(r_)); \
  } while (0)
#define CUDA_TRY(x)                                                                                        \
  do {                                                                                                    \
    cudaError_t e_ = (x);                                                                                 \
    if (e_ != cudaSuccess) return tri::set_error(TRI_ECUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

int tri_comm_unique_id(uint8_t* id) {
  if (!id) return tri::set_error(TRI_EINVAL, "id is NULL");
  if (!nccl().ok) return tri::set_error(TRI_EINTERNAL, "libnccl.so.2 not found");
  ncclUniqueId u;
  NCCL_TRY(nccl().get_unique_id(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return TRI_OK;
}

int tri_comm_init(const uint8_t* id, int32_t world, int32_t rank, int32_t device, tri_comm** out) {
  if (!id || !out) return tri::set_error(TRI_EINVAL, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return tri::set_error(TRI_EINVAL, "rank %d / world %d", rank, world);
  if (!nccl().ok) return tri::set_error(TRI_EINTERNAL, "libnccl.so.2 not found");
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  CUDA_TRY(cudaSetDevice(device));
  tri_comm* c = new tri_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  const ncclResult_t r = nccl().comm_init_rank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return tri::set_error(TRI_ECUDA, "ncclCommInitRank failed: %s", nccl().error_string(r));
  }
  *out = c;
  return TRI_OK;
}

int tri_comm_destroy(tri_comm* c) {
  if (!c) return TRI_OK;
  cudaSetDevice(c->device);
  for (auto& b : c->bufs) {
    cudaStreamSynchronize(b.st);
    cudaFree(b.local);
    cudaFree(b.all);
  }
  if (c->comm) nccl().comm_destroy(c->comm);
  delete c;
  return TRI_OK;
}

int tri_ivf_search_sharded(tri_ivf* v, tri_comm* c, const double* q, int32_t B, int32_t k, const int32_t* nprobe,
                           int32_t ldo, int64_t* ids, double* dists, void* stream) {
  if (!v || !c) return tri::set_error(TRI_EINVAL, "NULL handle");
  if (B < 0 || k < 1 || ldo < k) return tri::set_error(TRI_EINVAL, "bad shape: B=%d k=%d ldo=%d", B, k, ldo);
  if (B == 0) return TRI_OK;
  if ((long long)c->world * k > 8192) return tri::set_error(TRI_EINVAL, "world * k = %lld exceeds 8192", (long long)c->world * k);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tri_comm::Bufs* b = nullptr;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& x : c->bufs)
      if (x.st == st && x.B == B && x.k == k) b = &x;
    if (!b) {
      tri_comm::Bufs nb{st, B, k, nullptr, nullptr};
      CUDA_TRY(cudaSetDevice(c->device));
      CUDA_TRY(cudaMalloc(&nb.local, (size_t)2 * B * k * sizeof(int64_t)));
      CUDA_TRY(cudaMalloc(&nb.all, (size_t)c->world * 2 * B * k * sizeof(int64_t)));
      c->bufs.push_back(nb);
      b = &c->bufs.back();
    }
  }
  std::vector<int32_t> ks(B, k);
  const long long bk = (long long)B * k;
  int rc = tri_ivf_search_dev(v, q, B, ks.data(), nprobe, k, b->local, reinterpret_cast<double*>(b->local + bk), stream);
  if (rc) return rc;
  NCCL_TRY(nccl().all_gather(b->local, b->all, (size_t)(2 * bk), ncclInt64, c->comm, st));
  return tri_merge_topk_ld(reinterpret_cast<const double*>(b->all + bk), b->all, c->world, B, k, k, 2 * bk, k, dists,
                           ids, ldo, stream);
}

}  // extern "C"
