// The multi-GPU search's single collective in the C ABI (SURVEY §8(b),(e)):
// rh_minloc_allreduce replaces the torch.distributed all-gather of
// search.distributed_best for callers without torch.  NCCL has no MINLOC,
// so every rank all-gathers the 16-byte (score bits, index) pairs over NCCL
// and one device thread reduces them with the lexicographic (score, index)
// rule -- identical on every rank, bit-exact fp64, no host round trip.
//
// NCCL is resolved at run time (dlsym in the process, else dlopen of
// libnccl.so.2): the library does not link it, so a process that already
// loaded an NCCL (torch's) keeps exactly one copy.
#include <dlfcn.h>
#include <nccl.h>

#include <math_constants.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = RTLD_DEFAULT;
    if (!dlsym(h, "ncclAllGather")) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather;
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const Nccl& n = nccl();
  rh::set_error("%s: %s", what, n.error_string ? n.error_string(r) : "NCCL error");
  return RH_E_CUDA;
}

int need_nccl() {
  if (nccl().ok) return RH_OK;
  rh::set_error("NCCL is not available (libnccl.so.2 not loaded and not loadable)");
  return RH_E_INVALID;
}

// (a, ia) < (b, ib) lexicographically; an index < 0 is "no candidate"
__device__ __forceinline__ bool lex_less_pair(double a, long long ia, double b, long long ib) {
  if (ia < 0) return false;
  if (ib < 0) return true;
  return a < b || (a == b && ia < ib);
}

__global__ void minloc_gathered_kernel(const unsigned long long* pairs, int world, double* score,
                                       long long* index) {
  double best = CUDART_INF_F;
  long long bi = -1;
  for (int r = 0; r < world; ++r) {
    const double s = __longlong_as_double((long long)pairs[2 * r]);
    const long long i = (long long)pairs[2 * r + 1];
    if (lex_less_pair(s, i, best, bi)) {
      best = s;
      bi = i;
    }
  }
  *score = bi < 0 ? CUDART_INF : best;
  *index = bi;
}

}  // namespace

extern "C" {

int rh_nccl_unique_id(uint8_t* id_out) {
  if (!id_out) {
    rh::set_error("rh_nccl_unique_id: NULL output");
    return RH_E_INVALID;
  }
  if (int rc = need_nccl()) return rc;
  ncclUniqueId id;
  if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return RH_OK;
}

int rh_nccl_comm_create(rh_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id,
                        void** comm_out) {
  if (!ctx || !id || !comm_out || world < 1 || rank < 0 || rank >= world) {
    rh::set_error("rh_nccl_comm_create: invalid arguments");
    return RH_E_INVALID;
  }
  if (int rc = need_nccl()) return rc;
  rh::DeviceGuard guard(ctx);
  ncclUniqueId uid;
  memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  if (ncclResult_t r = nccl().comm_init_rank(&comm, world, uid, rank))
    return nccl_fail(r, "ncclCommInitRank");
  *comm_out = comm;
  return RH_OK;
}

int rh_nccl_comm_destroy(void* comm) {
  if (!comm) return RH_OK;
  if (int rc = need_nccl()) return rc;
  if (ncclResult_t r = nccl().comm_destroy(static_cast<ncclComm_t>(comm)))
    return nccl_fail(r, "ncclCommDestroy");
  return RH_OK;
}

int rh_minloc_allreduce(rh_ctx* ctx, void* comm, int32_t world, double* score, int64_t* index,
                        void* stream) {
  if (!ctx || !comm || world < 1 || !score || !index) {
    rh::set_error("rh_minloc_allreduce: invalid arguments");
    return RH_E_INVALID;
  }
  if (int rc = need_nccl()) return rc;
  rh::DeviceGuard guard(ctx);
  cudaStream_t st = rh::as_stream(stream);
  // scratch: this rank's pair, then the gathered pairs
  void* ws = nullptr;
  if (int rc = rh::workspace(ctx, 16 * ((size_t)world + 1), &ws, 4, st)) return rc;
  unsigned long long* mine = static_cast<unsigned long long*>(ws);
  unsigned long long* all = mine + 2;
  RH_CUDA(cudaMemcpyAsync(mine, score, 8, cudaMemcpyDeviceToDevice, st));
  RH_CUDA(cudaMemcpyAsync(mine + 1, index, 8, cudaMemcpyDeviceToDevice, st));
  if (ncclResult_t r = nccl().all_gather(mine, all, 2, ncclUint64, static_cast<ncclComm_t>(comm),
                                         st))
    return nccl_fail(r, "ncclAllGather");
  minloc_gathered_kernel<<<1, 1, 0, st>>>(all, world, score, reinterpret_cast<long long*>(index));
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

}  // extern "C"
