// dist.cu -- multi-GPU C-ABI (include/ctproj_b200.h, "multi-GPU" section):
// view-sharded SF back projection fused with the cross-rank reduction.
//
// north_star item 4 / SURVEY.md 8(e): every rank back-projects its view shard
// into a full-size partial volume; the partial volumes are summed so that rank
// r ends up owning z-slab r.  Instead of one blocking reduce-scatter after the
// whole back projection, the partial volume is produced in z-chunks
// (CTP_BACK_ZCHUNK slices = one back-kernel z-block) and each finished chunk
// is reduced to the ranks owning its slices (ncclReduce, grouped) on the
// communicator's own stream while the next chunk is being back-projected.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): inside a torch
// process this returns the copy torch already loaded (2.28.x), standalone it
// is the system library.  Only nccl.h's types are used at compile time.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "plan_internal.h"
#include "sf_launch.h"

using ctp_internal::cuda_fail;
using ctp_internal::DeviceGuard;
using ctp_internal::fail;

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string error;
  bool ok = false;
};

NcclApi load_nccl() {
  NcclApi a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return a;
  }
#define CTP_SYM(field, name)                                         \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));     \
  if (!a.field) {                                                    \
    a.error = std::string("libnccl.so.2 lacks ") + name;             \
    return a;                                                        \
  }
  CTP_SYM(get_unique_id, "ncclGetUniqueId")
  CTP_SYM(comm_init_rank, "ncclCommInitRank")
  CTP_SYM(comm_destroy, "ncclCommDestroy")
  CTP_SYM(reduce, "ncclReduce")
  CTP_SYM(group_start, "ncclGroupStart")
  CTP_SYM(group_end, "ncclGroupEnd")
  CTP_SYM(error_string, "ncclGetErrorString")
#undef CTP_SYM
  a.ok = true;
  return a;
}

const NcclApi& nccl() {
  static const NcclApi api = load_nccl();
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  return fail(CTP_ERR_CUDA, std::string(where) + ": " + nccl().error_string(r));
}

size_t align_up(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace

struct ctp_dist {
  ncclComm_t comm;
  int nranks, rank, device;
  cudaStream_t comm_stream;        // reductions run here, overlapped with the back projection
  std::vector<cudaEvent_t> chunk;  // chunk c of the partial volume is complete
  cudaEvent_t done;                // every reduction of the call has completed
};

extern "C" {

int ctp_dist_unique_id(unsigned char* id, size_t id_bytes) {
  if (!id || id_bytes < sizeof(ncclUniqueId)) return fail(CTP_ERR_INVALID_ARGUMENT, "id buffer too small (128 bytes)");
  if (!nccl().ok) return fail(CTP_ERR_CUDA, nccl().error);
  ncclUniqueId u;
  const ncclResult_t r = nccl().get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return CTP_OK;
}

int ctp_dist_create(const unsigned char* id, size_t id_bytes, int nranks, int rank, int device, ctp_dist** out) {
  if (!out) return fail(CTP_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (!id || id_bytes < sizeof(ncclUniqueId)) return fail(CTP_ERR_INVALID_ARGUMENT, "id buffer too small (128 bytes)");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CTP_ERR_INVALID_ARGUMENT, "bad rank / nranks");
  if (!nccl().ok) return fail(CTP_ERR_CUDA, nccl().error);
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  ctp_dist* d = new ctp_dist();
  d->nranks = nranks;
  d->rank = rank;
  cudaGetDevice(&d->device);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = nccl().comm_init_rank(&d->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete d;
    return nccl_fail(r, "ncclCommInitRank");
  }
  cudaError_t e = cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    nccl().comm_destroy(d->comm);
    delete d;
    return cuda_fail(e, "ctp_dist_create");
  }
  *out = d;
  return CTP_OK;
}

int ctp_dist_destroy(ctp_dist* d) {
  if (!d) return CTP_OK;
  DeviceGuard guard(d->device);
  cudaStreamSynchronize(d->comm_stream);
  if (nccl().ok) nccl().comm_destroy(d->comm);
  for (cudaEvent_t e : d->chunk) cudaEventDestroy(e);
  cudaEventDestroy(d->done);
  cudaStreamDestroy(d->comm_stream);
  delete d;
  return CTP_OK;
}

int ctp_dist_slab(const ctp_plan* plan, const ctp_dist* d, int rank, int* z_first, int* z_count) {
  if (!plan || !d || rank < 0 || rank >= d->nranks) return fail(CTP_ERR_INVALID_ARGUMENT, "bad arguments");
  const int nz = plan->gp.nz;
  const int S = (nz + d->nranks - 1) / d->nranks;
  if (z_first) *z_first = rank * S;
  if (z_count) *z_count = S;
  return CTP_OK;
}

size_t ctp_sf_back_sharded_workspace_bytes(const ctp_plan* plan, const ctp_dist* d, int batch) {
  if (!plan || !d || batch < 1) return 0;
  // transposed sinogram shard + the full partial volume
  return align_up(plan->sino_elems * sizeof(float) * (size_t)batch) +
         align_up(plan->vol_elems * sizeof(float) * (size_t)batch);
}

int ctp_sf_back_sharded(const ctp_plan* plan, ctp_dist* d, const float* sino, float* slab, int batch,
                        void* workspace, size_t workspace_bytes, void* stream) {
  if (!plan || !d) return fail(CTP_ERR_INVALID_ARGUMENT, "plan / dist is null");
  if (!sino || !slab) return fail(CTP_ERR_INVALID_ARGUMENT, "null data pointer");
  if (batch < 1) return fail(CTP_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (!plan->sf_ok) return fail(CTP_ERR_UNSUPPORTED_GEOMETRY, "SF does not support this geometry");
  const size_t need = ctp_sf_back_sharded_workspace_bytes(plan, d, batch);
  if (!workspace || workspace_bytes < need)
    return fail(CTP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  if (plan->device != d->device) return fail(CTP_ERR_INVALID_ARGUMENT, "plan and communicator on different devices");
  if (!nccl().ok) return fail(CTP_ERR_CUDA, nccl().error);
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const ctp::GridParams& gp = plan->gp;
  const int nz = gp.nz;
  const size_t plane = (size_t)gp.nx * gp.ny;
  const int S = (nz + d->nranks - 1) / d->nranks;
  float* yT = static_cast<float*>(workspace);
  float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) +
                                         align_up(plan->sino_elems * sizeof(float) * (size_t)batch));
  const int zch = CTP_BACK_ZCHUNK;
  const int nchunks = (nz + zch - 1) / zch;
  while ((int)d->chunk.size() < nchunks) {
    cudaEvent_t e;
    cudaError_t ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaEventCreate");
    d->chunk.push_back(e);
  }
  // the previous call's reductions read `part` of the caller's last workspace;
  // the caller's stream already waits for them (see the end of this function)
  cudaError_t e = ctp::launch_back_input(sino, yT, gp.nr, gp.nc, batch * gp.nv, s);
  if (e != cudaSuccess) return cuda_fail(e, "transpose_segscan_kernel");
  // slab rows past nz (the last owner's padding) are zero
  const int pad0 = nz - d->rank * S;  // first padded row of this rank's slab
  if (pad0 < S) {
    for (int b = 0; b < batch; ++b) {
      const int r0 = pad0 > 0 ? pad0 : 0;
      e = cudaMemsetAsync(slab + ((size_t)b * S + r0) * plane, 0, (size_t)(S - r0) * plane * sizeof(float), s);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(slab padding)");
    }
  }
  for (int c = 0; c < nchunks; ++c) {
    const int z0 = c * zch, z1 = z0 + zch < nz ? z0 + zch : nz;
    e = ctp::launch_back(gp, plan->d_coef, plan->d_ax, yT, part, batch, false, s, z0, z1);
    if (e != cudaSuccess) return cuda_fail(e, "sf_back_kernel (z-chunk)");
    e = cudaEventRecord(d->chunk[c], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d->comm_stream, d->chunk[c], 0);
    if (e != cudaSuccess) return cuda_fail(e, "chunk event");
    // reduce every owner's share of this chunk to its owner (same order on every rank)
    ncclResult_t r = nccl().group_start();
    for (int o = z0 / S; r == ncclSuccess && o < d->nranks && o * S < z1; ++o) {
      const int a = z0 > o * S ? z0 : o * S;
      const int bnd = z1 < (o + 1) * S ? z1 : (o + 1) * S;
      if (a >= bnd) continue;
      for (int b = 0; b < batch && r == ncclSuccess; ++b) {
        const float* src = part + ((size_t)b * nz + a) * plane;
        float* dst = o == d->rank ? slab + ((size_t)b * S + (a - o * S)) * plane : const_cast<float*>(src);
        r = nccl().reduce(src, dst, (size_t)(bnd - a) * plane, ncclFloat32, ncclSum, o, d->comm, d->comm_stream);
      }
    }
    const ncclResult_t r2 = nccl().group_end();
    if (r != ncclSuccess) return nccl_fail(r, "ncclReduce");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  }
  e = cudaEventRecord(d->done, d->comm_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, d->done, 0);
  if (e != cudaSuccess) return cuda_fail(e, "completion event");
  return CTP_OK;
}

}  // extern "C"
