// One-process multi-GPU collectives for the single-call drop-in
// `power_urv(a, ..., ngpus=N)` (one process, one host thread per GPU,
// ncclCommInitAll).  The reference has no multi-GPU path (it is NumPy on one host);
// this is the plumbing of the row-sharded PowerURV in distributed.py when it runs
// under one Python process instead of torchrun.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): inside a PyTorch process
// that is torch's own NCCL (already loaded, matched by soname), elsewhere the
// system one.  The library itself therefore loads on machines without NCCL; only
// these entry points report URV_NCCL_ERROR there.
#include "common.cuh"
#include "../../include/urv_b200.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <vector>

namespace urv {
namespace {

struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.CommInitAll, "ncclCommInitAll");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.AllGather, "ncclAllGather");
    sym(api.ReduceScatter, "ncclReduceScatter");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    api.ok = api.CommInitAll && api.CommDestroy && api.GetErrorString && api.AllReduce && api.Broadcast &&
             api.AllGather && api.ReduceScatter && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  if (!api.ok) {
    set_error("NCCL (libnccl.so.2) is not available in this process");
    throw CudaFailure{kNcclError};
  }
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    set_error("%s: %s", what, nccl().GetErrorString(r));
    throw CudaFailure{kNcclError};
  }
}

template <class F>
int nccl_guarded(F&& fn) {
  try {
    fn();
    return kOk;
  } catch (const CudaFailure& f) {
    return f.status;
  } catch (...) {
    set_error("unexpected host exception in the NCCL wrapper");
    return kNcclError;
  }
}

ncclComm_t as_comm(void* c) { return static_cast<ncclComm_t>(c); }
cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// dst(:, j) = src(:, idx[j]) (by_rows = 0) or dst(i, :) = src(idx[i], :) (by_rows = 1),
// column-major.  One pass that packs the blocks of a layout change into the contiguous
// per-peer order of an all-to-all send buffer (or unpacks a receive buffer).
__global__ void gather_kernel(const double* __restrict__ src, long long lds, long long rows, long long cols,
                              const long long* __restrict__ idx, int by_rows, double* __restrict__ dst,
                              long long ldd) {
  const long long total = rows * cols;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = t % rows, c = t / rows;
    const long long sr = by_rows ? idx[r] : r, sc = by_rows ? c : idx[c];
    dst[r + c * ldd] = src[sr + sc * lds];
  }
}

}  // namespace
}  // namespace urv

extern "C" {

int urv_gather_f64(const double* src, int64_t lds, int64_t rows, int64_t cols, const int64_t* idx, int by_rows,
                   double* dst, int64_t ldd, void* stream) {
  return urv::nccl_guarded([&] {
    if (rows <= 0 || cols <= 0) return;
    const long long total = static_cast<long long>(rows) * cols;
    const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    urv::gather_kernel<<<grid, 256, 0, urv::as_stream(stream)>>>(src, lds, rows, cols,
                                                                 reinterpret_cast<const long long*>(idx), by_rows,
                                                                 dst, ldd);
    URV_CHECK_LAUNCH();
  });
}

int urv_nccl_available(void) {
  try {
    (void)urv::nccl();
    return 1;
  } catch (...) {
    return 0;
  }
}

int urv_nccl_init_all(int ndev, const int* devices, void** comms) {
  return urv::nccl_guarded([&] {
    if (ndev < 1) {
      urv::set_error("urv_nccl_init_all: ndev must be >= 1");
      throw urv::CudaFailure{urv::kInvalid};
    }
    std::vector<ncclComm_t> c(ndev);
    urv::nccl_check(urv::nccl().CommInitAll(c.data(), ndev, devices), "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i) comms[i] = c[i];
  });
}

int urv_nccl_destroy(void* comm) {
  return urv::nccl_guarded([&] { urv::nccl_check(urv::nccl().CommDestroy(urv::as_comm(comm)), "ncclCommDestroy"); });
}

int urv_nccl_all_reduce_f64(void* comm, const double* send, double* recv, int64_t count, void* stream) {
  return urv::nccl_guarded([&] {
    urv::nccl_check(urv::nccl().AllReduce(send, recv, static_cast<size_t>(count), ncclFloat64, ncclSum,
                                          urv::as_comm(comm), urv::as_stream(stream)),
                    "ncclAllReduce");
  });
}

int urv_nccl_broadcast_f64(void* comm, double* buf, int64_t count, int root, void* stream) {
  return urv::nccl_guarded([&] {
    urv::nccl_check(urv::nccl().Broadcast(buf, buf, static_cast<size_t>(count), ncclFloat64, root,
                                          urv::as_comm(comm), urv::as_stream(stream)),
                    "ncclBroadcast");
  });
}

int urv_nccl_all_gather_f64(void* comm, const double* send, double* recv, int64_t count, void* stream) {
  return urv::nccl_guarded([&] {
    urv::nccl_check(urv::nccl().AllGather(send, recv, static_cast<size_t>(count), ncclFloat64, urv::as_comm(comm),
                                          urv::as_stream(stream)),
                    "ncclAllGather");
  });
}

int urv_nccl_reduce_scatter_f64(void* comm, const double* send, double* recv, int64_t count, void* stream) {
  return urv::nccl_guarded([&] {
    urv::nccl_check(urv::nccl().ReduceScatter(send, recv, static_cast<size_t>(count), ncclFloat64, ncclSum,
                                              urv::as_comm(comm), urv::as_stream(stream)),
                    "ncclReduceScatter");
  });
}

int urv_nccl_all_to_all_f64(void* comm, int nranks, const double* send, const int64_t* send_counts,
                            const int64_t* send_displs, double* recv, const int64_t* recv_counts,
                            const int64_t* recv_displs, void* stream) {
  return urv::nccl_guarded([&] {
    const auto& api = urv::nccl();
    urv::nccl_check(api.GroupStart(), "ncclGroupStart");
    try {
      for (int p = 0; p < nranks; ++p) {
        if (send_counts[p] > 0)
          urv::nccl_check(api.Send(send + send_displs[p], static_cast<size_t>(send_counts[p]), ncclFloat64, p,
                                   urv::as_comm(comm), urv::as_stream(stream)),
                          "ncclSend");
        if (recv_counts[p] > 0)
          urv::nccl_check(api.Recv(recv + recv_displs[p], static_cast<size_t>(recv_counts[p]), ncclFloat64, p,
                                   urv::as_comm(comm), urv::as_stream(stream)),
                          "ncclRecv");
      }
    } catch (...) {
      api.GroupEnd();
      throw;
    }
    urv::nccl_check(api.GroupEnd(), "ncclGroupEnd");
  });
}

}  // extern "C"
