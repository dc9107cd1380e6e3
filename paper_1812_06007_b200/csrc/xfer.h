// Host <-> HBM transfers of pageable matrices through pinned staging (xfer.cu).
#pragma once
#include "common.cuh"

namespace urv {

// Column-major rows x cols: pageable host src (ld lds) -> device dst (ld ldd), on stream cs.
// Returns once every chunk has been handed to the DMA engine (the copies may still run on cs).
void h2d_staged(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                cudaStream_t cs);
// device src -> pageable host dst; returns when dst is complete.
void d2h_staged(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                cudaStream_t cs);

// The same, ordered with stream st (H2D: st's later work waits; D2H: starts after st's
// pending work).  Both block the calling thread until the host side is done.
void h2d_ordered(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                 cudaStream_t st);
void d2h_ordered(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                 cudaStream_t st);

// D2H on a worker thread once `ready` has fired: the caller keeps enqueueing GPU
// work.  join() waits and rethrows a failure as CudaFailure.
class AsyncD2H {
 public:
  AsyncD2H(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
           cudaEvent_t ready, int device);
  ~AsyncD2H();
  AsyncD2H(const AsyncD2H&) = delete;
  AsyncD2H& operator=(const AsyncD2H&) = delete;
  void join();

 private:
  struct Impl;
  Impl* impl_;
};

}  // namespace urv
