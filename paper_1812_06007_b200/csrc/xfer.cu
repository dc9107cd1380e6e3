// Host <-> HBM transfers of pageable NumPy matrices through pinned staging.
//
// A pageable cudaMemcpy runs at ~11 GB/s on this box and blocks the calling
// thread; registering the caller's pages (cudaHostRegister) costs more than it
// saves for a single 2 GB matrix.  Instead the matrix moves in column chunks
// through a small ring of pinned buffers that is allocated once per process:
// the host side of chunk k (a memcpy split over several threads) overlaps the
// DMA of chunk k-1.  Transfers run on their own stream; the D2H side is driven
// by a worker thread so the caller keeps enqueueing GPU work meanwhile.
#include "xfer.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace urv {

namespace {

constexpr int NBUF = 3;

size_t chunk_bytes() {
  static const size_t v = [] {
    const char* e = getenv("URV_XFER_CHUNK_MB");
    const long mb = e ? atol(e) : 32;
    return static_cast<size_t>(std::max(1L, mb)) << 20;
  }();
  return v;
}

int copy_threads() {
  static const int v = [] {
    const char* e = getenv("URV_XFER_THREADS");
    const int t = e ? atoi(e) : 8;
    return std::max(1, std::min(t, 32));
  }();
  return v;
}

// One ring of pinned buffers; a process keeps a few and hands them out (two
// transfers can be in flight at once: an output D2H and the next one).
struct Ring {
  void* buf[NBUF] = {nullptr, nullptr, nullptr};
  cudaEvent_t done[NBUF] = {nullptr, nullptr, nullptr};  // events belong to `device`
  size_t bytes = 0;
  int device = 0;
};

std::mutex g_ring_mu;
std::vector<Ring*> g_free_rings[64];  // per device

Ring* acquire_ring() {
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    auto& pool = g_free_rings[dev & 63];
    if (!pool.empty()) {
      Ring* r = pool.back();
      pool.pop_back();
      return r;
    }
  }
  Ring* r = new Ring;
  r->bytes = chunk_bytes();
  r->device = dev;
  for (int i = 0; i < NBUF; ++i) {
    URV_CUDA(cudaHostAlloc(&r->buf[i], r->bytes, cudaHostAllocPortable));
    URV_CUDA(cudaEventCreateWithFlags(&r->done[i], cudaEventDisableTiming));
  }
  return r;
}

void release_ring(Ring* r) {
  for (int i = 0; i < NBUF; ++i) cudaEventSynchronize(r->done[i]);
  std::lock_guard<std::mutex> lk(g_ring_mu);
  g_free_rings[r->device & 63].push_back(r);
}

// dst/src column blocks: copy nc columns of `rows` doubles between two strided
// layouts, split over threads by columns (or by rows for a single wide column).
void host_copy(double* dst, long long ldd, const double* src, long long lds, long long rows, long long nc) {
  const int T = copy_threads();
  const long long total = rows * nc;
  if (T == 1 || total * 8 < (4 << 20)) {
    for (long long c = 0; c < nc; ++c) memcpy(dst + c * ldd, src + c * lds, static_cast<size_t>(rows) * 8);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  if (ldd == rows && lds == rows) {  // contiguous: split the flat range
    const long long per = (total + T - 1) / T;
    for (int t = 0; t < T; ++t) {
      const long long lo = t * per, hi = std::min(total, lo + per);
      if (lo >= hi) break;
      th.emplace_back([=] { memcpy(dst + lo, src + lo, static_cast<size_t>(hi - lo) * 8); });
    }
  } else {
    const long long per = (nc + T - 1) / T;
    for (int t = 0; t < T; ++t) {
      const long long lo = t * per, hi = std::min(nc, lo + per);
      if (lo >= hi) break;
      th.emplace_back([=] {
        for (long long c = lo; c < hi; ++c) memcpy(dst + c * ldd, src + c * lds, static_cast<size_t>(rows) * 8);
      });
    }
  }
  for (auto& t : th) t.join();
}

}  // namespace

void h2d_staged(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                cudaStream_t cs) {
  if (rows <= 0 || cols <= 0) return;
  Ring* r = acquire_ring();
  const long long cpc = std::max(1LL, static_cast<long long>(r->bytes / (rows * 8)));
  if (cpc < 1 || static_cast<size_t>(rows * 8) > r->bytes) {  // a single column larger than a chunk
    release_ring(r);
    URV_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, rows * 8, cols, cudaMemcpyHostToDevice, cs));
    return;
  }
  int k = 0;
  for (long long c0 = 0; c0 < cols; c0 += cpc, ++k) {
    const int s = k % NBUF;
    const long long nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaEventSynchronize(r->done[s]));  // the DMA that last read this buffer is done
    host_copy(static_cast<double*>(r->buf[s]), rows, src + c0 * lds, lds, rows, nc);
    URV_CUDA(cudaMemcpy2DAsync(dst + c0 * ldd, ldd * 8, r->buf[s], rows * 8, rows * 8, nc, cudaMemcpyHostToDevice,
                               cs));
    URV_CUDA(cudaEventRecord(r->done[s], cs));
  }
  release_ring(r);
}

void d2h_staged(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                cudaStream_t cs) {
  if (rows <= 0 || cols <= 0) return;
  Ring* r = acquire_ring();
  const long long cpc = std::max(1LL, static_cast<long long>(r->bytes / (rows * 8)));
  if (static_cast<size_t>(rows * 8) > r->bytes) {
    release_ring(r);
    URV_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, src, lds * 8, rows * 8, cols, cudaMemcpyDeviceToHost, cs));
    URV_CUDA(cudaStreamSynchronize(cs));
    return;
  }
  const long long nchunks = (cols + cpc - 1) / cpc;
  auto issue = [&](long long k) {
    const int s = static_cast<int>(k % NBUF);
    const long long c0 = k * cpc, nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaMemcpy2DAsync(r->buf[s], rows * 8, src + c0 * lds, lds * 8, rows * 8, nc, cudaMemcpyDeviceToHost,
                               cs));
    URV_CUDA(cudaEventRecord(r->done[s], cs));
  };
  for (long long k = 0; k < std::min<long long>(NBUF, nchunks); ++k) issue(k);
  for (long long k = 0; k < nchunks; ++k) {
    const int s = static_cast<int>(k % NBUF);
    const long long c0 = k * cpc, nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaEventSynchronize(r->done[s]));
    host_copy(dst + c0 * ldd, ldd, static_cast<const double*>(r->buf[s]), rows, rows, nc);
    if (k + NBUF < nchunks) issue(k + NBUF);
  }
  release_ring(r);
}

// Ordered with `st`: the copy starts after st's pending work (D2H) and st's later
// work waits for it (H2D).  Blocking on the host.
namespace {
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t e = nullptr;
  explicit SideStream(cudaStream_t st) {
    URV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    URV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    URV_CUDA(cudaEventRecord(e, st));
    URV_CUDA(cudaStreamWaitEvent(s, e, 0));
  }
  ~SideStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    if (e) cudaEventDestroy(e);
  }
};
}  // namespace

void h2d_ordered(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                 cudaStream_t st) {
  SideStream ss(st);
  h2d_staged(dst, ldd, src, lds, rows, cols, ss.s);
  URV_CUDA(cudaEventRecord(ss.e, ss.s));
  URV_CUDA(cudaStreamWaitEvent(st, ss.e, 0));
}

void d2h_ordered(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                 cudaStream_t st) {
  SideStream ss(st);
  d2h_staged(dst, ldd, src, lds, rows, cols, ss.s);
}

// ---- asynchronous D2H: a worker thread waits for `ready`, then copies ----
struct AsyncD2H::Impl {
  std::thread th;
  cudaStream_t cs = nullptr;
  int status = 0;
  char err[512] = {0};
};

AsyncD2H::AsyncD2H(double* dst, long long ldd, const double* src, long long lds, long long rows, long long cols,
                   cudaEvent_t ready, int device)
    : impl_(new Impl) {
  URV_CUDA(cudaStreamCreateWithFlags(&impl_->cs, cudaStreamNonBlocking));
  URV_CUDA(cudaStreamWaitEvent(impl_->cs, ready, 0));
  Impl* im = impl_;
  im->th = std::thread([=] {
    try {
      URV_CUDA(cudaSetDevice(device));
      d2h_staged(dst, ldd, src, lds, rows, cols, im->cs);
      URV_CUDA(cudaStreamSynchronize(im->cs));
    } catch (const CudaFailure& f) {
      im->status = f.status;
      snprintf(im->err, sizeof(im->err), "%s", last_error());
    } catch (...) {
      im->status = kCudaError;
      snprintf(im->err, sizeof(im->err), "output copy failed");
    }
  });
}

void AsyncD2H::join() {
  if (!impl_) return;
  if (impl_->th.joinable()) impl_->th.join();
  if (impl_->cs) {
    cudaStreamDestroy(impl_->cs);
    impl_->cs = nullptr;
  }
  const int st = impl_->status;
  if (st) {
    set_error("%s", impl_->err);
    delete impl_;
    impl_ = nullptr;
    throw CudaFailure{st};
  }
  delete impl_;
  impl_ = nullptr;
}

AsyncD2H::~AsyncD2H() {
  if (!impl_) return;
  if (impl_->th.joinable()) impl_->th.join();
  if (impl_->cs) cudaStreamDestroy(impl_->cs);
  delete impl_;
}

}  // namespace urv
