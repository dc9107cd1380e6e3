// Internal interface of the FP64 GEMM engine and the shared device workspace.
#pragma once
#include "common.cuh"

#include <vector>

namespace urv {

// Growable, stream-ordered device scratch buffer (the library's memory pool).
class Workspace {
 public:
  explicit Workspace(cudaStream_t s = nullptr) : stream_(s) {}
  ~Workspace() { release(); }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  void set_stream(cudaStream_t s) { stream_ = s; }
  double* get(size_t doubles) {
    if (doubles > cap_) {
      release();
      dev_alloc(reinterpret_cast<void**>(&ptr_), doubles * sizeof(double), stream_);
      cap_ = doubles;
    }
    return ptr_;
  }
  void release() {
    if (ptr_) cudaFreeAsync(ptr_, stream_);
    ptr_ = nullptr;
    cap_ = 0;
  }

 private:
  cudaStream_t stream_;
  double* ptr_ = nullptr;
  size_t cap_ = 0;
};

// Device buffer owned by one call, freed stream-ordered.
struct DevBuf {
  double* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t doubles, cudaStream_t st) : s(st) {
    if (doubles) dev_alloc(reinterpret_cast<void**>(&p), doubles * sizeof(double), st);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (p) cudaFreeAsync(p, s);
      p = o.p;
      s = o.s;
      o.p = nullptr;
    }
    return *this;
  }
};

// C = alpha op(A) op(B) + beta C.  Column-major; lda/ldb must be even (TMA).
// Uses deterministic split-K through `ws` when the tile grid under-fills the GPU.
void dgemm(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
           long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
           cudaStream_t stream, Workspace& ws);

// Low level: with splits > 1 the k-range is split and partial product z is
// written to columns [z*P, z*P + N) of C, P = gemm_split_cols(N) (ld ldc);
// alpha/beta are ignored in that mode and the caller reduces the partials.
// C must be 16-byte aligned with an even ldc (TMA store).
void dgemm_launch(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
                  long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
                  cudaStream_t stream, int splits);

int gemm_splits_for(long long M, long long N, long long K);
// Column stride (in columns) between split-K partial blocks in the partial buffer.
inline long long gemm_split_cols(long long N) { return (N + 127) / 128 * 128; }
int gemm_effective_splits(long long K, int splits);

inline long long round_up(long long x, long long a) { return (x + a - 1) / a * a; }

}  // namespace urv
