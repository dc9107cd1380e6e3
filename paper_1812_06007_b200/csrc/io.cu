// Streaming file <-> HBM transfer for the reference's URVK1 binary format
// (io.py:42-71: magic "URVK1", two little-endian u64 dims, then column-major
// little-endian float64).  The header is parsed by the caller (Python, so the
// reference's error messages are reproduced verbatim); these routines move the
// payload in column blocks through pinned staging buffers, overlapping pread /
// pwrite with the H2D / D2H copies, so a matrix never has to exist in host RAM
// as a whole (the 34 GB config-5 input).
#include "io.h"

#include "dgemm.h"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace urv {

namespace {

constexpr int NSTAGE = 3;

size_t chunk_bytes() {
  static const size_t v = [] {
    const char* e = getenv("URV_IO_CHUNK_MB");  // test hook: small chunks exercise the pipeline
    const long mb = e ? atol(e) : 64;
    return static_cast<size_t>(std::max(1L, mb)) << 20;
  }();
  return v;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

struct Staging {
  void* buf[NSTAGE] = {nullptr, nullptr, nullptr};
  cudaEvent_t done[NSTAGE] = {nullptr, nullptr, nullptr};
  explicit Staging(size_t bytes) {
    for (int i = 0; i < NSTAGE; ++i) {
      URV_CUDA(cudaHostAlloc(&buf[i], bytes, cudaHostAllocDefault));
      URV_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < NSTAGE; ++i) {
      if (done[i]) {
        cudaEventSynchronize(done[i]);
        cudaEventDestroy(done[i]);
      }
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};

bool full_pread(int fd, void* dst, size_t n, off_t off) {
  auto* p = static_cast<unsigned char*>(dst);
  while (n > 0) {
    const ssize_t r = pread(fd, p, n, off);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    n -= static_cast<size_t>(r);
    off += r;
  }
  return true;
}

bool full_pwrite(int fd, const void* src, size_t n, off_t off) {
  auto* p = static_cast<const unsigned char*>(src);
  while (n > 0) {
    const ssize_t r = pwrite(fd, p, n, off);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    p += r;
    n -= static_cast<size_t>(r);
    off += r;
  }
  return true;
}

}  // namespace

// rows x cols column-major float64 from `path` at byte `offset` into device dst (ld ldd).
void read_file_to_device(const char* path, long long offset, long long rows, long long cols, double* dst,
                         long long ldd, cudaStream_t st) {
  if (rows < 0 || cols < 0 || ldd < std::max(rows, 1LL) || offset < 0) {
    set_error("read_file_to_device: bad shape rows=%lld cols=%lld ld=%lld", rows, cols, ldd);
    throw CudaFailure{kInvalid};
  }
  if (rows == 0 || cols == 0) return;
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) {
    set_error("%s: cannot open (%s)", path, strerror(errno));
    throw CudaFailure{kInvalid};
  }
  struct stat sb;
  if (fstat(f.fd, &sb) != 0 || sb.st_size < offset + rows * cols * 8) {
    set_error("%s: file holds fewer than %lld entries after byte %lld", path, rows * cols, offset);
    throw CudaFailure{kInvalid};
  }
  const long long col_bytes = rows * 8;
  const long long cpc = std::max(1LL, static_cast<long long>(chunk_bytes()) / col_bytes);  // columns per chunk
  const size_t stage_bytes = static_cast<size_t>(std::min(cpc, cols) * col_bytes);
  Staging sg(stage_bytes);
  int k = 0;
  for (long long c0 = 0; c0 < cols; c0 += cpc, ++k) {
    const int s = k % NSTAGE;
    const long long nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaEventSynchronize(sg.done[s]));  // the copy that last used this buffer has landed
    if (!full_pread(f.fd, sg.buf[s], static_cast<size_t>(nc * col_bytes), offset + c0 * col_bytes)) {
      set_error("%s: read failed at column %lld (%s)", path, c0, strerror(errno));
      throw CudaFailure{kInvalid};
    }
    URV_CUDA(cudaMemcpy2DAsync(dst + c0 * ldd, ldd * 8, sg.buf[s], col_bytes, col_bytes, nc,
                               cudaMemcpyHostToDevice, st));
    URV_CUDA(cudaEventRecord(sg.done[s], st));
  }
  URV_CUDA(cudaStreamSynchronize(st));
}

// rows x cols column-major float64 from device src (ld lds) into `path` at byte
// `offset` (the file must exist; it is extended as needed).
void write_device_to_file(const char* path, long long offset, const double* src, long long rows, long long cols,
                          long long lds, cudaStream_t st) {
  if (rows < 0 || cols < 0 || lds < std::max(rows, 1LL) || offset < 0) {
    set_error("write_device_to_file: bad shape rows=%lld cols=%lld ld=%lld", rows, cols, lds);
    throw CudaFailure{kInvalid};
  }
  if (rows == 0 || cols == 0) return;
  Fd f;
  f.fd = open(path, O_WRONLY);
  if (f.fd < 0) {
    set_error("%s: cannot open for writing (%s)", path, strerror(errno));
    throw CudaFailure{kInvalid};
  }
  const long long col_bytes = rows * 8;
  const long long cpc = std::max(1LL, static_cast<long long>(chunk_bytes()) / col_bytes);
  const size_t stage_bytes = static_cast<size_t>(std::min(cpc, cols) * col_bytes);
  Staging sg(stage_bytes);
  const long long nchunks = (cols + cpc - 1) / cpc;
  // issue up to NSTAGE copies ahead, write each chunk once its copy has landed
  auto issue = [&](long long k) {
    const int s = static_cast<int>(k % NSTAGE);
    const long long c0 = k * cpc, nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaMemcpy2DAsync(sg.buf[s], col_bytes, src + c0 * lds, lds * 8, col_bytes, nc, cudaMemcpyDeviceToHost,
                               st));
    URV_CUDA(cudaEventRecord(sg.done[s], st));
  };
  for (long long k = 0; k < std::min<long long>(NSTAGE, nchunks); ++k) issue(k);
  for (long long k = 0; k < nchunks; ++k) {
    const int s = static_cast<int>(k % NSTAGE);
    const long long c0 = k * cpc, nc = std::min(cpc, cols - c0);
    URV_CUDA(cudaEventSynchronize(sg.done[s]));
    if (!full_pwrite(f.fd, sg.buf[s], static_cast<size_t>(nc * col_bytes), offset + c0 * col_bytes)) {
      set_error("%s: write failed at column %lld (%s)", path, c0, strerror(errno));
      throw CudaFailure{kInvalid};
    }
    if (k + NSTAGE < nchunks) issue(k + NSTAGE);
  }
}

}  // namespace urv
