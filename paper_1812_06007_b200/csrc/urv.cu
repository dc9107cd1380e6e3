// PowerURV driver and the C ABI of liburv_b200.so (include/urv_b200.h).
//
// Mirrors the reference's `power_urv` (factorizations.py:104-145), `_orth`
// (:70-83) and `_powered_sample` (:86-101) operation for operation, with every
// numeric step on the GPU: GEMMs on the TMA+DMMA engine, QRs on the cooperative
// Householder panel + compact-WY GEMM updates, norms / finiteness / nonzero /
// rank-deficiency checks as fixed-order device reductions.  The host only moves
// buffers and turns the per-stage diagnostics into the reference's exceptions
// and warnings (Python side).
#include "common.cuh"
#include "dgemm.h"
#include "qr.h"
#include "profile.h"
#include "rng.h"
#include "svd.h"
#include "io.h"
#include "xfer.h"
#include "../../include/urv_b200.h"

#include <atomic>
#include <memory>
#include <cstdarg>
#include <thread>
#include <mutex>
#include <utility>
#include <vector>

namespace urv {

// ------------------------------- errors -------------------------------------
namespace {
thread_local char g_err[1024] = "";
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

// ------------------------------ launch counter ------------------------------
namespace {
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------ device info ---------------------------------
cudaMemPool_t lib_pool() {
  static cudaMemPool_t pools[64] = {nullptr};
  static std::once_flag flags[64];
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  std::call_once(flags[dev & 63], [dev] {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return;
    // Keep up to a fifth of the device's memory cached between calls (36 GB on a B200):
    // a repeated config-4 call with host buffers needs ~13 GB of scratch, and re-mapping
    // what a smaller threshold released cost 0.37 s per call (e2e 3.55 s at 8 GB vs 3.18 s
    // at 16 GB, profiles/r02_e2e_pool.log); the rest goes back to the driver at the call's
    // final synchronisation, and urv_release_memory() drops everything.
    const char* e = getenv("URV_POOL_KEEP_MB");
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t keep = e ? static_cast<uint64_t>(atoll(e)) << 20 : static_cast<uint64_t>(total_b / 5);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev & 63] = pool;
  });
  if (!pools[dev & 63]) {
    set_error("cannot create the memory pool of device %d", dev);
    throw CudaFailure{kCudaError};
  }
  return pools[dev & 63];
}

void dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  URV_CUDA(cudaMallocFromPoolAsync(p, bytes, lib_pool(), st));
}

void trim_pool() {
  URV_CUDA(cudaDeviceSynchronize());
  URV_CUDA(cudaMemPoolTrimTo(lib_pool(), 0));
}

const DeviceInfo& device_info() {
  static DeviceInfo infos[64];
  static std::once_flag flags[64];
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  std::call_once(flags[dev & 63], [dev] {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
      infos[dev & 63].sms = p.multiProcessorCount;
      infos[dev & 63].max_smem_optin = static_cast<int>(p.sharedMemPerBlockOptin);
    }
  });
  if (infos[dev & 63].sms == 0) {
    set_error("cannot query device %d", dev);
    throw CudaFailure{kCudaError};
  }
  return infos[dev & 63];
}

// ------------------------------ stats registry ------------------------------
namespace {
struct StatRec {
  int dev;
  int cls;
  double flops, bytes;
  cudaEvent_t e0, e1;
  cudaStream_t stream;
};
std::mutex g_stats_mu;
std::vector<StatRec> g_stats;
std::vector<cudaEvent_t> g_stats_free[64];  // recycled events per device: no cudaEventCreate per launch once warm
bool g_stats_on = false;

int stats_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}
cudaEvent_t stats_event() {
  {
    auto& fl = g_stats_free[stats_device()];
    std::lock_guard<std::mutex> lk(g_stats_mu);
    if (!fl.empty()) {
      cudaEvent_t e = fl.back();
      fl.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  return cudaEventCreate(&e) == cudaSuccess ? e : nullptr;
}
}  // namespace

StatsScope::StatsScope(cudaStream_t s, int c, double f, double b)
    : stream(s), cls(c), flops(f), bytes(b), ev0(nullptr) {
  if (!g_stats_on) return;
  cudaEvent_t e = stats_event();
  if (!e) return;
  cudaEventRecord(e, s);
  ev0 = e;
}
StatsScope::~StatsScope() {
  if (!ev0) return;
  cudaEvent_t e1 = stats_event();
  if (!e1) return;
  cudaEventRecord(e1, stream);
  std::lock_guard<std::mutex> lk(g_stats_mu);
  g_stats.push_back({stats_device(), cls, flops, bytes, static_cast<cudaEvent_t>(ev0), e1, stream});
}

// ------------------------------ small kernels -------------------------------
namespace {

constexpr int STATS_BLOCKS = 296;  // fixed: keeps the reduction order device-independent
constexpr int STATS_THREADS = 256;

// Pass 1: per-block {sum of squares, #non-finite, #nonzero} over a column-major matrix.
__global__ void __launch_bounds__(STATS_THREADS) matrix_stats_partial(const double* __restrict__ A, long long lda,
                                                                      int rows, int cols,
                                                                      double* __restrict__ part) {
  __shared__ double s0[STATS_THREADS / 32], s1[STATS_THREADS / 32], s2[STATS_THREADS / 32];
  double ss = 0.0, nf = 0.0, nz = 0.0;
  const long long total = static_cast<long long>(rows) * cols;
  for (long long idx = blockIdx.x * static_cast<long long>(STATS_THREADS) + threadIdx.x; idx < total;
       idx += static_cast<long long>(STATS_BLOCKS) * STATS_THREADS) {
    const double x = A[idx % rows + (idx / rows) * lda];
    ss += x * x;
    nf += isfinite(x) ? 0.0 : 1.0;
    nz += (x != 0.0) ? 1.0 : 0.0;  // NaN != 0 counts as nonzero, like ndarray.any()
  }
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s0[w] = ss;
    s1[w] = nf;
    s2[w] = nz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int i = 0; i < STATS_THREADS / 32; ++i) {
      a += s0[i];
      b += s1[i];
      c += s2[i];
    }
    part[3 * blockIdx.x + 0] = a;
    part[3 * blockIdx.x + 1] = b;
    part[3 * blockIdx.x + 2] = c;
  }
}

// Pass 2: fixed-order sum of the block partials into stage slot out[0..2].
__global__ void matrix_stats_final(const double* __restrict__ part, double* __restrict__ out) {
  const int lane = threadIdx.x;
  double a = 0, b = 0, c = 0;
  for (int i = lane; i < STATS_BLOCKS; i += 32) {
    a += part[3 * i];
    b += part[3 * i + 1];
    c += part[3 * i + 2];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    out[0] = a;
    out[1] = b;
    out[2] = c;
  }
}

void matrix_stats(const double* A, long long lda, long long rows, long long cols, double* slot, double* part,
                  cudaStream_t st) {
  StatsScope scope(st, kKAux, 0.0, 8.0 * rows * cols);
  matrix_stats_partial<<<STATS_BLOCKS, STATS_THREADS, 0, st>>>(A, lda, static_cast<int>(rows),
                                                                 static_cast<int>(cols), part);
  URV_CHECK_LAUNCH();
  matrix_stats_final<<<1, 32, 0, st>>>(part, slot);
  URV_CHECK_LAUNCH();
}

// out (cols x rows) = in^T, in column-major rows x cols.  32x32 smem tiles.
__global__ void transpose_kernel(const double* __restrict__ in, long long ldi, long long rows, long long cols,
                                 double* __restrict__ out, long long ldo) {
  __shared__ double tile[32][33];
  const long long r0 = blockIdx.x * 32LL;
  // column tiles are strided over gridDim.y (at most 65535): any number of columns
  for (long long c0 = blockIdx.y * 32LL; c0 < cols; c0 += gridDim.y * 32LL) {
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const long long r = r0 + threadIdx.x, c = c0 + k;
      if (r < rows && c < cols) tile[k][threadIdx.x] = in[r + c * ldi];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const long long c = c0 + threadIdx.x, r = r0 + k;  // out(c, r)
      if (r < rows && c < cols) out[c + r * ldo] = tile[threadIdx.x][k];
    }
    __syncthreads();
  }
}

void transpose(const double* in, long long ldi, long long rows, long long cols, double* out, long long ldo,
               cudaStream_t st) {
  StatsScope scope(st, kKAux, 0.0, 16.0 * rows * cols);
  const long long gx = (rows + 31) / 32, gy = std::min<long long>((cols + 31) / 32, 65535);
  if (gx > 0x7fffffffLL) {
    set_error("transpose: %lld rows exceed the grid", rows);
    throw CudaFailure{kInvalid};
  }
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(std::max<long long>(gy, 1)));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, ldi, rows, cols, out, ldo);
  URV_CHECK_LAUNCH();
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  bool owned = false;
  explicit StreamGuard(void* user) {
    if (user) {
      s = static_cast<cudaStream_t>(user);
    } else {
      URV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      owned = true;
    }
  }
  ~StreamGuard() {
    if (owned) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};


// Work that contains cooperative panel launches must never co-reside with other such
// work on one device (the panels' spin barriers need every CTA resident).  Calls that
// return before their work completes (the asynchronous device entry points below) are
// therefore chained per device by an event, in host issue order: each one's stream waits
// for the previous one's work and records its own completion.
struct PanelOrder {
  cudaStream_t s;
  cudaEvent_t ev = nullptr;
  explicit PanelOrder(cudaStream_t st) : s(st) {
    static std::mutex mu;
    static cudaEvent_t evs[64] = {nullptr};
    int dev = 0;
    URV_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!evs[dev & 63]) URV_CUDA(cudaEventCreateWithFlags(&evs[dev & 63], cudaEventDisableTiming));
    ev = evs[dev & 63];
    URV_CUDA(cudaStreamWaitEvent(s, ev, 0));
  }
  ~PanelOrder() {
    if (ev) cudaEventRecord(ev, s);
  }
};

// Fresh host output buffers (np.empty) are not yet backed by pages; faulting
// 6 GB in during the D2H copy costs more than the copy.  Touch them on host
// threads while the GPU computes (joined before the copies; URV_PREFAULT=0 disables).
struct PrefaultPages {
  std::vector<std::thread> th;
  PrefaultPages(std::initializer_list<std::pair<void*, size_t>> ranges) {
    static const bool on = [] {
      const char* e = getenv("URV_PREFAULT");
      return !(e && e[0] == '0');
    }();
    if (!on) return;
    for (auto& r : ranges) {
      if (!r.first || r.second < (16u << 20)) continue;
      const size_t parts = 4, chunk = (r.second + parts - 1) / parts;
      for (size_t k = 0; k < parts; ++k) {
        char* lo = static_cast<char*>(r.first) + k * chunk;
        const size_t len = std::min(chunk, r.second - std::min(r.second, k * chunk));
        if (len) th.emplace_back([lo, len] {
          for (size_t off = 0; off < len; off += 4096) reinterpret_cast<volatile char*>(lo)[off] = 0;
        });
      }
    }
  }
  void join() {
    for (auto& t : th) t.join();
    th.clear();
  }
  ~PrefaultPages() { join(); }
};

// Matrix handed to the library: pointer, storage shape and leading dimension.
struct Operand {
  const double* p;
  long long rows, cols, ld;  // column-major storage
};

// Make a device-resident column-major copy with an even leading dimension
// unless the input already qualifies.
const double* stage_in(const Operand& in, int on_device, DevBuf& holder, long long& ld_out, cudaStream_t st) {
  if (on_device && in.ld % 2 == 0 && (reinterpret_cast<uintptr_t>(in.p) % 16) == 0) {
    ld_out = in.ld;
    return in.p;
  }
  ld_out = round_up(in.rows, 8);
  holder = DevBuf(static_cast<size_t>(ld_out) * in.cols, st);
  if (on_device)
    URV_CUDA(cudaMemcpy2DAsync(holder.p, ld_out * 8, in.p, in.ld * 8, in.rows * 8, in.cols,
                               cudaMemcpyDeviceToDevice, st));
  else
    h2d_ordered(holder.p, ld_out, in.p, in.ld, in.rows, in.cols, st);  // pinned staging (xfer.cu)
  return holder.p;
}

// Output destination: a device buffer with even ld (the user's, when possible).
struct OutBuf {
  double* dev = nullptr;
  long long ld = 0;
  DevBuf tmp;
  double* user = nullptr;
  long long user_ld = 0;
  int user_on_device = 0;
  long long rows = 0, cols = 0;
  void init(double* u, long long uld, int on_dev, long long r, long long c, cudaStream_t st) {
    user = u;
    user_ld = uld;
    user_on_device = on_dev;
    rows = r;
    cols = c;
    if (on_dev && uld % 2 == 0 && (reinterpret_cast<uintptr_t>(u) % 16) == 0) {
      dev = u;
      ld = uld;
    } else {
      ld = round_up(r, 8);
      tmp = DevBuf(static_cast<size_t>(ld) * c, st);
      dev = tmp.p;
    }
  }
  void finish(cudaStream_t st) {
    if (dev == user) return;
    if (user_on_device)
      URV_CUDA(cudaMemcpy2DAsync(user, user_ld * 8, dev, ld * 8, rows * 8, cols, cudaMemcpyDeviceToDevice, st));
    else
      d2h_ordered(user, user_ld, dev, ld, rows, cols, st);  // pinned staging (xfer.cu)
  }
};

}  // namespace

// ------------------------------ PowerURV driver ------------------------------
namespace {

void power_urv_impl(const double* A, long long m, long long n, long long lda, int a_rowmajor, int a_on_device,
                    const double* G, long long ldg, int g_on_device, unsigned long long seed,
                    unsigned long long rstream, int q, int reorth, int skip_redundant,
                    double* U, long long ldu, double* R, long long ldr, double* V, long long ldv,
                    int out_on_device, double* stage_info, long long n_stages, void* user_stream) {
  if (m < 1 || n < 1 || m < n || q < 0) {
    set_error("invalid shape/q: m=%lld n=%lld q=%d", m, n, q);
    throw CudaFailure{kInvalid};
  }
  if (stage_info && n_stages < 2LL * q + 3) {
    set_error("stage_info needs %d stages", 2 * q + 3);
    throw CudaFailure{kInvalid};
  }
  StreamGuard sg(user_stream);
  cudaStream_t st = sg.s;
  PanelOrder panel_order(st);
  Workspace ws(st);

  // ---- inputs ----
  DevBuf a_hold, g_hold;
  long long lda_d = 0, ldg_d = 0;
  const Operand a_in{A, a_rowmajor ? n : m, a_rowmajor ? m : n, lda};
  PrefaultPages prefault({{out_on_device ? nullptr : U, static_cast<size_t>(ldu) * n * 8},
                          {out_on_device ? nullptr : R, static_cast<size_t>(ldr) * n * 8},
                          {out_on_device ? nullptr : V, static_cast<size_t>(ldv) * n * 8}});
  int device = 0;
  URV_CUDA(cudaGetDevice(&device));
  // Host A: staged H2D (pinned ring, multi-threaded host copies) on a copy stream,
  // driven by a helper thread so the Gaussian draw below overlaps it.
  const double* dA = nullptr;
  cudaStream_t cs_a = nullptr;
  cudaEvent_t a_landed = nullptr;
  std::thread a_copier;
  int a_copy_status = 0;
  char a_copy_err[512] = {0};
  if (a_on_device) {
    dA = stage_in(a_in, a_on_device, a_hold, lda_d, st);
  } else {
    lda_d = round_up(a_in.rows, 8);
    a_hold = DevBuf(static_cast<size_t>(lda_d) * a_in.cols, st);
    dA = a_hold.p;
    URV_CUDA(cudaStreamCreateWithFlags(&cs_a, cudaStreamNonBlocking));
    URV_CUDA(cudaEventCreateWithFlags(&a_landed, cudaEventDisableTiming));
    URV_CUDA(cudaEventRecord(a_landed, st));  // the allocation above is ordered on st
    URV_CUDA(cudaStreamWaitEvent(cs_a, a_landed, 0));
    a_copier = std::thread([&, device] {
      try {
        URV_CUDA(cudaSetDevice(device));
        h2d_staged(a_hold.p, lda_d, A, lda, a_in.rows, a_in.cols, cs_a);
      } catch (const CudaFailure& f) {
        a_copy_status = f.status;
        snprintf(a_copy_err, sizeof(a_copy_err), "%s", last_error());
      } catch (...) {
        a_copy_status = kCudaError;
      }
    });
  }
  auto a_join = [&] {  // A resident before its first use on st
    if (!a_copier.joinable()) return;
    a_copier.join();
    if (a_copy_status) {
      set_error("%s", a_copy_err);
      throw CudaFailure{a_copy_status};
    }
    URV_CUDA(cudaEventRecord(a_landed, cs_a));
    URV_CUDA(cudaStreamWaitEvent(st, a_landed, 0));
  };
  struct CopyStreamGuard {  // joins the copier and releases the copy stream on every exit path
    std::thread& t;
    cudaStream_t& s;
    cudaEvent_t& e;
    ~CopyStreamGuard() {
      if (t.joinable()) t.join();
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
      if (e) cudaEventDestroy(e);
    }
  } copy_guard{a_copier, cs_a, a_landed};
  const char opAY = a_rowmajor ? 'T' : 'N';    // A . Y
  const char opAtY = a_rowmajor ? 'N' : 'T';   // A^T . Y

  const long long ldm = round_up(m, 8);
  const long long ns = 2LL * q + 3;
  DevBuf info(static_cast<size_t>(URV_STAGE_FIELDS) * ns, st);
  DevBuf part(3 * STATS_BLOCKS, st);
  URV_CUDA(cudaMemsetAsync(info.p, 0, sizeof(double) * URV_STAGE_FIELDS * ns, st));
  auto slot = [&](long long s) { return info.p + URV_STAGE_FIELDS * s; };

  // Buffer plan: the output buffers double as work buffers, so one call needs
  // A, Z (the A.Y product / QR work matrix) and U, R, V only -- 5 matrices, which
  // is what lets the 65536^2 configuration run on one GPU.
  //   V buffer: Y (G, then every re-orthonormalised sample), finally V
  //   U buffer: Q(A.Y) during the power steps, finally U
  //   R buffer: A^T Q during the power steps, finally R
  OutBuf u_out, r_out, v_out;
  u_out.init(U, ldu, out_on_device, m, n, st);
  r_out.init(R, ldr, out_on_device, n, n, st);
  v_out.init(V, ldv, out_on_device, n, n, st);
  DevBuf Z(static_cast<size_t>(ldm) * n, st);
  struct Mat {
    double* p;
    long long ld;
  };
  Mat Y{v_out.dev, v_out.ld}, Y2{r_out.dev, r_out.ld};
  const Mat Qm{u_out.dev, u_out.ld};

  if (G) {
    URV_CUDA(cudaMemcpy2DAsync(Y.p, Y.ld * 8, G, ldg * 8, n * 8, n,
                               g_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  } else if (!gaussian_device(seed, rstream, n, n, Y.p, Y.ld, st)) {  // random.py:52-61 on the device
    set_error("device Gaussian draw could not be resolved; pass G");
    throw CudaFailure{kInvalid};
  }

  // stage 0: validated_matrix(a)  (core.py:47-54)
  a_join();
  matrix_stats(dA, lda_d, a_in.rows, a_in.cols, slot(0), part.p, st);
  {
    // validated_matrix rejects a non-finite A before any arithmetic (core.py:52-53):
    // read stage 0 back now and end the call (the caller raises from stage_info)
    // instead of running the whole factorisation on NaNs.  One early sync; the
    // GPU is idle for a launch latency at most.
    double s0[URV_STAGE_FIELDS];
    URV_CUDA(cudaMemcpyAsync(s0, slot(0), sizeof(s0), cudaMemcpyDeviceToHost, st));
    URV_CUDA(cudaStreamSynchronize(st));
    if (s0[1] > 0) {
      if (stage_info) {
        std::fill(stage_info, stage_info + URV_STAGE_FIELDS * ns, 0.0);
        std::copy(s0, s0 + URV_STAGE_FIELDS, stage_info);
      }
      return;
    }
  }

  // ---- _powered_sample: factorizations.py:86-101 ----
  // Implicit-Q form (default): Q(Z) is only ever used as A^T Q(Z) and Q(Y) only as
  // A Q(Y), so neither is formed.  A^T Q(Z) = ((H_Z^T A)(:n, :))^T applies the
  // compact-WY reflectors of Z to a copy of A from the left, and A Q(Y) =
  // (A H_Y)(:, :n) applies those of Y from the right: 2mn^2 flops per product in
  // place of dorgqr (4mn^2 - 4/3 n^3) + a 2mn^2 GEMM.  Same stages, same stats.
  static const int implicit_q = [] {  // 0: explicit Q, 1: fused (default), 2: unfused apply
    const char* e = getenv("URV_IMPLICIT_Q");
    return e ? atoi(e) : 1;
  }();
  auto copy_a = [&](double* dst, long long ldd) {  // column-major m x n copy of A
    if (a_rowmajor)
      transpose(dA, lda_d, n, m, dst, ldd, st);
    else
      URV_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, dA, lda_d * 8, m * 8, n, cudaMemcpyDeviceToDevice, st));
  };
  auto copy_at = [&](double* dst, long long ldd) {  // column-major n x m copy of A^T
    if (a_rowmajor)
      URV_CUDA(cudaMemcpy2DAsync(dst, ldd * 8, dA, lda_d * 8, n * 8, m, cudaMemcpyDeviceToDevice, st));
    else
      transpose(dA, lda_d, m, n, dst, ldd, st);
  };
  // V deferred (fused path, reference sequence without the redundant QR): the last
  // Y step also carries A^T, so A V arrives with the factorisation and V = Q(Y) is
  // formed on a low-priority side stream while the final QR runs.
  QrFactors fy_last;
  static const bool vdefer_on = [] {
    const char* e = getenv("URV_VDEFER");
    return !(e && e[0] == '0');
  }();
  const bool v_deferred = vdefer_on && reorth && implicit_q == 1 && q > 0 && skip_redundant;
  if (reorth && implicit_q == 1 && q > 0) {
    // Fused: the copy of A (resp. A^T) rides along as extra trailing columns of the
    // QR of Z (resp. Y), so the reflectors reach it block by block and the
    // latency-bound panels of the last blocks stay hidden under its update.
    //   Z step: [Z | A]   -> H_Z^T A,   A^T Q(Z) = ((H_Z^T A)(:n, :))^T
    //   Y step: [Y | A^T] -> H_Y^T A^T, A Q(Y)   = (H_Y^T A^T)^T  (H_Y is n x n)
    const long long lde = round_up(n, 2);
    DevBuf e_hold;
    double* Et = Qm.p;  // the U buffer is free during the Y step
    if (lde * m > Qm.ld * n) {
      e_hold = DevBuf(static_cast<size_t>(lde) * m, st);
      Et = e_hold.p;
    }
    QrFactors fy;
    for (int i = 0; i < q; ++i) {
      const long long s1 = 1 + 2LL * i, s2 = 2 + 2LL * i;
      if (i == 0) dgemm(opAY, 'N', m, n, n, 1.0, dA, lda_d, Y.p, Y.ld, 0.0, Z.p, ldm, st, ws);  // a @ G
      matrix_stats(Z.p, ldm, m, n, slot(s1), part.p, st);
      QrFactors fz;
      copy_a(Qm.p, Qm.ld);
      qr_factor(Z.p, ldm, m, n, slot(s1), slot(s1) + 3, st, ws, fz, Qm.p, Qm.ld, n);
      transpose(Qm.p, Qm.ld, n, n, Y2.p, Y2.ld, st);  // a.T @ Q(Z)
      matrix_stats(Y2.p, Y2.ld, n, n, slot(s2), part.p, st);
      if (i + 1 < q || v_deferred) {
        copy_at(Et, lde);
        qr_factor(Y2.p, Y2.ld, n, n, slot(s2), slot(s2) + 3, st, ws, fy, Et, lde, m);
        transpose(Et, lde, n, m, Z.p, ldm, st);  // next a @ Q(Y)  (after the loop: a @ v)
      } else {
        qr_factor(Y2.p, Y2.ld, n, n, slot(s2), slot(s2) + 3, st, ws, fy);
      }
    }
    if (v_deferred)
      fy_last = std::move(fy);
    else
      qr_form_q(fy, Y.p, Y.ld, st, ws);  // the last Q(Y) is V: form it explicitly
  } else if (reorth && implicit_q == 2 && q > 0) {  // the same products, applied after each factorisation
    QrFactors fy;
    for (int i = 0; i < q; ++i) {
      const long long s1 = 1 + 2LL * i, s2 = 2 + 2LL * i;
      if (i == 0) {
        dgemm(opAY, 'N', m, n, n, 1.0, dA, lda_d, Y.p, Y.ld, 0.0, Z.p, ldm, st, ws);
      } else {
        copy_a(Z.p, ldm);
        qr_apply_q_right(fy, Z.p, ldm, m, st, ws);  // (a H_Y)(:, :n)
      }
      matrix_stats(Z.p, ldm, m, n, slot(s1), part.p, st);
      QrFactors fz;
      qr_factor(Z.p, ldm, m, n, slot(s1), slot(s1) + 3, st, ws, fz);
      copy_a(Qm.p, Qm.ld);
      qr_apply_qt_left(fz, Qm.p, Qm.ld, n, st, ws);  // H_Z^T a
      transpose(Qm.p, Qm.ld, n, n, Y2.p, Y2.ld, st);
      matrix_stats(Y2.p, Y2.ld, n, n, slot(s2), part.p, st);
      qr_factor(Y2.p, Y2.ld, n, n, slot(s2), slot(s2) + 3, st, ws, fy);
    }
    qr_form_q(fy, Y.p, Y.ld, st, ws);
  } else if (reorth) {
    for (int i = 0; i < q; ++i) {
      const long long s1 = 1 + 2LL * i, s2 = 2 + 2LL * i;
      dgemm(opAY, 'N', m, n, n, 1.0, dA, lda_d, Y.p, Y.ld, 0.0, Z.p, ldm, st, ws);        // a @ y
      matrix_stats(Z.p, ldm, m, n, slot(s1), part.p, st);
      householder_qr_device(Z.p, ldm, m, n, Qm.p, Qm.ld, nullptr, 0, slot(s1), slot(s1) + 3, st, ws);
      dgemm(opAtY, 'N', n, n, m, 1.0, dA, lda_d, Qm.p, Qm.ld, 0.0, Y2.p, Y2.ld, st, ws);  // a.T @ y
      matrix_stats(Y2.p, Y2.ld, n, n, slot(s2), part.p, st);
      householder_qr_device(Y2.p, Y2.ld, n, n, Y.p, Y.ld, nullptr, 0, slot(s2), slot(s2) + 3, st, ws);
    }
  } else {
    for (int i = 0; i < q; ++i) {
      dgemm(opAY, 'N', m, n, n, 1.0, dA, lda_d, Y.p, Y.ld, 0.0, Z.p, ldm, st, ws);
      dgemm(opAtY, 'N', n, n, m, 1.0, dA, lda_d, Z.p, ldm, 0.0, Y2.p, Y2.ld, st, ws);
      std::swap(Y, Y2);
    }
    if (q > 0) matrix_stats(Y.p, Y.ld, n, n, slot(1), part.p, st);
  }

  // ---- v = _orth(y, "right-factor QR"): factorizations.py:142 ----
  const long long sr = 2LL * q + 1;
  cudaStream_t sv = st;  // where V is final
  Workspace wsv(nullptr);
  DevBuf part_v;
  cudaEvent_t v_done = nullptr;
  // V late (device outputs): V = Q(Y) is formed while the final QR runs its tail, where
  // the panel chain outlasts the trailing updates and the GEMM engine would idle, instead
  // of competing with the QR's big updates from its start; R is extracted after U then
  // (fy_last lives in the R buffer).  Host outputs keep the early V, whose D2H overlaps
  // the final QR.  URV_VLATE=0 disables.
  static const int vlate_blocks = [] {
    const char* e = getenv("URV_VLATE");
    return e ? atoi(e) : 24;
  }();
  // only when the final QR has more outer blocks than the tail: for small n the host's
  // launch enqueue is the bottleneck and the early V starts sooner (config 1/2 regressed)
  const bool v_late = v_deferred && out_on_device && vlate_blocks > 0 &&
                      ceil_div(n, outer_block_width(m, n)) > vlate_blocks;
  cudaEvent_t v_tail = nullptr;
  auto form_v = [&] {
    qr_form_q(fy_last, Y.p, Y.ld, sv, wsv);
    matrix_stats(Y.p, Y.ld, n, n, slot(sr), part_v.p, sv);
    URV_CUDA(cudaEventRecord(v_done, sv));  // fy_last (in the R buffer) is no longer read
  };
  if (v_deferred) {
    int lo_prio = 0, hi_prio = 0;
    URV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    URV_CUDA(cudaStreamCreateWithPriority(&sv, cudaStreamNonBlocking, lo_prio));
    URV_CUDA(cudaEventCreateWithFlags(&v_done, cudaEventDisableTiming));
    URV_CUDA(cudaEventRecord(v_done, st));
    URV_CUDA(cudaStreamWaitEvent(sv, v_done, 0));
    wsv.set_stream(sv);
    part_v = DevBuf(3 * STATS_BLOCKS, sv);
    if (v_late)
      URV_CUDA(cudaEventCreateWithFlags(&v_tail, cudaEventDisableTiming));
    else
      form_v();
  } else {
    matrix_stats(Y.p, Y.ld, n, n, slot(sr), part.p, st);
  }
  if (!(reorth && q > 0 && skip_redundant)) {
    // QR of Y into the other n x n buffer (Y2), then make sure V ends in the V buffer
    householder_qr_device(Y.p, Y.ld, n, n, Y2.p, Y2.ld, nullptr, 0, slot(sr), slot(sr) + 3, st, ws);
    std::swap(Y, Y2);
  }  // else: Y already has orthonormal columns (Householder Q), V = Q(Y) = Y up to rounding
  if (Y.p != v_out.dev)
    URV_CUDA(cudaMemcpy2DAsync(v_out.dev, v_out.ld * 8, Y.p, Y.ld * 8, n * 8, n, cudaMemcpyDeviceToDevice, st));

  // Host outputs leave through worker threads (staged D2H) as soon as each is final:
  // V overlaps the last GEMM + QR, R overlaps the explicit-Q formation.
  cudaEvent_t v_ready = nullptr, r_ready = nullptr, u_ready = nullptr;
  struct EventGuard {
    cudaEvent_t* e[3];
    ~EventGuard() {
      for (auto* p : e)
        if (*p) cudaEventDestroy(*p);
    }
  } ev_guard{{&v_ready, &r_ready, &u_ready}};
  std::unique_ptr<AsyncD2H> d2h_v, d2h_r;
  prefault.join();
  if (!out_on_device) {
    URV_CUDA(cudaEventCreateWithFlags(&v_ready, cudaEventDisableTiming));
    URV_CUDA(cudaEventCreateWithFlags(&r_ready, cudaEventDisableTiming));
    URV_CUDA(cudaEventCreateWithFlags(&u_ready, cudaEventDisableTiming));
    URV_CUDA(cudaEventRecord(v_ready, sv));
    d2h_v.reset(new AsyncD2H(V, ldv, v_out.dev, v_out.ld, n, n, v_ready, device));
  }

  // ---- u, r = householder_qr(a @ v): factorizations.py:143 ----
  const long long sf = 2LL * q + 2;
  if (!v_deferred) dgemm(opAY, 'N', m, n, n, 1.0, dA, lda_d, v_out.dev, v_out.ld, 0.0, Z.p, ldm, st, ws);
  matrix_stats(Z.p, ldm, m, n, slot(sf), part.p, st);
  {
    QrFactors fz;
    qr_factor(Z.p, ldm, m, n, nullptr, nullptr, st, ws, fz, nullptr, 0, 0, 0, v_tail, vlate_blocks);
    if (v_late) {
      URV_CUDA(cudaStreamWaitEvent(sv, v_tail, 0));
      form_v();
      qr_form_q(fz, u_out.dev, u_out.ld, st, ws);
      URV_CUDA(cudaStreamWaitEvent(st, v_done, 0));  // R lands where fy_last lived
      qr_extract_r(fz, r_out.dev, r_out.ld, st);
    } else {
      if (v_deferred) URV_CUDA(cudaStreamWaitEvent(st, v_done, 0));  // R lands where fy_last lived
      qr_extract_r(fz, r_out.dev, r_out.ld, st);
      if (r_ready) URV_CUDA(cudaEventRecord(r_ready, st));
      qr_form_q(fz, u_out.dev, u_out.ld, st, ws);
    }
  }
  if (!out_on_device) {
    d2h_r.reset(new AsyncD2H(R, ldr, r_out.dev, r_out.ld, n, n, r_ready, device));
    URV_CUDA(cudaEventRecord(u_ready, st));
    URV_CUDA(cudaStreamWaitEvent(st, u_ready, 0));
    AsyncD2H d2h_u(U, ldu, u_out.dev, u_out.ld, m, n, u_ready, device);
    d2h_u.join();
    d2h_r->join();
    d2h_v->join();
  } else {
    u_out.finish(st);
    r_out.finish(st);
  }
  if (v_deferred) URV_CUDA(cudaStreamWaitEvent(st, v_done, 0));  // V and its stage stats are final
  if (out_on_device) v_out.finish(st);
  if (stage_info)
    URV_CUDA(cudaMemcpyAsync(stage_info, info.p, sizeof(double) * URV_STAGE_FIELDS * ns, cudaMemcpyDeviceToHost,
                             st));
  ws.release();
  URV_CUDA(cudaStreamSynchronize(st));
  if (v_deferred) {
    wsv.release();
    part_v = DevBuf();
    URV_CUDA(cudaStreamSynchronize(sv));
    cudaStreamDestroy(sv);
    cudaEventDestroy(v_done);
    if (v_tail) cudaEventDestroy(v_tail);
  }
}

// ------------------------------ rsvd driver ------------------------------
// factorizations.py:180-207: Y = powered sample of the first `ell` columns of
// the same Gaussian draw, Q = orth(A Y) (range finder), tall = A^T Q = Qt Rt
// (Householder QR), Rt = Ur diag(sigma) W^T (Jacobi, svd.cu); then
// v = Qt Ur and u = Q W.  Stages: 0 = A, 1..2q = power steps (reorth) or
// 1 = the final sample (no reorth), 2q+1 = range-finder QR.
void rsvd_impl(const double* A, long long m, long long n, long long lda, int a_rowmajor, int a_on_device,
               long long ell, const double* G, long long ldg, int g_on_device, unsigned long long seed,
               unsigned long long rstream, int q, int reorth, double* U, long long ldu, double* sigma, double* V,
               long long ldv, int out_on_device, double* stage_info, long long n_stages, void* user_stream) {
  if (m < 1 || n < 1 || ell < 1 || ell >= std::min(m, n) || q < 0) {
    set_error("invalid rsvd arguments: m=%lld n=%lld ell=%lld q=%d", m, n, ell, q);
    throw CudaFailure{kInvalid};
  }
  if (stage_info && n_stages < 2LL * q + 2) {
    set_error("stage_info needs %d stages", 2 * q + 2);
    throw CudaFailure{kInvalid};
  }
  StreamGuard sg(user_stream);
  cudaStream_t st = sg.s;
  PanelOrder panel_order(st);
  Workspace ws(st);
  DevBuf a_hold;
  long long lda_d = 0;
  const Operand a_in{A, a_rowmajor ? n : m, a_rowmajor ? m : n, lda};
  const double* dA = stage_in(a_in, a_on_device, a_hold, lda_d, st);
  const char opAY = a_rowmajor ? 'T' : 'N';
  const char opAtY = a_rowmajor ? 'N' : 'T';
  const long long ldm = round_up(m, 8), ldn = round_up(n, 8), ldl = round_up(ell, 8);
  const long long ns = 2LL * q + 2;
  DevBuf info(static_cast<size_t>(URV_STAGE_FIELDS) * ns, st), part(3 * STATS_BLOCKS, st);
  URV_CUDA(cudaMemsetAsync(info.p, 0, sizeof(double) * URV_STAGE_FIELDS * ns, st));
  auto slot = [&](long long s) { return info.p + URV_STAGE_FIELDS * s; };
  DevBuf Y(static_cast<size_t>(ldn) * ell, st), Y2(static_cast<size_t>(ldn) * ell, st);
  DevBuf Z(static_cast<size_t>(ldm) * ell, st), Qz(static_cast<size_t>(ldm) * ell, st);
  if (G) {
    URV_CUDA(cudaMemcpy2DAsync(Y.p, ldn * 8, G, ldg * 8, n * 8, ell,
                               g_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  } else if (!gaussian_device(seed, rstream, n, ell, Y.p, ldn, st)) {  // prefix of the n x n draw
    set_error("device Gaussian draw could not be resolved; pass G");
    throw CudaFailure{kInvalid};
  }
  matrix_stats(dA, lda_d, a_in.rows, a_in.cols, slot(0), part.p, st);
  // _powered_sample (factorizations.py:86-101); Q's are formed explicitly here:
  // for ell << n that is cheaper than carrying A along the QR (power_urv_impl)
  if (reorth) {
    for (int i = 0; i < q; ++i) {
      const long long s1 = 1 + 2LL * i, s2 = 2 + 2LL * i;
      dgemm(opAY, 'N', m, ell, n, 1.0, dA, lda_d, Y.p, ldn, 0.0, Z.p, ldm, st, ws);
      matrix_stats(Z.p, ldm, m, ell, slot(s1), part.p, st);
      householder_qr_device(Z.p, ldm, m, ell, Qz.p, ldm, nullptr, 0, slot(s1), slot(s1) + 3, st, ws);
      dgemm(opAtY, 'N', n, ell, m, 1.0, dA, lda_d, Qz.p, ldm, 0.0, Y2.p, ldn, st, ws);
      matrix_stats(Y2.p, ldn, n, ell, slot(s2), part.p, st);
      householder_qr_device(Y2.p, ldn, n, ell, Y.p, ldn, nullptr, 0, slot(s2), slot(s2) + 3, st, ws);
    }
  } else {
    for (int i = 0; i < q; ++i) {
      dgemm(opAY, 'N', m, ell, n, 1.0, dA, lda_d, Y.p, ldn, 0.0, Z.p, ldm, st, ws);
      dgemm(opAtY, 'N', n, ell, m, 1.0, dA, lda_d, Z.p, ldm, 0.0, Y2.p, ldn, st, ws);
      std::swap(Y, Y2);
    }
    if (q > 0) matrix_stats(Y.p, ldn, n, ell, slot(1), part.p, st);
  }
  // qq = _orth(a @ z, "range-finder QR")
  const long long sr = 2LL * q + 1;
  dgemm(opAY, 'N', m, ell, n, 1.0, dA, lda_d, Y.p, ldn, 0.0, Z.p, ldm, st, ws);
  matrix_stats(Z.p, ldm, m, ell, slot(sr), part.p, st);
  householder_qr_device(Z.p, ldm, m, ell, Qz.p, ldm, nullptr, 0, slot(sr), slot(sr) + 3, st, ws);
  // An error stage (collapse / non-finite) ends the call here: the caller raises
  // the reference's exception from stage_info, nothing else is meaningful.
  std::vector<double> hinfo(static_cast<size_t>(URV_STAGE_FIELDS) * ns);
  URV_CUDA(cudaMemcpyAsync(hinfo.data(), info.p, sizeof(double) * hinfo.size(), cudaMemcpyDeviceToHost, st));
  URV_CUDA(cudaStreamSynchronize(st));
  if (stage_info) std::copy(hinfo.begin(), hinfo.end(), stage_info);
  bool failed = hinfo[1] > 0;
  for (long long s = 1; s < ns; ++s) {
    const double* r = hinfo.data() + URV_STAGE_FIELDS * s;
    const bool orth_stage = reorth ? true : (s == sr);
    if (orth_stage && (r[0] == 0.0 || r[1] > 0)) failed = true;
    if (!reorth && q > 0 && s == 1 && r[2] == 0) failed = true;
  }
  if (failed) {
    ws.release();
    return;
  }
  // tall = (qq.T @ a).T = A^T Q  ->  Qt Rt  ->  SVD of Rt
  dgemm(opAtY, 'N', n, ell, m, 1.0, dA, lda_d, Qz.p, ldm, 0.0, Y.p, ldn, st, ws);
  DevBuf Rt(static_cast<size_t>(ldl) * ell, st), Ur(static_cast<size_t>(ldl) * ell, st),
      W(static_cast<size_t>(ldl) * ell, st), sig(ell, st);
  householder_qr_device(Y.p, ldn, n, ell, Y2.p, ldn, Rt.p, ldl, nullptr, nullptr, st, ws);
  jacobi_svd_device(Rt.p, ldl, static_cast<int>(ell), sig.p, Ur.p, ldl, W.p, ldl, st);
  OutBuf u_out, v_out, s_out;
  u_out.init(U, ldu, out_on_device, m, ell, st);
  v_out.init(V, ldv, out_on_device, n, ell, st);
  s_out.init(sigma, ell, out_on_device, ell, 1, st);
  dgemm('N', 'N', n, ell, ell, 1.0, Y2.p, ldn, Ur.p, ldl, 0.0, v_out.dev, v_out.ld, st, ws);  // v = Qt Ur
  dgemm('N', 'N', m, ell, ell, 1.0, Qz.p, ldm, W.p, ldl, 0.0, u_out.dev, u_out.ld, st, ws);   // u = Q W
  URV_CUDA(cudaMemcpyAsync(s_out.dev, sig.p, sizeof(double) * ell, cudaMemcpyDeviceToDevice, st));
  u_out.finish(st);
  v_out.finish(st);
  s_out.finish(st);
  ws.release();
  URV_CUDA(cudaStreamSynchronize(st));
}

void householder_qr_impl(const double* A, long long m, long long n, long long lda, int a_rowmajor,
                         int a_on_device, double* Q, long long ldq, double* R, long long ldr, int out_on_device,
                         double* stage_info, void* user_stream) {
  if (m < 1 || n < 1 || m < n) {
    set_error("householder_qr requires rows >= cols >= 1, got %lldx%lld", m, n);
    throw CudaFailure{kInvalid};
  }
  StreamGuard sg(user_stream);
  cudaStream_t st = sg.s;
  PanelOrder panel_order(st);
  Workspace ws(st);
  const long long ldm = round_up(m, 8);
  DevBuf W(static_cast<size_t>(ldm) * n, st);
  if (a_rowmajor) {
    // C-order m x n input = column-major n x m buffer: transpose on the device.
    DevBuf a_hold;
    long long lda_d = 0;
    const Operand a_in{A, n, m, lda};
    const double* dA = stage_in(a_in, a_on_device, a_hold, lda_d, st);
    transpose(dA, lda_d, n, m, W.p, ldm, st);
  } else if (a_on_device) {
    URV_CUDA(cudaMemcpy2DAsync(W.p, ldm * 8, A, lda * 8, m * 8, n, cudaMemcpyDeviceToDevice, st));
  } else {
    h2d_ordered(W.p, ldm, A, lda, m, n, st);
  }
  DevBuf info(URV_STAGE_FIELDS, st), part(3 * STATS_BLOCKS, st);
  URV_CUDA(cudaMemsetAsync(info.p, 0, sizeof(double) * URV_STAGE_FIELDS, st));
  matrix_stats(W.p, ldm, m, n, info.p, part.p, st);
  OutBuf q_out, r_out;
  q_out.init(Q, ldq, out_on_device, m, n, st);
  r_out.init(R, ldr, out_on_device, n, n, st);
  householder_qr_device(W.p, ldm, m, n, q_out.dev, q_out.ld, r_out.dev, r_out.ld, info.p, info.p + 3, st, ws);
  q_out.finish(st);
  r_out.finish(st);
  if (stage_info)
    URV_CUDA(cudaMemcpyAsync(stage_info, info.p, sizeof(double) * URV_STAGE_FIELDS, cudaMemcpyDeviceToHost, st));
  ws.release();
  URV_CUDA(cudaStreamSynchronize(st));
}

}  // namespace
}  // namespace urv

// --------------------------------- C ABI ------------------------------------
namespace {
// The cooperative panel kernel spins on a grid barrier, so two of them must never
// be resident at the same time: calls that factor (power_urv, householder_qr)
// hold a per-device lock until their stream has drained.
std::mutex& device_lock() {
  static std::mutex locks[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return locks[dev & 63];
}

template <class F>
int guarded(F&& fn) {
  try {
    // A host thread that has not touched the runtime yet has no current context,
    // and the driver-level tensor-map encoder needs one: bind this thread's device.
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaSetDevice(dev);
    fn();
    return urv::kOk;
  } catch (const urv::CudaFailure& f) {
    return f.status;
  } catch (const std::bad_alloc&) {
    urv::set_error("host allocation failed");
    return urv::kOutOfMemory;
  } catch (...) {
    urv::set_error("unexpected C++ exception");
    return urv::kCudaError;
  }
}
}  // namespace

extern "C" {

int urv_power_urv_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor, int a_on_device,
                      const double* G, int64_t ldg, int g_on_device, uint64_t seed, uint64_t rstream, int q,
                      int reorth, int skip_redundant_qr, double* U, int64_t ldu, double* R, int64_t ldr, double* V,
                      int64_t ldv, int out_on_device, double* stage_info, int64_t n_stages, void* stream) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(device_lock());
    urv::power_urv_impl(A, m, n, lda, a_rowmajor, a_on_device, G, ldg, g_on_device, seed, rstream, q, reorth,
                        skip_redundant_qr, U, ldu, R, ldr, V, ldv, out_on_device, stage_info, n_stages, stream);
  });
}

int urv_rsvd_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor, int a_on_device, int64_t ell,
                 const double* G, int64_t ldg, int g_on_device, uint64_t seed, uint64_t rstream, int q, int reorth,
                 double* U, int64_t ldu, double* sigma, double* V, int64_t ldv, int out_on_device,
                 double* stage_info, int64_t n_stages, void* stream) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(device_lock());
    urv::rsvd_impl(A, m, n, lda, a_rowmajor, a_on_device, ell, G, ldg, g_on_device, seed, rstream, q, reorth, U, ldu,
                   sigma, V, ldv, out_on_device, stage_info, n_stages, stream);
  });
}

int urv_read_f64_file(const char* path, int64_t offset, int64_t rows, int64_t cols, double* dst, int64_t ldd,
                      void* stream) {
  return guarded([&] {
    urv::StreamGuard sg(stream);
    urv::read_file_to_device(path, offset, rows, cols, dst, ldd, sg.s);
  });
}

int urv_write_f64_file(const char* path, int64_t offset, const double* src, int64_t rows, int64_t cols, int64_t lds,
                       void* stream) {
  return guarded([&] {
    urv::StreamGuard sg(stream);
    urv::write_device_to_file(path, offset, src, rows, cols, lds, sg.s);
  });
}

int urv_rng_set_tables(const double* wi, const double* fi, const uint64_t* ki, double r, double inv_r) {
  return guarded([&] {
    urv::rng_set_tables(wi, fi, reinterpret_cast<const unsigned long long*>(ki), r, inv_r);
  });
}

int urv_gaussian_f64(uint64_t seed, uint64_t rstream, int64_t rows, int64_t cols, double* out, int64_t ldo,
                     int out_on_device, void* stream) {
  return guarded([&] {
    if (rows < 1 || cols < 1) {
      urv::set_error("matrix dimensions must be positive, got %lldx%lld", (long long)rows, (long long)cols);
      throw urv::CudaFailure{urv::kInvalid};
    }
    urv::StreamGuard sg(stream);
    urv::OutBuf o;
    o.init(out, ldo, out_on_device, rows, cols, sg.s);
    if (!urv::gaussian_device(seed, rstream, rows, cols, o.dev, o.ld, sg.s)) {
      urv::set_error("device Gaussian draw could not be resolved");
      throw urv::CudaFailure{urv::kInvalid};
    }
    o.finish(sg.s);
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

int urv_householder_qr_f64(const double* A, int64_t m, int64_t n, int64_t lda, int a_rowmajor, int a_on_device,
                           double* Q, int64_t ldq, double* R, int64_t ldr, int out_on_device, double* stage_info,
                           void* stream) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(device_lock());
    urv::householder_qr_impl(A, m, n, lda, a_rowmajor, a_on_device, Q, ldq, R, ldr, out_on_device, stage_info,
                             stream);
  });
}

int urv_qr_factor_f64(double* W, int64_t m, int64_t n, int64_t ldw, double* tau, void* stream) {
  return guarded([&] {
    if (m < n || n < 1 || ldw % 2 || (reinterpret_cast<uintptr_t>(W) & 15)) {
      urv::set_error("urv_qr_factor_f64: need m >= n >= 1 and W 16-byte aligned with an even ldw");
      throw urv::CudaFailure{urv::kInvalid};
    }
    std::lock_guard<std::mutex> lk(device_lock());
    urv::StreamGuard sg(stream);
    urv::Workspace ws(sg.s);
    urv::qr_factor_tau(W, ldw, m, n, tau, sg.s, ws);
    ws.release();
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

int urv_geqrt_f64(double* W, int64_t m, int64_t k, int64_t ldw, double* T, int64_t ldt, void* stream) {
  return guarded([&] {
    if (ldw % 2 || (reinterpret_cast<uintptr_t>(W) & 15)) {
      urv::set_error("urv_geqrt_f64: W must be 16-byte aligned with an even ldw");
      throw urv::CudaFailure{urv::kInvalid};
    }
    std::lock_guard<std::mutex> lk(device_lock());
    urv::StreamGuard sg(stream);  // a private stream (NULL) is synchronised on return
    urv::PanelOrder order(sg.s);
    urv::Workspace ws(sg.s);
    urv::geqrt_device(W, ldw, m, k, T, ldt, sg.s, ws);
    ws.release();  // stream-ordered: asynchronous on the caller's stream
  });
}

int urv_larfb_f64(const double* P, int64_t ldp, int64_t m, int64_t k, const double* T, int64_t ldt, int trans,
                  double* C, int64_t ldc, int64_t ncols, void* stream) {
  return guarded([&] {
    if (ldc % 2 || (reinterpret_cast<uintptr_t>(C) & 15)) {
      urv::set_error("urv_larfb_f64: C must be 16-byte aligned with an even ldc");
      throw urv::CudaFailure{urv::kInvalid};
    }
    urv::StreamGuard sg(stream);
    urv::Workspace ws(sg.s);
    urv::apply_block_reflector(P, ldp, m, k, T, ldt, trans != 0, C, ldc, ncols, sg.s, ws);
    ws.release();  // stream-ordered: asynchronous on the caller's stream
  });
}

int urv_tail_sumsq_f64(const double* R, int64_t n, int64_t ldr, double* out, void* stream) {
  return guarded([&] {
    urv::StreamGuard sg(stream);
    urv::tail_sumsq_device(R, ldr, n, out, sg.s);
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

int urv_trmv_upper_f64(const double* R, int64_t ldr, int64_t k0, int64_t N, int trans, const double* x, double* y,
                       void* stream) {
  return guarded([&] {
    urv::StreamGuard sg(stream);
    urv::trmv_device(R, ldr, k0, N, trans, x, y, sg.s);
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

int urv_tri_inv_f64(const double* R, int64_t n, int64_t ldr, double* X, int64_t ldx, void* stream) {
  return guarded([&] {
    urv::StreamGuard sg(stream);
    urv::Workspace ws(sg.s);
    urv::tri_inv_device(R, ldr, n, X, ldx, sg.s, ws);
    ws.release();
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

int urv_dgemm_f64(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  return guarded([&] {
    if (lda % 2 || ldb % 2 || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) {
      urv::set_error("urv_dgemm_f64: A and B must be 16-byte aligned with even lda, ldb");
      throw urv::CudaFailure{urv::kInvalid};
    }
    urv::StreamGuard sg(stream);
    urv::Workspace ws(sg.s);
    urv::dgemm(ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, sg.s, ws);
    ws.release();  // stream-ordered: asynchronous on the caller's stream
  });
}

int urv_matrix_stats_f64(const double* A, int64_t rows, int64_t cols, int64_t lda, int a_on_device, double* out,
                         void* stream) {
  return guarded([&] {
    if (rows < 1 || cols < 1) {
      out[0] = out[1] = out[2] = 0.0;
      return;
    }
    urv::StreamGuard sg(stream);
    urv::DevBuf hold;
    long long ld = 0;
    const urv::Operand in{A, rows, cols, lda};
    const double* d = urv::stage_in(in, a_on_device, hold, ld, sg.s);
    urv::DevBuf slot(4, sg.s), part(3 * urv::STATS_BLOCKS, sg.s);
    urv::matrix_stats(d, ld, rows, cols, slot.p, part.p, sg.s);
    URV_CUDA(cudaMemcpyAsync(out, slot.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, sg.s));
    URV_CUDA(cudaStreamSynchronize(sg.s));
  });
}

void urv_stats_enable(int on) { urv::g_stats_on = on != 0; }

int urv_stats_timeline(double* out, int max_records) {
  std::lock_guard<std::mutex> lk(urv::g_stats_mu);
  if (urv::g_stats.empty()) return 0;
  std::vector<cudaStream_t> ids;
  const cudaEvent_t t0 = urv::g_stats.front().e0;
  int k = 0;
  for (auto& r : urv::g_stats) {
    if (k >= max_records) break;
    size_t id = 0;
    while (id < ids.size() && ids[id] != r.stream) ++id;
    if (id == ids.size()) ids.push_back(r.stream);
    float a = 0.f, b = 0.f;
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&a, t0, r.e0) != cudaSuccess ||
        cudaEventElapsedTime(&b, t0, r.e1) != cudaSuccess)
      return -1;
    double* o = out + 5 * k++;
    o[0] = r.cls;
    o[1] = static_cast<double>(id);
    o[2] = a;
    o[3] = b;
    o[4] = r.flops;
  }
  return k;
}

int urv_stats_read(double* out, int n_classes) {
  std::lock_guard<std::mutex> lk(urv::g_stats_mu);
  for (int i = 0; i < 4 * n_classes; ++i) out[i] = 0.0;
  int rc = 0;
  for (auto& r : urv::g_stats) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) rc = 3;
    if (r.cls < n_classes) {
      out[4 * r.cls + 0] += 1;
      out[4 * r.cls + 1] += r.flops;
      out[4 * r.cls + 2] += r.bytes;
      out[4 * r.cls + 3] += ms;
    }
    urv::g_stats_free[r.dev].push_back(r.e0);
    urv::g_stats_free[r.dev].push_back(r.e1);
  }
  urv::g_stats.clear();
  return rc;
}

int urv_set_device(int device) {
  return guarded([&] { URV_CUDA(cudaSetDevice(device)); });
}

int urv_release_memory(void) {
  return guarded([&] { urv::trim_pool(); });
}

int urv_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

long long urv_launch_count(void) { return urv::g_launches.load(); }

int urv_debug_panel_cycles(double* out, int n) {
  int r = 0;
  const int rc = guarded([&] { r = urv::debug_panel_cycles(out, n); });
  return rc == urv::kOk ? r : -rc;
}

const char* urv_last_error(void) { return urv::last_error(); }
const char* urv_version(void) { return "urv_b200 0.1.0 (sm_100a, fp64 tma+dmma)"; }

}  // extern "C"
