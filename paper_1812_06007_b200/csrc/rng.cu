// Device generator for the reference's Gaussian test matrix, bit-identical to
// NumPy's Generator(Philox(key=[seed, stream])).standard_normal(rows*cols)
// reshaped column-major (random.py:47-61 of the reference).
//
//  * Philox4x64-10 keyed by (seed, stream); the counter is incremented before
//    each block of four 64-bit words (NumPy's philox4x64_next).
//  * NumPy's 256-layer ziggurat (random_standard_normal): fast path
//    x = rabs * wi[idx] when rabs < ki[idx]; otherwise a wedge test with one
//    extra uniform, or for idx == 0 the tail loop with two uniforms per try.
//    The tables are NumPy's own (located and verified on the host, random.py).
//
// Each output consumes a data-dependent number of raw draws, so the stream is
// resolved in three passes over blocks of B raw positions:
//   1. zig_block_map : for every block and entry offset e < E, the draw chain
//                      from block start + e to the block end -> (exit offset
//                      into the next block, outputs emitted); chains from e > 0
//                      are followed only until they merge with the chain from 0;
//   2. zig_block_scan: one CTA composes those maps (chunked) and assigns each
//                      block its true entry offset and output base;
//   3. zig_emit      : every block replays its chain from the true entry and
//                      writes its outputs.  Tail outputs (|x| > r, ~2e-4 of all)
//                      are also logged so the host can recompute them with the
//                      C library's log1p, making the values bit-identical to NumPy.
#include "common.cuh"
#include "dgemm.h"

#include <cmath>
#include <mutex>
#include <vector>

namespace urv {

namespace {

struct ZigTables {
  double wi[256];
  double fi[256];
  unsigned long long ki[256];
  double r, inv_r;
};
__constant__ ZigTables c_zig;
bool g_zig_host_set = false;
ZigTables g_zig_host;
std::mutex g_zig_mu;

constexpr int ZIG_B = 2048;  // raw positions per block
constexpr int ZIG_E = 8;     // entry offsets tabulated per block

struct Philox {
  unsigned long long k0, k1;
  unsigned long long cached_block = ~0ull;
  unsigned long long w[4];
  __device__ __forceinline__ void block(unsigned long long b) {
    // counter = b + 1 (NumPy increments before generating); b < 2^62 here
    unsigned long long c0 = b + 1, c1 = 0, c2 = 0, c3 = 0, a0 = k0, a1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const unsigned long long hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0), lo0 = 0xD2E7470EE14C6C93ull * c0;
      const unsigned long long hi1 = __umul64hi(0xCA5A826395121157ull, c2), lo1 = 0xCA5A826395121157ull * c2;
      const unsigned long long n0 = hi1 ^ c1 ^ a0, n2 = hi0 ^ c3 ^ a1;
      c0 = n0;
      c1 = lo1;
      c2 = n2;
      c3 = lo0;
      if (r < 9) {
        a0 += 0x9E3779B97F4A7C15ull;
        a1 += 0xBB67AE8584CAA73Bull;
      }
    }
    w[0] = c0;
    w[1] = c1;
    w[2] = c2;
    w[3] = c3;
    cached_block = b;
  }
  __device__ __forceinline__ unsigned long long raw(unsigned long long p) {
    const unsigned long long b = p >> 2;
    if (b != cached_block) block(b);
    return w[p & 3];
  }
  __device__ __forceinline__ double uniform(unsigned long long p) {
    return __dmul_rn(static_cast<double>(raw(p) >> 11), 1.0 / 9007199254740992.0);
  }
};

// One try of random_standard_normal starting at raw position p.
// Returns the next try position; *emit = 1 and *x = value if it produced an output;
// *tail = 1 (with *u1 = the accepted first tail uniform, *neg = sign) for tail outputs.
__device__ __forceinline__ unsigned long long zig_step(Philox& ph, unsigned long long p, int* emit, double* x,
                                                       int* tail, double* u1, int* neg) {
  unsigned long long rr = ph.raw(p);
  const int idx = static_cast<int>(rr & 0xff);
  rr >>= 8;
  const int sign = static_cast<int>(rr & 1);
  const unsigned long long rabs = (rr >> 1) & 0x000fffffffffffffull;
  double v = __dmul_rn(static_cast<double>(rabs), c_zig.wi[idx]);
  if (sign) v = -v;
  *tail = 0;
  if (rabs < c_zig.ki[idx]) {
    *emit = 1;
    *x = v;
    return p + 1;
  }
  if (idx == 0) {
    unsigned long long q = p + 1;
    for (;;) {
      const double a = ph.uniform(q), b = ph.uniform(q + 1);
      q += 2;
      const double xx = __dmul_rn(-c_zig.inv_r, log1p(-a));
      const double yy = -log1p(-b);
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        const int ng = static_cast<int>((rabs >> 8) & 1);
        const double t = __dadd_rn(c_zig.r, xx);
        *emit = 1;
        *x = ng ? -t : t;
        *tail = 1;
        *u1 = a;
        *neg = ng;
        return q;
      }
    }
  }
  const double u = ph.uniform(p + 1);
  const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(c_zig.fi[idx - 1], -c_zig.fi[idx]), u), c_zig.fi[idx]);
  const double rhs = exp(__dmul_rn(__dmul_rn(-0.5, v), v));
  *emit = lhs < rhs ? 1 : 0;
  *x = v;
  return p + 2;
}

__global__ void zig_block_map(unsigned long long k0, unsigned long long k1, int nblocks, int* __restrict__ exit_off,
                              int* __restrict__ count) {
  // One thread per block.  The chain from offset 0 is walked in full, noting which
  // of the first 32 positions start a try (vis) and which of those tries emitted
  // (em).  A chain entering at e > 0 is walked only until it lands on a try start of
  // chain 0 (almost always within a step or two); from there both chains coincide.
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  Philox ph{k0, k1};
  const unsigned long long start = static_cast<unsigned long long>(blk) * ZIG_B, end = start + ZIG_B;
  unsigned int vis = 0, em = 0;
  unsigned long long p = start;
  int n0 = 0;
  while (p < end) {
    const unsigned long long off = p - start;
    int emit, tail, neg;
    double x, u1;
    p = zig_step(ph, p, &emit, &x, &tail, &u1, &neg);
    if (off < 32) {
      vis |= 1u << off;
      em |= static_cast<unsigned int>(emit) << off;
    }
    n0 += emit;
  }
  const int exit0 = static_cast<int>(p - end);
  exit_off[blk * ZIG_E] = exit0;
  count[blk * ZIG_E] = n0;
  for (int e = 1; e < ZIG_E; ++e) {
    unsigned long long q = start + e;
    int c = 0, ex = -1;
    while (q < end) {
      const unsigned long long off = q - start;
      if (off < 32 && ((vis >> off) & 1u)) {  // merged with chain 0
        c += n0 - __popc(em & ((1u << off) - 1u));
        ex = exit0;
        break;
      }
      int emit, tail, neg;
      double x, u1;
      q = zig_step(ph, q, &emit, &x, &tail, &u1, &neg);
      c += emit;
    }
    exit_off[blk * ZIG_E + e] = ex >= 0 ? ex : static_cast<int>(q - end);
    count[blk * ZIG_E + e] = c;
  }
}

// One CTA: chunk maps (entry -> exit, outputs) over CH consecutive blocks, a serial
// walk over chunks, then each chunk assigns its blocks' entries and output bases.
// status[0] = 0 ok, 1 an exit offset >= E occurred (host falls back), [1] = outputs.
__global__ void zig_block_scan(int nblocks, const int* __restrict__ exit_off, const int* __restrict__ count,
                               int* __restrict__ entry, long long* __restrict__ base, long long* __restrict__ status) {
  constexpr int THREADS = 512;
  __shared__ int cexit[THREADS][ZIG_E];
  __shared__ int ccount[THREADS][ZIG_E];  // < 2^31: a chunk spans < 2^31 raw positions
  __shared__ int centry[THREADS];
  __shared__ long long cbase[THREADS];
  __shared__ int bad;
  const int tid = threadIdx.x;
  const int ch = (nblocks + THREADS - 1) / THREADS;  // blocks per chunk
  const int b0 = min(nblocks, tid * ch), b1 = min(nblocks, b0 + ch);
  if (tid == 0) bad = 0;
  __syncthreads();
  {  // chunk map for every entry offset; the E chains are independent (ILP)
    int cur[ZIG_E];
    int n[ZIG_E];
#pragma unroll
    for (int e = 0; e < ZIG_E; ++e) {
      cur[e] = e;
      n[e] = 0;
    }
    for (int b = b0; b < b1; ++b) {
#pragma unroll
      for (int e = 0; e < ZIG_E; ++e) {
        if (cur[e] < ZIG_E) {
          const int k = b * ZIG_E + cur[e];
          n[e] += count[k];
          cur[e] = exit_off[k];
        }
      }
    }
#pragma unroll
    for (int e = 0; e < ZIG_E; ++e) {
      cexit[tid][e] = cur[e] < ZIG_E ? cur[e] : ZIG_E;  // ZIG_E marks "not representable"
      ccount[tid][e] = n[e];
    }
  }
  __syncthreads();
  if (tid == 0) {
    int cur = 0;
    long long n = 0;
    for (int c = 0; c < THREADS; ++c) {
      centry[c] = cur;
      cbase[c] = n;
      if (cur >= ZIG_E) {
        bad = 1;
        cur = 0;
      }
      n += ccount[c][cur];
      cur = cexit[c][cur];
    }
    status[1] = n;
  }
  __syncthreads();
  int cur = centry[tid];
  long long n = cbase[tid];
  for (int b = b0; b < b1; ++b) {
    if (cur >= ZIG_E) {
      bad = 1;
      break;
    }
    entry[b] = cur;
    base[b] = n;
    n += count[b * ZIG_E + cur];
    cur = exit_off[b * ZIG_E + cur];
  }
  __syncthreads();
  if (tid == 0) status[0] = bad;
}

struct TailRec {
  long long index;
  double u1;
  long long neg;
};

__global__ void zig_emit(unsigned long long k0, unsigned long long k1, int nblocks, const int* __restrict__ entry,
                         const long long* __restrict__ base, long long total, long long rows, double* __restrict__ out,
                         long long ld, TailRec* __restrict__ tails, int max_tails, int* __restrict__ ntails) {
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  long long i = base[blk];
  if (i >= total) return;
  Philox ph{k0, k1};
  const unsigned long long end = static_cast<unsigned long long>(blk + 1) * ZIG_B;
  unsigned long long p = static_cast<unsigned long long>(blk) * ZIG_B + entry[blk];
  while (p < end && i < total) {
    int emit, tail, neg;
    double x, u1;
    p = zig_step(ph, p, &emit, &x, &tail, &u1, &neg);
    if (emit) {
      out[(i % rows) + (i / rows) * ld] = x;
      if (tail) {
        const int slot = atomicAdd(ntails, 1);  // order of the log is irrelevant
        if (slot < max_tails) tails[slot] = TailRec{i, u1, neg};
      }
      ++i;
    }
  }
}

__global__ void scatter_values(const long long* __restrict__ idx, const double* __restrict__ val, int n, long long rows,
                               double* __restrict__ out, long long ld) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[(idx[t] % rows) + (idx[t] / rows) * ld] = val[t];
}

}  // namespace

void rng_set_tables(const double* wi, const double* fi, const unsigned long long* ki, double r, double inv_r) {
  std::lock_guard<std::mutex> lk(g_zig_mu);
  for (int i = 0; i < 256; ++i) {
    g_zig_host.wi[i] = wi[i];
    g_zig_host.fi[i] = fi[i];
    g_zig_host.ki[i] = ki[i];
  }
  g_zig_host.r = r;
  g_zig_host.inv_r = inv_r;
  g_zig_host_set = true;
}

bool rng_tables_ready() {
  std::lock_guard<std::mutex> lk(g_zig_mu);
  return g_zig_host_set;
}

// Column-major rows x cols N(0,1) matrix into device memory `out` (ld), bit-identical
// to NumPy's Generator(Philox(key=[seed, stream])).standard_normal(rows*cols).
// Returns false (nothing written reliably) if the chain could not be resolved.
bool gaussian_device(unsigned long long seed, unsigned long long stream, long long rows, long long cols, double* out,
                     long long ld, cudaStream_t st) {
  {
    std::lock_guard<std::mutex> lk(g_zig_mu);
    if (!g_zig_host_set) {
      set_error("device Gaussian generator: ziggurat tables not configured (urv_rng_set_tables)");
      throw CudaFailure{kInvalid};
    }
    static unsigned uploaded = 0;
    int dev = 0;
    URV_CUDA(cudaGetDevice(&dev));
    if (!(uploaded & (1u << dev))) {
      URV_CUDA(cudaMemcpyToSymbol(c_zig, &g_zig_host, sizeof(ZigTables)));
      uploaded |= 1u << dev;
    }
  }
  const long long total = rows * cols;
  // ~1.2% extra draws on average; 4% + 2 blocks of slack
  const long long raw_needed = total + total / 25 + 2LL * ZIG_B;
  const int nblocks = static_cast<int>((raw_needed + ZIG_B - 1) / ZIG_B);
  DevBuf exit_off((static_cast<size_t>(nblocks) * ZIG_E + 1) / 2 + 1, st);  // ints packed in doubles
  DevBuf count((static_cast<size_t>(nblocks) * ZIG_E + 1) / 2 + 1, st);
  DevBuf entry((static_cast<size_t>(nblocks) + 1) / 2 + 1, st);
  DevBuf base(static_cast<size_t>(nblocks) + 1, st);
  DevBuf status(2, st);
  const int max_tails = static_cast<int>(std::max<long long>(4096, total / 1000));
  DevBuf tails(static_cast<size_t>(max_tails) * 3, st);
  DevBuf ntails(1, st);
  URV_CUDA(cudaMemsetAsync(ntails.p, 0, sizeof(double), st));
  int* d_exit = reinterpret_cast<int*>(exit_off.p);
  int* d_count = reinterpret_cast<int*>(count.p);
  int* d_entry = reinterpret_cast<int*>(entry.p);
  long long* d_base = reinterpret_cast<long long*>(base.p);
  long long* d_status = reinterpret_cast<long long*>(status.p);
  {
    StatsScope sc(st, kKAux, 0.0, 8.0 * total);
    zig_block_map<<<ceil_div(nblocks, 128), 128, 0, st>>>(seed, stream, nblocks, d_exit, d_count);
    URV_CHECK_LAUNCH();
    zig_block_scan<<<1, 512, 0, st>>>(nblocks, d_exit, d_count, d_entry, d_base, d_status);
    URV_CHECK_LAUNCH();
    zig_emit<<<ceil_div(nblocks, 128), 128, 0, st>>>(seed, stream, nblocks, d_entry, d_base, total, rows, out, ld,
                                                   reinterpret_cast<TailRec*>(tails.p), max_tails,
                                                   reinterpret_cast<int*>(ntails.p));
    URV_CHECK_LAUNCH();
  }
  long long hstatus[2];
  int hnt = 0;
  URV_CUDA(cudaMemcpyAsync(hstatus, d_status, sizeof(hstatus), cudaMemcpyDeviceToHost, st));
  URV_CUDA(cudaMemcpyAsync(&hnt, ntails.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  URV_CUDA(cudaStreamSynchronize(st));
  if (hstatus[0] != 0 || hstatus[1] < total || hnt > max_tails) return false;
  // Tail values with the C library's log1p (NumPy's npy_log1p), patched on the device.
  if (hnt > 0) {
    std::vector<TailRec> h(hnt);
    URV_CUDA(cudaMemcpyAsync(h.data(), tails.p, sizeof(TailRec) * hnt, cudaMemcpyDeviceToHost, st));
    URV_CUDA(cudaStreamSynchronize(st));
    std::vector<long long> idx(hnt);
    std::vector<double> val(hnt);
    for (int k = 0; k < hnt; ++k) {
      const volatile double xx = -g_zig_host.inv_r * std::log1p(-h[k].u1);
      const double t = g_zig_host.r + xx;
      idx[k] = h[k].index;
      val[k] = h[k].neg ? -t : t;
    }
    DevBuf didx(hnt, st), dval(hnt, st);
    URV_CUDA(cudaMemcpyAsync(didx.p, idx.data(), sizeof(long long) * hnt, cudaMemcpyHostToDevice, st));
    URV_CUDA(cudaMemcpyAsync(dval.p, val.data(), sizeof(double) * hnt, cudaMemcpyHostToDevice, st));
    scatter_values<<<ceil_div(hnt, 256), 256, 0, st>>>(reinterpret_cast<long long*>(didx.p), dval.p, hnt, rows, out,
                                                       ld);
    URV_CHECK_LAUNCH();
    URV_CUDA(cudaStreamSynchronize(st));
  }
  return true;
}

}  // namespace urv
