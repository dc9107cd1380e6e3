// FP64 GEMM engine for sm_100a: TMA-fed, mbarrier-pipelined, DMMA.8x8x4 tensor cores.
//
// C = alpha * op(A) * op(B) + beta * C, column-major, op in {N, T}.
// Replaces the reference's OpenBLAS dgemm call sites on the hot path:
//   factorizations.py:91  a @ y          (A.Y)
//   factorizations.py:92  a.T @ y        (A^T.Y)
//   factorizations.py:143 a @ v          (A.V)
//   core.py:151 / :157    vs.T @ c, vs @ w  (compact-WY trailing update / Q formation)
//
// Design (B200-first):
//   * FP64 on sm_100a has no tcgen05 kind; the FP64 tensor path is warp-level
//     mma.sync m8n8k4 (SASS DMMA.8x8x4).  A probe on the box measured 37.15 TF/s
//     for DMMA vs 36.5 TF/s for DFMA (profiles/r01_fp64_peak_probe.log): same pipe,
//     but one DMMA is 256 FMAs per issue slot, leaving the issue port free.
//   * Operand tiles arrive by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle) into
//     a STAGES-deep ring guarded by full/empty mbarriers; one producer warp, the
//     other warps are DMMA consumers.  TMA zero-fills M/N/K tails, so there is
//     no boundary code in the main loop.
//   * Swizzle-aware fragment addressing keeps every 64-bit LDS at the 2-wavefront
//     minimum for both K-major and MN-major operands (MN-major tiles use a row
//     permutation inside each 16-row block, applied consistently to C).
//   * Deterministic split-K: partial tiles go to a workspace and are reduced in a
//     fixed order (no atomics), so results are bitwise reproducible.
#include "common.cuh"
#include "dgemm.h"

#include <cudaTypedefs.h>
#include <mutex>

namespace urv {

namespace {

constexpr int BK = 16;  // doubles per k-block: one 128-byte swizzle row

template <int BM_, int BN_, int WM_, int WN_, int STAGES_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int TM = BM / WM, TN = BN / WN;  // warp tile
  static constexpr int MI = TM / 8, NI = TN / 8;   // DMMA tiles per warp
  static constexpr int CONSUMERS = WM * WN;
  static constexpr int THREADS = CONSUMERS * 32;  // TMA issue folded into warp 0
  static constexpr int LOOKAHEAD = STAGES - 2;     // k-blocks in flight ahead of compute
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(TM % 16 == 0 && TN % 16 == 0, "warp tile must be a multiple of 16");
};

// Byte offset of element (mn, k) inside a K-major tile: rows of 16 k-values
// (128 B) per mn, 16-byte chunks XOR-swizzled by (mn & 7)  [TMA SWIZZLE_128B].
__device__ __forceinline__ uint32_t kmaj_off(int mn, int k) {
  return mn * 128 + ((((k >> 1) ^ (mn & 7)) << 4) | ((k & 1) << 3));
}
// Byte offset of (mn, k) inside an MN-major tile made of 16x16 TMA boxes (2 KB):
// box (mn >> 4), line k holds 16 mn-values, chunks swizzled by (k & 7).
__device__ __forceinline__ uint32_t mnmaj_off(int mn, int k) {
  return (mn >> 4) * 2048 + k * 128 + (((((mn & 15) >> 1) ^ (k & 7)) << 4) | ((mn & 1) << 3));
}
// Which physical row of the tile feeds fragment row g of DMMA tile `tile`.
template <bool KMAJ>
__device__ __forceinline__ int frag_row(int tile, int g) {
  if (KMAJ) return tile * 8 + g;
  // MN-major: tile pair (2p, 2p+1) shares one 16-row box; rows {0-3, 8-11} and
  // {4-7, 12-15} keep 4 k-lines of a fragment load on disjoint bank groups.
  return (tile >> 1) * 16 + (tile & 1) * 4 + (g & 3) + ((g >> 2) << 3);
}

template <class Cfg, bool A_KMAJ, bool B_KMAJ>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
    dgemm_tma_dmma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   int M, int N, int K, int shiftA, int shiftB, int k_per_split, double alpha,
                   double beta, double* __restrict__ C, long long ldc, double* __restrict__ ws,
                   long long ws_split_stride, int tiles_m, int tiles_n) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Grouped rasterisation: 8 M-tiles share their B column panel in L2.
  constexpr int GROUP = 8;
  const int bid = blockIdx.x;
  const int per_group = GROUP * tiles_n;
  const int first_m = (bid / per_group) * GROUP;
  const int gsize = min(tiles_m - first_m, GROUP);
  const int tm = first_m + (bid % per_group) % gsize;
  const int tn = (bid % per_group) / gsize;
  const int m0 = tm * Cfg::BM, n0 = tn * Cfg::BN;

  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int nk = (kend - kbeg + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::CONSUMERS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // TMA issue for k-block kb (one elected thread).  Slot reuse is guarded by the
  // `empty` barrier, which every consumer warp arrives on after its last read.
  auto issue = [&](int kb) {
    const int s = kb % Cfg::STAGES;
    const uint32_t par = (kb / Cfg::STAGES) & 1;
    mbar_wait(&empty[s], par ^ 1);
    mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
    unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
    unsigned char* sb = sa + Cfg::A_BYTES;
    const int k = kbeg + kb * BK;
    if (A_KMAJ) {
      tma_load_2d(sa, &mapA, k + shiftA, m0, &full[s]);
    } else {
#pragma unroll
      for (int b = 0; b < Cfg::BM / 16; ++b) tma_load_2d(sa + b * 2048, &mapA, m0 + b * 16 + shiftA, k, &full[s]);
    }
    if (B_KMAJ) {
      tma_load_2d(sb, &mapB, k + shiftB, n0, &full[s]);
    } else {
#pragma unroll
      for (int b = 0; b < Cfg::BN / 16; ++b) tma_load_2d(sb + b * 2048, &mapB, n0 + b * 16 + shiftB, k, &full[s]);
    }
  };
  const bool producer = (threadIdx.x == 0);
  if (producer) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int kb = 0; kb < min(nk, Cfg::LOOKAHEAD); ++kb) issue(kb);
  }

  // ------------------------------ DMMA consumers ------------------------------
  const int wm = warp % Cfg::WM, wn = warp / Cfg::WM;
  const int g = lane >> 2, t = lane & 3;

  double acc[Cfg::MI][Cfg::NI][2];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Per-thread fragment base offsets (k-step 0); later k-steps are XOR/add
  // adjustments known at compile time.
  uint32_t offA[Cfg::MI], offB[Cfg::NI];
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    const int mn = wm * Cfg::TM + frag_row<A_KMAJ>(i, g);
    offA[i] = A_KMAJ ? kmaj_off(mn, t) : mnmaj_off(mn, t);
  }
#pragma unroll
  for (int j = 0; j < Cfg::NI; ++j) {
    const int mn = wn * Cfg::TN + frag_row<B_KMAJ>(j, g);
    offB[j] = B_KMAJ ? kmaj_off(mn, t) : mnmaj_off(mn, t);
  }

  for (int kb = 0; kb < nk; ++kb) {
    if (producer && kb + Cfg::LOOKAHEAD < nk) issue(kb + Cfg::LOOKAHEAD);
    const int s = kb % Cfg::STAGES;
    const uint32_t par = (kb / Cfg::STAGES) & 1;
    mbar_wait(&full[s], par);
    // plain C++ shared loads (LDS.64): ordered after the mbarrier wait's memory clobber
    const unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
    const unsigned char* sb = sa + Cfg::A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double a[Cfg::MI], b[Cfg::NI];
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i) {
        const uint32_t o = A_KMAJ ? (offA[i] ^ (ks << 5))
                                  : ((offA[i] ^ ((ks & 1) << 6)) + (ks >> 1) * 1024 + (ks & 1) * 512);
        a[i] = *reinterpret_cast<const double*>(sa + o);
      }
#pragma unroll
      for (int j = 0; j < Cfg::NI; ++j) {
        const uint32_t o = B_KMAJ ? (offB[j] ^ (ks << 5))
                                  : ((offB[j] ^ ((ks & 1) << 6)) + (ks >> 1) * 1024 + (ks & 1) * 512);
        b[j] = *reinterpret_cast<const double*>(sb + o);
      }
#pragma unroll
      for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // --------------------------------- epilogue ---------------------------------
  double* out;
  long long ldo;
  const bool partial = ws != nullptr;
  if (partial) {
    out = ws + blockIdx.z * ws_split_stride;
    ldo = M;
  } else {
    out = C;
    ldo = ldc;
  }
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    const int m = m0 + wm * Cfg::TM + frag_row<A_KMAJ>(i, g);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn * Cfg::TN + frag_row<B_KMAJ>(j, 2 * t + h);
        if (n >= N) continue;
        double* p = out + m + static_cast<long long>(n) * ldo;
        if (partial) {
          *p = acc[i][j][h];
        } else if (beta == 0.0) {
          *p = alpha * acc[i][j][h];
        } else {
          *p = alpha * acc[i][j][h] + beta * *p;
        }
      }
    }
  }
}

// C = alpha * sum_z ws[z] + beta * C   (fixed summation order over z)
__global__ void splitk_reduce(const double* __restrict__ ws, long long split_stride, int splits, int M,
                              int N, double alpha, double beta, double* __restrict__ C, long long ldc) {
  const long long total = static_cast<long long>(M) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(idx % M);
    const long long n = idx / M;
    double s = ws[idx];
    for (int z = 1; z < splits; ++z) s += ws[idx + z * split_stride];
    double* p = C + m + n * ldc;
    *p = (beta == 0.0) ? alpha * s : alpha * s + beta * *p;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    throw CudaFailure{kCudaError};
  }
  return fn;
}

// Column-major matrix `rows x cols` with leading dimension ld (elements).
// box = {box0 (contiguous), box1}.  Returns the element shift applied to align
// the base address to 16 bytes.
int make_map(CUtensorMap* map, const double* ptr, long long rows, long long cols, long long ld, int box0,
             int box1) {
  // TMA needs a 16-byte aligned base and row pitch; a swizzled box must also
  // start on a 16-byte boundary, so misaligned operands are rejected (callers copy).
  if (ld % 2 != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15) != 0) {
    set_error("dgemm operand must be 16-byte aligned with an even leading dimension (ptr %p, ld %lld)",
              static_cast<const void*>(ptr), ld);
    throw CudaFailure{kInvalid};
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld", (int)r, rows, cols, ld);
    throw CudaFailure{kCudaError};
  }
  return 0;
}

using BigCfg = GemmCfg<128, 128, 2, 4, 4>;   // 8 DMMA warps (warp 0 also issues TMA), 128 KB ring
using SmallCfg = GemmCfg<64, 128, 1, 4, 6>;  // M <= 64 (W = V^T C of a 64-wide panel)

__global__ void scale_kernel(double* C, long long ldc, int M, int N, double beta) {
  const long long total = static_cast<long long>(M) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    double* p = C + idx % M + (idx / M) * ldc;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

template <class Cfg, bool AK, bool BK_>
void launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, int sa, int sb, int kps,
                int splits, double alpha, double beta, double* C, long long ldc, double* ws,
                long long wss, cudaStream_t st) {
  auto kern = dgemm_tma_dmma<Cfg, AK, BK_>;
  static unsigned attr_mask = 0;  // one bit per device
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (!(attr_mask & (1u << dev))) {
    URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr_mask |= 1u << dev;
  }
  const int tiles_m = ceil_div(M, Cfg::BM), tiles_n = ceil_div(N, Cfg::BN);
  dim3 grid(tiles_m * tiles_n, 1, splits);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(ma, mb, M, N, K, sa, sb, kps, alpha, beta, C, ldc, ws, wss,
                                               tiles_m, tiles_n);
  URV_CHECK_LAUNCH();
}

template <class Cfg>
void launch_any(bool ak, bool bk, const double* A, long long lda, const double* B, long long ldb, long long M,
                long long N, long long K, int kps, int splits, double alpha, double beta, double* C,
                long long ldc, double* ws, long long wss, cudaStream_t st) {
  CUtensorMap ma, mb;
  int sa, sb;
  if (ak)  // op(A) = A^T, A stored K x M: K-major tile, one box per stage
    sa = make_map(&ma, A, K, M, lda, BK, Cfg::BM);
  else  // A stored M x K: MN-major, 16x16 boxes
    sa = make_map(&ma, A, M, K, lda, 16, BK);
  if (bk)  // B stored K x N
    sb = make_map(&mb, B, K, N, ldb, BK, Cfg::BN);
  else  // op(B) = B^T, B stored N x K
    sb = make_map(&mb, B, N, K, ldb, 16, BK);
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  if (ak && bk)
    launch_cfg<Cfg, true, true>(ma, mb, m, n, k, sa, sb, kps, splits, alpha, beta, C, ldc, ws, wss, st);
  else if (ak && !bk)
    launch_cfg<Cfg, true, false>(ma, mb, m, n, k, sa, sb, kps, splits, alpha, beta, C, ldc, ws, wss, st);
  else if (!ak && bk)
    launch_cfg<Cfg, false, true>(ma, mb, m, n, k, sa, sb, kps, splits, alpha, beta, C, ldc, ws, wss, st);
  else
    launch_cfg<Cfg, false, false>(ma, mb, m, n, k, sa, sb, kps, splits, alpha, beta, C, ldc, ws, wss, st);
}

}  // namespace

int gemm_splits_for(long long M, long long N, long long K) {
  const int bm = M <= SmallCfg::BM ? SmallCfg::BM : BigCfg::BM;
  const int tiles = ceil_div(M, bm) * ceil_div(N, BigCfg::BN);
  const int sms = device_info().sms;
  if (tiles >= sms || K < 16 * BK) return 1;
  int splits = ceil_div(2LL * sms, tiles);
  const int max_by_k = static_cast<int>(K / (8 * BK));  // >= 8 k-blocks per split
  if (splits > max_by_k) splits = max_by_k;
  if (splits > 64) splits = 64;
  return splits < 1 ? 1 : splits;
}

int gemm_effective_splits(long long K, int splits) {
  if (splits <= 1) return 1;
  const int kps = ceil_div(ceil_div(K, BK), splits) * BK;
  return ceil_div(K, kps);
}

void dgemm_launch(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
                  long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
                  cudaStream_t stream, double* ws, int splits) {
  if (M <= 0 || N <= 0) return;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
    set_error("dgemm: dimension exceeds 2^31");
    throw CudaFailure{kInvalid};
  }
  if (K <= 0) {
    if (splits > 1) {
      URV_CUDA(cudaMemsetAsync(ws, 0, sizeof(double) * M * N * splits, stream));
      return;
    }
    scale_kernel<<<296, 256, 0, stream>>>(C, ldc, static_cast<int>(M), static_cast<int>(N), beta);
    URV_CHECK_LAUNCH();
    return;
  }
  const bool ak = (ta == 'T' || ta == 't');
  const bool bk = !(tb == 'T' || tb == 't');
  int kps = static_cast<int>(K);
  if (splits > 1) {
    kps = ceil_div(ceil_div(K, BK), splits) * BK;
    splits = ceil_div(K, kps);
  }
  const long long wss = M * N;
  double* wsp = (splits > 1) ? ws : nullptr;
  StatsScope scope(stream, kKGemm, 2.0 * M * N * K, 8.0 * (M * K + K * N + 2 * M * N));
  if (M <= SmallCfg::BM)
    launch_any<SmallCfg>(ak, bk, A, lda, B, ldb, M, N, K, kps, splits, alpha, beta, C, ldc, wsp, wss, stream);
  else
    launch_any<BigCfg>(ak, bk, A, lda, B, ldb, M, N, K, kps, splits, alpha, beta, C, ldc, wsp, wss, stream);
}

void dgemm(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
           long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
           cudaStream_t stream, Workspace& wsp) {
  if (M <= 0 || N <= 0) return;
  const int splits = gemm_splits_for(M, N, K);
  if (splits > 1) {
    const int eff = gemm_effective_splits(K, splits);
    double* ws = wsp.get(static_cast<size_t>(eff) * M * N);
    dgemm_launch(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, nullptr, 0, stream, ws, splits);
    StatsScope scope(stream, kKAux, 0.0, 8.0 * (eff + 2) * M * N);
    const long long total = M * N;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    splitk_reduce<<<blocks, 256, 0, stream>>>(ws, M * N, eff, static_cast<int>(M), static_cast<int>(N), alpha,
                                              beta, C, ldc);
    URV_CHECK_LAUNCH();
  } else {
    dgemm_launch(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, stream, nullptr, 1);
  }
}

}  // namespace urv
