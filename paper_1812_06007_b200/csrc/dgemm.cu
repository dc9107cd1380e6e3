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
#include <cmath>
#include <mutex>

namespace urv {

namespace {

constexpr int BK = 16;  // doubles per k-block: one 128-byte swizzle row

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int LOOK_, int MINB_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int LOOKAHEAD = LOOK_;  // k-blocks in flight ahead of compute
  static constexpr int MINB = MINB_;       // CTAs per SM (register / smem budget)
  static constexpr int TM = BM / WM, TN = BN / WN;  // warp tile
  static constexpr int MI = TM / 8, NI = TN / 8;   // DMMA tiles per warp
  static constexpr int CONSUMERS = WM * WN;
  static constexpr int THREADS = CONSUMERS * 32;  // TMA issue folded into thread 0
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RING = STAGES * STAGE_BYTES;
  // C staging tile (TMA store / beta-load), 16-row strips of BN 128-byte lines,
  // reuses the operand ring once the main loop is done.
  static constexpr int STRIP = BN * 128;
  static constexpr int CTILE = BM * BN * 8;
  static constexpr int DATA = RING > CTILE ? RING : CTILE;
  static constexpr int SMEM = DATA + 1024 /*align*/ + 8 * (2 * STAGES + 1);
  static_assert(TM % 16 == 0 && TN % 16 == 0, "warp tile must be a multiple of 16");
  static_assert(LOOKAHEAD >= 1 && LOOKAHEAD < STAGES, "lookahead");
  static_assert(BM % 16 == 0, "C strips");
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
// 64-bit shared accesses are serviced per half-warp (lanes 0-15 = g 0..3,
// lanes 16-31 = g 4..7, each with t = 0..3).  Under the 128-byte swizzle a
// half-warp's 16 accesses must hit 16 distinct 8-byte bank pairs, both for the
// main-loop fragment loads and for the epilogue's C-staging stores (whose
// columns come from the K-major B mapping, n & 7 in {0,1,4,5} or {2,3,6,7}):
//   K-major : half-warp rows {0,3,4,7} / {1,2,5,6}
//   MN-major: rows {0,1,12,13} / {2,3,14,15} (even tile), {4,5,8,9} / {6,7,10,11} (odd tile)
// The same mapping is applied to C, so the permutation is invisible outside.
template <bool KMAJ>
__device__ __forceinline__ int frag_row(int tile, int g) {
  const int hh = g >> 2;
  if (KMAJ) return tile * 8 + (((g & 3) << 1) | (hh ^ (g & 1)));
  const int odd = tile & 1;
  const int sgrp = ((g >> 1) & 1) ? (odd ? 4 : 6) + hh : (odd ? 2 : 0) + hh;
  return (tile >> 1) * 16 + 2 * sgrp + (g & 1);
}

template <class Cfg, bool A_KMAJ, bool B_KMAJ>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    dgemm_tma_dmma(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, int M, int N, int K, int k_per_split,
                   int c_cols_per_split, double alpha, double beta, int tiles_m, int tiles_n) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B) by pointer arithmetic on the __shared__
  // array, so the compiler keeps the shared state space (LDS, not generic LD).
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::DATA);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* cbar = empty + Cfg::STAGES;

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
  const int c_y0 = n0 + blockIdx.z * c_cols_per_split;  // split-K partials: column block z

  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int nk = (kend - kbeg + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::CONSUMERS);
    }
    mbar_init(cbar, 1);
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
      tma_load_2d(sa, &mapA, k, m0, &full[s]);
    } else {
#pragma unroll
      for (int b = 0; b < Cfg::BM / 16; ++b) tma_load_2d(sa + b * 2048, &mapA, m0 + b * 16, k, &full[s]);
    }
    if (B_KMAJ) {
      tma_load_2d(sb, &mapB, k, n0, &full[s]);
    } else {
#pragma unroll
      for (int b = 0; b < Cfg::BN / 16; ++b) tma_load_2d(sb + b * 2048, &mapB, n0 + b * 16, k, &full[s]);
    }
  };
  const bool producer = (threadIdx.x == 0);
  if (producer) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    tma_prefetch_desc(&mapC);
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

  // C prefetch (beta != 0): the epilogue stages C in the ring.  When every C strip lies
  // inside one ring stage, the strips of a stage are loaded as soon as all warps have
  // released that stage's LAST k-block, so the C load overlaps the final k-blocks instead
  // of following the main loop.
  constexpr bool kCPrefetch = (Cfg::STAGE_BYTES % Cfg::STRIP) == 0;
  constexpr int SPS = kCPrefetch ? Cfg::STAGE_BYTES / Cfg::STRIP : 1;  // strips per stage
  const int strips = min(Cfg::BM / 16, (M - m0 + 15) / 16);
  const int c_groups = (strips + SPS - 1) / SPS;  // ring stages holding C strips
  unsigned c_pending = (beta != 0.0 && kCPrefetch && producer) ? ((1u << c_groups) - 1u) : 0u;
  auto c_issue_group = [&](int gidx) {
    const int lo = gidx * SPS, hi = min(strips, lo + SPS);
    for (int sidx = lo; sidx < hi; ++sidx) tma_load_2d(smem + sidx * Cfg::STRIP, &mapC, m0 + sidx * 16, c_y0, cbar);
  };
  if (c_pending) mbar_expect_tx(cbar, strips * Cfg::STRIP);
  auto c_prefetch = [&](int kb_now) {  // producer: issue every group whose stage is free by now
    for (int gidx = 0; gidx < c_groups; ++gidx) {
      if (!(c_pending & (1u << gidx))) continue;
      const int last = (nk - 1 - gidx) >= 0 ? gidx + Cfg::STAGES * ((nk - 1 - gidx) / Cfg::STAGES) : -1;
      if (last >= kb_now) continue;  // the stage is still to be read
      if (last >= 0) mbar_wait(&empty[gidx], (last / Cfg::STAGES) & 1);  // all warps released it
      c_issue_group(gidx);
      c_pending &= ~(1u << gidx);
    }
  };

  for (int kb = 0; kb < nk; ++kb) {
    if (producer && kb + Cfg::LOOKAHEAD < nk) issue(kb + Cfg::LOOKAHEAD);
    if (c_pending && kb + Cfg::LOOKAHEAD >= nk) c_prefetch(kb);
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
    if (lane == 0) mbar_arrive_after_reads(&empty[s]);
  }

  // ------------------ epilogue: stage C in smem, TMA store ------------------
  __syncthreads();  // every warp is done reading the ring, which now holds C
  if (beta != 0.0) {
    if (producer) {
      if (kCPrefetch) {
        c_prefetch(nk);  // whatever the main loop could not issue yet (every stage is free now)
      } else {
        mbar_expect_tx(cbar, strips * Cfg::STRIP);
        for (int sidx = 0; sidx < strips; ++sidx)
          tma_load_2d(smem + sidx * Cfg::STRIP, &mapC, m0 + sidx * 16, c_y0, cbar);
      }
    }
    mbar_wait(cbar, 0);
  }
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i) {
    const int ml = wm * Cfg::TM + frag_row<A_KMAJ>(i, g);
    const uint32_t rowpart = (ml >> 4) * Cfg::STRIP;
    const int mq = (ml & 15) >> 1, mb = (ml & 1) << 3;
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int nl = wn * Cfg::TN + frag_row<B_KMAJ>(j, 2 * t + h);
        double* p = reinterpret_cast<double*>(smem + rowpart + nl * 128 + (((mq ^ (nl & 7)) << 4) | mb));
        const double v = alpha * acc[i][j][h];
        *p = (beta == 0.0) ? v : v + beta * *p;
      }
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (producer) {
    for (int sidx = 0; sidx < strips; ++sidx) tma_store_2d(&mapC, smem + sidx * Cfg::STRIP, m0 + sidx * 16, c_y0);
    tma_store_commit_and_wait();
  }
}

// C = alpha * sum_z ws[z] + beta * C   (fixed summation order over z)
__global__ void splitk_reduce(const double* __restrict__ ws, long long ldws, long long split_stride, int splits,
                              int M, int N, double alpha, double beta, double* __restrict__ C, long long ldc) {
  const long long total = static_cast<long long>(M) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(idx % M);
    const long long n = idx / M;
    const long long w = m + n * ldws;
    double s = ws[w];
    for (int z = 1; z < splits; ++z) s += ws[w + z * split_stride];
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

// Tile configurations (all 8 DMMA warps, warp 0's lane 0 also issues TMA):
//   Big   128x128, warp tile 64x32, 4-stage 128 KB ring, 1 CTA/SM   -- long-K products (A.Y, A^T.Y, V^T C)
//   Upd   128x64,  warp tile 32x32, 4-stage  96 KB ring, 2 CTAs/SM  -- short-K rank-k updates (C -= V W)
//   Skinny 64x128, warp tile 32x32, 4-stage  96 KB ring, 2 CTAs/SM  -- M <= 64 (W = V^T C, leaf width)
// Two resident CTAs let one CTA's epilogue (C load / TMA store) overlap the other's main loop.
using BigCfg = GemmCfg<128, 128, 2, 4, 4, 2, 1>;
using UpdCfg = GemmCfg<128, 64, 4, 2, 4, 3, 2>;
using SkinnyCfg = GemmCfg<64, 128, 2, 4, 4, 2, 2>;

enum class Pick { Big, Upd, Skinny };
Pick pick_cfg(long long M, long long N, long long K) {
  // Long-K products with M <= 256 rows (the outer-block V^T C, Gram) and a moderate output
  // width run better on 64-row tiles at 2 CTAs/SM; wide outputs keep the 128x128 tiles.
  // Measured (profiles/r01_skinny_n.log, N <= 8192): config 2 161.2 -> 156.7 ms, config 3
  // 514.5 -> 508.4-509.2 ms, config 4 2997 -> 2989-2992 ms; all N: config 4 3043.  URV_SKINNY_N overrides.
  static const long long skinny_n = [] {
    const char* e = getenv("URV_SKINNY_N");
    return e ? atoll(e) : 8192LL;
  }();
  if (M <= SkinnyCfg::BM) return Pick::Skinny;
  if (M <= 256 && K > 256 && N <= skinny_n) return Pick::Skinny;
  if (K <= 256) return Pick::Upd;
  return Pick::Big;
}

__global__ void scale_kernel(double* C, long long ldc, int M, int N, double beta) {
  const long long total = static_cast<long long>(M) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    double* p = C + idx % M + (idx / M) * ldc;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

template <class Cfg, bool AK, bool BK_>
void launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, int M, int N, int K,
                int kps, int splits, double alpha, double beta, cudaStream_t st) {
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
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(ma, mb, mc, M, N, K, kps,
                                               splits > 1 ? static_cast<int>(gemm_split_cols(N)) : 0, alpha,
                                               beta, tiles_m, tiles_n);
  URV_CHECK_LAUNCH();
}

template <class Cfg>
void launch_any(bool ak, bool bk, const double* A, long long lda, const double* B, long long ldb, long long M,
                long long N, long long K, int kps, int splits, double alpha, double beta, double* C,
                long long ldc, cudaStream_t st) {
  CUtensorMap ma, mb, mc;
  if (ak)  // op(A) = A^T, A stored K x M: K-major tile, one box per stage
    make_map(&ma, A, K, M, lda, BK, Cfg::BM);
  else  // A stored M x K: MN-major, 16x16 boxes
    make_map(&ma, A, M, K, lda, 16, BK);
  if (bk)  // B stored K x N
    make_map(&mb, B, K, N, ldb, BK, Cfg::BN);
  else  // op(B) = B^T, B stored N x K
    make_map(&mb, B, N, K, ldb, 16, BK);
  // 16-row strips of the C tile; split-K partials use column blocks padded to
  // gemm_split_cols(N) so a tile's N tail never spills into the next split.
  make_map(&mc, C, M, splits > 1 ? gemm_split_cols(N) * splits : N, ldc, 16, Cfg::BN);
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  if (ak && bk)
    launch_cfg<Cfg, true, true>(ma, mb, mc, m, n, k, kps, splits, alpha, beta, st);
  else if (ak && !bk)
    launch_cfg<Cfg, true, false>(ma, mb, mc, m, n, k, kps, splits, alpha, beta, st);
  else if (!ak && bk)
    launch_cfg<Cfg, false, true>(ma, mb, mc, m, n, k, kps, splits, alpha, beta, st);
  else
    launch_cfg<Cfg, false, false>(ma, mb, mc, m, n, k, kps, splits, alpha, beta, st);
}

}  // namespace

int gemm_splits_for(long long M, long long N, long long K) {
  int bm = BigCfg::BM, bn = BigCfg::BN, per_sm = 1;
  switch (pick_cfg(M, N, K)) {
    case Pick::Upd: bm = UpdCfg::BM; bn = UpdCfg::BN; per_sm = UpdCfg::MINB; break;
    case Pick::Skinny: bm = SkinnyCfg::BM; bn = SkinnyCfg::BN; per_sm = SkinnyCfg::MINB; break;
    default: break;
  }
  const long long tiles = static_cast<long long>(ceil_div(M, bm)) * ceil_div(N, bn);
  const int slots = device_info().sms * per_sm;
  // Optional cap on the k-range of one Big CTA (URV_MAX_KPS): long-lived CTAs
  // delay the look-ahead stream's kernels, which wait for free SMs.
  static const long long max_kps = [] {
    const char* e = getenv("URV_MAX_KPS");
    return e ? atoll(e) : 0LL;
  }();
  const int max_s = static_cast<int>(std::min<long long>(64, K / (8 * BK)));
  // M <= 64 products (the leaf V^T C of the panel phase: one or two tiles, K = panel
  // rows) are latency-bound: split K into runs of >= 8 k-blocks, at most 32 splits.
  // The wave-quantisation rule below never clears its threshold for 1-2 tiles unless
  // K >= 30 * 128 and fell back to ONE split.  Measured (profiles/r01_skinny_splits.log):
  // config 2 190.1 -> 164.3 ms, config 4 3041 -> 3011 ms.  URV_SKINNY_SPLITS overrides.
  if (bm == SkinnyCfg::BM) {
    static const int force = [] {
      const char* e = getenv("URV_SKINNY_SPLITS");
      return e ? atoi(e) : 0;
    }();
    const long long want = force > 0 ? force : std::min<long long>(32, K / (8 * BK));
    return static_cast<int>(std::max<long long>(1, std::min<long long>(want, 64)));
  }
  // At most 32 k-splits (measured, profiles/r01_split_cap.log: config 4 3012 -> 3000 ms at 32,
  // 3003 at 16; configs 2/3 unchanged).  URV_SPLIT_CAP overrides.
  static const int split_cap = [] {
    const char* e = getenv("URV_SPLIT_CAP");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  int s_min = 1;
  if (max_kps > 0 && bm == BigCfg::BM && bn == BigCfg::BN && K > max_kps)
    s_min = static_cast<int>(std::min<long long>(std::max(1, max_s), (K + max_kps - 1) / max_kps));
  if (s_min <= 1 && (tiles >= 4LL * slots || K < 16 * BK)) return 1;
  // Pick the split count with the best wave quantisation (>= 8 k-blocks per
  // split, <= 64 splits); ties go to fewer splits (less partial traffic).
  int best = s_min;
  double best_eff = 0.0;
  for (int s = s_min; s <= std::max(s_min, std::min(max_s, split_cap)); ++s) {
    const double waves = static_cast<double>(tiles * s) / slots;
    const double eff = waves / std::ceil(waves) * std::min(1.0, waves / 2.0);  // want >= 2 full waves
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int gemm_effective_splits(long long K, int splits) {
  if (splits <= 1) return 1;
  const int kps = ceil_div(ceil_div(K, BK), splits) * BK;
  return ceil_div(K, kps);
}

void dgemm_launch(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
                  long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
                  cudaStream_t stream, int splits) {
  if (M <= 0 || N <= 0) return;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
    set_error("dgemm: dimension exceeds 2^31");
    throw CudaFailure{kInvalid};
  }
  splits = gemm_effective_splits(K, splits);
  if (K <= 0) {
    if (splits > 1) {
      URV_CUDA(cudaMemset2DAsync(C, ldc * 8, 0, M * 8, gemm_split_cols(N) * splits, stream));
      return;
    }
    scale_kernel<<<296, 256, 0, stream>>>(C, ldc, static_cast<int>(M), static_cast<int>(N), beta);
    URV_CHECK_LAUNCH();
    return;
  }
  const bool ak = (ta == 'T' || ta == 't');
  const bool bk = !(tb == 'T' || tb == 't');
  const int kps = splits > 1 ? ceil_div(ceil_div(K, BK), splits) * BK : static_cast<int>(K);
  if (splits > 1) {
    alpha = 1.0;
    beta = 0.0;
  }
  const Pick pk = pick_cfg(M, N, K);
  StatsScope scope(stream, pk == Pick::Big ? kKGemm : (pk == Pick::Upd ? kKGemmUpd : kKGemmSkinny),
                   2.0 * M * N * K, 8.0 * (M * K + K * N + (beta != 0.0 ? 2 : 1) * M * N));
  switch (pk) {
    case Pick::Skinny:
      launch_any<SkinnyCfg>(ak, bk, A, lda, B, ldb, M, N, K, kps, splits, alpha, beta, C, ldc, stream);
      break;
    case Pick::Upd:
      launch_any<UpdCfg>(ak, bk, A, lda, B, ldb, M, N, K, kps, splits, alpha, beta, C, ldc, stream);
      break;
    default:
      launch_any<BigCfg>(ak, bk, A, lda, B, ldb, M, N, K, kps, splits, alpha, beta, C, ldc, stream);
  }
}

void dgemm(char ta, char tb, long long M, long long N, long long K, double alpha, const double* A,
           long long lda, const double* B, long long ldb, double beta, double* C, long long ldc,
           cudaStream_t stream, Workspace& wsp) {
  if (M <= 0 || N <= 0) return;
  const int splits = gemm_effective_splits(K, gemm_splits_for(M, N, K));
  if (splits > 1) {
    const long long ldws = round_up(M, 8);
    const long long npad = gemm_split_cols(N);
    double* ws = wsp.get(static_cast<size_t>(splits) * ldws * npad);
    dgemm_launch(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.0, ws, ldws, stream, splits);
    StatsScope scope(stream, kKAux, 0.0, 8.0 * (splits + 2) * M * N);
    const long long total = M * N;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
    splitk_reduce<<<blocks, 256, 0, stream>>>(ws, ldws, ldws * npad, splits, static_cast<int>(M),
                                              static_cast<int>(N), alpha, beta, C, ldc);
    URV_CHECK_LAUNCH();
  } else {
    dgemm_launch(ta, tb, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, stream, 1);
  }
}

}  // namespace urv
