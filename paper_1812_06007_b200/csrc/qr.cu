// Blocked Householder QR for sm_100a (FP64), diag(R) >= 0, explicit thin Q.
//
// Replaces the reference's `householder_qr` (core.py:112-158) and its helpers
// `_householder` (core.py:57-76), `_qr_panel` (core.py:79-98), `_wy_t`
// (core.py:101-109).  Same reflector convention: v(0) = 1, the reflector maps x
// to +||x|| e1 (Parlett's cancellation-free v0), sigma == 0 gives tau = 0 (x0 >= 0)
// or tau = 2 (x0 < 0), and R(j,j) is produced by the rank-1 update itself.
//
// Kernels:
//   panel_geqr2  cooperative kernel: the (m-j0) x nb panel is spread over up to
//                one CTA per SM and held in shared memory; each column costs two
//                grid barriers (norm, then the v^T A / V^T v dot products).  All
//                cross-CTA sums are fixed-order, so every CTA derives identical
//                reflectors and the result is bitwise deterministic.  CTA 0 also
//                builds the compact-WY T (dlarft forward/columnwise) in-kernel.
//   apply_t      reduces the split-K partials of V^T C and multiplies by T^T (QR
//                trailing update, core.py:151) or T (Q formation, core.py:157).
//   Trailing update / Q formation use the TMA+DMMA GEMM (dgemm.cu).
#include "common.cuh"
#include "dgemm.h"
#include "qr.h"

#include <algorithm>

namespace urv {

namespace {

constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of a[0..n) in a fixed order, computed by one warp; every lane returns
// the same bits (butterfly with commutative adds).
__device__ __forceinline__ double warp_fixed_sum(const double* a, int n, int lane) {
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += ld_cg(a + i);
  return warp_sum(s);
}

// Panel layout in shared memory: column-major S[c * rb + r], rb rows owned by
// this CTA.  Warp w owns columns {w, w + 8, w + 16, ...} (NB / 8 of them).
template <int NB>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
    panel_geqr2(double* __restrict__ P, long long ldp, int M, int ncols, int rb, double* __restrict__ Tout,
                double* __restrict__ part1, double* __restrict__ part2, double* __restrict__ x0slot,
                unsigned int* __restrict__ counter) {
  extern __shared__ __align__(16) double sm[];
  constexpr int CPW = NB / PANEL_WARPS;  // columns per warp
  double* S = sm;                          // NB * rb
  double* vloc = S + NB * rb;              // rb
  double* T = vloc + rb;                   // NB * NB (CTA 0)
  double* sdot = T + NB * NB;              // NB     (CTA 0)
  __shared__ double red[PANEL_WARPS];

  const int G = gridDim.x, c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = c * rb;
  const int nrows = max(0, min(rb, M - r0));
  unsigned int bar_target = 0;

  // ---- load the CTA's rows of the panel (coalesced along rows) ----
  for (int col = 0; col < NB; ++col) {
    for (int r = tid; r < rb; r += PANEL_THREADS) {
      double v = 0.0;
      if (col < ncols && r < nrows) v = P[(r0 + r) + col * ldp];
      S[col * rb + r] = v;
    }
  }
  if (c == 0)
    for (int i = tid; i < NB * NB; i += PANEL_THREADS) T[i] = 0.0;
  __syncthreads();

  // ---- norm partial of column 0 (rows > 0) ----
  {
    double s = 0.0;
    for (int r = tid; r < nrows; r += PANEL_THREADS)
      if (r0 + r > 0) s += S[r] * S[r];
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < PANEL_WARPS; ++w) t += red[w];
      part1[c] = t;
      if (r0 == 0 && nrows > 0) *x0slot = S[0];
    }
  }

  for (int j = 0; j < ncols; ++j) {
    // ================= barrier 1: norm partials of column j =================
    bar_target += G;
    if (G > 1) grid_barrier(counter, bar_target); else __syncthreads();

    // Reflector (identical in every CTA): core.py:57-76
    const double sigma = warp_fixed_sum(part1, G, lane);
    const double x0 = ld_cg(x0slot);
    double tau, v0 = 1.0;
    const bool flat = (sigma == 0.0);
    if (flat) {
      tau = (x0 >= 0.0) ? 0.0 : 2.0;
    } else {
      const double mu = sqrt(x0 * x0 + sigma);
      v0 = (x0 <= 0.0) ? (x0 - mu) : (-sigma / (x0 + mu));
      tau = 2.0 * v0 * v0 / (sigma + v0 * v0);
    }
    // v over this CTA's rows: 0 above j, 1 at j, x/v0 (or x when flat) below.
    for (int r = tid; r < rb; r += PANEL_THREADS) {
      const int gi = r0 + r;
      double v = 0.0;
      if (r < nrows) {
        if (gi == j) v = 1.0;
        else if (gi > j) v = flat ? S[j * rb + r] : S[j * rb + r] / v0;
      }
      vloc[r] = v;
    }
    __syncthreads();

    // Dot products s_k = sum_i v_i S(i,k) over this CTA's rows i >= j, all k.
    // (k < j: V(:,k)^T v_j for the T column; k >= j: v^T A for w.)
    const int lo = max(0, j - r0);
    {
      double acc[CPW];
#pragma unroll
      for (int q = 0; q < CPW; ++q) acc[q] = 0.0;
      for (int r = lo + lane; r < nrows; r += 32) {
        const double v = vloc[r];
#pragma unroll
        for (int q = 0; q < CPW; ++q) acc[q] += v * S[(warp + q * PANEL_WARPS) * rb + r];
      }
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        const double s = warp_sum(acc[q]);
        if (lane == 0) part2[c * NB + warp + q * PANEL_WARPS] = s;
      }
    }

    // ================= barrier 2: dot partials =================
    bar_target += G;
    if (G > 1) grid_barrier(counter, bar_target); else __syncthreads();

    // Fixed-order cross-CTA sums for this warp's columns: lane = (col q, chain h)
    double wcol[CPW];
    {
      constexpr int CHAINS = 32 / CPW;  // lanes per column
      const int q = lane % CPW, h = lane / CPW;
      const int col = warp + q * PANEL_WARPS;
      double s = 0.0;
      for (int cc = h; cc < G; cc += CHAINS) s += ld_cg(part2 + cc * NB + col);
#pragma unroll
      for (int o = CPW; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      // lanes with the same q now hold the same sum
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq) wcol[qq] = __shfl_sync(0xffffffffu, s, qq);
    }

    // CTA 0: T(:j, j) = -tau T(:j,:j) s(:j), T(j,j) = tau   (core.py:101-109)
    if (c == 0) {
      if (lane < CPW) sdot[warp + lane * PANEL_WARPS] = wcol[lane];
      __syncthreads();
      if (tid < j) {
        double s = 0.0;
        for (int l = tid; l < j; ++l) s += T[l * NB + tid] * sdot[l];
        T[j * NB + tid] = -tau * s;
      }
      if (tid == 0) T[j * NB + j] = tau;
    }

    // Rank-1 update of columns k >= j over rows i >= j: S(i,k) -= v_i * tau * s_k
    if (tau != 0.0) {
      for (int r = lo + lane; r < nrows; r += 32) {
        const double v = vloc[r];
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          const int col = warp + q * PANEL_WARPS;
          if (col >= j && col < ncols) S[col * rb + r] -= v * (tau * wcol[q]);
        }
      }
    }
    __syncwarp();
    // Column j: keep R(j,j) on row j, store v below it (LAPACK-style V storage).
    if ((j % PANEL_WARPS) == warp) {
      for (int r = lo + lane; r < nrows; r += 32)
        if (r0 + r > j) S[j * rb + r] = vloc[r];
    }
    // Norm partial of column j+1 (rows > j+1) from the warp that owns it.
    if (j + 1 < ncols && ((j + 1) % PANEL_WARPS) == warp) {
      const int col = j + 1;
      double s = 0.0;
      for (int r = lane; r < nrows; r += 32)
        if (r0 + r > col) s += S[col * rb + r] * S[col * rb + r];
      s = warp_sum(s);
      if (lane == 0) part1[c] = s;
      const int lr = col - r0;
      if (lr >= 0 && lr < nrows && lane == 0) *x0slot = S[col * rb + lr];
    }
    __syncthreads();
  }

  // ---- write back: R on/above the diagonal, V below it ----
  for (int col = 0; col < ncols; ++col)
    for (int r = tid; r < nrows; r += PANEL_THREADS) P[(r0 + r) + col * ldp] = S[col * rb + r];
  if (c == 0)
    for (int i = tid; i < NB * NB; i += PANEL_THREADS) Tout[i] = T[i];
}

// Explicit unit-lower V (M x nb, ld ldv) from the V stored below the diagonal.
__global__ void load_v(const double* __restrict__ P, long long ldp, int M, int nb, double* __restrict__ V,
                       long long ldv) {
  const long long total = static_cast<long long>(M) * nb;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % M), col = static_cast<int>(idx / M);
    double v;
    if (r < col) v = 0.0;
    else if (r == col) v = 1.0;
    else v = P[r + col * ldp];
    V[r + col * ldv] = v;
  }
}

// out(:, c) = op(T) * sum_z ws_z(:, c)   for the nb x N block W; op = T^T (trans) or T.
__global__ void apply_t(const double* __restrict__ ws, long long split_stride, int splits, int nb, int N,
                        const double* __restrict__ T, int ldt, int trans, double* __restrict__ out,
                        long long ldo) {
  extern __shared__ double smt[];
  double* Ts = smt;           // nb * nb
  double* Ws = Ts + nb * nb;  // nb * 32
  const int tid = threadIdx.x;
  for (int i = tid; i < nb * nb; i += blockDim.x) Ts[i] = T[(i % nb) + (i / nb) * ldt];
  const int c0 = blockIdx.x * 32;
  const int cols = min(32, N - c0);
  for (int i = tid; i < nb * 32; i += blockDim.x) {
    const int r = i % nb, cc = i / nb;
    double s = 0.0;
    if (cc < cols) {
      const long long idx = r + static_cast<long long>(c0 + cc) * nb;
      s = ws[idx];
      for (int z = 1; z < splits; ++z) s += ws[idx + z * split_stride];
    }
    Ws[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < nb * cols; i += blockDim.x) {
    const int r = i % nb, cc = i / nb;
    double s = 0.0;
    if (trans) {  // (T^T w)(r) = sum_{l <= r} T(l, r) w(l)
      for (int l = 0; l <= r; ++l) s += Ts[l + r * nb] * Ws[l + cc * nb];
    } else {  // (T w)(r) = sum_{l >= r} T(r, l) w(l)
      for (int l = r; l < nb; ++l) s += Ts[r + l * nb] * Ws[l + cc * nb];
    }
    out[r + static_cast<long long>(c0 + cc) * ldo] = s;
  }
}

__global__ void set_identity(double* Q, long long ldq, int m, int n) {
  const long long total = static_cast<long long>(m) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % m), col = static_cast<int>(idx / m);
    Q[r + col * ldq] = (r == col) ? 1.0 : 0.0;
  }
}

__global__ void extract_r(const double* __restrict__ W, long long ldw, int n, double* __restrict__ R,
                          long long ldr) {
  const long long total = static_cast<long long>(n) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % n), col = static_cast<int>(idx / n);
    R[r + col * ldr] = (r <= col) ? W[r + col * ldw] : 0.0;
  }
}

// deficient = #{ j : R(j,j) < eps * sqrt(sumsq) }   (factorizations.py:80)
__global__ void count_deficient(const double* __restrict__ W, long long ldw, int n,
                                const double* __restrict__ sumsq, double* __restrict__ out) {
  __shared__ long long cnt[32];
  const double thr = 2.220446049250313e-16 * sqrt(*sumsq);
  long long local = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) local += (W[j + j * ldw] < thr) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += cnt[w];
    *out = static_cast<double>(s);
  }
}

inline int grid_for(long long total) {
  const long long b = (total + 255) / 256;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, 148LL * 8)));
}

template <int NB>
void launch_panel(double* P, long long ldp, int M, int ncols, double* T, QrScratch& scr, unsigned int* counter,
                  cudaStream_t st) {
  const DeviceInfo& di = device_info();
  // rows per CTA: at least 64, at most what fits in shared memory
  const size_t fixed = static_cast<size_t>(NB) * NB * 8 + NB * 8;
  const int max_rb = static_cast<int>((static_cast<size_t>(di.max_smem_optin) - fixed - 2048) / ((NB + 1) * 8));
  int G = std::min(di.sms, std::max(1, ceil_div(M, 64)));
  int rb = ceil_div(M, G);
  if (rb > max_rb) {
    set_error("panel of %d rows does not fit in %d CTAs (rb=%d > %d)", M, G, rb, max_rb);
    throw CudaFailure{kInvalid};
  }
  G = ceil_div(M, rb);
  const size_t smem = (static_cast<size_t>(NB) * rb + rb + NB * NB + NB) * sizeof(double);
  auto kern = panel_geqr2<NB>;
  static unsigned attr_mask = 0;
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (!(attr_mask & (1u << dev))) {
    cudaFuncAttributes fa;
    URV_CUDA(cudaFuncGetAttributes(&fa, kern));
    URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  di.max_smem_optin - static_cast<int>(fa.sharedSizeBytes)));
    attr_mask |= 1u << dev;
  }
  // Level-2 flops of the panel (LAPACK dgeqr2: 2 M nb^2 - 2/3 nb^3) and the
  // bytes it must move (read + write the panel once).
  const double fl = 2.0 * M * ncols * ncols - 2.0 / 3.0 * ncols * ncols * ncols;
  StatsScope scope(st, kKPanel, fl, 16.0 * M * ncols);
  void* args[] = {&P, &ldp, &M, &ncols, &rb, &T, &scr.part1, &scr.part2, &scr.x0, &counter};
  URV_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(G), dim3(PANEL_THREADS), args, smem,
                                       st));
  count_launch();
}

}  // namespace

int qr_panel_width(long long m) {
  (void)m;
  return 64;
}

void householder_qr_device(double* W, long long ldw, long long m, long long n, double* Q, long long ldq,
                           double* R, long long ldr, const double* sumsq, double* deficient,
                           cudaStream_t st, Workspace& ws) {
  const int NB = qr_panel_width(m);
  const int npan = ceil_div(n, NB);
  const long long ldv = round_up(m, 8);
  DevBuf Vbuf(static_cast<size_t>(ldv) * NB, st);
  DevBuf Tall(static_cast<size_t>(npan) * NB * NB, st);
  const int sms = device_info().sms;
  DevBuf scratch(static_cast<size_t>(sms) * (NB + 1) + 8, st);
  unsigned int* counters = nullptr;
  URV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&counters), sizeof(unsigned int) * npan, st));
  URV_CUDA(cudaMemsetAsync(counters, 0, sizeof(unsigned int) * npan, st));
  QrScratch scr{scratch.p, scratch.p + sms, scratch.p + static_cast<size_t>(sms) * (NB + 1)};
  DevBuf Wt(static_cast<size_t>(NB) * n, st);

  try {
    // ---------------- factorisation: core.py:143-152 ----------------
    for (int p = 0; p < npan; ++p) {
      const long long j0 = static_cast<long long>(p) * NB;
      const int nb = static_cast<int>(std::min<long long>(NB, n - j0));
      const int M = static_cast<int>(m - j0);
      double* Pp = W + j0 + j0 * ldw;
      double* Tp = Tall.p + static_cast<size_t>(p) * NB * NB;
      launch_panel<64>(Pp, ldw, M, nb, Tp, scr, counters + p, st);
      if (j0 + nb < n) {
        const long long Nt = n - j0 - nb;
        double* Cp = W + j0 + (j0 + nb) * ldw;
        {
          StatsScope s2(st, kKAux, 0.0, 16.0 * M * nb);
          load_v<<<grid_for(static_cast<long long>(M) * nb), 256, 0, st>>>(Pp, ldw, M, nb, Vbuf.p, ldv);
          URV_CHECK_LAUNCH();
        }
        // W = V^T C (split-K partials) ; W = T^T W ; C -= V W
        const int splits = gemm_splits_for(nb, Nt, M);
        const int eff = gemm_effective_splits(M, splits);
        double* part = ws.get(static_cast<size_t>(eff) * nb * Nt);
        dgemm_launch('T', 'N', nb, Nt, M, 1.0, Vbuf.p, ldv, Cp, ldw, 0.0, part, nb, st, part, splits);
        {
          StatsScope s3(st, kKApplyT, 1.0 * nb * nb * Nt, 8.0 * (eff + 1) * nb * Nt);
          const size_t sm = (static_cast<size_t>(nb) * nb + nb * 32) * sizeof(double);
          apply_t<<<ceil_div(Nt, 32), 256, sm, st>>>(part, static_cast<long long>(nb) * Nt, eff,
                                                     nb, static_cast<int>(Nt), Tp, NB, 1, Wt.p, NB);
          URV_CHECK_LAUNCH();
        }
        dgemm_launch('N', 'N', M, Nt, nb, -1.0, Vbuf.p, ldv, Wt.p, NB, 1.0, Cp, ldw, st, nullptr, 1);
      }
    }
    // ---------------- deficiency count and R ----------------
    if (deficient) {
      StatsScope s4(st, kKAux, 0.0, 8.0 * n);
      count_deficient<<<1, 1024, 0, st>>>(W, ldw, static_cast<int>(n), sumsq, deficient);
      URV_CHECK_LAUNCH();
    }
    if (R) {
      StatsScope s5(st, kKAux, 0.0, 16.0 * n * n);
      extract_r<<<grid_for(n * n), 256, 0, st>>>(W, ldw, static_cast<int>(n), R, ldr);
      URV_CHECK_LAUNCH();
    }
    // ---------------- explicit Q: core.py:154-157 (live columns only) ----------------
    {
      StatsScope s6(st, kKAux, 0.0, 8.0 * m * n);
      set_identity<<<grid_for(m * n), 256, 0, st>>>(Q, ldq, static_cast<int>(m), static_cast<int>(n));
      URV_CHECK_LAUNCH();
    }
    for (int p = npan - 1; p >= 0; --p) {
      const long long j0 = static_cast<long long>(p) * NB;
      const int nb = static_cast<int>(std::min<long long>(NB, n - j0));
      const int M = static_cast<int>(m - j0);
      const long long Nq = n - j0;
      double* Pp = W + j0 + j0 * ldw;
      double* Tp = Tall.p + static_cast<size_t>(p) * NB * NB;
      double* Bq = Q + j0 + j0 * ldq;
      {
        StatsScope s2(st, kKAux, 0.0, 16.0 * M * nb);
        load_v<<<grid_for(static_cast<long long>(M) * nb), 256, 0, st>>>(Pp, ldw, M, nb, Vbuf.p, ldv);
        URV_CHECK_LAUNCH();
      }
      const int splits = gemm_splits_for(nb, Nq, M);
      const int eff = gemm_effective_splits(M, splits);
      double* part = ws.get(static_cast<size_t>(eff) * nb * Nq);
      dgemm_launch('T', 'N', nb, Nq, M, 1.0, Vbuf.p, ldv, Bq, ldq, 0.0, part, nb, st, part, splits);
      {
        StatsScope s3(st, kKApplyT, 1.0 * nb * nb * Nq, 8.0 * (eff + 1) * nb * Nq);
        const size_t sm = (static_cast<size_t>(nb) * nb + nb * 32) * sizeof(double);
        apply_t<<<ceil_div(Nq, 32), 256, sm, st>>>(part, static_cast<long long>(nb) * Nq, eff, nb,
                                                   static_cast<int>(Nq), Tp, NB, 0, Wt.p, NB);
        URV_CHECK_LAUNCH();
      }
      dgemm_launch('N', 'N', M, Nq, nb, -1.0, Vbuf.p, ldv, Wt.p, NB, 1.0, Bq, ldq, st, nullptr, 1);
    }
  } catch (...) {
    cudaFreeAsync(counters, st);
    throw;
  }
  URV_CUDA(cudaFreeAsync(counters, st));
}

}  // namespace urv
