// Blocked Householder QR for sm_100a (FP64), diag(R) >= 0, explicit thin Q.
//
// Replaces the reference's `householder_qr` (core.py:112-158) and its helpers
// `_householder` (core.py:57-76), `_qr_panel` (core.py:79-98), `_wy_t`
// (core.py:101-109).  Same reflector convention: v(0) = 1, the reflector maps x
// to +||x|| e1 (Parlett's cancellation-free v0), sigma == 0 gives tau = 0 (x0 >= 0)
// or tau = 2 (x0 < 0), and R(j,j) is produced by the rank-1 update itself.
//
// Structure (two-level blocking; the reference uses one level of 32):
//   outer blocks of NBO = 256 columns, each factored as 64-wide leaves:
//     panel_geqr2   cooperative kernel, one CTA per SM at most, the leaf panel
//                   held in shared memory; two grid barriers per column; all
//                   cross-CTA sums in a fixed order (bitwise deterministic);
//                   CTA 0 keeps V^T v and builds the leaf T after the loop.
//     leaf update   W = V^T C (split-K DMMA), W = T^T W (apply_t), C -= V W
//                   for the remaining columns of the outer block.
//   outer T         Gram V^T V (DMMA GEMM) + t_merge:  T12 = -T11 (V1^T V2) T22
//   trailing update C <- C - V T^T (V^T C)  as three DMMA GEMMs with K = 256
//   explicit Q      backward over outer blocks on the live columns (dorgqr):
//                   B <- B - V T (V^T B)
#include "common.cuh"
#include "dgemm.h"
#include "qr.h"

#include <algorithm>
#include <cstdlib>

namespace urv {

namespace {

constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;
constexpr int LEAF = 64;   // columns per cooperative panel
constexpr int NBO = 256;   // columns per outer block (trailing-update rank)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order sum of a[0..n) by one warp; every lane returns the same bits.
// Loads are issued in batches of 8 so L2 latency is paid once per batch.
__device__ __forceinline__ double warp_fixed_sum(const double* a, int n, int lane) {
  double s = 0.0;
  for (int base = lane; base < n; base += 32 * 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + 32 * u;
      v[u] = i < n ? ld_cg(a + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  return warp_sum(s);
}

// Panel layout in shared memory: column-major S[c * rb + r], rb rows owned by
// this CTA.  Warp w owns columns {w, w + 8, w + 16, ...} (NB / 8 of them).
template <int NB>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
    panel_geqr2(double* __restrict__ P, long long ldp, int M, int ncols, int rb, double* __restrict__ Tout,
                int ldt, double* __restrict__ part1, double* __restrict__ part2, double* __restrict__ x0slot,
                unsigned int* __restrict__ counter) {
  extern __shared__ __align__(16) double sm[];
  constexpr int CPW = NB / PANEL_WARPS;  // columns per warp
  double* S = sm;                          // NB * rb
  double* vloc = S + NB * rb;              // rb
  double* T = vloc + rb;                   // NB * NB  (CTA 0: Gram columns, then T)
  double* taus = T + NB * NB;              // NB       (CTA 0)
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
    if (c == 0 && tid == 0) taus[j] = tau;
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
    // (k < j: V(:,k)^T v_j for T; k >= j: v^T A for w.)
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

    // Fixed-order cross-CTA sums for this warp's columns: lane = (column q, chain h)
    double wcol[CPW];
    {
      constexpr int CHAINS = 32 / CPW;  // lanes per column
      const int q = lane % CPW, h = lane / CPW;
      const int col = warp + q * PANEL_WARPS;
      double s = 0.0;
      for (int base = h; base < G; base += CHAINS * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int cc = base + CHAINS * u;
          v[u] = cc < G ? ld_cg(part2 + cc * NB + col) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
#pragma unroll
      for (int o = CPW; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq) wcol[qq] = __shfl_sync(0xffffffffu, s, qq);
    }

    // CTA 0 keeps the Gram column V(:, :j)^T v_j for the T build after the loop.
    if (c == 0 && lane < CPW) {
      const int col = warp + lane * PANEL_WARPS;
      if (col < j) T[j * NB + col] = wcol[lane];
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
  if (c != 0) return;

  // ---- CTA 0: T from the Gram columns (core.py:101-109), in place ----
  // T(:j, j) = -tau_j T(:j, :j) g_j, T(j, j) = tau_j; column j of the array holds
  // g_j = V(:, :j)^T v_j above the diagonal until it is overwritten.
  __shared__ double tpart[4][NB];
  {
    const int r = tid % NB, p = tid / NB;  // 4 partial sums per row
    for (int j = 0; j < ncols; ++j) {
      double s = 0.0;
      if (r < j)
        for (int l = r + p; l < j; l += 4) s += T[l * NB + r] * T[j * NB + l];
      tpart[p][r] = s;
      __syncthreads();
      if (tid < j) {
        const double tot = (tpart[0][tid] + tpart[1][tid]) + (tpart[2][tid] + tpart[3][tid]);
        T[j * NB + tid] = -taus[j] * tot;
      }
      if (tid == 0) T[j * NB + j] = taus[j];
      __syncthreads();
    }
  }
  for (int i = tid; i < NB * NB; i += PANEL_THREADS) {
    const int r = i % NB, col = i / NB;
    Tout[r + static_cast<long long>(col) * ldt] = (r <= col && col < ncols) ? T[i] : 0.0;
  }
}

// Explicit unit-lower V columns [c0, c1) of an outer block: V(r, c) = 0 (r < c),
// 1 (r == c), P(r, c) (r > c), for rows [0, M).  P/V are relative to the block origin.
__global__ void load_v(const double* __restrict__ P, long long ldp, int M, int c0, int c1, double* __restrict__ V,
                       long long ldv) {
  const int nc = c1 - c0;
  const long long total = static_cast<long long>(M) * nc;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % M), col = c0 + static_cast<int>(idx / M);
    double v;
    if (r < col) v = 0.0;
    else if (r == col) v = 1.0;
    else v = P[r + static_cast<long long>(col) * ldp];
    V[r + static_cast<long long>(col) * ldv] = v;
  }
}

// out(:, c) = op(T) * sum_z part_z(:, c) for an nb x N block (nb <= 64); op = T^T
// (trans) or T.  Partial z lives at columns [z*pstride, z*pstride + N) (ld ldp).
__global__ void apply_t(const double* __restrict__ part, long long ldp, long long pstride, int splits, int nb,
                        int N, const double* __restrict__ T, int ldt, int trans, double* __restrict__ out,
                        long long ldo) {
  __shared__ double Ts[64 * 64];
  __shared__ double Ws[64 * 32];
  const int tid = threadIdx.x;
  for (int i = tid; i < nb * nb; i += blockDim.x) Ts[i] = T[(i % nb) + (i / nb) * ldt];
  const int c0 = blockIdx.x * 32;
  const int cols = min(32, N - c0);
  for (int i = tid; i < nb * 32; i += blockDim.x) {
    const int r = i % nb, cc = i / nb;
    double s = 0.0;
    if (cc < cols) {
      const long long idx = r + static_cast<long long>(c0 + cc) * ldp;
      s = part[idx];
      for (int z = 1; z < splits; ++z) s += part[idx + z * pstride * ldp];
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

// Fixed-order sum of split-K partials: out = sum_z part_z (nb x N).
__global__ void sum_partials(const double* __restrict__ part, long long ldp, long long pstride, int splits, int nb,
                             int N, double* __restrict__ out, long long ldo) {
  const long long total = static_cast<long long>(nb) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % nb);
    const long long col = idx / nb;
    const long long base = r + col * ldp;
    double s = part[base];
    for (int z = 1; z < splits; ++z) s += part[base + z * pstride * ldp];
    out[r + col * ldo] = s;
  }
}

// T merge for leaf k (columns [c0, c0 + nb) of the outer T, ld ldt):
//   X = Gram(0:c0, c0:c0+nb) T_kk      (step 0)
//   T(0:c0, c0:c0+nb) = -T(0:c0, 0:c0) X   (step 1, T upper triangular)
__global__ void t_merge(double* __restrict__ T, int ldt, const double* __restrict__ Gm, int ldg, int c0, int nb,
                        double* __restrict__ X, int step) {
  const int total = c0 * nb;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int r = idx % c0, cc = idx / c0;
    double s = 0.0;
    if (step == 0) {
      for (int l = 0; l <= cc; ++l) s += Gm[r + (c0 + l) * ldg] * T[(c0 + l) + (c0 + cc) * ldt];
      X[r + cc * c0] = s;
    } else {
      for (int l = r; l < c0; ++l) s += T[r + l * ldt] * X[l + cc * c0];
      T[r + (c0 + cc) * ldt] = -s;
    }
  }
}

__global__ void set_identity(double* Q, long long ldq, int m, int n) {
  const long long total = static_cast<long long>(m) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % m), col = static_cast<int>(idx / m);
    Q[r + static_cast<long long>(col) * ldq] = (r == col) ? 1.0 : 0.0;
  }
}

__global__ void extract_r(const double* __restrict__ W, long long ldw, int n, double* __restrict__ R,
                          long long ldr) {
  const long long total = static_cast<long long>(n) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % n), col = static_cast<int>(idx / n);
    R[r + static_cast<long long>(col) * ldr] = (r <= col) ? W[r + static_cast<long long>(col) * ldw] : 0.0;
  }
}

// deficient = #{ j : R(j,j) < eps * sqrt(sumsq) }   (factorizations.py:80)
__global__ void count_deficient(const double* __restrict__ W, long long ldw, int n,
                                const double* __restrict__ sumsq, double* __restrict__ out) {
  __shared__ long long cnt[32];
  const double thr = 2.220446049250313e-16 * sqrt(*sumsq);
  long long local = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) local += (W[j + static_cast<long long>(j) * ldw] < thr) ? 1 : 0;
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

// Rows-per-CTA floor for the cooperative panel (sets its grid size); URV_PANEL_MIN_ROWS overrides.
int panel_min_rows() {
  static const int v = [] {
    const char* e = getenv("URV_PANEL_MIN_ROWS");
    return e ? std::max(16, atoi(e)) : 128;
  }();
  return v;
}

template <int NB>
void launch_panel(double* P, long long ldp, int M, int ncols, double* T, int ldt, QrScratch& scr,
                  unsigned int* counter, cudaStream_t st) {
  const DeviceInfo& di = device_info();
  const size_t fixed = (static_cast<size_t>(NB) * NB + NB) * 8;
  const int max_rb = static_cast<int>((static_cast<size_t>(di.max_smem_optin) - fixed - 4096) / ((NB + 1) * 8));
  int G = std::min(di.sms, std::max(1, ceil_div(M, panel_min_rows())));
  int rb = ceil_div(M, G);
  if (rb > max_rb) {
    G = ceil_div(M, max_rb);
    rb = ceil_div(M, G);
  }
  if (G > di.sms) {
    set_error("panel of %d rows does not fit in %d CTAs of %d rows", M, di.sms, max_rb);
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
  // Level-2 flops of the panel (dgeqr2: 2 M nb^2 - 2/3 nb^3); reads + writes the panel once.
  const double fl = 2.0 * M * ncols * ncols - 2.0 / 3.0 * ncols * ncols * ncols;
  StatsScope scope(st, kKPanel, fl, 16.0 * M * ncols);
  void* args[] = {&P, &ldp, &M, &ncols, &rb, &T, &ldt, &scr.part1, &scr.part2, &scr.x0, &counter};
  URV_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(G), dim3(PANEL_THREADS), args, smem,
                                       st));
  count_launch();
}

// W(nb x N, ld ldwo) = op(T) V^T C, with V (M x nb, ld ldv), C (M x N, ld ldc).
// For nb <= 64 the T multiply is fused with the split-K reduction (apply_t);
// for wider blocks it is a DMMA GEMM with the (upper-triangular) T.
void vt_c_times_t(const double* V, long long ldv, const double* C, long long ldc, long long M, int nb, long long N,
                  const double* T, int ldt, bool trans, double* Wout, long long ldwo, double* Wtmp,
                  long long ldwt, cudaStream_t st, Workspace& ws) {
  const int splits = gemm_effective_splits(M, gemm_splits_for(nb, N, M));
  const long long ldp = round_up(nb, 8);
  const long long pstride = gemm_split_cols(N);
  if (nb <= 64) {
    double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
    dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, part, ldp, st, splits);
    StatsScope s3(st, kKApplyT, 1.0 * nb * nb * N, 8.0 * (splits + 1) * nb * N);
    apply_t<<<ceil_div(N, 32), 256, 0, st>>>(part, ldp, splits > 1 ? pstride : 0, splits, nb, static_cast<int>(N),
                                             T, ldt, trans ? 1 : 0, Wout, ldwo);
    URV_CHECK_LAUNCH();
    return;
  }
  // wide block: W0 = V^T C (reduced), then W = op(T) W0 on the tensor cores
  if (splits > 1) {
    double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
    dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, part, ldp, st, splits);
    StatsScope s3(st, kKApplyT, 0.0, 8.0 * (splits + 1) * nb * N);
    sum_partials<<<grid_for(static_cast<long long>(nb) * N), 256, 0, st>>>(part, ldp, pstride, splits, nb,
                                                                          static_cast<int>(N), Wtmp, ldwt);
    URV_CHECK_LAUNCH();
  } else {
    dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, Wtmp, ldwt, st, 1);
  }
  dgemm_launch(trans ? 'T' : 'N', 'N', nb, N, nb, 1.0, T, ldt, Wtmp, ldwt, 0.0, Wout, ldwo, st, 1);
}

}  // namespace

int qr_panel_width(long long m) {
  (void)m;
  return LEAF;
}

void householder_qr_device(double* W, long long ldw, long long m, long long n, double* Q, long long ldq,
                           double* R, long long ldr, const double* sumsq, double* deficient,
                           cudaStream_t st, Workspace& ws) {
  const int nouter = ceil_div(n, NBO);
  const long long ldv = round_up(m, 8);
  const int ldt = NBO;
  DevBuf Vbuf(static_cast<size_t>(ldv) * NBO, st);
  DevBuf Tall(static_cast<size_t>(nouter) * NBO * NBO, st);
  URV_CUDA(cudaMemsetAsync(Tall.p, 0, sizeof(double) * nouter * NBO * NBO, st));  // T is upper triangular
  const int sms = device_info().sms;
  DevBuf scratch(static_cast<size_t>(sms) * (LEAF + 1) + 8, st);
  const int nleaves = ceil_div(n, LEAF);
  unsigned int* counters = nullptr;
  URV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&counters), sizeof(unsigned int) * nleaves, st));
  URV_CUDA(cudaMemsetAsync(counters, 0, sizeof(unsigned int) * nleaves, st));
  QrScratch scr{scratch.p, scratch.p + sms, scratch.p + static_cast<size_t>(sms) * (LEAF + 1)};
  const long long ldwt = NBO;
  DevBuf Wt(static_cast<size_t>(ldwt) * n, st);
  DevBuf Wt2(static_cast<size_t>(ldwt) * n, st);
  DevBuf Gram(static_cast<size_t>(NBO) * NBO, st);
  DevBuf Xm(static_cast<size_t>(NBO) * LEAF, st);

  try {
    // ---------------- factorisation: core.py:143-152 ----------------
    for (int p = 0; p < nouter; ++p) {
      const long long j0 = static_cast<long long>(p) * NBO;
      const int nbo = static_cast<int>(std::min<long long>(NBO, n - j0));
      const int M = static_cast<int>(m - j0);
      double* Pp = W + j0 + j0 * ldw;  // outer block origin
      double* Tp = Tall.p + static_cast<size_t>(p) * NBO * NBO;
      for (int c0 = 0; c0 < nbo; c0 += LEAF) {
        const int nbl = std::min(LEAF, nbo - c0);
        const int Ml = M - c0;
        double* Pl = Pp + c0 + c0 * ldw;
        launch_panel<LEAF>(Pl, ldw, Ml, nbl, Tp + c0 + static_cast<long long>(c0) * ldt, ldt, scr,
                           counters + (j0 + c0) / LEAF, st);
        {
          StatsScope s2(st, kKAux, 0.0, 16.0 * M * nbl);
          load_v<<<grid_for(static_cast<long long>(M) * nbl), 256, 0, st>>>(Pp, ldw, M, c0, c0 + nbl, Vbuf.p, ldv);
          URV_CHECK_LAUNCH();
        }
        if (c0 + nbl < nbo) {  // update the rest of the outer block with this leaf
          const long long Nr = nbo - c0 - nbl;
          double* Cr = Pl + static_cast<long long>(nbl) * ldw;
          const double* Vl = Vbuf.p + c0 + static_cast<long long>(c0) * ldv;
          vt_c_times_t(Vl, ldv, Cr, ldw, Ml, nbl, Nr, Tp + c0 + static_cast<long long>(c0) * ldt, ldt, true, Wt.p,
                       ldwt, Wt2.p, ldwt, st, ws);
          dgemm_launch('N', 'N', Ml, Nr, nbl, -1.0, Vl, ldv, Wt.p, ldwt, 1.0, Cr, ldw, st, 1);
        }
      }
      // outer T from the leaf T's: T12 = -T11 (V1^T V2) T22, leaf by leaf
      if (nbo > LEAF) {
        dgemm('T', 'N', nbo, nbo, M, 1.0, Vbuf.p, ldv, Vbuf.p, ldv, 0.0, Gram.p, NBO, st, ws);
        for (int c0 = LEAF; c0 < nbo; c0 += LEAF) {
          const int nbl = std::min(LEAF, nbo - c0);
          StatsScope s4(st, kKApplyT, 2.0 * c0 * nbl * (c0 + nbl), 0.0);
          t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, st>>>(Tp, ldt, Gram.p, NBO, c0, nbl, Xm.p,
                                                                                0);
          URV_CHECK_LAUNCH();
          t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, st>>>(Tp, ldt, Gram.p, NBO, c0, nbl, Xm.p,
                                                                                1);
          URV_CHECK_LAUNCH();
        }
      }
      // trailing update: C <- C - V T^T (V^T C)   (core.py:149-151)
      if (j0 + nbo < n) {
        const long long Nt = n - j0 - nbo;
        double* Cp = W + j0 + (j0 + nbo) * ldw;
        vt_c_times_t(Vbuf.p, ldv, Cp, ldw, M, nbo, Nt, Tp, ldt, true, Wt.p, ldwt, Wt2.p, ldwt, st, ws);
        dgemm_launch('N', 'N', M, Nt, nbo, -1.0, Vbuf.p, ldv, Wt.p, ldwt, 1.0, Cp, ldw, st, 1);
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
    for (int p = nouter - 1; p >= 0; --p) {
      const long long j0 = static_cast<long long>(p) * NBO;
      const int nbo = static_cast<int>(std::min<long long>(NBO, n - j0));
      const int M = static_cast<int>(m - j0);
      const long long Nq = n - j0;
      double* Pp = W + j0 + j0 * ldw;
      double* Tp = Tall.p + static_cast<size_t>(p) * NBO * NBO;
      double* Bq = Q + j0 + j0 * ldq;
      {
        StatsScope s2(st, kKAux, 0.0, 16.0 * M * nbo);
        load_v<<<grid_for(static_cast<long long>(M) * nbo), 256, 0, st>>>(Pp, ldw, M, 0, nbo, Vbuf.p, ldv);
        URV_CHECK_LAUNCH();
      }
      vt_c_times_t(Vbuf.p, ldv, Bq, ldq, M, nbo, Nq, Tp, ldt, false, Wt.p, ldwt, Wt2.p, ldwt, st, ws);
      dgemm_launch('N', 'N', M, Nq, nbo, -1.0, Vbuf.p, ldv, Wt.p, ldwt, 1.0, Bq, ldq, st, 1);
    }
  } catch (...) {
    cudaFreeAsync(counters, st);
    throw;
  }
  URV_CUDA(cudaFreeAsync(counters, st));
}

}  // namespace urv
