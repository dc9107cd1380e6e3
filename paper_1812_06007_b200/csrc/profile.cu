// Device building blocks of the rank-revealing profiles (diagnostics.py:86-169 of
// the reference).  For a URV factorization A = U R V^T the rank-k
// truncation residual is U(:, k:) R(k:, k:) V^T up to the reconstruction error, so
//   abs_frobenius[k] = ||R(k:, k:)||_F        abs_spectral[k] = smax(R(k:, k:))
// (the reference forms and decomposes the m x n residual for every k, O(n^4)).
//   * row_tail_sumsq: s_i = sum_{j >= i} R(i, j)^2, from which every ||R(k:, k:)||_F
//     follows by a suffix sum (exact, O(n^2));
//   * trmv on a diagonal block of an upper-triangular matrix (and its transpose):
//     the matrix-vector products of the Golub-Kahan-Lanczos iteration that gives
//     smax(R(k:, k:)) and, on R^{-1}, smin(R(:k, :k));
//   * upper-triangular inverse (recursive 2 x 2 blocking on the DMMA GEMM engine,
//     64 x 64 diagonal blocks by substitution in shared memory).
// Every reduction has a fixed order (bitwise reproducible).
#include "common.cuh"
#include "dgemm.h"
#include "profile.h"

namespace urv {

namespace {

constexpr int PT = 256;  // 32 rows x 8 column phases

// out[i] = sum_{j >= i} R(i, j)^2 for i < n (column-major R, ld ldr).
__global__ void __launch_bounds__(PT) row_tail_sumsq(const double* __restrict__ R, long long ldr, int n,
                                                     double* __restrict__ out) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, ph = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (i < n)
    for (long long j = blockIdx.x * 32 + ph; j < n; j += 8)
      if (j >= i) {
        const double v = R[i + j * ldr];
        acc += v * v;
      }
  part[ph][lane] = acc;
  __syncthreads();
  if (ph == 0 && i < n) {
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p) s += part[p][lane];
    out[i] = s;
  }
}

// y = B x, B = R(k0 : k0+N, k0 : k0+N) upper triangular: y_i = sum_{j >= i} B(i, j) x_j.
__global__ void __launch_bounds__(PT) trmv_n(const double* __restrict__ R, long long ldr, long long k0, int N,
                                             const double* __restrict__ x, double* __restrict__ y) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, ph = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const double* B = R + k0 + k0 * ldr;
  double acc = 0.0;
  if (i < N)
    for (long long j = blockIdx.x * 32 + ph; j < N; j += 8)
      if (j >= i) acc += B[i + j * ldr] * x[j];
  part[ph][lane] = acc;
  __syncthreads();
  if (ph == 0 && i < N) {
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < 8; ++p) s += part[p][lane];
    y[i] = s;
  }
}

// y = B^T x: y_j = sum_{i <= j} B(i, j) x_i, one warp per column (coalesced).
__global__ void __launch_bounds__(PT) trmv_t(const double* __restrict__ R, long long ldr, long long k0, int N,
                                             const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= N) return;
  const double* col = R + k0 + (k0 + j) * ldr;
  double acc = 0.0;
  for (int i = lane; i <= j; i += 32) acc += col[i] * x[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[j] = acc;
}

// X = inverse of the nb x nb upper-triangular diagonal block (nb <= 64), one CTA:
// column c of X solves R x = e_c by back substitution; thread c owns column c.
constexpr int TB = 64;
__global__ void __launch_bounds__(TB) tri_inv_block(const double* __restrict__ R, long long ldr, int nb,
                                                    double* __restrict__ X, long long ldx) {
  __shared__ double Rs[TB][TB + 1];
  const int c = threadIdx.x;
  for (int idx = c; idx < nb * nb; idx += TB) {
    const int r = idx % nb, col = idx / nb;
    Rs[r][col] = R[r + static_cast<long long>(col) * ldr];
  }
  __syncthreads();
  if (c >= nb) return;
  double x[TB];
#pragma unroll
  for (int r = 0; r < TB; ++r) x[r] = 0.0;
  // rows c+1.. of the solution are zero (upper triangular inverse)
  for (int r = nb - 1; r >= 0; --r) {
    if (r > c) continue;
    double s = (r == c) ? 1.0 : 0.0;
    for (int l = r + 1; l <= c; ++l) s -= Rs[r][l] * x[l];
    x[r] = s / Rs[r][r];
  }
  for (int r = 0; r < nb; ++r) X[r + static_cast<long long>(c) * ldx] = (r <= c) ? x[r] : 0.0;
}

// X (n x n) = R^{-1}, R upper triangular; X's strictly lower part is zeroed by the caller.
//   inv([[A, B], [0, C]]) = [[A^-1, -A^-1 B C^-1], [0, C^-1]]
void tri_inv_rec(const double* R, long long ldr, long long n, double* X, long long ldx, double* tmp, long long ldt,
                 cudaStream_t st, Workspace& ws) {
  if (n <= TB) {
    tri_inv_block<<<1, TB, 0, st>>>(R, ldr, static_cast<int>(n), X, ldx);
    URV_CHECK_LAUNCH();
    return;
  }
  const long long h = (n / 2 + TB - 1) / TB * TB;  // multiple of 64: 16-byte aligned sub-blocks
  tri_inv_rec(R, ldr, h, X, ldx, tmp, ldt, st, ws);
  tri_inv_rec(R + h + h * ldr, ldr, n - h, X + h + h * ldx, ldx, tmp, ldt, st, ws);
  // tmp (h x (n-h)) = B C^-1, then X12 = -A^-1 tmp
  dgemm('N', 'N', h, n - h, n - h, 1.0, R + h * ldr, ldr, X + h + h * ldx, ldx, 0.0, tmp, ldt, st, ws);
  dgemm('N', 'N', h, n - h, h, -1.0, X, ldx, tmp, ldt, 0.0, X + h * ldx, ldx, st, ws);
}

__global__ void zero_strict_lower(double* X, long long ldx, int n) {
  const long long total = static_cast<long long>(n) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
    if (r > c) X[r + static_cast<long long>(c) * ldx] = 0.0;
  }
}

}  // namespace

void tail_sumsq_device(const double* R, long long ldr, long long n, double* out, cudaStream_t st) {
  StatsScope s(st, kKAux, 2.0 * n * n / 2, 8.0 * n * n / 2);
  row_tail_sumsq<<<static_cast<int>((n + 31) / 32), PT, 0, st>>>(R, ldr, static_cast<int>(n), out);
  URV_CHECK_LAUNCH();
}

void trmv_device(const double* R, long long ldr, long long k0, long long N, int trans, const double* x, double* y,
                 cudaStream_t st) {
  if (N <= 0) return;
  StatsScope s(st, kKAux, 1.0 * N * N, 4.0 * N * N);
  if (trans) {
    trmv_t<<<static_cast<int>((N + 7) / 8), PT, 0, st>>>(R, ldr, k0, static_cast<int>(N), x, y);
  } else {
    trmv_n<<<static_cast<int>((N + 31) / 32), PT, 0, st>>>(R, ldr, k0, static_cast<int>(N), x, y);
  }
  URV_CHECK_LAUNCH();
}

void tri_inv_device(const double* R, long long ldr, long long n, double* X, long long ldx, cudaStream_t st,
                    Workspace& ws) {
  if (n <= 0) return;
  if (ldr % 2 || ldx % 2 || (reinterpret_cast<uintptr_t>(R) & 15) || (reinterpret_cast<uintptr_t>(X) & 15)) {
    set_error("tri_inv: R and X must be 16-byte aligned with even leading dimensions");
    throw CudaFailure{kInvalid};
  }
  StatsScope s(st, kKAux, 2.0 * n * n * n / 3.0, 16.0 * n * n);
  const long long ldt = round_up(n, 8);
  DevBuf tmp(static_cast<size_t>(ldt) * n, st);
  tri_inv_rec(R, ldr, n, X, ldx, tmp.p, ldt, st, ws);
  zero_strict_lower<<<1184, 256, 0, st>>>(X, ldx, static_cast<int>(n));
  URV_CHECK_LAUNCH();
}

}  // namespace urv
