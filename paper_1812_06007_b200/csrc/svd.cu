// Small dense SVD on the device: one-sided (Hestenes) Jacobi.
//
// Used for the l x l core of rsvd (factorizations.py:180-207 of the reference,
// which calls `svd` = numpy/LAPACK gesdd, core.py:220-228): the tall n x l
// sample is first reduced by the blocked Householder QR (qr.cu), and the
// triangular factor R (l x l) is diagonalised here,
//     R J = X,  X(:, i) = sigma_i u_i,  so  R = U diag(sigma) J^T.
// One cooperative kernel runs all sweeps: the l/2 disjoint column pairs of a
// round-robin (circle-method) step are rotated by one warp each, steps are
// separated by a grid barrier, and the sweep loop ends when a sweep applies no
// rotation (|x_i . x_j| <= tol ||x_i|| ||x_j|| for every pair, a scale-invariant
// test, so even tiny singular values get orthogonal vectors).  Every reduction
// has a fixed order: results are bitwise reproducible.
#include "common.cuh"
#include "svd.h"

#include <algorithm>

namespace urv {

namespace {

constexpr int JT = 256;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pair k of round-robin step s over np (even) players: player 0 is fixed, the
// others rotate around a circle of np - 1.
__device__ __forceinline__ void rr_pair(int np, int s, int k, int& i, int& j) {
  if (k == 0) {
    i = 0;
    j = 1 + s % (np - 1);
  } else {
    i = 1 + (s + k) % (np - 1);
    j = 1 + ((s - k) % (np - 1) + (np - 1)) % (np - 1);
  }
}

__global__ void __launch_bounds__(JT) jacobi_sweeps(double* __restrict__ X, long long ldx, double* __restrict__ J,
                                                    long long ldj, int n, double tol, int max_sweeps,
                                                    unsigned int* __restrict__ bar, unsigned int* __restrict__ rot,
                                                    int* __restrict__ sweeps_done) {
  const int np = n + (n & 1);
  const int npairs = np / 2;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * JT + threadIdx.x) >> 5, nw = (gridDim.x * JT) >> 5;
  unsigned int target = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int s = 0; s < np - 1; ++s) {
      for (int k = gw; k < npairs; k += nw) {
        int i, j;
        rr_pair(np, s, k, i, j);
        if (i >= n || j >= n) continue;  // the dummy player of an odd n
        double* xi = X + static_cast<long long>(i) * ldx;
        double* xj = X + static_cast<long long>(j) * ldx;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int r = lane; r < n; r += 32) {
          const double u = xi[r], v = xj[r];
          a += u * u;
          b += v * v;
          g += u * v;
        }
        a = wsum(a);
        b = wsum(b);
        g = wsum(g);
        if (g != 0.0 && fabs(g) > tol * sqrt(a) * sqrt(b)) {
          const double z = (b - a) / (2.0 * g);
          const double t = (z >= 0.0 ? 1.0 : -1.0) / (fabs(z) + sqrt(1.0 + z * z));
          const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
          for (int r = lane; r < n; r += 32) {
            const double u = xi[r], v = xj[r];
            xi[r] = c * u - sn * v;
            xj[r] = sn * u + c * v;
          }
          double* ji = J + static_cast<long long>(i) * ldj;
          double* jj = J + static_cast<long long>(j) * ldj;
          for (int r = lane; r < n; r += 32) {
            const double u = ji[r], v = jj[r];
            ji[r] = c * u - sn * v;
            jj[r] = sn * u + c * v;
          }
          if (lane == 0) atomicAdd(rot + sweep, 1u);
        }
      }
      target += gridDim.x;
      grid_barrier(bar, target);
    }
    if (__ldcg(rot + sweep) == 0u) {  // same value in every CTA after the barrier
      if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_done = sweep + 1;
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_done = -1;
}

// sigma_i = ||X(:, i)||  (one warp per column)
__global__ void column_norms(const double* __restrict__ X, long long ldx, int n, double* __restrict__ s) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n) return;
  double a = 0.0;
  for (int r = lane; r < n; r += 32) {
    const double u = X[r + static_cast<long long>(w) * ldx];
    a += u * u;
  }
  a = wsum(a);
  if (lane == 0) s[w] = sqrt(a);
}

// Nonincreasing order, ties by index: rank_i = #{j : s_j > s_i or (s_j == s_i and j < i)}.
__global__ void sort_gather(const double* __restrict__ X, long long ldx, const double* __restrict__ J, long long ldj,
                            const double* __restrict__ s, int n, double* __restrict__ sigma, double* __restrict__ U,
                            long long ldu, double* __restrict__ W, long long ldw) {
  const int i = blockIdx.y;  // source column
  __shared__ int rank_s;
  if (threadIdx.x == 0) {
    int r = 0;
    const double si = s[i];
    for (int j = 0; j < n; ++j) r += (s[j] > si || (s[j] == si && j < i)) ? 1 : 0;
    rank_s = r;
    if (blockIdx.x == 0) sigma[r] = si;
  }
  __syncthreads();
  const int dst = rank_s;
  const double si = s[i];
  const double inv = si > 0.0 ? 1.0 / si : 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    U[r + static_cast<long long>(dst) * ldu] = X[r + static_cast<long long>(i) * ldx] * inv;
    W[r + static_cast<long long>(dst) * ldw] = J[r + static_cast<long long>(i) * ldj];
  }
}

// Exactly-zero singular values leave U(:, i) = 0: replace those columns by an
// orthonormal completion (Gram-Schmidt, twice, of unit vectors against every other
// column).  They sort last, so columns [first, n) are the ones to complete.
__global__ void complete_basis(double* __restrict__ U, long long ldu, int n, const double* __restrict__ sigma) {
  __shared__ double red[JT / 32];
  __shared__ double coef;
  __shared__ int first_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    int f = n;
    while (f > 0 && !(sigma[f - 1] > 0.0)) --f;
    first_s = f;
  }
  __syncthreads();
  const int first = first_s;
  auto block_sum = [&](double v) {
    v = wsum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < JT / 32; ++w) t += red[w];
      coef = t;
    }
    __syncthreads();
    return coef;
  };
  int cand = 0;
  for (int c = first; c < n; ++c) {
    double* uc = U + static_cast<long long>(c) * ldu;
    for (;; ++cand) {
      if (cand >= n) return;  // cannot happen for an orthonormal set of < n columns
      for (int r = tid; r < n; r += JT) uc[r] = (r == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int o = 0; o < c; ++o) {
          const double* uo = U + static_cast<long long>(o) * ldu;
          double d = 0.0;
          for (int r = tid; r < n; r += JT) d += uo[r] * uc[r];
          d = block_sum(d);
          for (int r = tid; r < n; r += JT) uc[r] -= d * uo[r];
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int r = tid; r < n; r += JT) nn += uc[r] * uc[r];
      nn = block_sum(nn);
      if (nn > 0.25) {
        const double inv = 1.0 / sqrt(nn);
        for (int r = tid; r < n; r += JT) uc[r] *= inv;
        __syncthreads();
        ++cand;
        break;
      }
    }
  }
}

__global__ void set_eye(double* J, long long ldj, int n) {
  const long long total = static_cast<long long>(n) * n;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
    J[r + static_cast<long long>(c) * ldj] = (r == c) ? 1.0 : 0.0;
  }
}

}  // namespace

void jacobi_svd_device(double* X, long long ldx, int n, double* sigma, double* U, long long ldu, double* W,
                       long long ldw, cudaStream_t st) {
  if (n < 1) return;
  const long long ldj = round_up(n, 2);
  DevBuf J(static_cast<size_t>(ldj) * n, st), s(n, st);
  const int max_sweeps = 64;
  unsigned int* ctr = nullptr;  // [0] barrier, [1..max_sweeps] rotations per sweep, then sweeps_done
  dev_alloc(reinterpret_cast<void**>(&ctr), sizeof(unsigned int) * (max_sweeps + 2), st);
  URV_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned int) * (max_sweeps + 2), st));
  int* done = reinterpret_cast<int*>(ctr + max_sweeps + 1);
  StatsScope scope(st, kKAux, 0.0, 16.0 * n * n);
  set_eye<<<std::max(1, std::min(1184, ceil_div(static_cast<long long>(n) * n, 256))), 256, 0, st>>>(J.p, ldj, n);
  URV_CHECK_LAUNCH();

  // co-resident grid: one warp per pair, capped by occupancy
  int per_sm = 0, dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  URV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_sweeps, JT, 0));
  const int pairs = (n + 1) / 2;
  const int grid = std::max(1, std::min(ceil_div(pairs, JT / 32), device_info().sms * std::max(1, per_sm)));
  const double tol = std::max(1, n) * 2.220446049250313e-16;
  int sweeps_cap = max_sweeps;
  unsigned int* bar = ctr;
  unsigned int* rot = ctr + 1;
  double* Jp = J.p;
  long long ldx_a = ldx, ldj_a = ldj;
  int n_a = n;
  double tol_a = tol;
  void* args[] = {&X, &ldx_a, &Jp, &ldj_a, &n_a, &tol_a, &sweeps_cap, &bar, &rot, &done};
  URV_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(jacobi_sweeps), dim3(grid), dim3(JT), args, 0, st));
  count_launch();
  int h_done = 0;
  URV_CUDA(cudaMemcpyAsync(&h_done, done, sizeof(int), cudaMemcpyDeviceToHost, st));
  column_norms<<<ceil_div(static_cast<long long>(n) * 32, 256), 256, 0, st>>>(X, ldx, n, s.p);
  URV_CHECK_LAUNCH();
  sort_gather<<<dim3(std::max(1, std::min(8, ceil_div(n, 256))), n), 256, 0, st>>>(X, ldx, J.p, ldj, s.p, n, sigma, U,
                                                                                    ldu, W, ldw);
  URV_CHECK_LAUNCH();
  complete_basis<<<1, JT, 0, st>>>(U, ldu, n, sigma);
  URV_CHECK_LAUNCH();
  URV_CUDA(cudaStreamSynchronize(st));
  URV_CUDA(cudaFreeAsync(ctr, st));
  if (h_done < 0) {
    set_error("Jacobi SVD did not converge in %d sweeps (n = %d)", max_sweeps, n);
    throw CudaFailure{kCudaError};
  }
}

}  // namespace urv
