// Device building blocks of the rank-revealing profiles (see profile.cu).
#pragma once
#include "dgemm.h"

namespace urv {

// out[i] = sum_{j >= i} R(i, j)^2, i < n (device out).
void tail_sumsq_device(const double* R, long long ldr, long long n, double* out, cudaStream_t st);
// y = B x (trans = 0) or B^T x (trans = 1), B = R(k0:k0+N, k0:k0+N) upper triangular (device vectors).
void trmv_device(const double* R, long long ldr, long long k0, long long N, int trans, const double* x, double* y,
                 cudaStream_t st);
// X = R^{-1} (n x n, upper triangular; zeros below).  16-byte aligned, even leading dimensions.
void tri_inv_device(const double* R, long long ldr, long long n, double* X, long long ldx, cudaStream_t st,
                    Workspace& ws);

}  // namespace urv
