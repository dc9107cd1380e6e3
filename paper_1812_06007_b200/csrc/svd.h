// Small dense SVD on the device (one-sided Jacobi), see svd.cu.
#pragma once

#include "common.cuh"
#include "dgemm.h"

namespace urv {

// X (n x n, ld ldx; destroyed) = U diag(sigma) W^T with sigma nonincreasing,
// U (n x n, ld ldu) and W (n x n, ld ldw) orthogonal.  Throws CudaFailure if the
// sweeps do not converge.  Synchronises `st`.
void jacobi_svd_device(double* X, long long ldx, int n, double* sigma, double* U, long long ldu, double* W,
                       long long ldw, cudaStream_t st);

}  // namespace urv
