// Internal interface of the device Householder QR.
#pragma once
#include "dgemm.h"

namespace urv {

struct QrScratch {
  double* part1;  // [G]        per-CTA norm partials
  double* part2;  // [G * NB]   per-CTA dot-product partials
  double* x0;     // [1]        current diagonal entry
};

int qr_panel_width(long long m);

// Householder QR of the m x n (m >= n) column-major W (overwritten with R above
// and V below the diagonal).  Writes the explicit thin Q (m x n) to Q and, when
// R != nullptr, the upper-triangular R (exact zeros below).  When deficient !=
// nullptr, stores #{j : R(j,j) < eps * sqrt(*sumsq)} there (device pointers).
// ldw and ldq must be even.
void householder_qr_device(double* W, long long ldw, long long m, long long n, double* Q, long long ldq,
                           double* R, long long ldr, const double* sumsq, double* deficient,
                           cudaStream_t st, Workspace& ws);

}  // namespace urv
