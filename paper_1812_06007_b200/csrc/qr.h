// Internal interface of the device Householder QR.
#pragma once
#include "dgemm.h"

namespace urv {

struct QrScratch {
  double* payload;  // [2][clusters][NB + 8] cluster partials of the panel's grid exchanges
};

int qr_panel_width(long long m);
int debug_panel_cycles(double* out, int n);

// Householder QR of the m x n (m >= n) column-major W (overwritten with R above
// and V below the diagonal).  Writes the explicit thin Q (m x n) to Q and, when
// R != nullptr, the upper-triangular R (exact zeros below).  When deficient !=
// nullptr, stores #{j : R(j,j) < eps * sqrt(*sumsq)} there (device pointers).
// ldw and ldq must be even.
// When r_ready != nullptr, an event is recorded on st as soon as R is final (before the
// explicit-Q phase) so a caller can start copying R out while Q is being formed.
void householder_qr_device(double* W, long long ldw, long long m, long long n, double* Q, long long ldq,
                           double* R, long long ldr, const double* sumsq, double* deficient,
                           cudaStream_t st, Workspace& ws, cudaEvent_t r_ready = nullptr);

}  // namespace urv
