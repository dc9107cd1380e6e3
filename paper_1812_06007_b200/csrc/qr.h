// Internal interface of the device Householder QR.
#pragma once
#include "dgemm.h"

namespace urv {

struct QrScratch {
  double* payload;  // [2][clusters][NB + 8] cluster partials of the panel's grid exchanges
};

int qr_panel_width(long long m);
// Outer block width (trailing-update rank) the QR uses for an m x n matrix.
int outer_block_width(long long m, long long n);

// A QR left in compact-WY form: V below the diagonal of W (m x n), R on and above
// it, and the upper-triangular T of every 256-column outer block (H_p = I - V_p T_p V_p^T).
struct QrFactors {
  double* W = nullptr;
  long long ldw = 0, m = 0, n = 0;
  DevBuf Tall;
  int nb = 256;  // outer block width (T blocks are nb x nb, ld nb)
};

// Factor W in place (panels, trailing updates, look-ahead); optional deficiency count.
// E (m x ne, optional) is carried along as extra trailing columns: on return it holds
// Q_full^T E, applied block by block so that it keeps the GPU busy under the panels.
// tail_ev (optional) is recorded on st when the factorisation enters its last tail_blocks
// outer blocks, where the panel chain outlasts the shrinking trailing updates and the
// GPU has room for other work (power_urv starts the deferred V formation there).
void qr_factor(double* W, long long ldw, long long m, long long n, const double* sumsq, double* deficient,
               cudaStream_t st, Workspace& ws, QrFactors& out, double* E = nullptr, long long lde = 0,
               long long ne = 0, int nb_force = 0, cudaEvent_t tail_ev = nullptr, int tail_blocks = 0);
void qr_extract_r(const QrFactors& f, double* R, long long ldr, cudaStream_t st);
// Explicit thin Q (m x n).
void qr_form_q(const QrFactors& f, double* Q, long long ldq, cudaStream_t st, Workspace& ws);
// B (m x ncols) <- Q_full^T B, Q_full = H_0 ... H_{P-1} (m x m).
void qr_apply_qt_left(const QrFactors& f, double* B, long long ldb, long long ncols, cudaStream_t st, Workspace& ws);
// B (nrows x m) <- B Q_full.
void qr_apply_q_right(const QrFactors& f, double* B, long long ldb, long long nrows, cudaStream_t st,
                      Workspace& ws);
int debug_panel_cycles(double* out, int n);
// Factor W in place and write tau_j = T(j, j) (the LAPACK (V, tau) form; device pointers).
void qr_factor_tau(double* W, long long ldw, long long m, long long n, double* tau, cudaStream_t st, Workspace& ws);

// Distributed-QR building blocks (column-block-cyclic Householder, distributed.py):
// factor an m x k panel (k <= 256) in place and return its T; apply H^T / H of such
// a factored panel to m x ncols columns.
void geqrt_device(double* W, long long ldw, long long m, long long k, double* T, long long ldt, cudaStream_t st,
                  Workspace& ws);
void apply_block_reflector(const double* P, long long ldp, long long m, long long k, const double* T, long long ldt,
                           bool trans, double* C, long long ldc, long long ncols, cudaStream_t st, Workspace& ws);

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
