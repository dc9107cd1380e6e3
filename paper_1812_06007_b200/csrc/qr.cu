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

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

namespace urv {

namespace {

constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;
constexpr int LEAF = 64;   // columns per cooperative panel
constexpr int NBO = 256;   // columns per outer block (trailing-update rank)
constexpr int MAX_PANEL_CTAS = 148;  // grid cap of the cooperative panel (B200 SM count)
constexpr int PANEL_CLUSTER = 16;    // max CTAs per thread-block cluster of the panel (8 portable, 16 opt-in)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sums a[0..N) over the 32 lanes of a warp by recursive halving (N a power of two
// <= 32): lanes q*(32/N) .. q*(32/N) + 32/N - 1 return the total of a[q], i.e. the
// column is q = lane >> (5 - log2 N).  N=8 takes 9 shuffles instead of 40 for eight
// butterfly sums.  Fixed order, so every CTA derives the same bits.
template <int N>
__device__ __forceinline__ double reduce_scatter(const double (&a)[N], int lane) {
  double cur[N];
#pragma unroll
  for (int k = 0; k < N; ++k) cur[k] = a[k];
  int mask = 16;
#pragma unroll
  for (int width = N; width > 1; width >>= 1, mask >>= 1) {
    const bool hi = lane & mask;
#pragma unroll
    for (int k = 0; k < width / 2; ++k) {
      const double send = hi ? cur[k] : cur[k + width / 2];
      const double keep = hi ? cur[k + width / 2] : cur[k];
      cur[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
    }
  }
  double v = cur[0];
  for (; mask > 0; mask >>= 1) v += __shfl_xor_sync(0xffffffffu, v, mask);
  return v;
}

}  // namespace
}  // namespace urv
#include "panel_cl.cuh"
#include "apply_cl.cuh"
namespace urv {
namespace {

// Cooperative Householder panel (core.py:57-98 per column, core.py:101-109 for T).
//
// Register-resident: CTA c owns rows [c*RB, c*RB + RB), RB = 32*(RPL+SPL); warp w
// owns columns {w, w+8, ...} (CPW = NB/8 of them) and lane l owns rows {l, l+32, ...},
// so every panel value lives in exactly one thread for the whole factorisation: rows
// i < RPL in registers S[i][q], rows RPL <= i < RPL+SPL in this thread's slice of
// dynamic shared memory (taller CTAs = fewer SMs held by the latency-bound panel
// while the trailing update runs beside it).  Shared memory otherwise only carries
// v_j (vloc), this CTA's partial payload and, on CTA 0, T.
//
// One all-reduce per column (plus an exact fallback, see below).  The payload of
// PW doubles per CTA:
//   [0, NB)   s_k = v_j^T A(:, k) over rows >= j        (w for k >= j, V^T v_j for k < j)
//   NB+0..2   ||x||^2, v_j^T x, ||v_j||^2 over rows > j+1, x = column j+1 before the update
//   NB+3..4   A(j+1, j+1) and v_j(j+1) (owner CTA only; others add 0)
//   NB+5..6   exact sigma / x0 partials (fallback exchange only)
// gives column j+1's sigma and x0 without a second exchange:
//   c = tau_j s_{j+1},  sigma' = ||x||^2 - 2 c v^T x + c^2 ||v||^2,  x0' = A(j+1,j+1) - c v_j(j+1).
// If the expansion shows cancellation (sigma' < (||x||^2 + c^2 ||v||^2) / 2) -- the same
// decision in every CTA -- sigma is recomputed exactly by one more exchange.
//
// The all-reduce is hierarchical and fixed-order (bitwise deterministic):
//   CTA partial -> cluster of 8 CTAs via DSMEM (rank order) -> cluster leaders exchange
//   through global memory behind a grid barrier among leaders only -> every CTA sums
//   the cluster partials in cluster order.  A single-cluster grid needs no global step.
// Row i >= RPL of a thread: CPW doubles strided by the CTA size (conflict-free).
struct SmRow {
  static constexpr bool kGlobal = false;
  double* b;
  __device__ __forceinline__ double& operator[](int q) const { return b[q * PANEL_THREADS]; }
};
// Row i >= RPL+SPL of a thread in the tall-panel variant (GROWS): the value stays in the
// panel matrix in global memory (L2) and is re-read every pass.  Cells outside the
// panel (rows >= M, columns >= ncols) alias a thread-local zero so no pass reads or
// writes memory that is not the panel's.
struct GmRow {
  static constexpr bool kGlobal = true;
  double* b;          // P + row + warp * ldp, or nullptr for a row past the panel
  long long stride;   // PANEL_WARPS * ldp (column q of this warp)
  int qmax;           // columns warp + 8q < ncols
  double* sink;
  __device__ __forceinline__ double& operator[](int q) const { return (b && q < qmax) ? b[q * stride] : *sink; }
};
template <class Row>
__device__ __forceinline__ constexpr bool row_is_global(const Row&) {
  return Row::kGlobal;
}
template <int N>
__device__ __forceinline__ constexpr bool row_is_global(const double (&)[N]) {
  return false;
}

template <int NB, int RPL, int SPL, bool GROWS>
__global__ void __launch_bounds__(PANEL_THREADS, 1)
    panel_geqr2(double* __restrict__ P, long long ldp, int M, int ncols, double* __restrict__ Tout, int ldt,
                double* __restrict__ Vout, long long ldv, int vzero_rows,
                double* __restrict__ gpay, unsigned int* __restrict__ counter,
                unsigned long long* __restrict__ prof, int exact_sigma, int gpl) {
  constexpr int CPW = NB / PANEL_WARPS;  // columns per warp
  constexpr int PW = NB + 8;             // payload doubles per CTA
  constexpr int RT = RPL + SPL;          // rows per lane held on chip
  constexpr int CHAINS = 32 / CPW;       // lanes summing one column
  // rows per CTA: RT per lane on chip, plus gpl per lane in global memory (GROWS only)
  const int RB = 32 * (RT + (GROWS ? gpl : 0));
  __shared__ double vloc_s[GROWS ? 1 : 32 * RT];
  __shared__ __align__(16) double pay[2][PW];
  __shared__ double T[NB * NB];          // CTA 0: Gram columns, then T
  __shared__ double taus[NB];
  __shared__ double red[PANEL_WARPS];
  __shared__ double pred[4];

  cg::cluster_group cl = cg::this_cluster();
  const int csz = static_cast<int>(cl.num_blocks());
  const int crank = static_cast<int>(cl.block_rank());
  const int G = gridDim.x, c = blockIdx.x;
  const int cid = c / csz, NCL = G / csz;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = c * RB;
  const int nrows = max(0, min(RB, M - r0));
  int ex = 0;

  // ---- load: row i, column q = A(r0 + lane + 32 i, warp + 8 q) ----
  double S[RPL][CPW];
  extern __shared__ double panel_dsm[];  // SPL * CPW * PANEL_THREADS doubles (+ vloc when GROWS)
  double* vloc = GROWS ? panel_dsm + SPL * CPW * PANEL_THREADS : vloc_s;
  double sink = 0.0;
  const int gqmax = (ncols - warp + PANEL_WARPS - 1) / PANEL_WARPS;
  auto for_rows = [&](auto&& body) {
#pragma unroll
    for (int i = 0; i < RPL; ++i) body(i, S[i]);
#pragma unroll
    for (int i = 0; i < SPL; ++i) body(RPL + i, SmRow{panel_dsm + i * CPW * PANEL_THREADS + tid});
    if constexpr (GROWS) {
#pragma unroll 1
      for (int i = RT; i < RT + gpl; ++i) {
        const int r = lane + 32 * i;
        double* b = (r < nrows) ? P + (r0 + r) + static_cast<long long>(warp) * ldp : nullptr;
        body(i, GmRow{b, PANEL_WARPS * ldp, gqmax, &sink});
      }
    }
  };
  for_rows([&](int i, auto&& row) {
    if (row_is_global(row)) return;  // already in place
    const int r = lane + 32 * i;
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int col = warp + q * PANEL_WARPS;
      row[q] = (col < ncols && r < nrows) ? P[(r0 + r) + static_cast<long long>(col) * ldp] : 0.0;
    }
  });
  if (c == 0)
    for (int k = tid; k < NB * NB; k += PANEL_THREADS) T[k] = 0.0;

  // row[q] with a run-time q (unrolled select keeps S in registers)
  auto colval = [&](auto&& row, int qsel) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < CPW; ++q)
      if (q == qsel) x = row[q];
    return x;
  };

  // All-reduce of pay[ex & 1] (filled by this CTA, visible after __syncthreads).
  // Multi-cluster: each cluster leader sums its 8 CTAs' partials over DSMEM and
  // writes the cluster partial to global memory (double-buffered by exchange
  // parity); the leaders then meet at a grid barrier (relaxed spin + one acquire
  // fence) and a second cluster barrier releases the other CTAs.  A single-cluster
  // grid reads its peers' partials straight from DSMEM.  The sums are read with
  // csum_part() / csum5_warp() until the next exchange.
  const double* gin = nullptr;
  unsigned int bar_target = 0;
  auto exchange = [&]() {
    const int b = ex & 1;
    cl.sync();
    if (NCL > 1) {
      double* gout = gpay + static_cast<long long>(b) * NCL * PW;
      bar_target += NCL;
      if (crank == 0) {  // leader: cluster partial -> global, then arrive (release)
        if (tid < PW) {
          double v[PANEL_CLUSTER];
#pragma unroll
          for (int r = 0; r < PANEL_CLUSTER; ++r) v[r] = r < csz ? *cl.map_shared_rank(&pay[b][tid], r) : 0.0;
          double sv = 0.0;
#pragma unroll
          for (int r = 0; r < PANEL_CLUSTER; ++r) sv += v[r];
          __stcg(gout + cid * PW + tid, sv);
        }
        __syncthreads();
        if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
      }
      // every CTA waits for all leaders itself (no second cluster barrier)
      if (tid == 0) {
        unsigned int v;
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        } while (v < bar_target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
      gin = gout;
    }
    ++ex;
  };
  // Fixed-order total of payload slot k over the grid, computed by this lane's
  // chain h in [0, nch); lanes of one chain group are combined by the caller.
  auto csum_part = [&](int k, int h, int nch) {
    double sv = 0.0;
    const int b = (ex - 1) & 1;
    if (NCL > 1) {
      constexpr int PER = (MAX_PANEL_CTAS / 8 + 3) / 4 + 1;  // >= max clusters / chains
      double v[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int cc = h + nch * u;
        v[u] = cc < NCL ? ld_cg(gin + cc * PW + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) sv += v[u];
    } else {
      double v[PANEL_CLUSTER];
#pragma unroll
      for (int u = 0; u < PANEL_CLUSTER; ++u) {
        const int r = h + nch * u;
        v[u] = r < csz ? *cl.map_shared_rank(&pay[b][k], r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PANEL_CLUSTER; ++u) sv += v[u];
    }
    return sv;
  };
  // Five consecutive slots k..k+4 at once (one batch of loads), full warp totals.
  auto csum5_warp = [&](int k, double* outv) {
    double sv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int b = (ex - 1) & 1;
    if (NCL > 1) {
      constexpr int PER = MAX_PANEL_CTAS / 8 / 32 + 1;
      double v[5][PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int cc = lane + 32 * u;
#pragma unroll
        for (int f = 0; f < 5; ++f) v[f][u] = cc < NCL ? ld_cg(gin + cc * PW + k + f) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PER; ++u)
#pragma unroll
        for (int f = 0; f < 5; ++f) sv[f] += v[f][u];
    } else if (lane < csz) {
      double v[5];
#pragma unroll
      for (int f = 0; f < 5; ++f) v[f] = *cl.map_shared_rank(&pay[b][k + f], lane);
#pragma unroll
      for (int f = 0; f < 5; ++f) sv[f] = v[f];
    }
#pragma unroll
    for (int f = 0; f < 5; ++f) outv[f] = warp_sum(sv[f]);
  };
  // Full fixed-order total of slot k by one warp (all lanes get the same bits).
  auto csum_warp = [&](int k) {
    double sv = csum_part(k, lane, 32);
    return warp_sum(sv);
  };

  // Exact sigma = ||A(col+1:, col)||^2 and x0 = A(col, col) via one exchange.
  auto exact_norm = [&](int col, double& sigma, double& x0) {
    if (warp == col % PANEL_WARPS) {
      const int qc = col / PANEL_WARPS;
      double sv = 0.0, xv = 0.0;
      for_rows([&](int i, auto&& row) {
        const int r = lane + 32 * i;
        const double x = colval(row, qc);
        if (r < nrows && r0 + r > col) sv += x * x;
        if (r < nrows && r0 + r == col) xv = x;
      });
      sv = warp_sum(sv);
      xv = warp_sum(xv);  // a single nonzero term
      if (lane == 0) {
        pay[ex & 1][NB + 5] = sv;
        pay[ex & 1][NB + 6] = xv;
      }
    }
    __syncthreads();
    exchange();
    sigma = csum_warp(NB + 5);
    x0 = csum_warp(NB + 6);
  };

  double sigma, x0;
  exact_norm(0, sigma, x0);
  const bool timing = prof != nullptr && tid == 0 && (c == 0 || c == G - 1);
  unsigned long long tph[6] = {0, 0, 0, 0, 0, 0}, tlast = timing ? clock64() : 0;
  unsigned long long nfallback = 0;
  auto tick = [&](int k) {
    if (timing) {
      const unsigned long long now = clock64();
      tph[k] += now - tlast;
      tlast = now;
    }
  };

  for (int j = 0; j < ncols; ++j) {
    // Reflector (identical in every CTA): core.py:57-76
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
    const int qj = j / PANEL_WARPS;
    const double rv0 = 1.0 / v0;
    if (warp == j % PANEL_WARPS) {  // v over this CTA's rows: 0 above j, 1 at j, x/v0 (or x) below
      for_rows([&](int i, auto&& row) {
        const int r = lane + 32 * i;
        const int gi = r0 + r;
        const double x = colval(row, qj);
        double v = 0.0;
        if (r < nrows) {
          if (gi == j) v = 1.0;
          else if (gi > j) v = flat ? x : x * rv0;
        }
        vloc[r] = v;
      });
    }
    __syncthreads();
    tick(0);

    // ---- this CTA's partials of the payload ----
    const int jn = j + 1;
    const int nwarp = jn % PANEL_WARPS, qn = jn / PANEL_WARPS;
    const int b = ex & 1;
    {
      double acc[CPW];
#pragma unroll
      for (int q = 0; q < CPW; ++q) acc[q] = 0.0;
      // v is read from vloc (zero above row j and past nrows) rather than cached in
      // registers: the taller variants need those registers for the panel itself
      for_rows([&](int i, auto&& row) {
        const double v = vloc[lane + 32 * i];
#pragma unroll
        for (int q = 0; q < CPW; ++q) acc[q] += v * row[q];
      });
      // recursive-halving reduce-scatter: lanes (32/CPW)q .. hold column q's sum
      {
        const double sv = reduce_scatter<CPW>(acc, lane);
        if ((lane & (32 / CPW - 1)) == 0) pay[b][warp + (lane / (32 / CPW)) * PANEL_WARPS] = sv;
      }
      if (warp == nwarp && jn < ncols) {
        double ex_x = 0.0, ex_p = 0.0, ex_v = 0.0, own_a = 0.0, own_v = 0.0;
        for_rows([&](int i, auto&& row) {
          const int r = lane + 32 * i;
          const double x = colval(row, qn);
          const double v = vloc[r];
          if (r < nrows && r0 + r > jn) {
            ex_x += x * x;
            ex_p += v * x;
            ex_v += v * v;
          }
          if (r < nrows && r0 + r == jn) {
            own_a = x;
            own_v = v;
          }
        });
        ex_x = warp_sum(ex_x);
        ex_p = warp_sum(ex_p);
        ex_v = warp_sum(ex_v);
        own_a = warp_sum(own_a);  // a single nonzero term
        own_v = warp_sum(own_v);
        if (lane == 0) {
          pay[b][NB + 0] = ex_x;
          pay[b][NB + 1] = ex_p;
          pay[b][NB + 2] = ex_v;
          pay[b][NB + 3] = own_a;
          pay[b][NB + 4] = own_v;
        }
      }
    }
    __syncthreads();
    tick(1);
    exchange();
    tick(2);

    // ---- grid sums of this warp's columns: lane = (column q, chain h) ----
    // The warp owning column j+1 fetches the five extras in the same batch of loads.
    double wcol[CPW];
    double sv;
    const bool predict = (jn < ncols && warp == nwarp);
    double e5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    {
      const int q = lane % CPW, h = lane / CPW;
      if (predict && NCL > 1) {
        constexpr int PER5 = MAX_PANEL_CTAS / 8 / 32 + 1;
        double xv[5][PER5];
#pragma unroll
        for (int u = 0; u < PER5; ++u) {
          const int cc = lane + 32 * u;
#pragma unroll
          for (int f = 0; f < 5; ++f) xv[f][u] = cc < NCL ? ld_cg(gin + cc * PW + NB + f) : 0.0;
        }
        sv = csum_part(warp + q * PANEL_WARPS, h, CHAINS);
#pragma unroll
        for (int u = 0; u < PER5; ++u)
#pragma unroll
          for (int f = 0; f < 5; ++f) e5[f] += xv[f][u];
#pragma unroll
        for (int f = 0; f < 5; ++f) e5[f] = warp_sum(e5[f]);
      } else {
        sv = csum_part(warp + q * PANEL_WARPS, h, CHAINS);
        if (predict) csum5_warp(NB, e5);
      }
#pragma unroll
      for (int o = CPW; o < 32; o <<= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq) wcol[qq] = __shfl_sync(0xffffffffu, sv, qq);
    }
    // The warp owning column j+1 predicts its sigma and x0 (identical in every CTA).
    if (predict) {
      const double pX = e5[0], pP = e5[1], pV = e5[2], pA = e5[3], pJ = e5[4];
      double sj = 0.0;
#pragma unroll
      for (int qq = 0; qq < CPW; ++qq)
        if (qq == qn) sj = wcol[qq];
      const double cc = tau * sj;
      const double sig = pX - 2.0 * cc * pP + cc * cc * pV;
      const bool ok = !exact_sigma && ((tau == 0.0) || (sig >= 0.5 * (pX + cc * cc * pV) && isfinite(sig)));
      if (lane == 0) {
        pred[0] = (tau == 0.0) ? pX : sig;
        pred[1] = (tau == 0.0) ? pA : pA - pJ * cc;
        pred[2] = ok ? 1.0 : 0.0;
      }
    }
    tick(3);
    // CTA 0 keeps the Gram column V(:, :j)^T v_j for T (lane q < CPW holds column warp + 8q).
    if (c == 0 && lane < CPW) {
      const int col = warp + lane * PANEL_WARPS;
      if (col < j) T[j * NB + col] = sv;
    }

    // Rank-1 update of columns k >= j over rows i >= j: A(i,k) -= v_i * tau * s_k
    if (tau != 0.0) {
      for_rows([&](int i, auto&& row) {
        const int r = lane + 32 * i;
        const double v = vloc[r];
        if (r < nrows && r0 + r >= j) {
          // load the whole row first: for shared-memory rows this issues the loads
          // back to back instead of a load/store chain per element
          double x[CPW];
#pragma unroll
          for (int q = 0; q < CPW; ++q) x[q] = row[q];
#pragma unroll
          for (int q = 0; q < CPW; ++q) {
            const int col = warp + q * PANEL_WARPS;
            if (col >= j && col < ncols) x[q] -= v * (tau * wcol[q]);
          }
#pragma unroll
          for (int q = 0; q < CPW; ++q) row[q] = x[q];
        }
      });
    }
    // Column j: R(j,j) stays on row j; v is stored below it (LAPACK-style V storage).
    if (warp == j % PANEL_WARPS) {
      for_rows([&](int i, auto&& row) {
        const int r = lane + 32 * i;
        if (r < nrows && r0 + r > j) {
          const double v = vloc[r];
#pragma unroll
          for (int q = 0; q < CPW; ++q)
            if (q == qj) row[q] = v;
        }
      });
    }
    __syncthreads();
    tick(4);
    if (jn < ncols) {
      if (pred[2] != 0.0) {
        sigma = pred[0];
        x0 = pred[1];
      } else {
        exact_norm(jn, sigma, x0);  // cancellation: recompute from the updated column
        ++nfallback;
      }
    }
    tick(5);
  }
  if (timing) {
    const int slot = (c == 0) ? 0 : 8;
#pragma unroll
    for (int k = 0; k < 6; ++k) atomicAdd(prof + slot + k, tph[k]);
    atomicAdd(prof + slot + 6, static_cast<unsigned long long>(ncols));
    atomicAdd(prof + slot + 7, c == 0 ? nfallback : static_cast<unsigned long long>(G));
  }

  // ---- write back: R on/above the diagonal, V below it ----
  for_rows([&](int i, auto&& row) {
    const int r = lane + 32 * i;
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int col = warp + q * PANEL_WARPS;
      if (col < ncols && r < nrows) {
        const int gi = r0 + r;
        P[gi + static_cast<long long>(col) * ldp] = row[q];
        // the explicit unit-lower V for the compact-WY updates (replaces a load_v pass)
        if (Vout) Vout[gi + static_cast<long long>(col) * ldv] = gi < col ? 0.0 : (gi == col ? 1.0 : row[q]);
      }
    }
  });
  if (Vout && c == 0)  // rows of the outer block above this leaf: V is zero there
    for (int idx = tid; idx < vzero_rows * ncols; idx += PANEL_THREADS)
      Vout[-vzero_rows + idx % vzero_rows + static_cast<long long>(idx / vzero_rows) * ldv] = 0.0;
  cl.sync();  // keep every CTA's shared memory alive until the leaders' DSMEM reads are done
  if (c != 0) return;

  // ---- CTA 0: T from the Gram columns (core.py:101-109), in place ----
  // T(:j, j) = -tau_j T(:j, :j) g_j, T(j, j) = tau_j; column j holds g_j = V(:, :j)^T v_j
  // above the diagonal until it is overwritten.
  __syncthreads();
  {
    constexpr int NP = PANEL_THREADS / NB;  // partial sums per row of T
    __shared__ double tp[NP][NB];
    const int r = tid % NB, p = tid / NB;
    for (int j = 0; j < ncols; ++j) {
      double s2 = 0.0;
      if (r < j)
        for (int l = r + p; l < j; l += NP) s2 += T[l * NB + r] * T[j * NB + l];
      tp[p][r] = s2;
      __syncthreads();
      if (tid < j) {
        double tot = 0.0;
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) tot += tp[pp][tid];
        T[j * NB + tid] = -taus[j] * tot;
      }
      if (tid == 0) T[j * NB + j] = taus[j];
      __syncthreads();
    }
  }
  for (int k = tid; k < NB * NB; k += PANEL_THREADS) {
    const int r = k % NB, col = k / NB;
    Tout[r + static_cast<long long>(col) * ldt] = (r <= col && col < ncols) ? T[k] : 0.0;
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
  constexpr int CC = 8;  // columns per CTA
  __shared__ double Ts[64 * 64];
  __shared__ double Ws[64 * CC];
  const int tid = threadIdx.x;
  for (int i = tid; i < nb * nb; i += blockDim.x) Ts[i] = T[(i % nb) + (i / nb) * ldt];
  const int c0 = blockIdx.x * CC;
  const int cols = min(CC, N - c0);
  for (int i = tid; i < nb * CC; i += blockDim.x) {
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

// Fixed-order pairwise (binary-tree) sum of split-K partials, for the accurate mode:
// the rounding of a long-K product then grows with log(splits), not with splits.
__device__ __forceinline__ double tree_sum(const double* p, long long stride, int n) {
  double v[64];
#pragma unroll 1
  for (int z = 0; z < n; ++z) v[z] = p[z * stride];
#pragma unroll 1
  for (int w = 1; w < n; w <<= 1)
#pragma unroll 1
    for (int z = 0; z + w < n; z += 2 * w) v[z] += v[z + w];
  return v[0];
}

__global__ void sum_partials_tree(const double* __restrict__ part, long long ldp, long long pstride, int splits,
                                  int nb, int N, double* __restrict__ out, long long ldo) {
  const long long total = static_cast<long long>(nb) * N;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx % nb);
    const long long col = idx / nb;
    out[r + col * ldo] = tree_sum(part + r + col * ldp, pstride * ldp, splits);
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

// Debug hook: URV_PANEL_PROF=1 makes every panel launch accumulate per-phase
// clock64 cycles (CTA 0 and the last CTA) into a device buffer read by
// urv_debug_panel_cycles().  Off (nullptr) by default.
unsigned long long* g_prof[64] = {nullptr};
unsigned long long* panel_prof_buffer() {
  static const bool on = getenv("URV_PANEL_PROF") != nullptr;
  if (!on) return nullptr;
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (!g_prof[dev & 63]) {
    URV_CUDA(cudaMalloc(reinterpret_cast<void**>(&g_prof[dev & 63]), 16 * sizeof(unsigned long long)));
    URV_CUDA(cudaMemset(g_prof[dev & 63], 0, 16 * sizeof(unsigned long long)));
  }
  return g_prof[dev & 63];
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

int panel_cluster_size() {
  static const int v = env_int("URV_PANEL_CLUSTER", 8) >= 16 ? 16 : 8;
  return v;
}

template <int NB, int SPL>
constexpr int panel_dyn_smem() {
  return SPL * (NB / PANEL_WARPS) * PANEL_THREADS * static_cast<int>(sizeof(double));
}
// Dynamic shared memory of a launch: the shared-memory rows, plus v for every row of
// the CTA in the tall-panel (GROWS) variant, whose row count is a launch parameter.
template <int NB, int RPL, int SPL, bool GROWS>
int panel_dyn_bytes(int gpl) {
  return panel_dyn_smem<NB, SPL>() + (GROWS ? 32 * (RPL + SPL + gpl) * static_cast<int>(sizeof(double)) : 0);
}

// Per-device one-time function attributes (non-portable cluster size, dynamic smem:
// everything the device allows beside the static shared memory for GROWS).
template <int NB, int RPL, int SPL, bool GROWS>
int panel_attrs() {
  static unsigned mask = 0;
  static int max_dyn[64] = {0};
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (mask & (1u << dev)) return max_dyn[dev & 63];
  auto kern = panel_geqr2<NB, RPL, SPL, GROWS>;
  if (panel_cluster_size() > 8) URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  int dyn = panel_dyn_smem<NB, SPL>();
  if (GROWS) {
    cudaFuncAttributes fa;
    URV_CUDA(cudaFuncGetAttributes(&fa, kern));
    dyn = device_info().max_smem_optin - static_cast<int>(fa.sharedSizeBytes);
  }
  if (dyn > 0) URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  max_dyn[dev & 63] = dyn;
  mask |= 1u << dev;
  return dyn;
}

template <int NB, int RPL, int SPL, bool GROWS>
void launch_panel_v(double* P, long long ldp, int M, int ncols, double* T, int ldt, double* Vout, long long ldv,
                    int vzero_rows, QrScratch& scr, unsigned int* counter, cudaStream_t st, int G, int gpl) {
  panel_attrs<NB, RPL, SPL, GROWS>();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(PANEL_THREADS);
  cfg.dynamicSmemBytes = panel_dyn_bytes<NB, RPL, SPL, GROWS>(gpl);
  cfg.stream = st;
  // Plain cluster launch: the spin barrier among cluster leaders needs every
  // cluster co-resident, which launch_panel guarantees by capping the grid at
  // cudaOccupancyMaxActiveClusters (one CTA per SM; nothing else is resident on
  // this stream while the panel runs).
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = panel_cluster_size();
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  unsigned long long* prof = panel_prof_buffer();
  static const int exact_sigma = env_int("URV_PANEL_EXACT", 0);
  URV_CUDA(cudaLaunchKernelEx(&cfg, panel_geqr2<NB, RPL, SPL, GROWS>, P, ldp, M, ncols, T, ldt, Vout, ldv,
                              vzero_rows, scr.payload, counter, prof, exact_sigma, gpl));
  count_launch();
}

// Maximum co-resident clusters of one panel variant at a given dynamic shared memory
// size (queried once per device and size).
template <int NB, int RPL, int SPL, bool GROWS>
int panel_max_clusters_v(int gpl) {
  static int cache[64] = {0};
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (GROWS || !cache[dev & 63]) {
    const int max_dyn = panel_attrs<NB, RPL, SPL, GROWS>();
    if (GROWS && panel_dyn_bytes<NB, RPL, SPL, GROWS>(gpl) > max_dyn) return 0;
    const int csz = panel_cluster_size();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csz * 8);
    cfg.blockDim = dim3(PANEL_THREADS);
    cfg.dynamicSmemBytes = panel_dyn_bytes<NB, RPL, SPL, GROWS>(gpl);
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = csz;
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = 1;
    cfg.attrs = &a;
    cfg.numAttrs = 1;
    int n = 0;
    URV_CUDA(cudaOccupancyMaxActiveClusters(&n, panel_geqr2<NB, RPL, SPL, GROWS>, &cfg));
    if (GROWS) return std::max(0, n);
    cache[dev & 63] = std::max(1, n);
  }
  return cache[dev & 63];
}

struct PanelVariant {
  int nb, rpl, spl;  // leaf width, register rows and shared-memory rows per lane
  void (*launch)(double*, long long, int, int, double*, int, double*, long long, int, QrScratch&, unsigned int*,
                 cudaStream_t, int, int);
  int (*max_clusters)(int);
};
#define URV_PANEL_VARIANT(NB, R, S) \
  {NB, R, S, launch_panel_v<NB, R, S, false>, panel_max_clusters_v<NB, R, S, false>}
// ascending rows per lane within each leaf width
const PanelVariant kPanelVariants[] = {
    URV_PANEL_VARIANT(64, 1, 0),  URV_PANEL_VARIANT(64, 2, 0),  URV_PANEL_VARIANT(64, 4, 0),
    URV_PANEL_VARIANT(64, 5, 0),  URV_PANEL_VARIANT(64, 6, 0),  URV_PANEL_VARIANT(64, 6, 2),
    URV_PANEL_VARIANT(64, 6, 6),  URV_PANEL_VARIANT(64, 6, 10), URV_PANEL_VARIANT(32, 8, 0),
    URV_PANEL_VARIANT(32, 12, 0), URV_PANEL_VARIANT(32, 16, 0), URV_PANEL_VARIANT(32, 16, 8),
    URV_PANEL_VARIANT(32, 16, 20)};
#undef URV_PANEL_VARIANT
// Panels taller than every on-chip variant (about 138k rows at 64 columns):
// 16 register rows per lane on chip, the rest of each CTA's rows re-read from global
// memory (L2) every pass.  Slower per column, no row limit short of shared memory for v.
const PanelVariant kTallVariants[] = {
    {64, 6, 0, launch_panel_v<64, 6, 0, true>, panel_max_clusters_v<64, 6, 0, true>},
    {32, 16, 0, launch_panel_v<32, 16, 0, true>, panel_max_clusters_v<32, 16, 0, true>}};

// Leaf width for an M-row panel: 64 while 64 columns fit the co-resident clusters
// (15 on this B200) at the tallest 64-wide variant (16 rows per lane), else 32.
// In a tall factorisation (m >= 2n) the trailing updates are thin and the panel chain is
// exposed, so panels above 8192 rows use 32-wide leaves (shorter per-leaf chain): config 3
// 522.5 / 522.1 -> 514.8 / 513.2 ms; for square ones 64 stays (config 4 2993 ms vs 2977 / 3051
// with 32, noisy) -- profiles/r01_leaf_width.log.  URV_LEAF32_ROWS overrides the threshold.
int panel_leaf_width(long long M, long long m_total, long long n_total) {
  // Round 2: leaves of up to 7168 rows run 64 wide on the single-cluster panel; above that the
  // cooperative panel is faster per column at 32 columns (3.3 vs 6 us) and that now wins for
  // square factorisations as well (config 4 2865.9 -> 2846.5 ms, config 5 164.5 -> 164.0 s:
  // profiles/r02_tune_c4.log).  URV_LEAF32_ROWS overrides the threshold.
  (void)m_total;
  (void)n_total;
  static const int force = env_int("URV_LEAF32_ROWS", -1);
  const long long thresh = force >= 0 ? force : 7168;
  return M > thresh ? 32 : 64;
}

// ---- single-cluster panel (panel_cl.cuh) ----
struct ClVariant {
  int rt;  // rows per lane
  void (*launch)(int, double*, long long, int, int, double*, int, double*, long long, int, cudaStream_t);
};
template <int RTR, int RTS>
void launch_cl_v(int csz, double* P, long long ldp, int M, int ncols, double* T, int ldt, double* Vout,
                 long long ldv, int vzero_rows, cudaStream_t st) {
  auto kern = panel_cl<RTR, RTS>;
  static unsigned mask = 0;
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (!(mask & (1u << dev))) {
    URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    URV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, panel_cl_smem_bytes<RTR, RTS>()));
    mask |= 1u << dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csz);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = panel_cl_smem_bytes<RTR, RTS>();
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = csz;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  // bit 0: exact sigma every column; bits 1-2: URV_CL_LAZY (0, 1, 2: where a step's lazy work sits, panel_cl.cuh)
  static const int exact_sigma = (env_int("URV_PANEL_EXACT", 0) ? 1 : 0) | ((env_int("URV_CL_LAZY", 0) & 3) << 1);
  URV_CUDA(cudaLaunchKernelEx(&cfg, kern, P, ldp, M, ncols, T, ldt, Vout, ldv, vzero_rows, exact_sigma,
                              panel_prof_buffer()));
  count_launch();
}
const ClVariant kClVariants[] = {{1, launch_cl_v<1, 0>}, {2, launch_cl_v<2, 0>},  {4, launch_cl_v<4, 0>},
                                 {6, launch_cl_v<6, 0>}, {8, launch_cl_v<6, 2>},  {10, launch_cl_v<6, 4>},
                                 {12, launch_cl_v<6, 6>}, {14, launch_cl_v<6, 8>}};
constexpr int kClMaxRt = 14;

// The single-cluster panel takes leaves of up to 64 columns whose rows fit one cluster:
// CL_MAXC CTAs x 32 lanes x 14 rows = 7168 rows.  URV_PANEL_CL=0 disables it; URV_CL_CSZ
// forces the cluster size (1, 2, 4, 8, 16), URV_CL_MAXC caps it.
bool launch_panel_cl(double* P, long long ldp, int M, int ncols, double* T, int ldt, double* Vout, long long ldv,
                     int vzero_rows, cudaStream_t st) {
  static const bool on = env_int("URV_PANEL_CL", 1) != 0;
  static const int force_csz = env_int("URV_CL_CSZ", 0);
  static const int maxc = std::min(CL_MAXC, std::max(1, env_int("URV_CL_MAXC", CL_MAXC)));
  if (!on || ncols > CL_NB || M > maxc * 32 * kClMaxRt) return false;
  // 16 CTAs (fewest rows per lane) unless forced to 8; the lazy reduction needs 8 or 16
  int csz = (force_csz == 8 || maxc < 16) ? 8 : 16;
  if (ceil_div(M, 32 * csz) > kClMaxRt) csz = 16;
  if (csz > maxc || ceil_div(M, 32 * csz) > kClMaxRt) return false;
  const int rt_need = ceil_div(M, 32 * csz);
  for (const ClVariant& v : kClVariants) {
    if (v.rt >= rt_need) {
      const double fl = 2.0 * M * ncols * ncols - 2.0 / 3.0 * ncols * ncols * ncols;
      StatsScope scope(st, kKPanel, fl, 16.0 * M * ncols);
      v.launch(csz, P, ldp, M, ncols, T, ldt, Vout, ldv, vzero_rows, st);
      return true;
    }
  }
  return false;
}

// Rows per lane for an M-row panel: the fewest that fit URV_PANEL_CLUSTERS clusters
// (default 6: the panel is latency-bound, so beyond that extra SMs mostly take work
// away from the concurrent trailing update -- config 4 measured 3.15 s at 13
// clusters, 3.06 s at 8, 3.04 s at 6 and 4; profiles/r01_panel_clusters.log), within
// the co-resident cap.  URV_PANEL_RPL forces a total rows-per-lane.
void launch_panel(double* P, long long ldp, int M, int ncols, double* T, int ldt, double* Vout, long long ldv,
                  int vzero_rows, QrScratch& scr, unsigned int* counter, cudaStream_t st, long long n_total) {
  if (launch_panel_cl(P, ldp, M, ncols, T, ldt, Vout, ldv, vzero_rows, st)) return;
  static const int force = env_int("URV_PANEL_RPL", 0);
  // Clusters for the panel grid: the latency-bound panel of a small factorisation likes more
  // CTAs (fewer rows per lane); in a large one extra SMs mostly take work from the concurrent
  // trailing update.  Measured (profiles/r01_panel_clusters2.log): 4000^2 161.3 ms at 8 vs
  // 163.5 at 6; 16384^2 2996.3 at 4-5 vs 3001.2 at 6 and 3019.1 at 8.
  static const int force_target = env_int("URV_PANEL_CLUSTERS", 0);
  const int target = force_target > 0 ? force_target : (n_total <= 8192 ? 8 : 5);
  const int csz = panel_cluster_size();
  const int NB = ncols > 32 ? 64 : 32;
  auto nclusters = [&](int rt) { return ceil_div(ceil_div(M, 32 * rt), csz); };
  const PanelVariant* pick = nullptr;
  for (int pass = 0; pass < 2 && !pick; ++pass) {
    for (const PanelVariant& v : kPanelVariants) {
      if (v.nb != NB) continue;
      const int rt = v.rpl + v.spl;
      const int cap = std::min(MAX_PANEL_CTAS / csz, v.max_clusters(0));
      const bool ok = pass == 0 ? (force ? (rt == force && nclusters(rt) <= cap) : nclusters(rt) <= std::min(target, cap))
                                : nclusters(rt) <= cap;
      if (ok) {
        pick = &v;
        break;
      }
    }
  }
  const double fl = 2.0 * M * ncols * ncols - 2.0 / 3.0 * ncols * ncols * ncols;
  if (!pick) {  // taller than every on-chip variant: rows beyond the chip stay in L2/HBM
    for (const PanelVariant& v : kTallVariants) {
      if (v.nb != NB) continue;
      const int rt = v.rpl + v.spl;
      int ncl = std::min(MAX_PANEL_CTAS / csz, v.max_clusters(0));
      for (; ncl >= 1; --ncl) {
        const int G = ncl * csz;
        const int gpl = std::max(0, ceil_div(M, 32LL * G) - rt);
        if (v.max_clusters(gpl) >= ncl) {
          StatsScope scope(st, kKPanel, fl, 16.0 * M * ncols);
          v.launch(P, ldp, M, ncols, T, ldt, Vout, ldv, vzero_rows, scr, counter, st, G, gpl);
          return;
        }
      }
    }
    set_error("householder panel of %d rows x %d columns exceeds the device (shared memory for v of every "
              "row: at most about %d rows)", M, ncols, 18 * 8 * 32 * 800);
    throw CudaFailure{kUnsupported};
  }
  const int G = nclusters(pick->rpl + pick->spl) * csz;
  StatsScope scope(st, kKPanel, fl, 16.0 * M * ncols);
  pick->launch(P, ldp, M, ncols, T, ldt, Vout, ldv, vzero_rows, scr, counter, st, G, 0);
}

// Fused C <- C - V op(T) V^T C for a narrow block (apply_cl.cuh): nb <= 64 and at most
// URV_FUSED_ROWS rows (default 8192: up to two staged chunks per CTA; beyond that the
// split-K GEMM chain is the better tool).  URV_FUSED_APPLY=0 disables it.
long long fused_apply_max_rows() {  // 0: disabled
  static const bool on = env_int("URV_FUSED_APPLY", 1) != 0;
  static const int max_rows = env_int("URV_FUSED_ROWS", 8192);
  return on ? max_rows : 0;
}
// leafw < nb: V holds several leaves (explicit zeros above each leaf's diagonal) whose block
// reflectors, with their T's on the diagonal of T, are applied one after the other inside the
// kernel while the strip of C stays in shared memory (at most 16 x 256 rows).
bool fused_block_apply(const double* V, long long ldv, const double* T, int ldt, bool trans, double* C,
                       long long ldc, long long M, int nb, long long N, cudaStream_t st, int leafw = 0) {
  if (leafw <= 0 || leafw > nb) leafw = nb;
  if (leafw > 64 || nb < 1 || N <= 0 || M <= 0 || M > fused_apply_max_rows()) return false;
  if (leafw < nb && M > 16 * AP_CH) return false;
  const long long strips = (N + AP_NS - 1) / AP_NS;
  if (strips > 65535) return false;
  int cs = 1;
  while (cs < 16 && ceil_div(M, cs) > AP_CH) cs *= 2;
  const int rows_per_cta = static_cast<int>(round_up(ceil_div(M, cs), 8));
  static unsigned mask = 0;
  int dev = 0;
  URV_CUDA(cudaGetDevice(&dev));
  if (!(mask & (1u << dev))) {
    URV_CUDA(cudaFuncSetAttribute(block_apply_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    URV_CUDA(cudaFuncSetAttribute(block_apply_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, apply_cl_smem_bytes()));
    mask |= 1u << dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs, static_cast<unsigned>(strips));
  cfg.blockDim = dim3(AP_THREADS);
  cfg.dynamicSmemBytes = apply_cl_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cs;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  StatsScope scope(st, kKApplyCl, 4.0 * M * nb * N + 2.0 * nb * nb * N, 16.0 * M * N + 8.0 * M * nb);
  URV_CUDA(cudaLaunchKernelEx(&cfg, block_apply_cl, V, ldv, T, ldt, trans ? 1 : 0, C, ldc, static_cast<int>(M),
                              static_cast<int>(N), nb, leafw, rows_per_cta));
  count_launch();
  return true;
}

// W(nb x N, ld ldwo) = op(T) V^T C, with V (M x nb, ld ldv), C (M x N, ld ldc).
// For nb <= 64 the T multiply is fused with the split-K reduction (apply_t);
// for wider blocks it is a DMMA GEMM with the (upper-triangular) T.
// Accurate long-K accumulation: a V^T C product (K = panel rows) split into runs of
// at most `acc` rows whose partials are added pairwise, so its rounding grows with
// log(M / acc) instead of M.  Switches (rows; 0 = the engine's own split-K):
//   URV_ACC_CHUNK  every V^T C (trailing updates, Q formation, Gram)
//   URV_FORMQ_ACC  the explicit-Q formation's V^T B only
//   URV_GRAM_CHUNK the outer-block Gram V^T V of the T merge only
int acc_chunk() {
  static const int v = env_int("URV_ACC_CHUNK", 0);
  return v;
}
// The Q formation and the Gram default to 1024-row runs: with one long accumulation
// the explicit Q's ||Q^T Q - I||_F grew to 2.7e-12 at 65536^2 (the gate is 1e-12);
// with runs of 1024 rows it is 6.8e-13 at no measurable cost (profiles/r02_orth_summary.md).
int formq_acc() {
  static const int v = env_int("URV_FORMQ_ACC", acc_chunk() > 0 ? acc_chunk() : 1024);
  return v;
}
int gram_chunk() {
  static const int v = env_int("URV_GRAM_CHUNK", acc_chunk() > 0 ? acc_chunk() : 1024);
  return v;
}

void vt_c_times_t(const double* V, long long ldv, const double* C, long long ldc, long long M, int nb, long long N,
                  const double* T, int ldt, bool trans, double* Wout, long long ldwo, double* Wtmp,
                  long long ldwt, cudaStream_t st, Workspace& ws, int acc = -1) {
  if (acc < 0) acc = acc_chunk();
  int splits_want = gemm_splits_for(nb, N, M);
  if (acc > 0) splits_want = std::min(64, std::max(splits_want, ceil_div(M, acc)));
  const int splits = gemm_effective_splits(M, splits_want);
  const bool tree = acc > 0;
  // The accurate mode's partials (splits x nb x N) can reach GBs for wide C (65536
  // columns: 8.6 GB at 64 splits); keep them under ~1 GB by going over C in column
  // chunks (same arithmetic per column, so the result does not depend on the chunking).
  constexpr long long kPartBudget = 1LL << 27;  // doubles
  if (tree && splits > 1 && static_cast<long long>(splits) * round_up(nb, 8) * gemm_split_cols(N) > kPartBudget) {
    const long long cols = std::max<long long>(128, kPartBudget / (splits * round_up(nb, 8)) / 128 * 128);
    for (long long c0 = 0; c0 < N; c0 += cols) {
      const long long nc = std::min(cols, N - c0);
      vt_c_times_t(V, ldv, C + c0 * ldc, ldc, M, nb, nc, T, ldt, trans, Wout + c0 * ldwo, ldwo, Wtmp + c0 * ldwt,
                   ldwt, st, ws, acc);
    }
    return;
  }
  const long long ldp = round_up(nb, 8);
  const long long pstride = gemm_split_cols(N);
  if (nb <= 64) {
    // narrow leaf block: fixed-order split-K reduction over the whole grid, then a
    // small T multiply (apply_t on the reduced W0, 16 columns per CTA)
    double* w0 = Wtmp;
    if (splits > 1) {
      double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
      dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, part, ldp, st, splits);
      StatsScope s3(st, kKApplyT, 0.0, 8.0 * (splits + 1) * nb * N);
      if (tree)
        sum_partials_tree<<<grid_for(static_cast<long long>(nb) * N), 256, 0, st>>>(part, ldp, pstride, splits, nb,
                                                                                 static_cast<int>(N), w0, ldwt);
      else
        sum_partials<<<grid_for(static_cast<long long>(nb) * N), 256, 0, st>>>(part, ldp, pstride, splits, nb,
                                                                              static_cast<int>(N), w0, ldwt);
      URV_CHECK_LAUNCH();
    } else {
      dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, w0, ldwt, st, 1);
    }
    StatsScope s3(st, kKApplyT, 1.0 * nb * nb * N, 16.0 * nb * N);
    apply_t<<<ceil_div(N, 8), 256, 0, st>>>(w0, ldwt, 0, 1, nb, static_cast<int>(N), T, ldt, trans ? 1 : 0, Wout,
                                             ldwo);
    URV_CHECK_LAUNCH();
    return;
  }
  // wide block: W0 = V^T C (reduced), then W = op(T) W0 on the tensor cores
  if (splits > 1) {
    double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
    dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, part, ldp, st, splits);
    StatsScope s3(st, kKApplyT, 0.0, 8.0 * (splits + 1) * nb * N);
    if (tree)
      sum_partials_tree<<<grid_for(static_cast<long long>(nb) * N), 256, 0, st>>>(part, ldp, pstride, splits, nb,
                                                                               static_cast<int>(N), Wtmp, ldwt);
    else
      sum_partials<<<grid_for(static_cast<long long>(nb) * N), 256, 0, st>>>(part, ldp, pstride, splits, nb,
                                                                            static_cast<int>(N), Wtmp, ldwt);
    URV_CHECK_LAUNCH();
  } else {
    dgemm_launch('T', 'N', nb, N, M, 1.0, V, ldv, C, ldc, 0.0, Wtmp, ldwt, st, 1);
  }
  dgemm_launch(trans ? 'T' : 'N', 'N', nb, N, nb, 1.0, T, ldt, Wtmp, ldwt, 0.0, Wout, ldwo, st, 1);
}

// Gram V^T V (nb x nb, K = M rows) of an outer block for its T merge.  With
// URV_ACC_CHUNK the K range is split into runs of at most that many rows and the
// partials are added pairwise (accurate mode); otherwise the engine's own split-K.
void gram_vtv(const double* V, long long ldv, long long M, int nb, double* G, long long ldg, cudaStream_t st,
              Workspace& ws) {
  if (gram_chunk() <= 0) {
    dgemm('T', 'N', nb, nb, M, 1.0, V, ldv, V, ldv, 0.0, G, ldg, st, ws);
    return;
  }
  const int splits = gemm_effective_splits(M, std::min(64, std::max(1, ceil_div(M, gram_chunk()))));
  if (splits <= 1) {
    dgemm_launch('T', 'N', nb, nb, M, 1.0, V, ldv, V, ldv, 0.0, G, ldg, st, 1);
    return;
  }
  const long long ldp = round_up(nb, 8), pstride = gemm_split_cols(nb);
  double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
  dgemm_launch('T', 'N', nb, nb, M, 1.0, V, ldv, V, ldv, 0.0, part, ldp, st, splits);
  StatsScope s3(st, kKApplyT, 0.0, 8.0 * (splits + 1) * nb * nb);
  sum_partials_tree<<<grid_for(static_cast<long long>(nb) * nb), 256, 0, st>>>(part, ldp, pstride, splits, nb, nb,
                                                                            G, ldg);
  URV_CHECK_LAUNCH();
}

// One block column of that Gram: G(0:c0, c0:c0+nb) = V(:, :c0)^T V(:, c0:c0+nb) (rows above c0
// of V(:, c0:) are zero, so K starts at row c0), for the leaf-by-leaf T merge.
void gram_vtv_block(const double* V, long long ldv, long long M, int c0, int nb, double* G, long long ldg,
                    cudaStream_t st, Workspace& ws) {
  const double* A = V + c0;
  const double* B = V + c0 + static_cast<long long>(c0) * ldv;
  double* Gb = G + static_cast<long long>(c0) * ldg;
  const long long K = M - c0;
  if (gram_chunk() <= 0) {
    dgemm('T', 'N', c0, nb, K, 1.0, A, ldv, B, ldv, 0.0, Gb, ldg, st, ws);
    return;
  }
  const int splits = gemm_effective_splits(K, std::min(64, std::max(1, ceil_div(K, gram_chunk()))));
  if (splits <= 1) {
    dgemm_launch('T', 'N', c0, nb, K, 1.0, A, ldv, B, ldv, 0.0, Gb, ldg, st, 1);
    return;
  }
  const long long ldp = round_up(c0, 8), pstride = gemm_split_cols(nb);
  double* part = ws.get(static_cast<size_t>(splits) * ldp * pstride);
  dgemm_launch('T', 'N', c0, nb, K, 1.0, A, ldv, B, ldv, 0.0, part, ldp, st, splits);
  StatsScope s3(st, kKApplyT, 0.0, 8.0 * (splits + 1) * c0 * nb);
  sum_partials_tree<<<grid_for(static_cast<long long>(c0) * nb), 256, 0, st>>>(part, ldp, pstride, splits, c0, nb, Gb,
                                                                            ldg);
  URV_CHECK_LAUNCH();
}

}  // namespace

int debug_panel_cycles(double* out, int n) {
  unsigned long long* b = panel_prof_buffer();
  for (int i = 0; i < n; ++i) out[i] = 0.0;
  if (!b) return 0;
  unsigned long long h[16];
  URV_CUDA(cudaDeviceSynchronize());
  URV_CUDA(cudaMemcpy(h, b, sizeof(h), cudaMemcpyDeviceToHost));
  URV_CUDA(cudaMemset(b, 0, sizeof(h)));
  for (int i = 0; i < n && i < 16; ++i) out[i] = static_cast<double>(h[i]);
  return 16;
}

int qr_panel_width(long long m) {
  (void)m;
  return LEAF;
}

// Outer block width (the rank of the trailing updates).  256 keeps the big updates
// efficient on the tensor pipe; up to n = 1024 the factorisation is latency-bound and
// single-leaf 64-column blocks (no leaf updates, no T merge) are faster.  Measured
// (profiles/r01_outer_block_sweep.log): config 1 20.97 -> 18.90 ms with 64; configs 2/3
// are fastest at 256 (189.6 / 526.5 ms vs 234.1 / 653.9 at 64).  URV_NBO overrides.
int outer_block_width(long long m, long long n) {
  (void)m;
  static const int force = env_int("URV_NBO", 0);
  if (force == 64 || force == 128 || force == 256) return force;
  if (n <= 1024) return 64;
  // Leafwise-mode factorisations (at most URV_FUSED_ROWS rows) of up to 4096 columns: with the
  // leaf split the panel chain waits for the main stream only at the outer-block boundaries, and
  // 128-column blocks (two leaves) halve what is pending there (config 2 80.0 -> 76.7 ms; 6144^2
  // and 8192^2 are 1-2% faster with 256: profiles/r02_nbo_leafwise.log).  URV_NBO_LW=256: off.
  static const int nbo_lw = env_int("URV_NBO_LW", 128);
  if ((nbo_lw == 128 || nbo_lw == 64) && m <= fused_apply_max_rows() && n <= 4096) return nbo_lw;
  return NBO;
}

void qr_factor(double* W, long long ldw, long long m, long long n, const double* sumsq, double* deficient,
               cudaStream_t st, Workspace& ws, QrFactors& out, double* E, long long lde, long long ne, int nb_force,
               cudaEvent_t tail_ev, int tail_blocks) {
  if (!E) ne = 0;
  int nb_pick = nb_force > 0 ? nb_force : outer_block_width(m, n);  // trailing-update rank
  // many attached columns (config 3's 4096^2 QRs carry A^T: 32768 of them) keep the main stream busy
  // with large updates either way: 256 stays faster there (config 3 477.5 vs 480.4 ms with 128)
  if (nb_force <= 0 && nb_pick == 128 && ne > 4 * n) nb_pick = NBO;
  const int NB_ = nb_pick;
  const int nouter = ceil_div(n, NB_);
  const long long ldv = round_up(m, 8);
  const int ldt = NB_;
  DevBuf Vbuf(static_cast<size_t>(ldv) * NB_, st);
  DevBuf Tall(static_cast<size_t>(nouter) * NB_ * NB_, st);
  URV_CUDA(cudaMemsetAsync(Tall.p, 0, sizeof(double) * nouter * NB_ * NB_, st));  // T is upper triangular
  const int sms = device_info().sms;
  // panel exchange buffer: 2 parities x clusters x (LEAF + 8) doubles; one barrier counter per leaf
  DevBuf scratch(static_cast<size_t>(2) * (MAX_PANEL_CTAS / 8 + 1) * (LEAF + 8), st);
  (void)sms;
  const int nleaves = ceil_div(n, 32);  // one barrier counter per (up to) 32-column leaf
  unsigned int* counters = nullptr;
  dev_alloc(reinterpret_cast<void**>(&counters), sizeof(unsigned int) * nleaves, st);
  URV_CUDA(cudaMemsetAsync(counters, 0, sizeof(unsigned int) * nleaves, st));
  QrScratch scr{scratch.p};
  const long long ldwt = NB_;
  const long long wcols = std::max(n, ne);
  DevBuf Wt(static_cast<size_t>(ldwt) * wcols, st), Wt2(static_cast<size_t>(ldwt) * wcols, st);
  DevBuf WtL(static_cast<size_t>(ldwt) * NB_, st), Wt2L(static_cast<size_t>(ldwt) * NB_, st);
  DevBuf VbufB(static_cast<size_t>(ldv) * NB_, st);
  DevBuf Gram(static_cast<size_t>(NB_) * NB_, st);
  DevBuf Xm(static_cast<size_t>(NB_) * LEAF, st);
  // Leafwise look-ahead (factorisations whose leaf updates run on the fused kernel, i.e. at
  // most URV_FUSED_ROWS rows): the next outer block receives block p's reflectors leaf by
  // leaf (four fused launches on L) instead of waiting for the outer T (Gram + six merges)
  // and a four-launch rank-256 update -- about 320 us per outer block on the panel chain
  // of a 4000^2 factorisation (profiles/r02_timeline_c2_fused.txt).  The Gram, the T merge
  // and the rank-256 update of everything beyond the next block move to the main stream,
  // which now runs one block behind; V is multi-buffered for that.  URV_LEAFWISE=0: off.
  static const bool leafwise_on = env_int("URV_LEAFWISE", 1) != 0;
  // The mode is chosen per factorisation (by its row count).  Switching to it for the last
  // blocks of a large factorisation works (the events of both schemes mean the same thing:
  // evN[q] = block q's columns carry every update the main stream owes them) but gains nothing
  // there -- config 4 2847.6 vs 2846.5 ms -- because the large trailing updates hide the panel
  // chain anyway; lw_at() keeps the per-block form for experiments (URV_LEAFWISE=2).
  const long long lw_rows = leafwise_on ? fused_apply_max_rows() : 0;
  static const bool lw_per_block = env_int("URV_LEAFWISE", 1) == 2;
  static const bool lw_single = env_int("URV_LW_SINGLE", 0) != 0;
  auto lw_at = [&](int p) {
    const long long Mp = lw_per_block ? m - static_cast<long long>(p) * NB_ : m;
    // URV_LW_SINGLE=1 (experiment, off): single-leaf outer blocks (n <= 1024) on the same schedule --
    // the block's reflectors onto the next block on the panel stream, the main stream one block
    // behind, the attached columns on their own stream.  Measured slower: config 1 7.94 -> 8.28 ms.
    return nouter > 1 && Mp <= lw_rows && (panel_leaf_width(Mp, m, n) < NB_ || lw_single);
  };
  const bool lw_any = lw_at(nouter - 1);
  // V buffers of the leafwise mode: block p's explicit V lives until the attached-column stream
  // (lowest priority, several blocks behind in the first part of a QR) has used it.  With three
  // buffers the panel stream waited 140-240 us per outer block for evE[p-3] at 4000^2
  // (profiles/r02_final_timeline_c2.txt); URV_LW_VBUFS (3..8, default 8) buffers of ldv x 256.
  static const int lw_vbufs = std::min(8, std::max(3, env_int("URV_LW_VBUFS", 8)));
  const int nvb = lw_any ? lw_vbufs : 2;
  DevBuf VbufC(lw_any ? static_cast<size_t>(ldv) * NB_ * (nvb - 2) : 0, st);
  double* vbufs[8] = {Vbuf.p, VbufB.p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int i = 2; i < nvb; ++i) vbufs[i] = VbufC.p + static_cast<size_t>(i - 2) * ldv * NB_;
  std::vector<cudaEvent_t> evN(nouter + 3, nullptr);  // block q's columns updated through block q-2 (main stream)

  // Look-ahead: the panel phase of outer block p+1 (leaves, leaf updates, T) runs on
  // a high-priority stream L as soon as block p's reflectors have been applied to
  // block p+1's columns; the rest of block p's trailing update proceeds on `st`.
  static const bool lookahead = [] {
    const char* e = getenv("URV_LOOKAHEAD");
    return !(e && e[0] == '0');
  }();
  cudaStream_t L = st;
  std::vector<cudaEvent_t> evs;
  auto new_event = [&]() {
    cudaEvent_t e;
    URV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
    return e;
  };
  if (lookahead && nouter > 1) {
    int lo_prio = 0, hi_prio = 0;
    URV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    URV_CUDA(cudaStreamCreateWithPriority(&L, cudaStreamNonBlocking, hi_prio));
    cudaEvent_t e0 = new_event();  // allocations / memsets above are ordered on st
    URV_CUDA(cudaEventRecord(e0, st));
    URV_CUDA(cudaStreamWaitEvent(L, e0, 0));
  }
  // Leafwise mode: the attached columns get their own stream and buffers (their rank-256
  // update is a four-launch chain of its own; on the main stream it made that stream the
  // longest chain of the factorisation)
  // ... and the outer T (Gram + merges: small kernels) a stream of its own, so that it neither
  // sits on the panel chain nor leaves bubbles between the main stream's large updates
  cudaStream_t Xs = st;
  if (lw_any && L != st) {
    int lo_prio = 0, hi_prio = 0;  // small kernels on the way to t_ready: panel-stream priority
    URV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    URV_CUDA(cudaStreamCreateWithPriority(&Xs, cudaStreamNonBlocking, hi_prio));
    URV_CUDA(cudaStreamWaitEvent(Xs, evs.back(), 0));  // e0: allocations ordered on st
  }
  Workspace wsXs(Xs);
  cudaStream_t Es = st;
  if (lw_any && ne > 0 && L != st) {
    URV_CUDA(cudaStreamCreateWithFlags(&Es, cudaStreamNonBlocking));
    URV_CUDA(cudaStreamWaitEvent(Es, evs.back(), 0));  // e0: allocations ordered on st
  }
  DevBuf WtE(Es != st ? static_cast<size_t>(ldwt) * ne : 0, st), Wt2E(Es != st ? static_cast<size_t>(ldwt) * ne : 0, st);
  Workspace wsEs(Es);
  // Leaf split (URV_LEAFSPLIT=0: off): in leafwise mode the panel chain L only carries what the
  // NEXT leaf needs -- a leaf's reflectors go onto the next leaf's columns on L (4 strips) and
  // onto everything else up to the end of the next outer block on a side stream S, one panel
  // ahead of their use.  Before: each leaf's update of the whole rest of its block (8-12
  // strips: two waves of 16-CTA clusters) and a four-leaf launch onto the next block's 256
  // columns (about 140 us) sat between two panels.
  static const bool leaf_split_on = env_int("URV_LEAFSPLIT", 1) != 0;
  const bool split = leaf_split_on && lw_any && !lw_per_block && L != st;
  cudaStream_t S = st;
  int side_prio = 0;  // the side streams run at the panel stream's priority: their 16-CTA clusters need whole
  if (split) {        // SMs and would otherwise queue behind the main stream's GEMM tiles for 300-500 us
    int lo_prio = 0;
    URV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &side_prio));
    URV_CUDA(cudaStreamCreateWithPriority(&S, cudaStreamNonBlocking, side_prio));
    URV_CUDA(cudaStreamWaitEvent(S, evs.back(), 0));  // e0: allocations ordered on st
  }
  cudaStream_t S2 = st;
  if (split) {
    URV_CUDA(cudaStreamCreateWithPriority(&S2, cudaStreamNonBlocking, side_prio));
    URV_CUDA(cudaStreamWaitEvent(S2, evs.back(), 0));
  }
  // ... and the main stream's work (outer-T consumers: the rank-256 updates that release evN)
  // moves to an internal stream of middle priority, above the attached-column stream Es: in
  // the first outer blocks of a 4000^2 power-step QR the attached columns' updates (37% of
  // all flops) otherwise compete with the updates the panel chain is waiting for.
  // URV_MAIN_PRIO=0: off.
  static const bool main_prio_on = env_int("URV_MAIN_PRIO", 1) != 0;
  cudaStream_t Ms = st;
  if (split && main_prio_on) {
    int lo_prio = 0, hi_prio = 0;
    URV_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    URV_CUDA(cudaStreamCreateWithPriority(&Ms, cudaStreamNonBlocking, (lo_prio + hi_prio) / 2));
    URV_CUDA(cudaStreamWaitEvent(Ms, evs.back(), 0));  // e0: allocations ordered on st
  }
  Workspace wsMs(Ms);
  Workspace& wsM = (Ms == st) ? ws : wsMs;
  DevBuf WtS(split ? static_cast<size_t>(ldwt) * NB_ : 0, st), Wt2S(split ? static_cast<size_t>(ldwt) * NB_ : 0, st);
  DevBuf WtS2(split ? static_cast<size_t>(ldwt) * NB_ : 0, st), Wt2S2(split ? static_cast<size_t>(ldwt) * NB_ : 0, st);
  Workspace wsS(S), wsS2(S2);
  cudaEvent_t evS = nullptr, evS2 = nullptr;  // the side streams' latest applies (S: within the block, S2: next block)
  int nb_sent = 0;  // reflectors of the current block already applied to the next block's columns
  std::vector<cudaEvent_t> evE(nouter + 3, nullptr);  // block q's attached-column update done (Es)
  Workspace wsL(L);
  Workspace& wsP = (L == st) ? ws : wsL;
  double* wtP = (L == st) ? Wt.p : WtL.p;
  double* wt2P = (L == st) ? Wt2.p : Wt2L.p;

  // update columns [c_lo, c_hi) of W (rows j0..m) with block p's reflectors on stream s
  auto block_update = [&](int p, long long c_lo, long long c_hi, double* V, cudaStream_t s, Workspace& w) {
    const long long j0 = static_cast<long long>(p) * NB_;
    const int nbo = static_cast<int>(std::min<long long>(NB_, n - j0));
    const int M = static_cast<int>(m - j0);
    const long long Nt = c_hi - c_lo;
    if (Nt <= 0) return;
    double* Cp = W + j0 + c_lo * ldw;
    double* Tp = Tall.p + static_cast<size_t>(p) * NB_ * NB_;
    if (fused_block_apply(V, ldv, Tp, ldt, true, Cp, ldw, M, nbo, Nt, s)) return;
    vt_c_times_t(V, ldv, Cp, ldw, M, nbo, Nt, Tp, ldt, true, Wt.p, ldwt, Wt2.p, ldwt, s, w);
    dgemm_launch('N', 'N', M, Nt, nbo, -1.0, V, ldv, Wt.p, ldwt, 1.0, Cp, ldw, s, 1);
  };

  // one leaf's block reflector onto N columns at C on stream s (fused kernel, else the GEMM chain)
  auto leaf_apply = [&](const double* Vl, const double* Tl, double* C, long long ldc, long long Ml, int nbl,
                        long long N, cudaStream_t s, double* wt, double* wt2, Workspace& w) {
    if (N <= 0) return;
    if (fused_block_apply(Vl, ldv, Tl, ldt, true, C, ldc, Ml, nbl, N, s)) return;
    vt_c_times_t(Vl, ldv, C, ldc, Ml, nbl, N, Tl, ldt, true, wt, ldwt, wt2, ldwt, s, w);
    dgemm_launch('N', 'N', Ml, N, nbl, -1.0, Vl, ldv, wt, ldwt, 1.0, C, ldc, s, 1);
  };

  // leaves [r0, r1) of an outer block (V, T at the block's origin, M rows) onto N columns at C
  // (block rows): one multi-leaf launch where the rows allow it, else leaf by leaf.  The split
  // and the unsplit leafwise schedules issue the same sequence of these (bitwise-equal results).
  auto next_block_apply = [&](const double* V, const double* T, double* C, long long M, int r0, int r1, int leafw,
                              long long N, cudaStream_t s, double* wt, double* wt2, Workspace& w) {
    if (r1 <= r0 || N <= 0) return;
    const double* V0 = V + r0 + static_cast<long long>(r0) * ldv;
    const double* T0 = T + r0 + static_cast<long long>(r0) * ldt;
    if (r1 - r0 > leafw && fused_block_apply(V0, ldv, T0, ldt, true, C + r0, ldw, M - r0, r1 - r0, N, s, leafw)) return;
    for (int d0 = r0; d0 < r1; d0 += leafw)
      leaf_apply(V + d0 + static_cast<long long>(d0) * ldv, T + d0 + static_cast<long long>(d0) * ldt, C + d0, ldw,
                 M - d0, std::min(leafw, r1 - d0), N, s, wt, wt2, w);
  };

  // Outer T, leaf by leaf (core.py:101-109 blocked): once leaf [c0, c0 + nbl) of an outer block is
  // factored, T(0:c0, c0:c0+nbl) = -T(0:c0, 0:c0) (V(:, :c0)^T V(:, c0:c0+nbl)) T_leaf.  Every
  // schedule issues these same launches; the split schedule issues them as the leaves finish, so
  // only the last leaf's piece is left when the block's panels are done.
  auto outer_t_leaf = [&](const double* Vb, double* Tp, long long M, int c0, int nbl, cudaStream_t s, Workspace& w) {
    gram_vtv_block(Vb, ldv, M, c0, nbl, Gram.p, NB_, s, w);
    StatsScope s4(s, kKApplyT, 2.0 * c0 * nbl * (c0 + nbl), 0.0);
    t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, s>>>(Tp, ldt, Gram.p, NB_, c0, nbl, Xm.p, 0);
    URV_CHECK_LAUNCH();
    t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, s>>>(Tp, ldt, Gram.p, NB_, c0, nbl, Xm.p, 1);
    URV_CHECK_LAUNCH();
  };

  try {
    // ---------------- factorisation: core.py:143-152 ----------------
    cudaEvent_t upd_prev = nullptr, t_ready = nullptr, e_on_st = nullptr;
    for (int p = 0; p < nouter; ++p) {
      const long long j0 = static_cast<long long>(p) * NB_;
      const int nbo = static_cast<int>(std::min<long long>(NB_, n - j0));
      const int M = static_cast<int>(m - j0);
      double* Pp = W + j0 + j0 * ldw;  // outer block origin
      double* Tp = Tall.p + static_cast<size_t>(p) * NB_ * NB_;
      const bool lw = lw_at(p);
      double* Vb = vbufs[(L == st) ? 0 : (lw_any ? p % nvb : (p & 1))];
      // ---- panel phase of block p on L ----
      if (lw) {
        if (evN[p]) URV_CUDA(cudaStreamWaitEvent(L, evN[p], 0));
        if (p >= nvb && evE[p - nvb]) URV_CUDA(cudaStreamWaitEvent(L, evE[p - nvb], 0));  // V buffer p % nvb is free
      } else if (upd_prev) {
        URV_CUDA(cudaStreamWaitEvent(L, upd_prev, 0));
      }
      const int leafw = panel_leaf_width(M, m, n);
      for (int c0 = 0; c0 < nbo; c0 += leafw) {
        const int nbl = std::min(leafw, nbo - c0);
        const int Ml = M - c0;
        double* Pl = Pp + c0 + c0 * ldw;
        // the panel also writes the leaf's explicit V into Vb (rows 0..M of the outer block)
        launch_panel(Pl, ldw, Ml, nbl, Tp + c0 + static_cast<long long>(c0) * ldt, ldt,
                     Vb + c0 + static_cast<long long>(c0) * ldv, ldv, c0, scr, counters + (j0 + c0) / 32, L, n);
        if (lw && split) {
          const double* Vl = Vb + c0 + static_cast<long long>(c0) * ldv;
          const double* Tl = Tp + c0 + static_cast<long long>(c0) * ldt;
          const bool has_next = j0 + nbo < n;
          const long long c1 = j0 + nbo;
          const long long Nn = has_next ? std::min<long long>(NB_, n - c1) : 0;
          const int nl = ceil_div(nbo, leafw), k = c0 / leafw;
          cudaEvent_t ev_panel = new_event();
          URV_CUDA(cudaEventRecord(ev_panel, L));
          if (k >= 1) {  // this leaf's block column of the outer T, beside the next panel
            URV_CUDA(cudaStreamWaitEvent(Xs, ev_panel, 0));
            outer_t_leaf(Vb, Tp, M, c0, nbl, Xs, wsXs);
          }
          if (k == nl - 1) {  // the block's panels are done: the main stream may go on
            URV_CUDA(cudaStreamWaitEvent(Ms, ev_panel, 0));
            if (nl == 1) URV_CUDA(cudaStreamWaitEvent(Xs, ev_panel, 0));
          }
          if (k < nl - 1) {
            const int nb2 = std::min(leafw, nbo - c0 - nbl);  // the next leaf
            double* Cr = Pl + static_cast<long long>(nbl) * ldw;
            // these columns carry the earlier leaves through S (and, for the block's first
            // leaf, the previous block through S2)
            if (evS) URV_CUDA(cudaStreamWaitEvent(L, evS, 0));
            if (k == 0 && evS2) URV_CUDA(cudaStreamWaitEvent(L, evS2, 0));
            leaf_apply(Vl, Tl, Cr, ldw, Ml, nbl, nb2, L, wtP, wt2P, wsP);
            const long long Nrest = nbo - c0 - nbl - nb2;
            if (Nrest > 0) {  // the rest of the block on S
              URV_CUDA(cudaStreamWaitEvent(S, ev_panel, 0));
              if (k == 0 && evS2) URV_CUDA(cudaStreamWaitEvent(S, evS2, 0));
              leaf_apply(Vl, Tl, Cr + static_cast<long long>(nb2) * ldw, ldw, Ml, nbl, Nrest, S, WtS.p, Wt2S.p, wsS);
              evS = new_event();
              URV_CUDA(cudaEventRecord(evS, S));
            }
            if (has_next && k >= nl - 3) {
              // the leaves not yet sent go onto the next block's columns on S2, well before the
              // block's last panel is done
              URV_CUDA(cudaStreamWaitEvent(S2, ev_panel, 0));
              if (evN[p + 1]) URV_CUDA(cudaStreamWaitEvent(S2, evN[p + 1], 0));
              next_block_apply(Vb, Tp, W + j0 + c1 * ldw, M, nb_sent, c0 + nbl, leafw, Nn, S2, WtS2.p, Wt2S2.p, wsS2);
              nb_sent = c0 + nbl;
              evS2 = new_event();
              URV_CUDA(cudaEventRecord(evS2, S2));
            }
          } else if (has_next) {
            // the block's last leaf: onto the next block's first leaf on L, onto the rest of it on S2
            const long long nb2 = std::min<long long>(panel_leaf_width(M - nbo, m, n), Nn);
            double* Cn = W + (j0 + c0) + c1 * ldw;
            if (evN[p + 1]) URV_CUDA(cudaStreamWaitEvent(L, evN[p + 1], 0));
            if (evS2) URV_CUDA(cudaStreamWaitEvent(L, evS2, 0));
            leaf_apply(Vl, Tl, Cn, ldw, Ml, nbl, nb2, L, wtP, wt2P, wsP);
            if (Nn > nb2) {
              URV_CUDA(cudaStreamWaitEvent(S2, ev_panel, 0));
              if (evN[p + 1]) URV_CUDA(cudaStreamWaitEvent(S2, evN[p + 1], 0));
              leaf_apply(Vl, Tl, Cn + nb2 * ldw, ldw, Ml, nbl, Nn - nb2, S2, WtS2.p, Wt2S2.p, wsS2);
              evS2 = new_event();
              URV_CUDA(cudaEventRecord(evS2, S2));
            }
            nb_sent = 0;
          }
        } else if (c0 + nbl < nbo) {  // update the rest of the outer block with this leaf
          const long long Nr = nbo - c0 - nbl;
          double* Cr = Pl + static_cast<long long>(nbl) * ldw;
          const double* Vl = Vb + c0 + static_cast<long long>(c0) * ldv;
          const double* Tl = Tp + c0 + static_cast<long long>(c0) * ldt;
          if (!fused_block_apply(Vl, ldv, Tl, ldt, true, Cr, ldw, Ml, nbl, Nr, L)) {
            vt_c_times_t(Vl, ldv, Cr, ldw, Ml, nbl, Nr, Tl, ldt, true, wtP, ldwt, wt2P, ldwt, L, wsP);
            dgemm_launch('N', 'N', Ml, Nr, nbl, -1.0, Vl, ldv, wtP, ldwt, 1.0, Cr, ldw, L, 1);
          }
        }
      }
      // outer T from the leaf T's: T12 = -T11 (V1^T V2) T22, leaf by leaf
      // Leafwise mode: the per-leaf pieces (every leafwise schedule issues these same launches).
      // Otherwise one Gram of the whole block, then the merges: three smaller Gram products on the
      // panel stream cost config 3 478.6 -> 490.2 ms and config 4 2827 -> 2848 ms.
      auto outer_t = [&](cudaStream_t s, Workspace& w) {
        if (nbo <= leafw) return;
        if (lw) {
          for (int c0 = leafw; c0 < nbo; c0 += leafw) outer_t_leaf(Vb, Tp, M, c0, std::min(leafw, nbo - c0), s, w);
          return;
        }
        gram_vtv(Vb, ldv, M, nbo, Gram.p, NB_, s, w);
        for (int c0 = leafw; c0 < nbo; c0 += leafw) {
          const int nbl = std::min(leafw, nbo - c0);
          StatsScope s4(s, kKApplyT, 2.0 * c0 * nbl * (c0 + nbl), 0.0);
          t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, s>>>(Tp, ldt, Gram.p, NB_, c0, nbl, Xm.p, 0);
          URV_CHECK_LAUNCH();
          t_merge<<<grid_for(static_cast<long long>(c0) * nbl), 256, 0, s>>>(Tp, ldt, Gram.p, NB_, c0, nbl, Xm.p, 1);
          URV_CHECK_LAUNCH();
        }
      };
      if (!lw) outer_t(L, wsP);
      if (L != st && !(lw && split)) {
        cudaEvent_t done = new_event();
        URV_CUDA(cudaEventRecord(done, L));
        URV_CUDA(cudaStreamWaitEvent(st, done, 0));
        if (lw) URV_CUDA(cudaStreamWaitEvent(Xs, done, 0));
      }
      if (lw && !split && j0 + nbo < n) {
        // block p's leaves onto the next block's columns, on L (they were updated through
        // block p-1 by the main stream: evN[p+1]; L's own earlier applies are in order)
        if (evN[p + 1]) URV_CUDA(cudaStreamWaitEvent(L, evN[p + 1], 0));
        const long long c1 = j0 + nbo;
        const long long Nn = std::min<long long>(NB_, n - c1);
        // the same launches as the split schedule issues: leaves up to the third from last in
        // one launch (while the block's rows fit one staged chunk per CTA), then leaf by leaf
        const int nl = ceil_div(nbo, leafw);
        const int r1 = std::max(0, nl - 2) * leafw, r2 = std::max(0, nl - 1) * leafw;
        double* Cn = W + j0 + c1 * ldw;
        next_block_apply(Vb, Tp, Cn, M, 0, std::min(r1, nbo), leafw, Nn, L, wtP, wt2P, wsP);
        next_block_apply(Vb, Tp, Cn, M, std::min(r1, nbo), std::min(r2, nbo), leafw, Nn, L, wtP, wt2P, wsP);
        next_block_apply(Vb, Tp, Cn, M, std::min(r2, nbo), nbo, leafw, Nn, L, wtP, wt2P, wsP);
      }
      // the caller's "tail reached" event: the last tail_blocks blocks follow
      if (tail_ev && p == std::max(0, nouter - tail_blocks)) URV_CUDA(cudaEventRecord(tail_ev, Ms));
      upd_prev = nullptr;
      if (lw) {
        // ---- main stream, one block behind: outer T, then the block after the next first ----
        if (Xs != st) {
          if (!split) outer_t(Xs, wsXs);
          t_ready = new_event();
          URV_CUDA(cudaEventRecord(t_ready, Xs));
          URV_CUDA(cudaStreamWaitEvent(Ms, t_ready, 0));
        } else {
          outer_t(st, ws);
        }
        if (j0 + nbo < n) {
          const long long c2 = std::min<long long>(n, j0 + 2LL * NB_), c3 = std::min<long long>(n, c2 + NB_);
          block_update(p, c2, c3, Vb, Ms, wsM);
          if (L != st && p + 2 < nouter) {
            evN[p + 2] = new_event();
            URV_CUDA(cudaEventRecord(evN[p + 2], Ms));
          }
          block_update(p, c3, n, Vb, Ms, wsM);
        }
      } else if (j0 + nbo < n) {
        // ---- trailing update of block p on st: next block's columns first ----
        const long long c1 = j0 + nbo, c2 = std::min<long long>(n, c1 + NB_);
        block_update(p, c1, c2, Vb, st, ws);
        if (L != st) {
          upd_prev = new_event();
          URV_CUDA(cudaEventRecord(upd_prev, st));
          evN[p + 1] = upd_prev;
        }
        block_update(p, c2, n, Vb, st, ws);
        if (L != st && lw_any && p + 2 < nouter) {  // the next block may run leafwise
          evN[p + 2] = new_event();
          URV_CUDA(cudaEventRecord(evN[p + 2], st));
        }
      }
      if (ne > 0) {  // the attached columns: E(j0:, :) <- H_p^T E(j0:, :)
        double* Ep = E + j0;
        if (Es != st && lw) {  // after the outer T, beside the main stream's trailing update
          URV_CUDA(cudaStreamWaitEvent(Es, t_ready, 0));
          if (e_on_st) {  // the blocks before the switch updated E on the main stream
            URV_CUDA(cudaStreamWaitEvent(Es, e_on_st, 0));
            e_on_st = nullptr;
          }
          if (!fused_block_apply(Vb, ldv, Tp, ldt, true, Ep, lde, M, nbo, ne, Es)) {
            vt_c_times_t(Vb, ldv, Ep, lde, M, nbo, ne, Tp, ldt, true, WtE.p, ldwt, Wt2E.p, ldwt, Es, wsEs);
            dgemm_launch('N', 'N', M, ne, nbo, -1.0, Vb, ldv, WtE.p, ldwt, 1.0, Ep, lde, Es, 1);
          }
          evE[p] = new_event();
          URV_CUDA(cudaEventRecord(evE[p], Es));
        } else {
          if (!fused_block_apply(Vb, ldv, Tp, ldt, true, Ep, lde, M, nbo, ne, st)) {
            vt_c_times_t(Vb, ldv, Ep, lde, M, nbo, ne, Tp, ldt, true, Wt.p, ldwt, Wt2.p, ldwt, st, ws);
            dgemm_launch('N', 'N', M, ne, nbo, -1.0, Vb, ldv, Wt.p, ldwt, 1.0, Ep, lde, st, 1);
          }
          if (Es != st && p + 1 < nouter && lw_at(p + 1)) {  // the next block updates E on Es
            e_on_st = new_event();
            URV_CUDA(cudaEventRecord(e_on_st, st));
          }
        }
      }
    }
    if (Ms != st) {  // join the internal main stream
      cudaEvent_t m_done = new_event();
      URV_CUDA(cudaEventRecord(m_done, Ms));
      URV_CUDA(cudaStreamWaitEvent(st, m_done, 0));
    }
    if (S != st) {  // join the leaf-split side streams (L has waited for all of their work already)
      cudaEvent_t s_done = new_event(), s2_done = new_event();
      URV_CUDA(cudaEventRecord(s_done, S));
      URV_CUDA(cudaStreamWaitEvent(st, s_done, 0));
      URV_CUDA(cudaEventRecord(s2_done, S2));
      URV_CUDA(cudaStreamWaitEvent(st, s2_done, 0));
    }
    if (Es != st) {  // join the attached-column stream
      cudaEvent_t e_done = new_event();
      URV_CUDA(cudaEventRecord(e_done, Es));
      URV_CUDA(cudaStreamWaitEvent(st, e_done, 0));
    }
    // ---------------- deficiency count (factorizations.py:80) ----------------
    if (deficient) {
      StatsScope s4(st, kKAux, 0.0, 8.0 * n);
      count_deficient<<<1, 1024, 0, st>>>(W, ldw, static_cast<int>(n), sumsq, deficient);
      URV_CHECK_LAUNCH();
    }
  } catch (...) {
    cudaFreeAsync(counters, st);
    for (auto e : evs) cudaEventDestroy(e);
    if (L != st) cudaStreamDestroy(L);
    if (S != st) cudaStreamDestroy(S);
    if (S2 != st) cudaStreamDestroy(S2);
    if (Ms != st) cudaStreamDestroy(Ms);
    if (Es != st) cudaStreamDestroy(Es);
    if (Xs != st) cudaStreamDestroy(Xs);
    throw;
  }
  URV_CUDA(cudaFreeAsync(counters, st));
  for (auto e : evs) cudaEventDestroy(e);  // released once their work completes
  if (S != st) {
    wsS.release();
    cudaStreamDestroy(S);
  }
  if (S2 != st) {
    wsS2.release();
    cudaStreamDestroy(S2);
  }
  if (Ms != st) {
    wsMs.release();
    cudaStreamDestroy(Ms);
  }
  if (Es != st) {
    wsEs.release();
    cudaStreamDestroy(Es);
  }
  if (Xs != st) {
    wsXs.release();
    cudaStreamDestroy(Xs);
  }
  if (L != st) {
    wsL.release();
    cudaStreamDestroy(L);
  }
  out.W = W;
  out.ldw = ldw;
  out.m = m;
  out.n = n;
  out.Tall = std::move(Tall);
  out.nb = NB_;
}

void qr_extract_r(const QrFactors& f, double* R, long long ldr, cudaStream_t st) {
  StatsScope s5(st, kKAux, 0.0, 16.0 * f.n * f.n);
  extract_r<<<grid_for(f.n * f.n), 256, 0, st>>>(f.W, f.ldw, static_cast<int>(f.n), R, ldr);
  URV_CHECK_LAUNCH();
}

// Explicit thin Q = H_0 H_1 ... H_{P-1} I(:, :n): core.py:154-157, backward over the
// outer blocks on the live columns only (dorgqr).
void qr_form_q(const QrFactors& f, double* Q, long long ldq, cudaStream_t st, Workspace& ws) {
  const long long m = f.m, n = f.n;
  const int nouter = ceil_div(n, f.nb);
  const long long ldv = round_up(m, 8), ldwt = f.nb;
  DevBuf Vbuf(static_cast<size_t>(ldv) * f.nb, st);
  DevBuf Wt(static_cast<size_t>(ldwt) * n, st), Wt2(static_cast<size_t>(ldwt) * n, st);
  {
    StatsScope s6(st, kKAux, 0.0, 8.0 * m * n);
    set_identity<<<grid_for(m * n), 256, 0, st>>>(Q, ldq, static_cast<int>(m), static_cast<int>(n));
    URV_CHECK_LAUNCH();
  }
  // URV_FORMQ_NB = 64: apply the 64-column diagonal blocks of each outer T (the leaf
  // block reflectors) one by one instead of the whole 256-column block (experiment).
  static const int formq_nb = env_int("URV_FORMQ_NB", 0);
  for (int p = nouter - 1; p >= 0; --p) {
    const long long j0 = static_cast<long long>(p) * f.nb;
    const int nbo = static_cast<int>(std::min<long long>(f.nb, n - j0));
    const int M = static_cast<int>(m - j0);
    const long long Nq = n - j0;
    const double* Pp = f.W + j0 + j0 * f.ldw;
    const double* Tp = f.Tall.p + static_cast<size_t>(p) * f.nb * f.nb;
    double* Bq = Q + j0 + j0 * ldq;
    {
      StatsScope s2(st, kKAux, 0.0, 16.0 * M * nbo);
      load_v<<<grid_for(static_cast<long long>(M) * nbo), 256, 0, st>>>(Pp, f.ldw, M, 0, nbo, Vbuf.p, ldv);
      URV_CHECK_LAUNCH();
    }
    if (formq_nb > 0 && formq_nb < nbo) {
      for (int c0 = ((nbo - 1) / formq_nb) * formq_nb; c0 >= 0; c0 -= formq_nb) {
        const int kb = std::min(formq_nb, nbo - c0);
        const double* Vl = Vbuf.p + c0 + static_cast<long long>(c0) * ldv;
        const double* Tl = Tp + c0 + static_cast<long long>(c0) * f.nb;
        double* Bl = Bq + c0 + static_cast<long long>(c0) * ldq;
        vt_c_times_t(Vl, ldv, Bl, ldq, M - c0, kb, Nq - c0, Tl, f.nb, false, Wt.p, ldwt, Wt2.p, ldwt, st, ws,
                     formq_acc());
        dgemm_launch('N', 'N', M - c0, Nq - c0, kb, -1.0, Vl, ldv, Wt.p, ldwt, 1.0, Bl, ldq, st, 1);
      }
      continue;
    }
    if (fused_block_apply(Vbuf.p, ldv, Tp, f.nb, false, Bq, ldq, M, nbo, Nq, st)) continue;
    vt_c_times_t(Vbuf.p, ldv, Bq, ldq, M, nbo, Nq, Tp, f.nb, false, Wt.p, ldwt, Wt2.p, ldwt, st, ws, formq_acc());
    dgemm_launch('N', 'N', M, Nq, nbo, -1.0, Vbuf.p, ldv, Wt.p, ldwt, 1.0, Bq, ldq, st, 1);
  }
}

// tau_j = T(j, j) of every outer block (debug / cross-checks: LAPACK-style (V, tau)).
__global__ void extract_tau(const double* __restrict__ Tall, int nb, int n, double* __restrict__ tau) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int p = j / nb, jj = j % nb;
    tau[j] = Tall[static_cast<long long>(p) * nb * nb + jj + static_cast<long long>(jj) * nb];
  }
}

void qr_factor_tau(double* W, long long ldw, long long m, long long n, double* tau, cudaStream_t st, Workspace& ws) {
  QrFactors f;
  qr_factor(W, ldw, m, n, nullptr, nullptr, st, ws, f);
  extract_tau<<<grid_for(n), 256, 0, st>>>(f.Tall.p, f.nb, static_cast<int>(n), tau);
  URV_CHECK_LAUNCH();
}

// B (m x ncols) <- H^T B = H_{P-1}^T ... H_0^T B  (block p: B(j0:, :) -= V T^T (V^T B(j0:, :))).
void qr_apply_qt_left(const QrFactors& f, double* B, long long ldb, long long ncols, cudaStream_t st,
                      Workspace& ws) {
  const long long m = f.m, n = f.n;
  const int nouter = ceil_div(n, f.nb);
  const long long ldv = round_up(m, 8), ldwt = f.nb;
  DevBuf Vbuf(static_cast<size_t>(ldv) * f.nb, st);
  DevBuf Wt(static_cast<size_t>(ldwt) * ncols, st), Wt2(static_cast<size_t>(ldwt) * ncols, st);
  for (int p = 0; p < nouter; ++p) {
    const long long j0 = static_cast<long long>(p) * f.nb;
    const int nbo = static_cast<int>(std::min<long long>(f.nb, n - j0));
    const int M = static_cast<int>(m - j0);
    const double* Pp = f.W + j0 + j0 * f.ldw;
    const double* Tp = f.Tall.p + static_cast<size_t>(p) * f.nb * f.nb;
    double* Bp = B + j0;
    {
      StatsScope s2(st, kKAux, 0.0, 16.0 * M * nbo);
      load_v<<<grid_for(static_cast<long long>(M) * nbo), 256, 0, st>>>(Pp, f.ldw, M, 0, nbo, Vbuf.p, ldv);
      URV_CHECK_LAUNCH();
    }
    vt_c_times_t(Vbuf.p, ldv, Bp, ldb, M, nbo, ncols, Tp, f.nb, true, Wt.p, ldwt, Wt2.p, ldwt, st, ws);
    dgemm_launch('N', 'N', M, ncols, nbo, -1.0, Vbuf.p, ldv, Wt.p, ldwt, 1.0, Bp, ldb, st, 1);
  }
}

// B (nrows x m) <- B H = B H_0 H_1 ... H_{P-1}  (block p: B(:, j0:) -= (B(:, j0:) V) T V^T).
void qr_apply_q_right(const QrFactors& f, double* B, long long ldb, long long nrows, cudaStream_t st,
                      Workspace& ws) {
  const long long m = f.m, n = f.n;
  const int nouter = ceil_div(n, f.nb);
  const long long ldv = round_up(m, 8), ldx = round_up(nrows, 8);
  DevBuf Vbuf(static_cast<size_t>(ldv) * f.nb, st);
  DevBuf X(static_cast<size_t>(ldx) * f.nb, st), X2(static_cast<size_t>(ldx) * f.nb, st);
  for (int p = 0; p < nouter; ++p) {
    const long long j0 = static_cast<long long>(p) * f.nb;
    const int nbo = static_cast<int>(std::min<long long>(f.nb, n - j0));
    const int M = static_cast<int>(m - j0);
    const double* Pp = f.W + j0 + j0 * f.ldw;
    const double* Tp = f.Tall.p + static_cast<size_t>(p) * f.nb * f.nb;
    double* Bp = B + j0 * ldb;
    {
      StatsScope s2(st, kKAux, 0.0, 16.0 * M * nbo);
      load_v<<<grid_for(static_cast<long long>(M) * nbo), 256, 0, st>>>(Pp, f.ldw, M, 0, nbo, Vbuf.p, ldv);
      URV_CHECK_LAUNCH();
    }
    dgemm('N', 'N', nrows, nbo, M, 1.0, Bp, ldb, Vbuf.p, ldv, 0.0, X.p, ldx, st, ws);      // X = B V
    dgemm_launch('N', 'N', nrows, nbo, nbo, 1.0, X.p, ldx, Tp, f.nb, 0.0, X2.p, ldx, st, 1);  // X T
    dgemm_launch('N', 'T', nrows, M, nbo, -1.0, X2.p, ldx, Vbuf.p, ldv, 1.0, Bp, ldb, st, 1);  // B -= X T V^T
  }
}

// One compact-WY block for the distributed (column-block-cyclic) QR: factor the
// m x k panel W in place (R on/above the diagonal, V below it, diag(R) >= 0) and
// write its k x k upper-triangular T (H = I - V T V^T).  k <= NBO, m >= k.
void geqrt_device(double* W, long long ldw, long long m, long long k, double* T, long long ldt, cudaStream_t st,
                  Workspace& ws) {
  if (k < 1 || k > NBO || m < k) {
    set_error("geqrt: need 1 <= k <= %d and m >= k, got %lld x %lld", NBO, m, k);
    throw CudaFailure{kInvalid};
  }
  QrFactors f;
  qr_factor(W, ldw, m, k, nullptr, nullptr, st, ws, f, nullptr, 0, 0, NBO);  // one block: a single T
  URV_CUDA(cudaMemcpy2DAsync(T, ldt * 8, f.Tall.p, static_cast<size_t>(f.nb) * 8, k * 8, k, cudaMemcpyDeviceToDevice,
                             st));
}

// C (m x ncols) <- H^T C (trans) or H C with H = I - V T V^T, V the unit-lower part of
// the factored m x k panel P (as left by geqrt_device / qr_factor).  core.py:149-151
// (trans, the trailing update) and core.py:154-157 (no trans, explicit Q).
void apply_block_reflector(const double* P, long long ldp, long long m, long long k, const double* T, long long ldt,
                           bool trans, double* C, long long ldc, long long ncols, cudaStream_t st, Workspace& ws) {
  if (ncols <= 0 || m <= 0 || k <= 0) return;
  if (k > NBO || m < k) {
    set_error("apply_block_reflector: need k <= %d and m >= k, got %lld x %lld", NBO, m, k);
    throw CudaFailure{kInvalid};
  }
  const long long ldv = round_up(m, 8), ldwt = round_up(k, 8);
  DevBuf Vbuf(static_cast<size_t>(ldv) * k, st);
  DevBuf Tc(static_cast<size_t>(ldwt) * k, st);
  DevBuf Wt(static_cast<size_t>(ldwt) * ncols, st), Wt2(static_cast<size_t>(ldwt) * ncols, st);
  {
    StatsScope s2(st, kKAux, 0.0, 16.0 * m * k);
    load_v<<<grid_for(m * k), 256, 0, st>>>(P, ldp, static_cast<int>(m), 0, static_cast<int>(k), Vbuf.p, ldv);
    URV_CHECK_LAUNCH();
  }
  // T with an even, 16-byte aligned leading dimension for the TMA operand maps
  URV_CUDA(cudaMemcpy2DAsync(Tc.p, ldwt * 8, T, ldt * 8, k * 8, k, cudaMemcpyDeviceToDevice, st));
  if (fused_block_apply(Vbuf.p, ldv, Tc.p, static_cast<int>(ldwt), trans, C, ldc, m, static_cast<int>(k), ncols, st))
    return;
  vt_c_times_t(Vbuf.p, ldv, C, ldc, m, static_cast<int>(k), ncols, Tc.p, static_cast<int>(ldwt), trans, Wt.p, ldwt,
               Wt2.p, ldwt, st, ws);
  dgemm_launch('N', 'N', m, ncols, k, -1.0, Vbuf.p, ldv, Wt.p, ldwt, 1.0, C, ldc, st, 1);
}

void householder_qr_device(double* W, long long ldw, long long m, long long n, double* Q, long long ldq,
                           double* R, long long ldr, const double* sumsq, double* deficient,
                           cudaStream_t st, Workspace& ws, cudaEvent_t r_ready) {
  QrFactors f;
  qr_factor(W, ldw, m, n, sumsq, deficient, st, ws, f);
  if (R) {
    qr_extract_r(f, R, ldr, st);
    if (r_ready) URV_CUDA(cudaEventRecord(r_ready, st));
  }
  qr_form_q(f, Q, ldq, st, ws);
}

}  // namespace urv
