// Single-cluster Householder panel (round 2): the 64-column leaf of core.py:57-109
// factored by ONE thread-block cluster (up to 16 CTAs) that talks only through
// distributed shared memory -- no global-memory barrier, no fences.  Included by qr.cu.
//
// Why: the cooperative panel_geqr2 pays a grid exchange through global memory per column
// (about 2200-2800 cycles on B200 whatever the protocol: profiles/r02_xchg_experiment.log)
// inside a dependent chain of about 10k cycles per column.  Here a column costs one
// st.async all-to-all (about 1000 cycles) and one __syncthreads, and everything that is
// not needed for the next reflector is taken off that chain:
//
//  * Same data layout as panel_geqr2: CTA c owns rows [c*RB, c*RB + RB), RB = 32*RT; warp w
//    owns columns {w, w+8, ...}, lane l rows {l, l+32, ...}; rows i < RTR in registers,
//    the rest in this thread's slice of shared memory.
//  * Inner blocks of 8 columns (one per warp).  Within an inner block only its own
//    columns get the rank-1 update of every step (the "active" column of each warp,
//    kept in registers); the later ("stale") columns receive the block's 8 reflectors
//    at once when the block is done:  C -= V (T^T V^T C), with T^T V^T C built by the
//    recurrence  z_t = w_t - sum_{u<t} tau_u (v_u^T v_t) z_u  from the raw products
//    w_t = v_t^T C that ride along with every step.
//  * Two pushes per step.  CRITICAL (waited for at once): the dot products of v_j with the
//    active columns and the five sums that predict column j+1's sigma and x0 (as in
//    panel_geqr2: one exchange per column, exact fallback on cancellation).  LAZY
//    (triple-buffered, consumed one step later, i.e. hidden behind the next exchange):
//    v_j^T V(:, :j) for T and v_j^T C for the stale columns.
//  * Every sum over lanes, CTAs and steps has a fixed order: bitwise deterministic, and
//    every CTA derives identical reflector scalars.
//
// Reflector convention, R(j,j) from the update itself, tau = 0 / 2 for sigma == 0: as
// panel_geqr2 (core.py:57-76).  T: core.py:101-109 from the Gram columns, on CTA 0.
#pragma once

namespace urv {
namespace {

constexpr int CL_THREADS = 256;
constexpr int CL_MAXC = 16;   // CTAs per cluster (8 portable, 16 opt-in)
constexpr int CL_XW = 16;     // critical payload slots per step
constexpr int CL_NB = 64;     // leaf width

// ((a0+a1)+(a2+a3)) + ... over 16 consecutive doubles (16-byte aligned), fixed order
__device__ __forceinline__ double sum16(const double* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a0 = q[0], a1 = q[1], a2 = q[2], a3 = q[3], a4 = q[4], a5 = q[5], a6 = q[6], a7 = q[7];
  const double s0 = (a0.x + a0.y) + (a1.x + a1.y), s1 = (a2.x + a2.y) + (a3.x + a3.y);
  const double s2 = (a4.x + a4.y) + (a5.x + a5.y), s3 = (a6.x + a6.y) + (a7.x + a7.y);
  return (s0 + s1) + (s2 + s3);
}

// Push `v` into [slot] of CTAs rank0 .. rank0+3 (those below csz) of the cluster.
__device__ __forceinline__ void push4(double* slot, uint64_t* bar, int rank0, int csz, double v) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (rank0 + r < csz) dsmem_push_f64(slot, bar, rank0 + r, v);
}

struct ClScalars {
  double tau, rv0;
};
// core.py:57-76 from sigma = ||x(1:)||^2 and x0, arranged so that the two divisions do not
// depend on each other (the scalars sit on the per-column critical path: sqrt 101 + division
// 134 cycles instead of sqrt + two dependent divisions).  With mu = sqrt(x0^2 + sigma) and
// v0 = x0 - mu:  sigma + v0^2 = -2 mu v0, so  tau = 2 v0^2 / (sigma + v0^2) = -v0 / mu;
// for x0 > 0 the cancellation-free v0 = -sigma / (x0 + mu) gives
// tau = sigma / ((x0 + mu) mu)  and  1 / v0 = -(x0 + mu) / sigma.
__device__ __forceinline__ ClScalars cl_reflector(double sigma, double x0) {
  ClScalars s;
  if (sigma == 0.0) {
    s.tau = (x0 >= 0.0) ? 0.0 : 2.0;
    s.rv0 = 1.0;
  } else {
    const double mu = sqrt(x0 * x0 + sigma);
    if (x0 <= 0.0) {
      const double v0 = x0 - mu;
      s.tau = -v0 / mu;
      s.rv0 = 1.0 / v0;
    } else {
      const double d = x0 + mu;
      s.tau = sigma / (d * mu);
      s.rv0 = -d / sigma;
    }
  }
  return s;
}

// packed strict upper triangle: entry (k, j), k < j
__device__ __forceinline__ int tri(int k, int j) { return j * (j - 1) / 2 + k; }

template <int RTR, int RTS>
constexpr int panel_cl_smem_bytes() {
  constexpr int RT = RTR + RTS, RB = 32 * RT;
  return (2 * CL_XW * 16 + 2 * 2 * 16 + 3 * 8 * 16 + 3 * CL_NB + 1024 + CL_NB * (CL_NB - 1) / 2 + 8 * CL_NB + 8 * RB + RB +
          RTS * 8 * CL_THREADS + 8 * 8 * 8 + CL_NB + 8) *
             static_cast<int>(sizeof(double)) +
         12 * static_cast<int>(sizeof(uint64_t));
}

template <int RTR, int RTS>
__global__ void __launch_bounds__(CL_THREADS, 1)
    panel_cl(double* __restrict__ P, long long ldp, int M, int ncols, double* __restrict__ Tout, int ldt,
             double* __restrict__ Vout, long long ldv, int vzero_rows, int exact_sigma,
             unsigned long long* __restrict__ prof) {
  constexpr int RT = RTR + RTS, RB = 32 * RT, NB = CL_NB;
  extern __shared__ __align__(16) double cl_dyn[];
  // ---- shared memory carve-up (doubles) ----
  double* xin = cl_dyn;                       // [2][CL_XW][16]  critical inbox: [parity][slot][rank]
  double* nin = xin + 2 * CL_XW * 16;         // [2][2][16]      exact-norm inbox
  double* pin = nin + 2 * 2 * 16;             // [3][8][16]      lazy partials of the values this CTA owns: [buffer][k / csz][rank]
  double* tin = pin + 3 * 8 * 16;             // [3][NB]         lazy totals
  double* Xs = tin + 3 * NB;                  // [1024]          scratch of the T build
  double* Gp = Xs + 1024;             // packed (k < j): v_k^T v_j, then T(k, j) on CTA 0
  double* Wz = Gp + NB * (NB - 1) / 2;        // [8][NB]         w_t[k] = v_t^T C(:, k), stale columns
  double* vbuf = Wz + 8 * NB;                 // [8][RB]         v of the inner block's reflectors
  double* xcur = vbuf + 8 * RB;               // [RB]            the next column to be factored
  double* srow = xcur + RB;                   // [RTS][8][256]   shared-memory rows
  double* Cz = srow + RTS * 8 * CL_THREADS;   // [8 warps][8 t][8 q]  tau_t z_t of the warp's columns
  double* taus = Cz + 8 * 8 * 8;              // [NB]
  double* pred = taus + NB;                   // [8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(pred + 8);
  uint64_t* xbar = bars;                      // [2]
  uint64_t* nbar = bars + 2;                  // [2]
  uint64_t* pbar = bars + 4;                  // [3]
  uint64_t* tbar = bars + 7;                  // [3]

  cg::cluster_group cl = cg::this_cluster();
  const int csz = static_cast<int>(cl.num_blocks());  // 8 or 16
  const int lcsz = (csz == 16) ? 4 : 3;
  const int crank = static_cast<int>(cl.block_rank());
  // bits 1-2: where the lazy work of a step sits.  0: products, owner sums and total take-up all before
  // the critical wait (behind the exchange); 1: all of it after the update, beside the next owner's
  // scalars (measured slower: the exchange latency, ~500 cycles, is then exposed: 3968 vs 3788 cycles
  // per column at 512 rows); 2: products before the wait, owner sums + take-up after the update.
  const int lazy_mode = (exact_sigma >> 1) & 3;
  const bool lazy_late = lazy_mode == 1, drain_late = lazy_mode != 0;
  exact_sigma &= 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = crank * RB;
  const int nrows = max(0, min(RB, M - r0));
  // URV_PANEL_PROF: cycles per phase seen by thread 0 of CTA 0 (slots 0-7) and of the last CTA (8-15)
  const bool timing = prof != nullptr && tid == 0 && crank == 0;
  unsigned long long tph[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tlast = timing ? clock64() : 0;
  auto tick = [&](int k) {
    if (timing) {
      const unsigned long long now = clock64();
      tph[k] += now - tlast;
      tlast = now;
    }
  };

  // ---- init: inboxes zero (ranks >= csz stay zero), barriers ----
  for (int k = tid; k < 2 * CL_XW * 16 + 2 * 2 * 16 + 3 * 8 * 16; k += CL_THREADS) xin[k] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 10; ++b) mbar_init(&bars[b], 1);
    mbar_fence_init();
  }

  // ---- load ----
  double S[RTR > 0 ? RTR : 1][8];
  auto srow_at = [&](int i, int q) -> double& { return srow[((i - RTR) * 8 + q) * CL_THREADS + tid]; };
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = lane + 32 * i;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int col = warp + 8 * q;
      const double x = (col < ncols && r < nrows) ? P[(r0 + r) + static_cast<long long>(col) * ldp] : 0.0;
      if (i < RTR) S[i][q] = x;
      else srow_at(i, q) = x;
    }
  }
  auto getS = [&](int i, int q) -> double {  // compile-time i, q after unrolling
    if (i < RTR) return S[i][q];
    return srow_at(i, q);
  };
  auto setS = [&](int i, int q, double x) {
    if (i < RTR) S[i][q] = x;
    else srow_at(i, q) = x;
  };
  cl.sync();  // barriers and zeroed inboxes of every CTA exist before the first push

  tick(7);
  int cnt_x = 0, cnt_n = 0;  // critical / exact-norm exchanges so far (parity, phase)
  double act[RT];            // the warp's column of the current inner block

  // Exact sigma = ||A(col+1:, col)||^2 and x0 = A(col, col); col is an active column.
  auto exact_norm = [&](int col, double& sigma, double& x0) {
    const int b = cnt_n & 1;
    const uint32_t phase = (cnt_n >> 1) & 1;
    if (tid == 0) mbar_expect_tx(&nbar[b], static_cast<uint32_t>(csz) * 2 * 8);
    if (warp == (col & 7)) {
      double sv = 0.0, xv = 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int gi = r0 + lane + 32 * i;  // padded rows hold zeros
        if (gi > col) sv += act[i] * act[i];
        if (gi == col) xv = act[i];
      }
      sv = warp_sum(sv);
      xv = warp_sum(xv);  // a single nonzero term
      if (lane < csz) {
        dsmem_push_f64(&nin[(b * 2 + 0) * 16 + crank], &nbar[b], lane, sv);
        dsmem_push_f64(&nin[(b * 2 + 1) * 16 + crank], &nbar[b], lane, xv);
      }
    }
    mbar_wait_cluster(&nbar[b], phase);
    sigma = sum16(&nin[(b * 2 + 0) * 16]);
    x0 = sum16(&nin[(b * 2 + 1) * 16]);
    ++cnt_n;
  };

  // Lazy payload of step jl, two hops one step apart (an all-to-all of 64 values costs 1024
  // remote stores per CTA and step; this costs 128): value k is summed by its owner CTA
  // k % csz (reduce_partials, one step after the partials were pushed), which pushes the total
  // to everybody (consume_totals, another step later) -> Gp / Wz.
  int next_p = 0, next_t = 0;  // next lazy step to reduce at its owners / whose totals to take
  // Both run on warps away from the step's owner and next owner (jl + 4 .. jl + 6 mod 8).
  auto reduce_partials = [&](int jl) {
    if (warp != ((jl + 4) & 7)) return;
    const int bl = jl % 3;
    mbar_wait_cluster(&pbar[bl], static_cast<uint32_t>((jl / 3) & 1));
#pragma unroll
    for (int u = 0; u < 2; ++u) {  // NB = (NB / csz) owned values x csz destinations
      const int idx = lane + 32 * u;
      const int kl = idx >> lcsz, r = idx & (csz - 1);
      const double tot = sum16(&pin[(bl * 8 + kl) * 16]);
      dsmem_push_f64(&tin[bl * NB + (kl << lcsz) + crank], &tbar[bl], r, tot);
    }
  };
  auto consume_totals = [&](int jl) {
    const int w = (warp - jl - 5) & 7;  // warps jl + 5 and jl + 6 take 32 columns each
    if (w > 1) return;
    const int bl = jl % 3;
    mbar_wait_cluster(&tbar[bl], static_cast<uint32_t>((jl / 3) & 1));
    const int k = 32 * w + lane;
    const double tot = tin[bl * NB + k];
    if (k < jl) Gp[tri(k, jl)] = tot;
    else if ((k >> 3) > (jl >> 3)) Wz[(jl & 7) * NB + k] = tot;
  };

  for (int qb = 0; 8 * qb < ncols; ++qb) {
    // ---- inner block qb: its columns become active ----
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      double x = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q == qb) x = getS(i, q);
      act[i] = x;
    }
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < RT; ++i) xcur[lane + 32 * i] = act[i];
    }
    __syncthreads();
    double sigma, x0;
    exact_norm(8 * qb, sigma, x0);
    ClScalars sc = cl_reflector(sigma, x0);
    tick(5);
    const int jend = min(ncols, 8 * qb + 8);

    for (int j = 8 * qb; j < jend; ++j) {
      const int wj = j & 7, jn = j + 1;
      const bool has_next = jn < jend;
      const double tau = sc.tau;
      if (tid == 0) taus[j] = tau;
      const int b = cnt_x & 1;
      const uint32_t phase = (cnt_x >> 1) & 1;
      const int bl = j % 3;
      if (tid == 0) mbar_expect_tx(&xbar[b], static_cast<uint32_t>(csz) * (has_next ? 13 : 8) * 8);
      if (tid == 32) mbar_expect_tx(&pbar[bl], NB * 8);
      if (tid == 64) mbar_expect_tx(&tbar[bl], NB * 8);
      // v over this thread's rows: 0 above j (and on padded rows, where x = 0), 1 at j.
      // Loads first, then selects: no branches (a branch per row serialises the loads).
      double v[RT];
      {
        double xc[RT];
#pragma unroll
        for (int i = 0; i < RT; ++i) xc[i] = xcur[lane + 32 * i];
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const int gi = r0 + lane + 32 * i;
          const double t = xc[i] * sc.rv0;
          v[i] = (gi > j) ? t : ((gi == j) ? 1.0 : 0.0);
        }
      }
      // ---- critical: v^T (active column), and the sums that predict column j+1 ----
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i) sacc += v[i] * act[i];
      if (has_next && warp == wj + 1) {
        double e[8] = {sacc, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const int gi = r0 + lane + 32 * i;
          const double xm = (gi > jn) ? act[i] : 0.0, vm = (gi > jn) ? v[i] : 0.0;
          e[1] += xm * xm;
          e[2] += vm * xm;
          e[3] += vm * vm;
          e[4] = (gi == jn) ? act[i] : e[4];
          e[5] = (gi == jn) ? v[i] : e[5];
        }
        const double t = reduce_scatter<8>(e, lane);
        const int f = lane >> 2;
        if (f < 6)
          push4(&xin[(b * CL_XW + (f == 0 ? warp : 8 + f)) * 16 + crank], &xbar[b], 4 * (lane & 3), csz, t);
      } else {
        const double t = (warp >= wj) ? warp_sum(sacc) : 0.0;
        if (lane < csz) dsmem_push_f64(&xin[(b * CL_XW + warp) * 16 + crank], &xbar[b], lane, t);
      }
      tick(0);
      // ---- lazy: v^T (finished columns) for T, v^T (stale columns) for the block update ----
      // Only the next owner does them here, behind its exchange; every other warp does them after
      // the update below, while the next owner computes the next reflector's scalars (they used
      // to idle at the step's __syncthreads for that long).  Same arithmetic either way.
      auto lazy_products = [&]() {
        double lz[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double a = 0.0;
#pragma unroll
          for (int i = 0; i < RT; ++i) a += v[i] * getS(i, q);
          lz[q] = a;
        }
        // the active column of a warp below wj is a finished column of this inner block
        // (its S copy is stale: take the registers); at and above wj it went the critical way
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q == qb) lz[q] = (warp < wj) ? sacc : 0.0;
        const double t = reduce_scatter<8>(lz, lane);
        if ((lane & 3) == 0) {
          const int k = warp + 8 * (lane >> 2);
          dsmem_push_f64(&pin[(bl * 8 + (k >> lcsz)) * 16 + crank], &pbar[bl], k & (csz - 1), t);
        }
      };
      const bool lazy_now = !lazy_late || (has_next && warp == wj + 1);
      if (lazy_now) lazy_products();
      tick(8);
      if (!drain_late) {
        while (next_p < j) reduce_partials(next_p++);
        tick(9);
        while (next_t < j - 1) consume_totals(next_t++);
      }
      tick(1);
      // ---- wait for the critical totals ----
      mbar_wait_cluster(&xbar[b], phase);
      ++cnt_x;
      tick(2);
      const double s = sum16(&xin[(b * CL_XW + warp) * 16]);
      if (warp >= wj && tau != 0.0) {
        const double ts = tau * s;
#pragma unroll
        for (int i = 0; i < RT; ++i) act[i] -= v[i] * ts;  // v = 0 above row j
      }
      if (warp == wj) {  // R(j,j) stays on row j; v is stored below it
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const int r = lane + 32 * i;
          if (r0 + r > j) act[i] = v[i];
          vbuf[wj * RB + r] = v[i];
        }
      }
      if (has_next && warp == wj + 1) {
        // the next owner: column j+1 for everybody, its predicted sigma / x0 and -- when the
        // prediction holds -- its reflector scalars, so that the other warps only read them
#pragma unroll
        for (int i = 0; i < RT; ++i) xcur[lane + 32 * i] = act[i];
        const double pX = sum16(&xin[(b * CL_XW + 9) * 16]), pP = sum16(&xin[(b * CL_XW + 10) * 16]);
        const double pV = sum16(&xin[(b * CL_XW + 11) * 16]), pA = sum16(&xin[(b * CL_XW + 12) * 16]);
        const double pJ = sum16(&xin[(b * CL_XW + 13) * 16]);
        const double cc = tau * s;
        const double sig = pX - 2.0 * cc * pP + cc * cc * pV;
        const bool ok = !exact_sigma && ((tau == 0.0) || (sig >= 0.5 * (pX + cc * cc * pV) && isfinite(sig)));
        const double psig = (tau == 0.0) ? pX : sig, px0 = (tau == 0.0) ? pA : pA - pJ * cc;
        const ClScalars nsc = cl_reflector(psig, px0);
        if (lane == 0) {
          pred[0] = psig;
          pred[1] = px0;
          pred[2] = ok ? 1.0 : 0.0;
          pred[3] = nsc.tau;
          pred[4] = nsc.rv0;
        }
      }
      if (!lazy_now) lazy_products();
      if (drain_late) {
        while (next_p < j) reduce_partials(next_p++);
        while (next_t < j - 1) consume_totals(next_t++);
      }
      tick(3);
      __syncthreads();
      if (has_next) {
        if (pred[2] != 0.0) {
          sc.tau = pred[3];
          sc.rv0 = pred[4];
        } else {
          exact_norm(jn, sigma, x0);  // cancellation: recompute from the updated column
          sc = cl_reflector(sigma, x0);
        }
      }
      tick(4);
    }

    // ---- inner block done: registers back to the panel, reflectors onto the stale columns ----
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q == qb) setS(i, q, act[i]);
    while (next_p < jend) reduce_partials(next_p++);
    while (next_t < jend) consume_totals(next_t++);
    if (jend >= ncols) break;
    __syncthreads();  // Gp entries of this block (written by their columns' warps), vbuf, taus
    // c_t = tau_t z_t,  z_t = w_t - sum_{u<t} (v_u^T v_t) c_u   (H_0 first, as core.py:149-151
    // applies them): lane q > qb of each warp does its column warp + 8 q
    if (lane < 8 && lane > qb) {
      const int k = warp + 8 * lane;
      double c[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        double a = Wz[t * NB + k];
#pragma unroll
        for (int u = 0; u < t; ++u) a -= Gp[tri(8 * qb + u, 8 * qb + t)] * c[u];
        c[t] = taus[8 * qb + t] * a;
        Cz[(warp * 8 + t) * 8 + lane] = c[t];
      }
    }
    __syncwarp();
    // C(:, k) -= sum_t v_t c_t[k] for the stale columns of this warp, four reflectors a pass
#pragma unroll 1
    for (int t0 = 0; t0 < 8; t0 += 4) {
      double c4[4][8];
#pragma unroll
      for (int tt = 0; tt < 4; ++tt)
#pragma unroll
        for (int q = 0; q < 8; ++q) c4[tt][q] = (q > qb) ? Cz[(warp * 8 + t0 + tt) * 8 + q] : 0.0;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int r = lane + 32 * i;
        double vt[4];
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) vt[tt] = vbuf[(t0 + tt) * RB + r];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q > qb) {
            double x = getS(i, q);
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) x -= vt[tt] * c4[tt][q];
            setS(i, q, x);
          }
        }
      }
    }
  }

  tick(5);
  // ---- write back: R on/above the diagonal, V below it; the explicit unit-lower V ----
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = lane + 32 * i;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int col = warp + 8 * q;
      if (col < ncols && r < nrows) {
        const int gi = r0 + r;
        const double x = getS(i, q);
        P[gi + static_cast<long long>(col) * ldp] = x;
        if (Vout) Vout[gi + static_cast<long long>(col) * ldv] = gi < col ? 0.0 : (gi == col ? 1.0 : x);
      }
    }
  }
  if (Vout && crank == 0)  // rows of the outer block above this leaf: V is zero there
    for (int idx = tid; idx < vzero_rows * ncols; idx += CL_THREADS)
      Vout[-vzero_rows + idx % vzero_rows + static_cast<long long>(idx / vzero_rows) * ldv] = 0.0;
  cl.sync();  // nobody leaves while a peer may still push into its shared memory
  tick(7);
  if (crank != 0) return;

  // ---- CTA 0: T (core.py:101-109) from the Gram columns, in place in the packed triangle ----
  // The column recurrence T(:j, j) = -tau_j T(:j, :j) g_j is T = (D + striu(V^T V))^-1 with
  // D = diag(1 / tau); blocked it reads T12 = -T11 (V1^T V2) T22, done here level by level
  // (blocks of 2, 4, ... 64 columns, all blocks of a level at once): about 2k cycles instead
  // of 64 dependent steps.
  {
    double* X = Xs;  // [blocks][half][half] scratch
    for (int sb = 2; sb <= NB; sb <<= 1) {
      const int half = sb >> 1, hh = half * half;
      const int total = (NB / sb) * hh;
      // X = G12 T22:  X(r, c) = sum_{l <= c} G(c0 + r, c1 + l) T(c1 + l, c1 + c),  c1 = c0 + half
      const int lh = 31 - __clz(half), lhh = 2 * lh;
      for (int e = tid; e < total; e += CL_THREADS) {
        const int c0 = (e >> lhh) * sb, c1 = c0 + half;
        const int r = e & (half - 1), c = (e & (hh - 1)) >> lh;
        double a = 0.0;
        if (c1 + c < ncols) {
          int ig = tri(c0 + r, c1);          // G(c0 + r, c1 + l): next column is c1 + l further on
          const double* tc = &Gp[tri(c1, c1 + c)];  // T(c1 + l, c1 + c), contiguous in l
#pragma unroll 4
          for (int l = 0; l < c; ++l) {
            a += Gp[ig] * tc[l];
            ig += c1 + l;
          }
          a += Gp[ig] * taus[c1 + c];
        }
        X[e] = a;
      }
      __syncthreads();
      // T12(r, c) = -sum_{l >= r} T(c0 + r, c0 + l) X(l, c)
      for (int e = tid; e < total; e += CL_THREADS) {
        const int blk = e >> lhh, c0 = blk * sb, c1 = c0 + half;
        const int r = e & (half - 1), c = (e & (hh - 1)) >> lh;
        if (c1 + c < ncols) {
          const double* Xb = X + blk * hh + c * half;
          double a = taus[c0 + r] * Xb[r];
          int it = tri(c0 + r, c0 + r + 1);  // T(c0 + r, c0 + l)
#pragma unroll 4
          for (int l = r + 1; l < half; ++l) {
            a += Gp[it] * Xb[l];
            it += c0 + l;
          }
          Gp[tri(c0 + r, c1 + c)] = -a;
        }
      }
      __syncthreads();
    }
  }
  for (int k = tid; k < NB * NB; k += CL_THREADS) {
    const int r = k % NB, col = k / NB;
    double t = 0.0;
    if (col < ncols) {
      if (r == col) t = taus[col];
      else if (r < col) t = Gp[tri(r, col)];
    }
    Tout[r + static_cast<long long>(col) * ldt] = t;
  }
  tick(6);
  if (timing) {
#pragma unroll
    for (int k = 0; k < 16; ++k) atomicAdd(prof + k, tph[k]);
  }
}

}  // namespace
}  // namespace urv
