// Fused block-reflector application for narrow blocks (round 2):
//     C <- C - V op(T) (V^T C),   V: M x nb (nb <= 64), T: nb x nb upper, C: M x N
// i.e. core.py:149-151 (op(T) = T^T, the trailing / leaf update) and core.py:154-157
// (op(T) = T, explicit Q) in ONE kernel.  Included by qr.cu.
//
// The unfused chain (split-K DMMA GEMM for V^T C, sum_partials, apply_t, DMMA GEMM for
// C -= V W) costs four launches of 25-40 us each on the latency-bound panel chain of the
// small and mid-size factorisations (profiles/r02_timeline_c2_cl.txt); this kernel does the
// same arithmetic in about the time of one of them:
//   * one cluster of CS <= 16 CTAs per strip of NS = 16 columns of C; CTA r of the cluster
//     owns a row block of V and C, staged once in shared memory (256-row chunks);
//   * phase 1: W_r = V_r^T C_r on the FP64 tensor cores (mma.m8n8k4: warp w owns rows
//     8w..8w+7 of W), accumulated over the CTA's chunks;
//   * all-reduce over the cluster in two hops through distributed shared memory: column n
//     of W is owned by one CTA, which adds the CS partials in rank order, multiplies by
//     op(T) and pushes the 64 results to every CTA (fixed order: bitwise deterministic);
//   * phase 2: C_r -= V_r W on the tensor cores, coalesced write-back.
#pragma once

namespace urv {
namespace {

constexpr int AP_THREADS = 256;
constexpr int AP_NS = 16;         // columns of C per cluster
constexpr int AP_CH = 256;        // rows per staged chunk
constexpr int AP_LD = AP_CH + 4;  // leading dimension of the staged chunks (conflict-free fragments)
constexpr int AP_LDW = 68;        // leading dimension of W (64 + 4)
constexpr int AP_LDT = 65;        // leading dimension of T in shared memory

constexpr int apply_cl_smem_bytes() {
  return (64 * AP_LD + AP_NS * AP_LD + AP_NS * AP_LDW + 64 * AP_LDT + 64 * AP_NS + 64 * AP_NS) *
             static_cast<int>(sizeof(double)) +
         2 * static_cast<int>(sizeof(uint64_t));
}

__global__ void __launch_bounds__(AP_THREADS, 1)
    block_apply_cl(const double* __restrict__ V, long long ldv, const double* __restrict__ T, int ldt, int trans,
                   double* __restrict__ C, long long ldc, int M, int N, int nb, int leafw, int rows_per_cta) {
  extern __shared__ __align__(16) double ap_dyn[];
  double* Vs = ap_dyn;                    // [64][AP_LD]   V chunk, column-major
  double* Cs = Vs + 64 * AP_LD;           // [NS][AP_LD]   C chunk, column-major
  double* Ws = Cs + AP_NS * AP_LD;        // [NS][AP_LDW]  W = op(T) V^T C (totals), column-major
  double* Ts = Ws + AP_NS * AP_LDW;       // [64][AP_LDT]  T
  double* inb = Ts + 64 * AP_LDT;         // [CS][cols_owned * 64] partials of the columns this CTA owns
  double* w0 = inb + 64 * AP_NS;          // [cols_owned * 64] their sums
  uint64_t* bars = reinterpret_cast<uint64_t*>(w0 + 64 * AP_NS);  // [0] partials, [1] totals

  cg::cluster_group cl = cg::this_cluster();
  const int CS = static_cast<int>(cl.num_blocks());
  const int crank = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.y * AP_NS;
  const int ncols = min(AP_NS, N - n0);
  const int cols_owned = AP_NS / CS;  // columns of W this CTA sums (CS divides NS)
  const int rbeg = crank * rows_per_cta;
  const int rows_cta = max(0, min(rows_per_cta, M - rbeg));
  const int nchunks = (rows_cta + AP_CH - 1) / AP_CH;
  const int nleaves = (nb + leafw - 1) / leafw;
  const int lr = lane >> 2, lc = lane & 3;  // fragment coordinates

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  // columns of the staged C beyond the strip stay zero
  for (int c = ncols; c < AP_NS; ++c) Cs[c * AP_LD + tid] = 0.0;
  cl.sync();  // every barrier of the cluster exists before the first push

  // Rows [chunk*CH, +CH) of this CTA's V (nbl columns from column vc0) and C into shared
  // memory: thread = row, one asynchronous 8-byte copy per element, all in flight (a loop of
  // dependent global loads made this the longest phase of the kernel).  Rows past the CTA's
  // rows and V columns past nbl are zero.
  auto stage = [&](int chunk, int vc0, int nbl, bool with_c) {
    const int cb = chunk * AP_CH;
    const int ch = min(AP_CH, rows_cta - cb);
    if (tid < ch) {
      const double* vrow = V + (rbeg + cb + tid) + static_cast<long long>(vc0) * ldv;
#pragma unroll 8
      for (int c = 0; c < nbl; ++c) cp_async_f64(&Vs[c * AP_LD + tid], vrow + static_cast<long long>(c) * ldv);
      if (with_c) {
        const double* crow = C + (rbeg + cb + tid) + static_cast<long long>(n0) * ldc;
#pragma unroll 8
        for (int c = 0; c < ncols; ++c) cp_async_f64(&Cs[c * AP_LD + tid], crow + static_cast<long long>(c) * ldc);
      }
    } else {
      for (int c = 0; c < nbl; ++c) Vs[c * AP_LD + tid] = 0.0;
      if (with_c)
        for (int c = 0; c < ncols; ++c) Cs[c * AP_LD + tid] = 0.0;
    }
    for (int c = nbl; c < 64; ++c) Vs[c * AP_LD + tid] = 0.0;
    cp_async_wait_all();
  };

  // The leaves of the block one after the other (H = H_0 H_1 ...: H^T C applies leaf 0 first,
  // H C the last leaf first); with one chunk per CTA the strip of C stays in shared memory.
  for (int li = 0; li < nleaves; ++li) {
    const int l = trans ? li : nleaves - 1 - li;
    const int c0 = l * leafw;
    const int nbl = min(leafw, nb - c0);
    const uint32_t parity = li & 1;
    if (tid == 0) {
      mbar_expect_tx(&bars[0], static_cast<uint32_t>(CS) * cols_owned * 64 * 8);
      mbar_expect_tx(&bars[1], 64 * AP_NS * 8);
    }
    // T of the leaf by asynchronous copies (needed only after phase 1); zeros outside nbl x nbl
    {
      const double* Tl = T + c0 + static_cast<long long>(c0) * ldt;
#pragma unroll 4
      for (int idx = tid; idx < 64 * 64; idx += AP_THREADS) {
        const int r = idx & 63, c = idx >> 6;
        if (r < nbl && c < nbl) cp_async_f64(&Ts[r + c * AP_LDT], &Tl[r + static_cast<long long>(c) * ldt]);
        else Ts[r + c * AP_LDT] = 0.0;
      }
    }
    // ---- phase 1: W_r(8w.., :) = V_r(:, 8w..)^T C_r over the chunks ----
    double acc[AP_NS / 8][2];
#pragma unroll
    for (int t = 0; t < AP_NS / 8; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      if (chunk > 0 || li > 0) __syncthreads();
      stage(chunk, c0, nbl, li == 0 || nchunks > 1);
      __syncthreads();
      if (8 * warp < nbl) {
        const double* va = Vs + (8 * warp + lr) * AP_LD + lc;
        const double* cb0 = Cs + lr * AP_LD + lc;
        const int kend = (min(AP_CH, rows_cta - chunk * AP_CH) + 3) & ~3;  // rows past the chunk are zero
#pragma unroll 4
        for (int k = 0; k < kend; k += 4) {
          const double a = va[k];
#pragma unroll
          for (int t = 0; t < AP_NS / 8; ++t) dmma_8x8x4(acc[t][0], acc[t][1], a, cb0[8 * t * AP_LD + k]);
        }
      }
    }
    if (nchunks == 0) cp_async_wait_all();  // T (a CTA without rows still owns columns of W)
    // partials to the owners of the columns: lane holds W_r(8w + lr, 8t + 2 lc + {0, 1})
#pragma unroll
    for (int t = 0; t < AP_NS / 8; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 8 * t + 2 * lc + e, i = 8 * warp + lr;
        const int owner = n / cols_owned, nl = n % cols_owned;
        dsmem_push_f64(&inb[crank * cols_owned * 64 + nl * 64 + i], &bars[0], owner, acc[t][e]);
      }
    // ---- owners: sum in rank order, multiply by op(T), push the totals to everybody ----
    mbar_wait_cluster(&bars[0], parity);
    for (int idx = tid; idx < cols_owned * 64; idx += AP_THREADS) {
      double sv = 0.0;
      for (int r = 0; r < CS; ++r) sv += inb[r * cols_owned * 64 + idx];
      w0[idx] = sv;
    }
    __syncthreads();  // w0, and T (every thread waited for its own copies)
    for (int idx = tid; idx < cols_owned * 64; idx += AP_THREADS) {
      const int nl = idx >> 6, i = idx & 63;
      const double* w = w0 + nl * 64;
      double sv = 0.0;
      if (trans) {  // (T^T w)(i) = sum_{l <= i} T(l, i) w(l)
        for (int k = 0; k <= i; ++k) sv += Ts[k + i * AP_LDT] * w[k];
      } else {  // (T w)(i) = sum_{l >= i} T(i, l) w(l)
        for (int k = i; k < 64; ++k) sv += Ts[i + k * AP_LDT] * w[k];
      }
      const int n = crank * cols_owned + nl;
      for (int r = 0; r < CS; ++r) dsmem_push_f64(&Ws[n * AP_LDW + i], &bars[1], r, sv);
    }
    mbar_wait_cluster(&bars[1], parity);

    // ---- phase 2: C_r -= V_r W ----
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      if (nchunks > 1) {  // a single chunk is still staged
        __syncthreads();
        stage(chunk, c0, nbl, true);
        __syncthreads();
      }
      const int cb = chunk * AP_CH;
      const int ch = min(AP_CH, rows_cta - cb);
      for (int rt = warp; 8 * rt < ch; rt += AP_THREADS / 32) {
        const int rr = 8 * rt + lr;
        double d[AP_NS / 8][2];
#pragma unroll
        for (int t = 0; t < AP_NS / 8; ++t) {
          d[t][0] = Cs[(8 * t + 2 * lc) * AP_LD + rr];
          d[t][1] = Cs[(8 * t + 2 * lc + 1) * AP_LD + rr];
        }
        for (int k = 0; k < nbl; k += 4) {
          const double a = -Vs[(k + lc) * AP_LD + rr];
#pragma unroll
          for (int t = 0; t < AP_NS / 8; ++t) dmma_8x8x4(d[t][0], d[t][1], a, Ws[(8 * t + lr) * AP_LDW + k + lc]);
        }
#pragma unroll
        for (int t = 0; t < AP_NS / 8; ++t) {
          Cs[(8 * t + 2 * lc) * AP_LD + rr] = d[t][0];
          Cs[(8 * t + 2 * lc + 1) * AP_LD + rr] = d[t][1];
        }
      }
      __syncthreads();
      if (nchunks > 1 || li == nleaves - 1) {
        for (int idx = tid; idx < AP_NS * AP_CH; idx += AP_THREADS) {
          const int r = idx & (AP_CH - 1), c = idx >> 8;
          if (r < ch && c < ncols) C[(rbeg + cb + r) + static_cast<long long>(n0 + c) * ldc] = Cs[c * AP_LD + r];
        }
      }
    }
  }
  cl.sync();  // nobody leaves while a peer may still push into its shared memory
}

}  // namespace
}  // namespace urv
