// Latency probe (round 2, session 3) for the panel's per-column all-reduce of PW = 72
// doubles, the way the panel would use it (one dependent round after another):
//   A. hierarchical: every CTA st.async-pushes its partials into the cluster leader's
//      shared memory (mbarrier complete_tx), the leader sums them in rank order and
//      publishes the cluster partial as LL lines {lo32,tag | hi32,tag}; every CTA polls
//      the NCL lines of each value it needs with all loads in flight at once.
//   B. flat LL: every CTA publishes its own partial, every CTA polls G lines per value.
//   C. single cluster: all-to-all st.async push, sums from local shared memory.
// Prints cycles per round seen by CTA 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 xchg_latency.cu -o xchg_latency
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;
constexpr int ITER = 2000;
constexpr int PW = 72;
constexpr int CSZ_MAX = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ll_store(unsigned long long* p, double v, unsigned int gen) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned long long w0 = (static_cast<unsigned long long>(gen) << 32) | (bits & 0xffffffffull);
  const unsigned long long w1 = (static_cast<unsigned long long>(gen) << 32) | (bits >> 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ void ll_ld(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ bool ll_ok(unsigned long long w0, unsigned long long w1, unsigned int gen) {
  return static_cast<unsigned int>(w0 >> 32) == gen && static_cast<unsigned int>(w1 >> 32) == gen;
}
__device__ __forceinline__ double ll_val(unsigned long long w0, unsigned long long w1) {
  return __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
}
__device__ __forceinline__ void push_f64(double* local_slot, uint64_t* local_bar, int rank, double v) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_slot)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// mode 0: hierarchical (A); mode 1: flat LL (B); mode 2: single-cluster all-to-all (C)
// staged = 1: partials go through pay[] + __syncthreads first (as the panel does today)
template <int MODE>
__global__ void k_xchg(unsigned long long* out, unsigned long long* gll, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  const int csz = cl.num_blocks(), crank = cl.block_rank();
  const int G = gridDim.x, c = blockIdx.x, cid = c / csz, NCL = G / csz;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ __align__(16) double slot[2][CSZ_MAX][PW];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double pay[2][PW];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  double carry = 0.0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) {
    const int b = i & 1;
    const uint32_t phase = (i >> 1) & 1;
    const unsigned int tag = i + 1;
    // partial payload (depends on the previous round's totals)
    if (tid < PW) pay[b][tid] = carry * 1e-9 + c + tid * 1e-3;
    __syncthreads();
    unsigned long long* lines = gll + static_cast<long long>(b) * 148 * PW * 2;
    if (MODE == 0) {
      if (crank == 0 && tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(csz * PW * 8)
                     : "memory");
      if (tid < PW) push_f64(&slot[b][crank][tid], &bar[b], 0, pay[b][tid]);
      if (crank == 0 && tid < PW) {
        bar_wait(&bar[b], phase);
        double sv = 0.0;
        for (int r = 0; r < csz; ++r) sv += slot[b][r][tid];
        ll_store(lines + 2 * (cid * PW + tid), sv, tag);
      }
    } else if (MODE == 1) {
      if (tid < PW) ll_store(lines + 2 * (c * PW + tid), pay[b][tid], tag);
    } else {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(csz * PW * 8)
                     : "memory");
      if (tid < PW) {
        const double v = pay[b][tid];
        for (int r = 0; r < csz; ++r) push_f64(&slot[b][crank][tid], &bar[b], r, v);
      }
    }
    // totals of this warp's 8 values: lane = (q, h), q = lane % 8 the value, h = lane / 8 the chain
    const int q = lane & 7, h = lane >> 3, k = warp + 8 * q;
    double sv = 0.0;
    if (MODE == 2) {
      bar_wait(&bar[b], phase);
      for (int r = h; r < csz; r += 4) sv += slot[b][r][k];
    } else {
      const int n = (MODE == 0) ? NCL : G;
      constexpr int PER = 10;  // up to 40 partials over 4 chains
      unsigned long long w0[PER], w1[PER];
      bool done;
      do {
        done = true;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int cc = h + 4 * u;
          if (cc < n) ll_ld(lines + 2 * (cc * PW + k), w0[u], w1[u]);
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int cc = h + 4 * u;
          if (cc < n && !ll_ok(w0[u], w1[u], tag)) done = false;
        }
      } while (!done);
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int cc = h + 4 * u;
        if (cc < n) sv += ll_val(w0[u], w1[u]);
      }
    }
    sv += __shfl_xor_sync(0xffffffffu, sv, 8);
    sv += __shfl_xor_sync(0xffffffffu, sv, 16);
    carry = sv;
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (c == 0 && tid == 0) out[0] = (t1 - t0) / ITER;
  cl.sync();
  sink[c * blockDim.x + tid] = carry;
}

template <class K, class... A>
void launch_cluster(K kern, int grid, int csz, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = csz;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (csz > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
}

int main() {
  unsigned long long *out, *gll;
  double* sink;
  cudaMalloc(&out, 8 * sizeof(unsigned long long));
  cudaMalloc(&sink, 148 * 256 * sizeof(double));
  cudaMalloc(&gll, 2 * 148 * PW * 2 * sizeof(unsigned long long));
  auto run = [&](const char* name, auto kern, int grid, int csz) {
    unsigned long long h = 0;
    cudaMemset(gll, 0, 2 * 148 * PW * 2 * sizeof(unsigned long long));
    cudaMemset(out, 0, 64);
    launch_cluster(kern, grid, csz, out, gll, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %3d CTAs (clusters of %2d): %5llu cycles/round (%s)\n", name, grid, csz, h, cudaGetErrorString(e));
  };
  for (int ncl : {2, 3, 5, 8}) run("A hierarchical push+LL", k_xchg<0>, ncl * 8, 8);
  for (int ncl : {2, 4}) run("A hierarchical push+LL", k_xchg<0>, ncl * 16, 16);
  for (int g : {16, 24, 40}) run("B flat LL", k_xchg<1>, g, 8);
  run("C single-cluster all-to-all push", k_xchg<2>, 8, 8);
  run("C single-cluster all-to-all push", k_xchg<2>, 16, 16);
  run("C single-cluster all-to-all push", k_xchg<2>, 4, 4);
  run("C single-cluster all-to-all push", k_xchg<2>, 2, 2);
  return 0;
}
