// Latency probe for the panel's per-column exchange primitives on B200 (sm_100a):
//   1. cluster barrier (barrier.cluster.arrive.release + wait.acquire), 8 / 16 CTAs
//   2. DSMEM pull: cl.sync, then every CTA loads one double from each peer
//   3. DSMEM push: every CTA st.async's one double into every peer's smem with
//      mbarrier complete_tx, then waits on its own mbarrier (no cluster barrier)
//   4. grid barrier among G CTAs: red.release.gpu add + relaxed spin + acq_rel fence
// Each test loops ITER rounds inside one kernel; prints cycles per round (CTA 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 sync_latency.cu -o sync_latency
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;
constexpr int ITER = 2000;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_cluster_sync(unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) cl.sync();
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / ITER;
}

__global__ void k_dsmem_pull(unsigned long long* out, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double val[2];
  const int csz = cl.num_blocks();
  double acc = 0.0;
  cl.sync();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) {
    if (threadIdx.x == 0) val[i & 1] = i + blockIdx.x;
    cl.sync();
    if (threadIdx.x < csz) acc += *cl.map_shared_rank(&val[i & 1], threadIdx.x);
    acc = __shfl_sync(0xffffffffu, acc, 0) + acc * 1e-300;  // use it (dependency)
  }
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / ITER;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_dsmem_push(unsigned long long* out, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  const int csz = cl.num_blocks();
  const int rank = cl.block_rank();
  __shared__ __align__(8) double inbox[2][16];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  double acc = 0.0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) {
    const int b = i & 1;
    const uint32_t phase = (i >> 1) & 1;
    if (threadIdx.x == 0)  // expect csz doubles this round
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])),
                   "r"(csz * 8) : "memory");
    // every CTA must have armed its barrier before peers' bytes land: arming precedes
    // the remote stores of THIS round only via the previous round's wait (double buffer)
    if (threadIdx.x < csz) {
      const double v = i + rank;
      // remote addresses of peer threadIdx.x's inbox slot [rank] and its mbarrier
      const uint32_t la = smem_u32(&inbox[b][rank]), lb = smem_u32(&bar[b]);
      uint32_t ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(threadIdx.x));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(threadIdx.x));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                   "d"(v), "r"(rb) : "memory");
    }
    // wait for csz doubles to land in my inbox[b]
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar[b])), "r"(phase) : "memory");
    if (threadIdx.x < csz) acc += inbox[b][threadIdx.x];
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2] = (t1 - t0) / ITER;
  cl.sync();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_grid_barrier(unsigned long long* out, unsigned int* counter) {
  unsigned int target = 0;
  const int G = gridDim.x;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) {
    target += G;
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
      unsigned int v;
      do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      } while (v < target);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[3] = (t1 - t0) / ITER;
}

// LL-style exchange (NCCL's "LL" idea): every CTA writes W doubles as 16-byte lines
// {lo32, tag, hi32, tag} (each 8-byte half single-copy atomic), every CTA polls all G*W
// lines until both tags of each equal the round: no fences, no separate flag or atomic.
__global__ void k_ll_exchange(unsigned long long* out, uint4* lines, int W, double* sink) {
  const int G = gridDim.x;
  double acc = 0.0;
  const unsigned long long t0 = clock64();
  for (int i = 1; i <= ITER; ++i) {
    uint4* buf = lines + static_cast<long long>(i & 1) * G * W;
    if (threadIdx.x < W) {
      const double v = i * 1e-3 + blockIdx.x + threadIdx.x;
      const unsigned long long b = __double_as_longlong(v);
      uint4* dst = buf + blockIdx.x * W + threadIdx.x;
      asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"((unsigned)(b & 0xffffffffu)),
                   "r"((unsigned)i), "r"((unsigned)(b >> 32)), "r"((unsigned)i) : "memory");
    }
    if (threadIdx.x < W) {
      for (int c = 0; c < G; ++c) {
        const uint4* src = buf + c * W + threadIdx.x;
        unsigned a0, f0, a1, f1;
        do {
          asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(f0), "=r"(a1), "=r"(f1)
                       : "l"(src) : "memory");
        } while (f0 != (unsigned)i || f1 != (unsigned)i);
        acc += __longlong_as_double((static_cast<long long>(a1) << 32) | a0);
      }
    }
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[4] = (t1 - t0) / ITER;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
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
  unsigned long long* out;
  double* sink;
  unsigned int* ctr;
  cudaMalloc(&out, 8 * sizeof(unsigned long long));
  cudaMalloc(&sink, 148 * 256 * sizeof(double));
  cudaMalloc(&ctr, sizeof(unsigned int));
  for (int csz : {8, 16}) {
    unsigned long long h[8] = {0};
    cudaMemset(out, 0, 64);
    launch_cluster(k_cluster_sync, csz, csz, out);
    launch_cluster(k_dsmem_pull, csz, csz, out, sink);
    launch_cluster(k_dsmem_push, csz, csz, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("cluster %2d: cluster.sync %llu cycles, sync+DSMEM pull %llu, st.async push + mbarrier %llu  (%s)\n", csz,
           h[0], h[1], h[2], cudaGetErrorString(e));
  }
  for (int G : {8, 16, 40, 64, 148}) {
    unsigned long long h[8] = {0};
    cudaMemset(ctr, 0, 4);
    k_grid_barrier<<<G, 256>>>(out, ctr);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
    printf("grid barrier over %3d CTAs: %llu cycles (%s)\n", G, h[3], cudaGetErrorString(e));
  }
  uint4* lines;
  cudaMalloc(&lines, 2 * 148 * 80 * sizeof(uint4));
  for (int G : {2, 5, 8, 16}) {
    for (int W : {72, 40}) {
      unsigned long long h[8] = {0};
      cudaMemset(lines, 0xff, 2 * 148 * 80 * sizeof(uint4));
      k_ll_exchange<<<G, 256>>>(out, lines, W, sink);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
      printf("LL exchange, %2d CTAs x %d doubles: %llu cycles (%s)\n", G, W, h[4], cudaGetErrorString(e));
    }
  }
  return 0;
}
