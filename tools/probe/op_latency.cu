// Dependent-chain latencies (cycles per op, one warp) of the operations on the panel's
// per-column critical path on B200: DFMA, DADD, double shuffle, sqrt, division, LDS,
// __syncthreads (8 warps), st.async self-push + mbarrier wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 op_latency.cu -o op_latency
#include <cstdio>
#include <cstdint>
constexpr int N = 4096;
__global__ void k(double* out, unsigned long long* cyc, double a, double b) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i + 1) % 1024;
  __syncthreads();
  double x = a + threadIdx.x;
  unsigned long long t0, t1;
  auto rec = [&](int slot) { if (threadIdx.x == 0) cyc[slot] = (t1 - t0); };
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, b, a);
  t1 = clock64(); rec(0);
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64(); rec(1);
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
  t1 = clock64(); rec(2);
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = sqrt(x + 2.0);
  t1 = clock64(); rec(3);
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = a / (x + 3.0);
  t1 = clock64(); rec(4);
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) idx = static_cast<int>(sm[idx & 1023]);
  t1 = clock64(); rec(5);
  x += idx;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) __syncthreads();
  t1 = clock64(); rec(6);
  // x + shuffle + add butterfly stage (what a warp_sum stage costs)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
  t1 = clock64(); rec(7);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
int main() {
  double* out; unsigned long long* cyc;
  cudaMalloc(&out, 256 * 8); cudaMalloc(&cyc, 64);
  k<<<1, 256>>>(out, cyc, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  unsigned long long h[8];
  cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DADD", "double SHFL", "sqrt(x+2)", "a/(x+3)", "LDS (dependent)", "__syncthreads (8 warps)", "SHFL+DADD stage"};
  for (int i = 0; i < 8; ++i) printf("%-26s %7.1f cycles\n", names[i], (double)h[i] / N);
  printf("(8 warps running the same chain: the FP64 numbers include pipe sharing)\n");
  k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 8; ++i) printf("1 warp: %-18s %7.1f cycles\n", names[i], (double)h[i] / N);
  return 0;
}
