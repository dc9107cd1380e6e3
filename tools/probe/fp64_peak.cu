// FP64 throughput probe: DMMA (mma.sync m8n8k4 f64) vs DFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters) {
  double acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = i;
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz smem/blk optin=%zu regs/SM=%d L2=%d\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.l2CacheSize);
  double* out; cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    int grid = p.multiProcessorCount * bpsm, iters = 20000;
    dmma_loop<<<grid, 256>>>(out, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); dmma_loop<<<grid, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8 * iters * (grid * 8.0);  // per warp-mma 256 FMA
    printf("DMMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
    dfma_loop<<<grid, 256>>>(out, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); dfma_loop<<<grid, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)grid * 256;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
