// Shared device/host helpers for the B200 PowerURV library (sm_100a, FP64).
//
// Everything here is plumbing: error handling, mbarrier / TMA / DMMA PTX
// wrappers, the deterministic grid barrier used by the cooperative panel
// kernel, and the per-kernel timing registry that bench.py reads.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

namespace urv {

// ---------------------------------------------------------------------------
// Status codes of the C ABI (include/urv_b200.h)
// ---------------------------------------------------------------------------
enum Status : int {
  kOk = 0,
  kInvalid = 1,       // -> ValueError
  kCollapse = 2,      // -> RankCollapseError
  kCudaError = 3,     // -> RuntimeError
  kNcclError = 4,     // -> RuntimeError
  kOutOfMemory = 5,   // -> MemoryError
  kUnsupported = 6,   // -> NotImplementedError (a size beyond what the device path handles)
};

void set_error(const char* fmt, ...);
const char* last_error();

struct CudaFailure {
  int status;
};

#define URV_CUDA(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::urv::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,                \
                       cudaGetErrorString(_e));                                     \
      throw ::urv::CudaFailure{_e == cudaErrorMemoryAllocation ? ::urv::kOutOfMemory \
                                                               : ::urv::kCudaError}; \
    }                                                                               \
  } while (0)

void count_launch();
#define URV_CHECK_LAUNCH()          \
  do {                              \
    ::urv::count_launch();          \
    URV_CUDA(cudaGetLastError());   \
  } while (0)

// ---------------------------------------------------------------------------
// Kernel timing registry (optional; enabled by urv_stats_enable)
// ---------------------------------------------------------------------------
enum KernelClass : int {
  kKGemm = 0,       // dgemm_tma_dmma, 128x128 tiles (long-K products)
  kKPanel = 1,      // panel_geqr2 (cooperative Householder panel)
  kKApplyT = 2,     // split-K reduce + T / T^T multiply
  kKAux = 3,        // norms, copies, identity, R extraction, deficiency count
  kKGemmUpd = 4,    // dgemm_tma_dmma, 128x64 tiles (short-K rank-k updates)
  kKGemmSkinny = 5, // dgemm_tma_dmma, 64x128 tiles (M <= 64)
  kKApplyCl = 6,    // block_apply_cl: fused C -= V op(T) V^T C for narrow blocks (one cluster per strip)
  kKNumClasses = 7,
};

struct StatsScope {
  StatsScope(cudaStream_t s, int cls, double flops, double bytes);
  ~StatsScope();
  cudaStream_t stream;
  int cls;
  double flops, bytes;
  void* ev0;
};

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer release of a ring slot read with LDS: ptxas does not make a (release)
// mbarrier arrive wait for the warp's outstanding shared-memory loads, so the
// producer's next TMA could overwrite the slot before they have read it.  The
// CTA-scope fence forces those loads to complete first.
__device__ __forceinline__ void mbar_arrive_after_reads(uint64_t* bar) {
  asm volatile(
      "fence.acq_rel.cta;\n"
      "mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "URV_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra URV_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2-D TMA tile load global -> shared, completion signalled on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// 2-D TMA tile store shared -> global (bulk group; clipped at the tensor bounds).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
// Waits only until the bulk stores have READ the shared-memory source (the CTA may then
// exit and its shared memory be reused); the global writes complete before the grid does.
__device__ __forceinline__ void tma_store_commit_and_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Generic-proxy shared-memory writes -> visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core (SASS: DMMA.8x8x4).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double ld_shared_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// Grid-wide barrier for cooperative kernels.  `counter` is zeroed before the
// launch; the k-th barrier waits until it reaches k * gridDim.x.  The spin uses
// relaxed loads and a single acquire fence afterwards (an ld.acquire per spin
// iteration would invalidate L1 every time).
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int target) {
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

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// LL ("low-latency") publication of one double between CTAs: two 8-byte words
// {low/high 32 bits of the value, 32-bit generation}, written with one vector
// store.  Each 8-byte word is single-copy atomic, so a reader that sees the
// expected generation in both words has the value -- no flag, no fence.
__device__ __forceinline__ void ll_store(unsigned long long* p, double v, unsigned int gen) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned long long w0 = (static_cast<unsigned long long>(gen) << 32) | (bits & 0xffffffffull);
  const unsigned long long w1 = (static_cast<unsigned long long>(gen) << 32) | (bits >> 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ bool ll_load(const unsigned long long* p, unsigned int gen, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
  v = __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
  return static_cast<unsigned int>(w0 >> 32) == gen && static_cast<unsigned int>(w1 >> 32) == gen;
}

__device__ __forceinline__ void ll_load_raw(const unsigned long long* p, unsigned long long& w0,
                                            unsigned long long& w1) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ bool ll_tag_ok(unsigned long long w0, unsigned long long w1, unsigned int gen) {
  return static_cast<unsigned int>(w0 >> 32) == gen && static_cast<unsigned int>(w1 >> 32) == gen;
}
__device__ __forceinline__ double ll_value(unsigned long long w0, unsigned long long w1) {
  return __longlong_as_double(static_cast<long long>((w1 << 32) | (w0 & 0xffffffffull)));
}

// One double into CTA `rank`'s copy of `local_slot` (distributed shared memory of the
// cluster), completion counted in bytes on that CTA's copy of `local_bar`.
__device__ __forceinline__ void dsmem_push_f64(double* local_slot, uint64_t* local_bar, int rank, double v) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_slot)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}
// `bytes` (a multiple of 16) of this CTA's shared memory at `src` into CTA `rank`'s copy of
// `local_dst`, completion counted on that CTA's copy of `local_bar` (one bulk-copy instruction).
__device__ __forceinline__ void dsmem_push_bulk(double* local_dst, uint64_t* local_bar, int rank, const double* src,
                                                uint32_t bytes) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ra),
               "r"(smem_u32(src)), "r"(bytes), "r"(rb)
               : "memory");
}
// 8-byte asynchronous copy global -> shared (LDGSTS): no register staging, every copy of a
// thread in flight at once; cp_async_wait_all() before the data is read.
__device__ __forceinline__ void cp_async_f64(double* smem_dst, const double* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// Wait for a phase of an mbarrier whose transactions come from other CTAs of the cluster.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "URV_WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra URV_WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Device properties cached per device.
struct DeviceInfo {
  int sms = 0;
  int max_smem_optin = 0;
};
const DeviceInfo& device_info();

// Stream-ordered allocation from the library's own memory pool on the current
// device (one pool per device, created on first use).  The pool keeps at most
// URV_POOL_KEEP_MB (default: a fifth of the device memory) of freed memory cached
// across calls and hands the rest back to the driver at the next synchronisation;
// urv_release_memory() returns all of it (for callers that need the memory back).
cudaMemPool_t lib_pool();
void dev_alloc(void** p, size_t bytes, cudaStream_t st);
// Return every cached (free) byte of this device's pool to the driver.
void trim_pool();

}  // namespace urv
