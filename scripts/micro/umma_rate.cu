// tcgen05.mma kind::f16 (bf16) issue/execution rate on sm_100a for the small
// N shapes of the kmeans pipeline: one thread per CTA (one CTA per SM) issues
// R back-to-back MMAs of shape M x N x 16 from shared-memory operands into
// TMEM; prints SM cycles per MMA.  A MN-major or K-major (SWIZZLE_128B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128) rate(int M, int N, int amn, int R, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (su32(sm) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t mb;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    const uint32_t sA = su32(base), sB = su32(base + 32768);
    const uint32_t id = idesc(M, N, amn != 0);
    const uint64_t a = amn ? desc(sA, 8192, 1024) : desc(sA, 16, 1024);
    const uint64_t b = desc(sB, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < R; r++)
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tb),
                   "l"(a), "l"(b), "r"(id), "r"(1)
                   : "memory");
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mb))
                 : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&mb))
                   : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      cyc[0] = t1 - t0;
      cyc[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 16);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int R = 4096;
  for (int amn = 0; amn < 2; amn++)
    for (int M : {64, 128})
      for (int N : {16, 32, 64, 128, 256}) {
        if (amn && M == 64) continue;
        rate<<<148, 128, 70 * 1024>>>(M, N, amn, 64, cyc);
        rate<<<148, 128, 70 * 1024>>>(M, N, amn, R, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
        printf("M=%3d N=%3d K=16 A %s: issue %.1f, complete %.1f SM cycles per MMA (%s)\n", M, N, amn ? "MN" : "K ",
               (double)h[0] / R, (double)h[1] / R, cudaGetErrorString(e));
      }
  return 0;
}
