// DRAM bandwidth of the kmeans tile pattern: a feature-major array
// f[l * npts + p] (32 rows of npts floats) streamed in tiles of P points x 32
// rows (32 chunks of 4P contiguous bytes, 64 MB apart) by 1D bulk copies into
// a shared-memory ring; consumers only release the slots.  Varies P (chunk
// 512 B .. 4 KB) and the ring depth.  Prints TB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tile_bw tile_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) stream(const float* f, long long npts, int P, int S, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  float* ring = reinterpret_cast<float*>(sm + 256);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; s++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntile = npts / P;
  const uint32_t tb = 32u * P * 4u;
  if (tid == 0) {  // producer
    int n = 0;
    for (long long i = blockIdx.x; i < ntile; i += gridDim.x, n++) {
      const int s = n % S;
      if (n >= S) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done)
                       : "r"(su32(&empty[s])), "r"(((n / S) - 1) & 1)
                       : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(tb) : "memory");
      for (int l = 0; l < 32; l++)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(ring + (size_t)s * 32 * P + l * P)),
            "l"(f + (long long)l * npts + i * P), "r"(P * 4), "r"(su32(&full[s]))
            : "memory");
    }
  } else if (tid == 32) {  // consumer: touch one value, release
    float acc = 0.f;
    int n = 0;
    for (long long i = blockIdx.x; i < ntile; i += gridDim.x, n++) {
      const int s = n % S;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(su32(&full[s])), "r"((n / S) & 1)
                     : "memory");
      acc += ring[(size_t)s * 32 * P];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  const long long npts = 1 << 24;
  float *f, *sink;
  cudaMalloc(&f, npts * 32 * 4);
  cudaMemset(f, 0, npts * 32 * 4);
  cudaMalloc(&sink, 4096 * 4);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int P : {128, 256, 512, 1024})
    for (int S : {2, 4, 8, 12}) {
      const size_t smem = 256 + (size_t)S * 32 * P * 4;
      if (smem > 220 * 1024 || S > 16) continue;
      for (int ctas : {1, 2}) {
        if (smem * ctas > 220 * 1024) continue;
        stream<<<148 * ctas, 64, smem>>>(f, npts, P, S, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; r++) stream<<<148 * ctas, 64, smem>>>(f, npts, P, S, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("P=%4d (chunk %5d B) stages %2d ctas/SM %d: %.3f ms, %.2f TB/s (%s)\n", P, P * 4, S, ctas, ms / 3,
               npts * 128.0 / (ms / 3 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
