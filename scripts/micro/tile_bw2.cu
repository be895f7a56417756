// DRAM bandwidth of the kmeans tile pattern through TMA tensor copies: a
// feature-major array f[l * npts + p] (32 rows) read in tiles of P points x 32
// rows by ONE cp.async.bulk.tensor per tile (3D map {256, P/256, 32} for
// P > 256 so every feature row of a tile is one contiguous 4P-byte run), one
// CTA per SM, S-stage ring.  Prints TB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tile_bw2 tile_bw2.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, long long npts, int P, int S,
                                                float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  unsigned char* ring = sm + ((1024u - (su32(sm) & 1023u)) & 1023u) + 1024;
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
  if (tid == 0) {
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
      if (P <= 256)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(ring + (size_t)s * tb)),
            "l"(&tm), "r"((int)(i * P)), "r"(0), "r"(su32(&full[s]))
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                su32(ring + (size_t)s * tb)),
            "l"(&tm), "r"(0), "r"((int)(i * P / 256)), "r"(0), "r"(su32(&full[s]))
            : "memory");
    }
  } else if (tid == 32) {
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
      acc += reinterpret_cast<float*>(ring + (size_t)s * tb)[0];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    sink[blockIdx.x] = acc;
  }
}

__global__ void fill(float* f, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    f[i] = (float)(x >> 8) * (1.0f / 16777216.0f);
  }
}

int main() {
  const long long npts = 1 << 24;
  float *f, *sink;
  cudaMalloc(&f, npts * 32 * 4);
  fill<<<148 * 8, 256>>>(f, npts * 32);  // non-zero data (a zero-filled buffer reads faster than the copy peak)
  cudaMalloc(&sink, 4096 * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int P : {128, 256, 512, 1024})
    for (int S : {2, 3, 4, 6, 8, 12}) {
      const size_t smem = 2048 + (size_t)S * 32 * P * 4;
      if (smem > 225 * 1024) continue;
      CUtensorMap tm;
      CUresult r;
      if (P <= 256) {
        cuuint64_t dims[2] = {(cuuint64_t)npts, 32};
        cuuint64_t strides[1] = {(cuuint64_t)npts * 4};
        cuuint32_t box[2] = {(cuuint32_t)P, 32}, es[2] = {1, 1};
        r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, f, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[3] = {256, (cuuint64_t)npts / 256, 32};
        cuuint64_t strides[2] = {1024, (cuuint64_t)npts * 4};
        cuuint32_t box[3] = {256, (cuuint32_t)P / 256, 32}, es[3] = {1, 1, 1};
        r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, f, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r != CUDA_SUCCESS) {
        printf("P=%d encode failed %d\n", P, (int)r);
        continue;
      }
      stream<<<148, 64, smem>>>(tm, npts, P, S, sink);
      cudaEventRecord(e0);
      for (int k = 0; k < 3; k++) stream<<<148, 64, smem>>>(tm, npts, P, S, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("TMA P=%4d (row %5d B) stages %2d: %.3f ms, %.2f TB/s (%s)\n", P, P * 4, S, ms / 3,
             npts * 128.0 / (ms / 3 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
