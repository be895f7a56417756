// Layout probe for tcgen05.mma kind::tf32 with SWIZZLE_NONE operands:
// one MMA, D dumped from all 128 TMEM lanes x 16 columns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// mode 0: M=64, A MN-major, B MN-major (the kmeans sums GEMM)
// mode 1: M=128, A K-major, B K-major (the distance GEMM)
// mode 2: M=64, A MN-major, B K-major
// mode 3: M=128, A MN-major, B MN-major
__global__ void probe(float* out, int mode, int swap) {
  __shared__ __align__(128) float A[64 * 64];   // up to 128 x 8 (or 64 x 8) elements, padded
  __shared__ __align__(128) float B[16 * 8 * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  const int M = (mode == 0 || mode == 2) ? 64 : 128;
  const bool amn = (mode == 0 || mode == 2 || mode == 3 || mode == 5), bmn = (mode == 0 || mode == 3 || mode == 4);
  for (int i = tid; i < 64 * 64; i += blockDim.x) A[i] = 0.f;
  for (int i = tid; i < 16 * 8 * 4; i += blockDim.x) B[i] = 0.f;
  __syncthreads();
  // A[m][k] = m + 1000 k (k < 8); B[k][n] = (k == n % 8) ? (1 + n / 8) : 0  => D[m][n] = (1 + n/8) * A[m][n%8]
  for (int i = tid; i < M * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    float v = (float)m + 128.f * k;
    int off;  // bytes
    if (amn) off = (m % 4) * 4 + (m / 4) * 128 + (k % 8) * 16;          // MN-major: SBO=128 (group of 4 m), k rows 16 B
    else off = (m % 8) * 16 + (m / 8) * 128 + (k / 4) * 2048 + (k % 4) * 4;  // K-major: SBO=128, LBO=2048
    A[off / 4] = v;
  }
  for (int i = tid; i < 8 * 16; i += blockDim.x) {
    int k = i / 16, n = i % 16;
    float v = (k == n % 8) ? (float)(1 + n / 8) : 0.f;
    int off;
    if (bmn) off = (n % 4) * 4 + (n / 4) * 128 + (k % 8) * 16;          // MN-major: SBO=128, k rows 16 B
    else off = (n % 8) * 16 + (n / 8) * 128 + (k / 4) * 256 + (k % 4) * 4;  // K-major: SBO=128, LBO=256
    B[off / 4] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tb = slot;
  if (tid == 0) {
    // swap: for MN-major operands put the MN-group stride into LBO
    uint64_t da = amn ? (swap ? desc(su32(A), 128, 2048) : desc(su32(A), 2048, 128)) : desc(su32(A), 2048, 128);
    uint64_t db = bmn ? (swap ? desc(su32(B), 128, 256) : desc(su32(B), 256, 128)) : desc(su32(B), 256, 128);
    uint32_t id = idesc(M, 16, amn, bmn);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                 :: "r"(tb), "l"(da), "l"(db), "r"(id), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
  }
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(su32(&bar)), "r"(0u) : "memory");
  } while (!done);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  const int warp = tid / 32;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tb + ((uint32_t)(32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int c = 0; c < 16; c++) out[tid * 16 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tb));
}
int main() {
  float* d; cudaMalloc(&d, 128 * 16 * 4);
  static float h[128 * 16];
  FILE* fo = fopen("gpurun_out/umma_probe.txt", "w");
  for (int mode = 0; mode < 6; mode++) {
    cudaMemset(d, 0, 128 * 16 * 4);
    probe<<<1, 128>>>(d, mode, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(fo, "mode %d err %s\n", mode, cudaGetErrorString(e));
    for (int lane = 0; lane < 128; lane++) {
      fprintf(fo, "%d", lane);
      for (int c = 0; c < 16; c++) fprintf(fo, " %.0f", h[lane * 16 + c]);
      fprintf(fo, "\n");
    }
  }
  fclose(fo);
  return 0;
}
