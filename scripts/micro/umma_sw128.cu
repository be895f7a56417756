// Layout probe for the kmeans tcgen05 pipeline (k_kmeans.cu kmeans_t5):
//  (1) distance GEMM  D[p][c] = sum_l F[l][p] C[c][l]  (M = 128 points, N = 16,
//      K = 32 features): A = the feature tile as loaded by a 2D TMA box
//      {32 points, 32 features} with SWIZZLE_128B = MN-major SW128 operand;
//      B = centroids K-major SWIZZLE_NONE (the round-1 layout).
//  (2) sums GEMM  S[l][c] = sum_p F[l][p] onehot[p][c]  (M = 128 rows of which
//      the 32 feature rows count, N = 16, K = 128 points): A = the same tile
//      read as K-major SW128 (rows = features), B = one-hot K-major SW128
//      written by threads.
// Several descriptor variants per GEMM; prints which ones match the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_sw128 umma_sw128.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// variant: [0] A lbo, [1] A sbo, [2] A layout, [3] sums-A lbo, [4] sums-A sbo, [5] sums-B sbo, [6] sums k-step bytes
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap tmap, const float* cent,
                                             const int* best, float* dout, float* sout, const int* var, const float* F, float* d2out,
                                             float* s2out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  // 1 KB-aligned: tile 16 KB (4 point blocks x 32 features x 128 B), one-hot 8 KB, B 2 KB
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  float* tile = (float*)base;
  float* oh = (float*)(base + 16384);
  float* Bc = (float*)(base + 16384 + 8192);
  float* t2 = (float*)(base + 32768);  // F again, K-major SW128: row p = point, 128 B = 32 features
  __shared__ __align__(8) uint64_t bar, mb;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // centroids K-major SWIZZLE_NONE: (c, l) at (c%8)*16 + (c/8)*128 + (l/4)*256 + (l%4)*4
  for (int i = tid; i < 16 * 32; i += 128) {
    const int c = i / 32, l = i % 32;
    Bc[((c & 7) * 16 + (c >> 3) * 128 + (l >> 2) * 256) / 4 + (l & 3)] = cent[i];
  }
  // one-hot K-major SW128: row c (cluster), 32 points of block b per 128 B row;
  // 16 B chunk index XOR (row % 8)
  const int vs = var[6];
  for (int i = tid; i < 16 * 128; i += 128) {
    const int c = i / 128, p = i % 128, b = p / 32, q = p % 32;
    const int off = b * 2048 + (c >> 3) * 1024 + (c & 7) * 128 + (((q >> 2) ^ (c & 7)) << 4) + (q & 3) * 4;
    oh[off / 4] = best[p] == c ? 1.f : 0.f;
  }
  {
    const int p = tid;  // thread p writes its point's row with 16 B stores
    for (int j = 0; j < 8; j++) {
      float4 v = make_float4(F[(4 * j + 0) * 256 + p], F[(4 * j + 1) * 256 + p], F[(4 * j + 2) * 256 + p],
                             F[(4 * j + 3) * 256 + p]);
      *reinterpret_cast<float4*>(t2 + ((p >> 3) * 1024 + (p & 7) * 128 + ((j ^ (p & 7)) << 4)) / 4) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16384) : "memory");
    for (int b = 0; b < 4; b++)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(base + b * 4096)),
          "l"(&tmap), "r"(b * 32), "r"(0), "r"(su32(&bar))
          : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&bar))
                   : "memory");
  }
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t sA = su32(tile), sB = su32(Bc);
    for (int kt = 0; kt < 4; kt++) {  // distance: K = 8 features per MMA
      const uint64_t a = desc(sA + kt * 1024, var[0], var[1], var[2]);
      const uint64_t b = desc(sB + kt * 512, 256, 128, 0);
      mma(tb, a, b, idesc(128, 16, true, false), kt > 0);
    }
    const uint32_t sO = su32(oh);
    for (int b = 0; b < 4; b++)      // sums: K = 128 points in 4 blocks of 32
      for (int kk = 0; kk < 4; kk++) {  // K = 8 points per MMA
        const uint64_t a = desc(sA + b * 4096 + kk * vs, var[3], var[4], 2);
        const uint64_t bb = desc(sO + b * 2048 + kk * vs, 16, var[5], 2);
        mma(tb + 32, a, bb, idesc(128, 16, false, false), b > 0 || kk > 0);
      }
    const uint32_t sT2 = su32(t2);
    for (int kt = 0; kt < 4; kt++) {  // distance from the K-major tile
      const uint64_t a = desc(sT2 + kt * 32, 16, 1024, 2);
      const uint64_t b = desc(sB + kt * 512, 256, 128, 0);
      mma(tb + 64, a, b, idesc(128, 16, false, false), kt > 0);
    }
    for (int b = 0; b < 4; b++)        // sums from the K-major tile read MN-major (M = features)
      for (int kk = 0; kk < 4; kk++) {  // K = 8 points = 8 rows of 128 B
        const uint64_t a = desc(sT2 + b * 4096 + kk * 1024, var[7], var[8], 2);
        const uint64_t bb = desc(sO + b * 2048 + kk * vs, 16, var[5], 2);
        mma(tb + 96, a, bb, idesc(128, 16, true, false), b > 0 || kk > 0);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mb))
                 : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&mb))
                   : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  ld16(tb + ((uint32_t)(32 * warp) << 16), v);
  for (int c = 0; c < 16; c++) dout[tid * 16 + c] = v[c];
  ld16(tb + 32 + ((uint32_t)(32 * warp) << 16), v);
  for (int c = 0; c < 16; c++) sout[tid * 16 + c] = v[c];
  ld16(tb + 64 + ((uint32_t)(32 * warp) << 16), v);
  for (int c = 0; c < 16; c++) d2out[tid * 16 + c] = v[c];
  ld16(tb + 96 + ((uint32_t)(32 * warp) << 16), v);
  for (int c = 0; c < 16; c++) s2out[tid * 16 + c] = v[c];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

static float tf32t(float x) {  // the tensor core's truncation to TF32
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xffffe000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int npts = 256, nf = 32;
  std::vector<float> F(nf * npts), C(16 * nf);
  std::vector<int> best(128);
  srand(7);
  for (auto& x : F) x = tf32t((float)(rand() % 2000) / 1000.f - 1.f);
  for (auto& x : C) x = tf32t((float)(rand() % 2000) / 1000.f - 1.f);
  for (auto& b : best) b = rand() % 16;
  float *dF, *dC, *dD, *dS, *dD2, *dS2;
  int *dB, *dV;
  cudaMalloc(&dF, F.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMalloc(&dB, 128 * 4);
  cudaMalloc(&dD, 128 * 16 * 4);
  cudaMalloc(&dS, 128 * 16 * 4);
  cudaMalloc(&dV, 16 * 4);
  cudaMalloc(&dD2, 128 * 16 * 4);
  cudaMalloc(&dS2, 128 * 16 * 4);
  cudaMemcpy(dF, F.data(), F.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, best.data(), 128 * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)npts, (cuuint64_t)nf};
  cuuint64_t strides[1] = {(cuuint64_t)npts * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dF, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  // CPU references
  std::vector<double> Dw(128 * 16), Sw(32 * 16, 0.0);
  for (int p = 0; p < 128; p++)
    for (int c = 0; c < 16; c++) {
      double s = 0;
      for (int l = 0; l < nf; l++) s += (double)F[l * npts + p] * C[c * nf + l];
      Dw[p * 16 + c] = s;
    }
  for (int l = 0; l < 32; l++)
    for (int p = 0; p < 128; p++) Sw[l * 16 + best[p]] += F[l * npts + p];
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  int variants[][9] = {
      {4096, 1024, 2, 16, 1024, 1024, 32, 4096, 1024}, {1024, 4096, 2, 16, 1024, 1024, 32, 1024, 4096},
      {4096, 1024, 1, 0, 1024, 1024, 32, 4096, 128}, {1024, 4096, 1, 4096, 1024, 1024, 32, 128, 4096},
  };
  std::vector<float> D(128 * 16), S(128 * 16), D2(128 * 16), S2(128 * 16);
  for (auto& v : variants) {
    cudaMemcpy(dV, v, sizeof(v), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 128 * 16 * 4);
    probe<<<1, 128, 60 * 1024>>>(tm, dC, dB, dD, dS, dV, dF, dD2, dS2);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d %d %d: %s\n", v[0], v[1], v[2], cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(D2.data(), dD2, D2.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(S2.data(), dS2, S2.size() * 4, cudaMemcpyDeviceToHost);
    double ed = 0, es2 = 0, ed2 = 0, ess2 = 0;
    for (int i = 0; i < 128 * 16; i++) ed = fmax(ed, fabs(D[i] - Dw[i]));
    for (int i = 0; i < 32 * 16; i++) es2 = fmax(es2, fabs(S[i] - Sw[i]));
    for (int i = 0; i < 128 * 16; i++) ed2 = fmax(ed2, fabs(D2[i] - Dw[i]));
    for (int i = 0; i < 32 * 16; i++) ess2 = fmax(ess2, fabs(S2[i] - Sw[i]));
    printf("  K-major tile: dist max err %.3g | sums (MN view lbo=%d sbo=%d) max err %.3g\n", ed2, v[7], v[8], ess2);
    printf("dist A(lbo=%d sbo=%d layout=%d): max err %.3g | sums A(lbo=%d sbo=%d) B(sbo=%d) kstep %d: max err %.3g\n",
           v[0], v[1], v[2], ed, v[3], v[4], v[5], v[6], es2);
    if (ed > 1e-3) {
      printf("  D[0..3][0..3] got %g %g %g %g / want %g %g %g %g; D[33][0] %g / %g\n", D[0], D[1], D[16], D[17], Dw[0],
             Dw[1], Dw[16], Dw[17], D[33 * 16], Dw[33 * 16]);
    }
  }
  return 0;
}
