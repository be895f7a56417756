// Layout probe for the bf16 tcgen05 kmeans (k_kmeans.cu kmeans_tg):
//  (1) distance GEMM  D[p][c'] (M = 128 points, K = 32 features):
//      A = feature planes written by threads, MN-major SWIZZLE_128B
//      (atom = 8 feature rows x 64 points x bf16; plane P, feature group fg,
//      point half ph at P*4096... see plane_off), B = centroid rows (Ch | Cl)
//      K-major SW128; MMA 1: A = Fh, B = rows 0..31 (N = 32) -> cols 0..31;
//      MMA 2: A = Fl, B = rows 0..15 (N = 16) -> cols 16..31 (accumulate).
//  (2) sums GEMM  S[r][c] (M = 64 rows = Fh features, Fl features; K = 128
//      points; N = 16): A = the same planes read K-major, B = one-hot
//      [cluster][point] K-major SW128.  M = 64 accumulator rows live in lanes
//      (r % 16) + 32 (r / 16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_bf16 umma_bf16.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {  // SWIZZLE_128B
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d),
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
// byte offset of (row r, element q) inside a SW128 atom of 8 rows x 64 bf16
__host__ __device__ constexpr uint32_t sw128(int r, int q) {
  return (uint32_t)(r * 128 + ((((q >> 3) ^ r) & 7) << 4) + (q & 7) * 2);
}
// feature planes: plane P (0 = hi, 1 = lo), feature l, point p of the tile
__host__ __device__ constexpr uint32_t plane_off(int P, int l, int p) {
  return (uint32_t)((p >> 6) * 8192 + (P * 4 + (l >> 3)) * 1024) + sw128(l & 7, p & 63);
}
__host__ __device__ constexpr uint32_t cent_off(int R, int l) {  // row R (0..15 hi, 16..31 lo)
  return (uint32_t)((R >> 3) * 1024) + sw128(R & 7, l);
}
__host__ __device__ constexpr uint32_t onehot_off(int c, int p) {
  return (uint32_t)((p >> 6) * 2048 + (c >> 3) * 1024) + sw128(c & 7, p & 63);
}

__global__ void __launch_bounds__(128) probe(const float* F, const float* C, const int* best, float* dout, float* sout) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  unsigned char* planes = base;              // 16 KB
  unsigned char* cb = base + 16384;          // 4 KB
  unsigned char* oh = base + 16384 + 4096;   // 4 KB
  __shared__ __align__(8) uint64_t mb;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < 8192; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0;  // 32 KB
  __syncthreads();
  {
    const int p = tid;
    for (int l = 0; l < 32; l++) {
      const float x = F[l * 128 + p];
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(h));
      *reinterpret_cast<__nv_bfloat16*>(planes + plane_off(0, l, p)) = h;
      *reinterpret_cast<__nv_bfloat16*>(planes + plane_off(1, l, p)) = lo;
    }
    for (int c = 0; c < 16; c++)
      *reinterpret_cast<__nv_bfloat16*>(oh + onehot_off(c, p)) = __float2bfloat16_rn(best[p] == c ? 1.f : 0.f);
  }
  for (int i = tid; i < 16 * 32; i += 128) {
    const int c = i / 32, l = i % 32;
    const float x = C[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(h));
    *reinterpret_cast<__nv_bfloat16*>(cb + cent_off(c, l)) = h;
    *reinterpret_cast<__nv_bfloat16*>(cb + cent_off(16 + c, l)) = lo;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (tid == 0) {
    const uint32_t sP = su32(planes), sC = su32(cb), sO = su32(oh);
    for (int kk = 0; kk < 2; kk++)  // hi planes x (Ch | Cl): K = 16 features per MMA
      mma(tb, desc(sP + kk * 2048, 8192, 1024), desc(sC + kk * 32, 16, 1024), idesc(128, 32, true, false), kk > 0);
    for (int kk = 0; kk < 2; kk++)  // lo planes x Ch -> cols 16..31
      mma(tb + 16, desc(sP + 4096 + kk * 2048, 8192, 1024), desc(sC + kk * 32, 16, 1024), idesc(128, 16, true, false), 1);
    for (int ph = 0; ph < 2; ph++)
      for (int kk = 0; kk < 4; kk++)  // K = 16 points per MMA
        mma(tb + 64, desc(sP + ph * 8192 + kk * 32, 16, 1024), desc(sO + ph * 2048 + kk * 32, 16, 1024),
            idesc(64, 16, false, false), ph > 0 || kk > 0);
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
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  ld16(tb + lane_base, v);
  for (int c = 0; c < 16; c++) dout[tid * 32 + c] = v[c];
  ld16(tb + 16 + lane_base, v);
  for (int c = 0; c < 16; c++) dout[tid * 32 + 16 + c] = v[c];
  ld16(tb + 64 + lane_base, v);
  for (int c = 0; c < 16; c++) sout[tid * 16 + c] = v[c];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

static float bf(float x) {  // RN to bf16
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x7fff + ((u >> 16) & 1)) & 0xffff0000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  std::vector<float> F(32 * 128), C(16 * 32);
  std::vector<int> best(128);
  srand(7);
  for (auto& x : F) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto& x : C) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto& b : best) b = rand() % 16;
  float *dF, *dC, *dD, *dS;
  int* dB;
  cudaMalloc(&dF, F.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMalloc(&dB, 128 * 4);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMalloc(&dS, 128 * 16 * 4);
  cudaMemcpy(dF, F.data(), F.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, best.data(), 128 * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  probe<<<1, 128, 40 * 1024>>>(dF, dC, dB, dD, dS);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("probe: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> D(128 * 32), S(128 * 16);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
  double ehh = 0, ecr = 0, etot = 0;
  for (int p = 0; p < 128; p++)
    for (int c = 0; c < 16; c++) {
      double hh = 0, cr = 0, ex = 0;
      for (int l = 0; l < 32; l++) {
        const float x = F[l * 128 + p], y = C[c * 32 + l];
        const float xh = bf(x), xl = bf(x - xh), yh = bf(y), yl = bf(y - yh);
        hh += (double)xh * yh;
        cr += (double)xh * yl + (double)xl * yh;
        ex += (double)x * y;
      }
      ehh = fmax(ehh, fabs(D[p * 32 + c] - hh));
      ecr = fmax(ecr, fabs(D[p * 32 + 16 + c] - cr));
      etot = fmax(etot, fabs(D[p * 32 + c] + D[p * 32 + 16 + c] - ex));
    }
  printf("distance: |hh - ref| %.3g  |cross - ref| %.3g  |hh + cross - exact| %.3g\n", ehh, ecr, etot);
  double es = 0;
  int bad = 0;
  for (int r = 0; r < 64; r++) {
    const int lane = (r % 16) + 32 * (r / 16), P = r / 32, l = r % 32;
    for (int c = 0; c < 16; c++) {
      double want = 0;
      for (int p = 0; p < 128; p++)
        if (best[p] == c) {
          const float x = F[l * 128 + p], xh = bf(x);
          want += P == 0 ? xh : bf(x - xh);
        }
      const double err = fabs(S[lane * 16 + c] - want);
      es = fmax(es, err);
      bad += err > 1e-4;
    }
  }
  printf("sums (M=64 rows at lanes r%%16 + 32(r/16)): max err %.3g, %d bad\n", es, bad);
  printf("%s\n", ehh < 1e-4 && ecr < 1e-5 && etot < 1e-4 && bad == 0 ? "PROBE OK" : "PROBE FAILED");
  return 0;
}
