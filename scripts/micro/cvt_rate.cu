// Throughput of f32 -> f64 conversion: F2F vs integer bit manipulation,
// and f64 add for reference.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double f2d_int(float f) {
  const unsigned b = __float_as_uint(f);
  // normal numbers only (the probe data is normal)
  const unsigned hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
  const unsigned lo = b << 29;
  return __hiloint2double((int)hi, (int)lo);
}
template <int MODE>
__global__ void k(const float* in, double* out, int iters) {
  float x[8];
  for (int j = 0; j < 8; j++) x[j] = in[(threadIdx.x + j) & 255];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      double d;
      if (MODE == 0) d = (double)x[j];
      else if (MODE == 1) d = f2d_int(x[j]);
      else d = (double)j;
      acc[j] = MODE == 2 ? __dadd_rn(acc[j], 1.000001) : __dadd_rn(acc[j], d);
      x[j] = __int_as_float(__float_as_int(x[j]) ^ 1);
    }
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* in; double* out;
  cudaMalloc(&in, 1024); cudaMalloc(&out, 148 * 8 * 256 * 8);
  float h[256]; for (int i = 0; i < 256; i++) h[i] = 1.0f + i * 0.37f;
  cudaMemcpy(in, h, 1024, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2048;
  for (int m = 0; m < 3; m++) for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    if (m == 0) k<0><<<148 * 8, 256>>>(in, out, iters);
    else if (m == 1) k<1><<<148 * 8, 256>>>(in, out, iters);
    else k<2><<<148 * 8, 256>>>(in, out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double n = 148.0 * 8 * 256 * iters * 8;
    if (rep) printf("%s: %.3f ms, %.1f G elem/s (per SM per clk %.1f)\n", m == 0 ? "F2F.F64.F32 + DADD" : m == 1 ? "int bits + DADD" : "DADD only",
                    ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
