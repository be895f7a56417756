// Issue rates on one B200 SM of the f64 operations the hotspot cell uses:
// F2F.F64.F32 (f32 -> f64), F2F.F32.F64 (f64 -> f32, RN), DADD, DMUL, and
// the integer-pipe f32 -> f64 widening (normal inputs).  8 independent
// chains per thread, 8 warps x 8 CTAs per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double f2d_int(float f) {
  const unsigned b = __float_as_uint(f);
  const unsigned hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
  return __hiloint2double((int)hi, (int)(b << 29));
}
template <int MODE>
__global__ void k(const float* in, double* out, int iters) {
  float x[8];
  double acc[8];
  for (int j = 0; j < 8; j++) {
    x[j] = in[(threadIdx.x + j) & 255];
    acc[j] = x[j];
  }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (MODE == 0) {  // F2F up
        acc[j] = (double)x[j];
        x[j] = __int_as_float(__float_as_int(x[j]) ^ (int)__double2hiint(acc[j]) & 1);
      } else if (MODE == 1) {  // int widening
        acc[j] = f2d_int(x[j]);
        x[j] = __int_as_float(__float_as_int(x[j]) ^ (int)__double2hiint(acc[j]) & 1);
      } else if (MODE == 2) {  // F2F down
        x[j] = __double2float_rn(acc[j]);
        acc[j] = __hiloint2double(__float_as_int(x[j]) | 0x3ff00000, i);
      } else if (MODE == 3) {
        acc[j] = __dadd_rn(acc[j], 1.000001);
      } else if (MODE == 4) {
        acc[j] = __dmul_rn(acc[j], 1.000001);
      } else {
        acc[j] = fma(acc[j], 1.000001, 1e-9);
      }
    }
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += acc[j] + x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* in;
  double* out;
  cudaMalloc(&in, 1024);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  float h[256];
  for (int i = 0; i < 256; i++) h[i] = 1.0f + i * 0.37f;
  cudaMemcpy(in, h, 1024, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  const char* names[] = {"F2F.F64.F32 (+xor)", "int widen (+xor)", "F2F.F32.F64 (+int)", "DADD", "DMUL", "DFMA"};
  for (int m = 0; m < 6; m++)
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      switch (m) {
        case 0: k<0><<<148 * 8, 256>>>(in, out, iters); break;
        case 1: k<1><<<148 * 8, 256>>>(in, out, iters); break;
        case 2: k<2><<<148 * 8, 256>>>(in, out, iters); break;
        case 3: k<3><<<148 * 8, 256>>>(in, out, iters); break;
        case 4: k<4><<<148 * 8, 256>>>(in, out, iters); break;
        default: k<5><<<148 * 8, 256>>>(in, out, iters); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double n = 148.0 * 8 * 256 * iters * 8;
      if (rep) printf("%-20s %.3f ms  per SM per clk %.2f\n", names[m], ms, n / (ms * 1e-3) / 148 / 1.965e9);
    }
  return 0;
}
