// Microbenchmark: legacy mma.sync throughput on sm_100a (tf32 m16n8k8, bf16 m16n8k16).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float d[8][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; j++) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float d[8][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; j++) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 4096;
  for (int w = 4; w <= 16; w *= 2) {
    for (int kind = 0; kind < 2; kind++) {
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        if (kind == 0) tf32_loop<<<148 * 2, w * 32>>>(out, iters);
        else bf16_loop<<<148 * 2, w * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 148.0 * 2 * w * iters * 8 * (kind == 0 ? 16 * 8 * 8 : 16 * 8 * 16) * 2.0;
        if (rep) printf("%s warps/CTA %d (2 CTA/SM): %.3f ms, %.1f TFLOP/s, %.2f mma/clk/SM\n", kind ? "bf16 m16n8k16" : "tf32 m16n8k8", w, ms,
               flops / ms / 1e9, (148.0 * 2 * w * iters * 8) / (ms * 1e-3 * 1.92e9) / 148);
      }
    }
  }
  return 0;
}
