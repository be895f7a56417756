// Host cost of one launch: a raw <<<>>> of an empty kernel, a raw launch of a
// vecadd-shaped kernel, and bf_launch (the C ABI) of vecadd PR1 (2^20, grid
// 4096 x 256), each timed over 20k back-to-back calls with the wall clock.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o launch_cost launch_cost.cu \
//        -I../../include -L../../paper_2206_07896_b200 -lbfgpu -Xlinker -rpath=...
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "bfgpu.h"

__global__ void empty_kernel() {}
__global__ void add_kernel(const float* a, const float* b, float* c, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) c[i] = a[i] + b[i];
}

template <class F>
double time_us(F f, int n = 20000) {
  for (int i = 0; i < 200; i++) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; i++) f();
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int n = 1 << 20;
  float *a, *b, *c;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4);
  printf("raw empty<<<1,32>>>            %7.3f us\n", time_us([&] { empty_kernel<<<1, 32, 0, s>>>(); }));
  printf("raw add<<<4096,256>>>          %7.3f us\n", time_us([&] { add_kernel<<<4096, 256, 0, s>>>(a, b, c, n); }));
  printf("raw add + cudaGetLastError     %7.3f us\n", time_us([&] { add_kernel<<<4096, 256, 0, s>>>(a, b, c, n); cudaGetLastError(); }));
  bf_arena* ar; bf_arena_create(0, &ar);
  uint32_t h[3];
  for (int i = 0; i < 3; i++) bf_alloc(ar, BF_F32, n, &h[i]);
  bf_runtime* rt; bf_runtime_create(ar, 1, 0, 0.0, 0, &rt);
  bf_slot sl[4] = {};
  for (int i = 0; i < 3; i++) { sl[i].kind = BF_SLOT_HANDLE; sl[i].v.handle = h[i]; }
  sl[3].kind = BF_SLOT_I32; sl[3].v.i32 = n;
  int32_t g[3] = {4096, 1, 1}, bl[3] = {256, 1, 1};
  uint64_t tid;
  printf("bf_launch vecadd PR1           %7.3f us\n", time_us([&] { bf_launch(rt, "vecadd", g, bl, 0, sl, 4, 0, 4096, &tid); }));
  bf_fault f;
  bf_synchronize(rt, &f);
  printf("bf_synchronize (idle)          %7.3f us\n", time_us([&] { bf_synchronize(rt, &f); }, 5000));
  printf("bf_launch + bf_synchronize     %7.3f us\n", time_us([&] { bf_launch(rt, "vecadd", g, bl, 0, sl, 4, 0, 4096, &tid); bf_synchronize(rt, &f); }, 5000));
  printf("raw add + cudaStreamSynchronize %6.3f us\n", time_us([&] { add_kernel<<<4096, 256, 0, s>>>(a, b, c, n); cudaStreamSynchronize(s); }, 5000));
  bf_shutdown(rt);
  return 0;
}
