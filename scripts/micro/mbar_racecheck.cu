// Does compute-sanitizer racecheck follow a warp's writes through __syncwarp
// and one lane's mbarrier arrive (the kmeans_tg split -> screen pattern)?
// Warp 0 writes shared memory (every lane), __syncwarp, lane 0 arrives
// (count 1); warp 1 waits on the phase and reads.  With every lane arriving
// (count 32) racecheck reports nothing; with this pattern it reports a hazard:
// a limitation of the tool (bar.warp.sync orders the lanes' writes before the
// release), not a race.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int* out) {
  __shared__ int buf[32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    buf[threadIdx.x] = threadIdx.x * 3;
    __syncwarp();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
  } else {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
    out[threadIdx.x - 32] = buf[threadIdx.x - 32];
  }
}
int main() {
  int* d;
  cudaMalloc(&d, 128);
  k<<<1, 64>>>(d);
  int h[32];
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("h[5] = %d (%s)\n", h[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
