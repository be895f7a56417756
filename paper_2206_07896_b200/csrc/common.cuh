// Device-side helpers shared by every sm_100a kernel of the launch runtime.
//
// A launch of the reference runtime hands a worker a contiguous range of
// *logical* blocks [first, first+count) of a (grid, block) geometry
// (runtime.py:175-201, 323-350).  On the GPU that range is executed by a
// physical grid sized for the B200 (148 SMs); the logical geometry is carried
// in KDesc and decoded exactly as the reference does (syntax.py:61-71).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "bf_internal.h"

namespace bf {

// Device fault word; first fault wins (runtime.py:340-341).
struct DevFault {
  int kind;
  int pad;
  long long block;
  unsigned long long task;
  int* host_flag;  // host-mapped pinned word set after a fault: a synchronize
                   // copies the record only when it is set
};

// Logical launch descriptor passed by value to every kernel.
struct KDesc {
  int gx, gy, gz;          // logical gridDim
  int bx, by, bz;          // logical blockDim
  long long first, count;  // logical block range of this fetch
  int* executed;           // per-task run counts (BF_FLAG_INSTRUMENT), nullable
  DevFault* fault;
  unsigned long long task;
};

__device__ __forceinline__ void record_fault(const KDesc& d, int kind, long long block) {
  if (atomicCAS(&d.fault->kind, 0, kind) == 0) {
    d.fault->block = block;
    d.fault->task = d.task;
    __threadfence_system();
    if (d.fault->host_flag) *(volatile int*)d.fault->host_flag = 1;
  }
}

// KernelTask.executed[b] += 1 for every block of the fetch (runtime.py:345).
// Called by every CTA of the kernel that executed the range; the counts are
// only observable after the stream drained, so the placement in the kernel
// does not matter.
__device__ __forceinline__ void mark_executed(const KDesc& d) {
  if (d.executed == nullptr) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = d.first + (long long)blockIdx.x * blockDim.x + threadIdx.x;
       b < d.first + d.count; b += stride)
    atomicAdd(d.executed + b, 1);
}

// ---- device-side block fetching (DevFetch, bf_internal.h) -------------------
// CTA-uniform claim loop:
//   FetchCursor fc = dev_fetch_cursor();
//   long long f = dev_fetch_first(F, fc);
//   while (f < F.nfetch) { const long long nx = dev_fetch_issue(F, fc); ...blocks of f...;
//                          dev_fetch_done(F, b0, b1); f = dev_fetch_take(nx); }
// Thread 0 issues the next claim's atomic before the current fetch's work, so
// its round trip overlaps the work; dev_fetch_take publishes it to the CTA.
// Sub-range j of the fetches is [j*F/S, (j+1)*F/S); thread 0's cursor starts
// on sub-range blockIdx.x % S and moves on when one is drained.
// thread 0's claim state; the CTA's claim and block counts are flushed once,
// at the end (dev_fetch_flush), not per claim: per-claim atomics on one
// statistics word would serialise every CTA of a fine-grained launch
struct FetchCursor {
  int sub, tried;
  unsigned long long claims, blocks;
};
__device__ __forceinline__ FetchCursor dev_fetch_cursor() {
  return FetchCursor{(int)(blockIdx.x % kFetchSubs), 0, 0ull, 0ull};
}
__device__ __forceinline__ long long dev_fetch_sub_start(const DevFetch& F, int j) {
  return (F.nfetch * j) / kFetchSubs;
}
__device__ __forceinline__ long long dev_fetch_claim(const DevFetch& F, FetchCursor& c) {
  while (c.tried < kFetchSubs) {
    const int j = c.sub;
    const long long lo = dev_fetch_sub_start(F, j), n = dev_fetch_sub_start(F, j + 1) - lo;
    const long long f = (long long)atomicAdd(F.cursor + j, 1ull);
    if (f < n) {
      c.claims++;
      return lo + f;
    }
    c.sub = (j + 1) % kFetchSubs;
    c.tried++;
  }
  return F.nfetch;
}
__device__ __forceinline__ long long dev_fetch_take(long long mine) {
  __shared__ long long s_claim;
  __syncthreads();  // every thread is done with the previous fetch
  if (threadIdx.x == 0) s_claim = mine;
  __syncthreads();
  return s_claim;
}
__device__ __forceinline__ long long dev_fetch_first(const DevFetch& F, FetchCursor& c) {
  return dev_fetch_take(threadIdx.x == 0 ? dev_fetch_claim(F, c) : 0);
}
__device__ __forceinline__ long long dev_fetch_issue(const DevFetch& F, FetchCursor& c) {
  return threadIdx.x == 0 ? dev_fetch_claim(F, c) : 0;
}
__device__ __forceinline__ void dev_fetch_range(const DevFetch& F, long long f, long long& b0, long long& b1) {
  b0 = F.first + f * F.grain;
  b1 = b0 + F.grain < F.first + F.total ? b0 + F.grain : F.first + F.total;
}
// blocks [b0, b1) of a fetch ran: busy/executed counters (runtime.py:344-348)
__device__ __forceinline__ void dev_fetch_done(const DevFetch& F, FetchCursor& c, long long b0, long long b1) {
  if (threadIdx.x == 0) c.blocks += (unsigned long long)(b1 - b0);
  if (F.executed)
    for (long long b = b0 + threadIdx.x; b < b1; b += blockDim.x) atomicAdd(F.executed + b, 1);
}
// the CTA's totals into its worker slot's statistics (call once, after the loop)
__device__ __forceinline__ void dev_fetch_flush(const DevFetch& F, const FetchCursor& c) {
  if (threadIdx.x == 0 && c.claims) {
    atomicAdd(F.stats + 2 * (blockIdx.x % F.slots), c.claims);
    atomicAdd(F.stats + 2 * (blockIdx.x % F.slots) + 1, c.blocks);
  }
}

// i32 wrapping multiply-add, as `blockIdx.x * blockDim.x + threadIdx.x` is
// evaluated with wrap_int after every operator (interp.py:89-90, arena.py:39-41).
__device__ __forceinline__ int wrap_mad(int a, int b, int c) {
  return (int)((unsigned)a * (unsigned)b + (unsigned)c);
}

// f64 arithmetic that must never be contracted into an FMA: the reference
// rounds every binary operator result to double (Python float arithmetic).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

}  // namespace bf

// ---- mbarrier + bulk-copy (TMA 1D) helpers, sm_90+ PTX --------------------
namespace bf {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {  // try_wait with a suspend-time hint: the warp sleeps until the phase flips
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000)
        : "memory");
  } while (!done);
}
// waiting loop for a single producer thread: back off so it does not steal
// issue slots from the consumer warps of its SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000)
        : "memory");
    if (done) return;
    __nanosleep(128);
  }
}
// global -> shared bulk copy completing `bytes` of transaction on `bar`
// (16 B aligned addresses, bytes % 16 == 0); streamed (L2 evict-first)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// shared -> global bulk copy (bulk-group completion), 16 B aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) accesses of the same memory
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
}  // namespace bf
