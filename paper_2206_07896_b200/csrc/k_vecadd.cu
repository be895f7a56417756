// vecadd — corpus/vecadd.kn:2-7 (`if (id < n) c[id] = a[id] + b[id]`).
//
// Semantics: the reference adds two f32 values as Python doubles and rounds
// once at the f32 store (interp.py:58-91, arena.py:111-116).  The exact sum of
// two f32 values rounded to f64 and then to f32 equals the correctly rounded
// f32 sum (53 >= 2*24+2), so a plain FADD is bit-exact.
//
// B200 mapping: the covered element range of a fetch is a union of at most
// two intervals [x0*bx, x1*bx) ∩ [0, n); each is streamed with 128-bit
// loads/stores (evict-first, single use) by a grid sized to the SM count.
// Algorithmic traffic: 12 B/element.
#include <climits>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

__global__ void __launch_bounds__(256) vecadd_stream(const float* a, const float* b, float* c,
                                                     long long lo, long long hi) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // scalar head up to 16 B alignment, float4 body, scalar tail
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) c[lo + tid] = a[lo + tid] + b[lo + tid];
  if (tid < hi - vhi) c[vhi + tid] = a[vhi + tid] + b[vhi + tid];
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* c4 = reinterpret_cast<float4*>(c);
  long long i = vlo / 4 + tid;
  const long long end = vhi / 4;
  // two independent 16 B loads per operand in flight per thread
  for (; i + stride < end; i += 2 * stride) {
    float4 x0 = __ldcs(a4 + i), y0 = __ldcs(b4 + i);
    float4 x1 = __ldcs(a4 + i + stride), y1 = __ldcs(b4 + i + stride);
    __stcs(c4 + i, make_float4(x0.x + y0.x, x0.y + y0.y, x0.z + y0.z, x0.w + y0.w));
    __stcs(c4 + i + stride, make_float4(x1.x + y1.x, x1.y + y1.y, x1.z + y1.z, x1.w + y1.w));
  }
  if (i < end) {
    float4 x0 = __ldcs(a4 + i), y0 = __ldcs(b4 + i);
    __stcs(c4 + i, make_float4(x0.x + y0.x, x0.y + y0.y, x0.z + y0.z, x0.w + y0.w));
  }
}

static int launch_vecadd(LaunchCtx& ctx) {
  const ArgVal& A = ctx.args[0];
  const ArgVal& B = ctx.args[1];
  const ArgVal& C = ctx.args[2];
  const long long n = ctx.args[3].i32;
  const long long bx = ctx.block[0];
  long long minlen = A.len;
  if (B.len < minlen) minlen = B.len;
  if (C.len < minlen) minlen = C.len;
  for (auto& xi : ctx.x_intervals()) {
    long long lo = xi.first * bx;
    long long hi = xi.second * bx;
    if (hi > n) hi = n;
    if (lo >= hi) continue;
    // id = blockIdx.x*blockDim.x + threadIdx.x wraps to a negative i32 past
    // INT_MAX; `id < n` then holds and the load traps (arena.py:104-108)
    if (hi - 1 > (long long)INT_MAX) {
      long long x = ((long long)INT_MAX + 1) / bx;
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(x),
                    "load index wraps past i32 range");
      hi = (long long)INT_MAX + 1;
    }
    if (hi > minlen) {
      long long x = (lo > minlen ? lo : minlen) / bx;
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(x),
                    "load index " + std::to_string(lo > minlen ? lo : minlen) +
                        " out of range [0, " + std::to_string(minlen) + ")");
      hi = minlen;
    }
    if (lo >= hi) continue;
    int grid = wave_grid(vecadd_stream, 256, 0, (hi - lo + 3) / 4, 256 * 2, ctx.num_sms, 8);
    vecadd_stream<<<grid, 256, 0, ctx.stream>>>((const float*)A.ptr, (const float*)B.ptr,
                                                (float*)C.ptr, lo, hi);
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_vecadd("vecadd",
                            {{BF_SLOT_HANDLE, BF_F32, "a"},
                             {BF_SLOT_HANDLE, BF_F32, "b"},
                             {BF_SLOT_HANDLE, BF_F32, "c"},
                             {BF_SLOT_I32, BF_I32, "n"}},
                            launch_vecadd);

}  // namespace bf
