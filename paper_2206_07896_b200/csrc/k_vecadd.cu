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

// Device-side fetching (BF_FLAG_DEVICE_FETCH): one persistent grid; each CTA
// claims `grain` logical blocks at a time and streams their elements
// [b0*bx, b1*bx) with 16 B vectors (1D grids, bx % 4 == 0).
__global__ void __launch_bounds__(256) vecadd_fetch(const float* a, const float* b, float* c, long long n,
                                                    long long bx, DevFetch F) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* c4 = reinterpret_cast<float4*>(c);
  FetchCursor fc = dev_fetch_cursor();
  long long f = dev_fetch_first(F, fc);
  while (f < F.nfetch) {
    const long long nx = dev_fetch_issue(F, fc);
    long long b0, b1;
    dev_fetch_range(F, f, b0, b1);
    const long long lo = b0 * bx, hi = b1 * bx < n ? b1 * bx : n;
    const long long vhi = lo + ((hi > lo ? hi - lo : 0) & ~3LL);
    for (long long i = lo / 4 + threadIdx.x; i < vhi / 4; i += blockDim.x) {
      const float4 x = __ldcs(a4 + i), y = __ldcs(b4 + i);
      __stcs(c4 + i, make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w));
    }
    for (long long i = vhi + threadIdx.x; i < hi; i += blockDim.x) c[i] = a[i] + b[i];
    dev_fetch_done(F, fc, b0, b1);
    f = dev_fetch_take(nx);
  }
  dev_fetch_flush(F, fc);
}

static int launch_vecadd_fetch(LaunchCtx& ctx) {
  const DevFetch& F = *ctx.dfetch;
  const ArgVal& A = ctx.args[0];
  const ArgVal& B = ctx.args[1];
  const ArgVal& C = ctx.args[2];
  const long long n = ctx.args[3].i32;
  const long long bx = ctx.block[0];
  const long long hi = std::min((F.first + F.total) * bx, n);
  // 1D geometry, aligned blocks, no host-detected trap (those keep host fetches)
  if ((long long)ctx.grid[1] * ctx.grid[2] * ctx.block[1] * ctx.block[2] != 1 || bx % 4 != 0 ||
      hi - 1 > (long long)INT_MAX || hi > std::min(A.len, std::min(B.len, C.len)))
    return BF_E_UNSUPPORTED;
  // a CTA as wide as one fetch's float4 (32..256 threads): fine grains get
  // more, narrower CTAs, i.e. more fetches in flight per SM
  const int threads = (int)std::min<long long>(256, std::max<long long>(32, (F.grain * bx / 4 + 31) / 32 * 32));
  const int grid = (int)std::min<long long>(
      F.nfetch, (long long)resident_ctas((const void*)vecadd_fetch, threads, 0) * ctx.num_sms);
  vecadd_fetch<<<grid, threads, 0, ctx.stream>>>((const float*)A.ptr, (const float*)B.ptr, (float*)C.ptr, n, bx,
                                                  F);
  BF_CUDA_LAUNCH_CHECK(ctx);
  ctx.dfetch_grid = grid;
  return BF_OK;
}

static int launch_vecadd(LaunchCtx& ctx) {
  if (ctx.dfetch) return launch_vecadd_fetch(ctx);
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
                            launch_vecadd, /*dev_fetch=*/true);

}  // namespace bf
