// nn — paper_2206_07896_b200/kernels/nn.kn (Rodinia nn "euclid").
//
// d[id] = sqrt((ll[2id] - x)^2 + (ll[2id+1] - y)^2) for id < n, evaluated in
// f64 operator by operator (interp.py:58-91, 147-150: math.sqrt is the
// correctly rounded IEEE sqrt == __dsqrt_rn) and rounded to f32 at the store.
// Records are {lat, lng} f32 pairs (array of structs, as Rodinia's LatLong).
//
// B200 mapping: 4 records per thread step = two 16 B loads + one 16 B store,
// streaming cache hints; 12 B per record.  Bound: HBM (f64 sqrt is a handful
// of DFMA per record, well under the FP64 roof at this intensity).
#include <climits>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

__device__ __forceinline__ float nn_dist(float lat, float lng, double x, double y) {
  const double a = dsub((double)lat, x);
  const double b = dsub((double)lng, y);
  return __double2float_rn(__dsqrt_rn(dadd(dmul(a, a), dmul(b, b))));
}

__global__ void __launch_bounds__(256) nn_stream(const float* __restrict__ ll,
                                                 float* __restrict__ d, long long lo, long long hi,
                                                 double x, double y) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) d[lo + tid] = nn_dist(ll[2 * (lo + tid)], ll[2 * (lo + tid) + 1], x, y);
  if (tid < hi - vhi) d[vhi + tid] = nn_dist(ll[2 * (vhi + tid)], ll[2 * (vhi + tid) + 1], x, y);
  const float4* l4 = reinterpret_cast<const float4*>(ll);
  float4* d4 = reinterpret_cast<float4*>(d);
  long long g = vlo / 4 + tid;
  const long long end = vhi / 4;
  for (; g + stride < end; g += 2 * stride) {  // 4 x 16 B loads in flight
    const float4 p0 = __ldcs(l4 + 2 * g), q0 = __ldcs(l4 + 2 * g + 1);
    const float4 p1 = __ldcs(l4 + 2 * (g + stride)), q1 = __ldcs(l4 + 2 * (g + stride) + 1);
    __stcs(d4 + g, make_float4(nn_dist(p0.x, p0.y, x, y), nn_dist(p0.z, p0.w, x, y),
                               nn_dist(q0.x, q0.y, x, y), nn_dist(q0.z, q0.w, x, y)));
    __stcs(d4 + g + stride, make_float4(nn_dist(p1.x, p1.y, x, y), nn_dist(p1.z, p1.w, x, y),
                                        nn_dist(q1.x, q1.y, x, y), nn_dist(q1.z, q1.w, x, y)));
  }
  if (g < end) {
    const float4 p = __ldcs(l4 + 2 * g), q = __ldcs(l4 + 2 * g + 1);
    __stcs(d4 + g, make_float4(nn_dist(p.x, p.y, x, y), nn_dist(p.z, p.w, x, y),
                               nn_dist(q.x, q.y, x, y), nn_dist(q.z, q.w, x, y)));
  }
}

static int launch_nn(LaunchCtx& ctx) {
  const ArgVal& L = ctx.args[0];
  const ArgVal& D = ctx.args[1];
  const long long n = ctx.args[2].i32;
  const double x = ctx.args[3].f64, y = ctx.args[4].f64;
  const long long bx = ctx.block[0];
  for (auto& xi : ctx.x_intervals()) {
    long long lo = xi.first * bx, hi = std::min(xi.second * bx, n);
    if (lo >= hi) continue;
    if (2 * (hi - 1) + 1 > (long long)INT_MAX) {
      // 2*id wraps to a negative i32 index in the DSL: the load traps
      long long bad = ((long long)INT_MAX + 1) / 2;
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(std::max(lo, bad) / bx),
                    "record index 2*id beyond i32");
      hi = std::max(lo, bad);
    }
    long long safe = std::min(L.len / 2, D.len);
    if (hi > safe) {
      long long bad = std::max(lo, safe);
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(bad / bx),
                    "load index " + std::to_string(bad) + " out of range");
      hi = bad;
    }
    if (lo >= hi) continue;
    int grid = stream_grid((hi - lo + 3) / 4, 256, ctx.num_sms, 8);
    nn_stream<<<grid, 256, 0, ctx.stream>>>((const float*)L.ptr, (float*)D.ptr, lo, hi, x, y);
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_nn("nn",
                        {{BF_SLOT_HANDLE, BF_F32, "ll"},
                         {BF_SLOT_HANDLE, BF_F32, "d"},
                         {BF_SLOT_I32, BF_I32, "n"},
                         {BF_SLOT_F32, BF_F32, "x"},
                         {BF_SLOT_F32, BF_F32, "y"}},
                        launch_nn);

}  // namespace bf
