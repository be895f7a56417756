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
#include <cstdlib>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

// RN_f32(RN_f64(sqrt(s))) without the ~30-op f64 sqrt sequence.
// f = sqrtf((float)s) is within one f32 ulp of the answer.  The f32
// midpoints m = f +- ulp/2 have <= 25 significant bits, so m*m is exact in
// f64 and s - m*m (an FMA) has the sign of sqrt(s) - m.  Pick the neighbour
// whose rounding interval holds sqrt(s); then emulate the double rounding:
// if RN_f64(sqrt(s)) == m exactly (|s - m*m| <= m * ulp64(m)), the f32
// rounding of m is a tie and goes to the even neighbour.  Values outside
// [2^-60, 2^60] (and s <= 0, NaN) take the exact f64 path.
// midpoints of the f32 rounding interval of f (f positive normal), exact in
// f64: f +- half an f32 ulp (a quarter below a power of two)
__device__ __forceinline__ void f32_midpoints(float f, double& mh, double& ml) {
  const int fb = __float_as_int(f);
  const long long e = (fb >> 23) & 0xff;  // biased f32 exponent
  const double hu = __longlong_as_double((e - 127 - 24 + 1023) << 52);  // ulp/2
  const double fd = (double)f;
  mh = fd + hu;
  ml = fd - ((fb & 0x7fffff) ? hu : 0.5 * hu);
}

__device__ __forceinline__ float sqrt_f64_to_f32(double s) {
  if (!(s >= 0x1p-60 && s <= 0x1p60)) return __double2float_rn(__dsqrt_rn(s));
  float f = sqrtf(__double2float_rn(s));  // within one f32 ulp of the answer
  double mh, ml;
  f32_midpoints(f, mh, ml);
  double eh = fma(-mh, mh, s), el = fma(-ml, ml, s);  // exact near the answer
  if (eh > 0.0 || el < 0.0) {  // sqrt(s) lies in a neighbour's interval
    f = __int_as_float(__float_as_int(f) + (eh > 0.0 ? 1 : -1));
    f32_midpoints(f, mh, ml);
    eh = fma(-mh, mh, s);
    el = fma(-ml, ml, s);
  }
  // double rounding: RN64(sqrt(s)) == m exactly iff sqrt(s) is within half
  // an f64 ulp of m, i.e. -m*u < s - m^2 <= m*u with u = ulp64(m) (f64 ties
  // go to m: it has <= 25 significant bits); then the f32 rounding of m is a
  // tie and goes to the even neighbour
  // m * ulp64(m): add ulp64's exponent to m's (exact, integer pipe)
  auto times_ulp = [](double m) {
    const long long b = __double_as_longlong(m);
    const long long e = (b >> 52) & 0x7ff;
    return __longlong_as_double(b + ((e - 1075) << 52));
  };
  const double th = times_ulp(mh), tl = times_ulp(ml);
  const bool even = (__float_as_int(f) & 1) == 0;
  if (eh > -th && eh <= th) return even ? f : __int_as_float(__float_as_int(f) + 1);
  if (el > -tl && el <= tl) return even ? f : __int_as_float(__float_as_int(f) - 1);
  return f;
}

template <bool EMU>
__device__ __forceinline__ float nn_dist(float lat, float lng, double x, double y) {
  const double a = dsub((double)lat, x);
  const double b = dsub((double)lng, y);
  const double s = dadd(dmul(a, a), dmul(b, b));
  return EMU ? sqrt_f64_to_f32(s) : __double2float_rn(__dsqrt_rn(s));
}

template <bool EMU>
__global__ void __launch_bounds__(256) nn_stream(const float* __restrict__ ll,
                                                 float* __restrict__ d, long long lo, long long hi,
                                                 double x, double y) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) d[lo + tid] = nn_dist<EMU>(ll[2 * (lo + tid)], ll[2 * (lo + tid) + 1], x, y);
  if (tid < hi - vhi) d[vhi + tid] = nn_dist<EMU>(ll[2 * (vhi + tid)], ll[2 * (vhi + tid) + 1], x, y);
  const float4* l4 = reinterpret_cast<const float4*>(ll);
  float4* d4 = reinterpret_cast<float4*>(d);
  long long g = vlo / 4 + tid;
  const long long end = vhi / 4;
  // 4 x 16 B loads per step, software-pipelined: the next step's loads are
  // in flight while this step's eight f64 distances (DSQRT) are computed
  if (g + stride < end) {
    float4 p0 = __ldcs(l4 + 2 * g), q0 = __ldcs(l4 + 2 * g + 1);
    float4 p1 = __ldcs(l4 + 2 * (g + stride)), q1 = __ldcs(l4 + 2 * (g + stride) + 1);
    for (;;) {
      const long long gn = g + 2 * stride;
      const bool more = gn + stride < end;
      float4 np0, nq0, np1, nq1;
      if (more) {
        np0 = __ldcs(l4 + 2 * gn);
        nq0 = __ldcs(l4 + 2 * gn + 1);
        np1 = __ldcs(l4 + 2 * (gn + stride));
        nq1 = __ldcs(l4 + 2 * (gn + stride) + 1);
      }
      __stcs(d4 + g, make_float4(nn_dist<EMU>(p0.x, p0.y, x, y), nn_dist<EMU>(p0.z, p0.w, x, y),
                                 nn_dist<EMU>(q0.x, q0.y, x, y), nn_dist<EMU>(q0.z, q0.w, x, y)));
      __stcs(d4 + g + stride, make_float4(nn_dist<EMU>(p1.x, p1.y, x, y), nn_dist<EMU>(p1.z, p1.w, x, y),
                                          nn_dist<EMU>(q1.x, q1.y, x, y), nn_dist<EMU>(q1.z, q1.w, x, y)));
      g = gn;
      if (!more) break;
      p0 = np0;
      q0 = nq0;
      p1 = np1;
      q1 = nq1;
    }
  }
  if (g < end) {
    const float4 p = __ldcs(l4 + 2 * g), q = __ldcs(l4 + 2 * g + 1);
    __stcs(d4 + g, make_float4(nn_dist<EMU>(p.x, p.y, x, y), nn_dist<EMU>(p.z, p.w, x, y),
                               nn_dist<EMU>(q.x, q.y, x, y), nn_dist<EMU>(q.z, q.w, x, y)));
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
    static int emu = -1;
    if (emu < 0) {
      const char* e = getenv("BF_NN_SQRT_EMU");
      emu = e ? atoi(e) : 0;
    }
    const int grid = emu ? wave_grid(nn_stream<true>, 256, 0, (hi - lo + 3) / 4, 256, ctx.num_sms, 8)
                         : wave_grid(nn_stream<false>, 256, 0, (hi - lo + 3) / 4, 256, ctx.num_sms, 8);
    if (emu)
      nn_stream<true><<<grid, 256, 0, ctx.stream>>>((const float*)L.ptr, (float*)D.ptr, lo, hi, x, y);
    else
      nn_stream<false><<<grid, 256, 0, ctx.stream>>>((const float*)L.ptr, (float*)D.ptr, lo, hi, x, y);
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
