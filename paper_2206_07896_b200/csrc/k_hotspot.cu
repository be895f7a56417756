// hotspot — paper_2206_07896_b200/kernels/hotspot.kn (Rodinia-style 5-point
// thermal stencil, one iteration per launch, clamped borders).
//
// Semantics (bit-exact with the reference interpreter): temperatures and
// power are f32 in memory; every operator is evaluated in f64 in source order
// (interp.py:58-91) and the result is rounded to f32 once at the store
// (arena.py:111-116).  The f32 scalar params carry doubles (hostprog.py:
// 390-414).  No FMA contraction: dadd/dsub/dmul are the _rn intrinsics.
//
// B200 mapping (fast path): a warp owns a 128-column x band-row strip; each
// lane holds a float4 of the north/centre/south rows in registers and slides
// down the strip, so every row of `src` is loaded once per strip (+2 halo
// rows per band, served by L2).  West/east neighbours come from warp shuffles;
// lanes at the strip edge load one scalar.  Algorithmic traffic per cell and
// iteration: 12 B (read src + power, write dst).
#include <climits>
#include <cstdlib>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

struct HsConst {
  double sdc, rx1, ry1, rz1, amb;
};

__device__ __forceinline__ float hs_cell(float tcf, float tnf, float tsf, float twf, float tef,
                                         float pf, const HsConst& k) {
  const double tc = tcf, tn = tnf, ts = tsf, tw = twf, te = tef, p = pf;
  const double two_tc = dmul(2.0, tc);
  const double a = dsub(dadd(ts, tn), two_tc);  // (ts + tn - 2.0*tc)
  const double b = dsub(dadd(te, tw), two_tc);  // (te + tw - 2.0*tc)
  const double c = dsub(k.amb, tc);             // (amb - tc)
  double acc = dadd(p, dmul(a, k.ry1));
  acc = dadd(acc, dmul(b, k.rx1));
  acc = dadd(acc, dmul(c, k.rz1));
  const double delta = dmul(k.sdc, acc);
  return __double2float_rn(dadd(tc, delta));
}

// Work split: the cell rectangle is cut into G column groups of 128 columns
// (one warp wide) and `bands` row bands; warp w owns (band w / G, group
// w % G), so neighbouring column groups run on neighbouring warps at the same
// time (their shared edge columns hit L1/L2) and every warp gets the same
// number of rows to within one: no tail wave (grid = resident warps).
// The row loop is software-pipelined one row ahead: the south row, power
// row and edge scalars of row r+1 are in flight while row r is computed.
template <int PF>
__global__ void __launch_bounds__(128) hotspot_band(const float* __restrict__ src,
                                                    const float* __restrict__ power,
                                                    float* __restrict__ dst, int rows, int cols,
                                                    int r_lo, int r_hi, int c_lo, int c_hi,
                                                    int groups, int bands, HsConst k) {
  // programmatic dependent launch (hotspot_pdl): this grid may be scheduled
  // while the previous kernel in the stream drains; wait for it (and its
  // memory) before the first load, and let the next launch get scheduled
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (w >= groups * bands) return;  // warp-uniform
  const int band = w / groups, g = w % groups;
  const long long nr = r_hi - r_lo;
  const int r_start = r_lo + (int)(nr * band / bands);
  const int r_end = r_lo + (int)(nr * (band + 1) / bands);
  if (r_start >= r_end) return;
  const int c0 = c_lo + g * 128 + lane * 4;
  const bool active = c0 < c_hi;
  const bool west_scalar = lane == 0;
  const bool east_scalar = (lane == 31) || (c0 + 4 >= c_hi);
  const long long colsl = cols;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);

  auto row4 = [&](int r) -> float4 {
    return active ? __ldg(reinterpret_cast<const float4*>(src + r * colsl + c0)) : zero;
  };
  auto pow4 = [&](int r) -> float4 {
    return active ? __ldcs(reinterpret_cast<const float4*>(power + r * colsl + c0)) : zero;
  };
  auto west_of = [&](int r) -> float {
    return (active && west_scalar && c0 > 0) ? __ldg(src + r * colsl + c0 - 1) : 0.f;
  };
  auto east_of = [&](int r) -> float {
    return (active && east_scalar && c0 + 4 < cols) ? __ldg(src + r * colsl + c0 + 4) : 0.f;
  };
  auto clamp_row = [&](int r) { return r < r_end ? r : r_end - 1; };

  // ring of PF rows in flight: slot i holds (south row of r+i, power/edges of r+i)
  float4 north = row4(r_start > 0 ? r_start - 1 : 0);
  float4 center = row4(r_start);
  float4 sq[PF], pq[PF];
  float wq[PF], eq[PF];
#pragma unroll
  for (int i = 0; i < PF; i++) {
    const int rr = clamp_row(r_start + i);
    sq[i] = row4(rr + 1 < rows ? rr + 1 : rows - 1);
    pq[i] = pow4(rr);
    wq[i] = west_of(rr);
    eq[i] = east_of(rr);
  }
  for (int r = r_start; r < r_end; r++) {
    const float4 south = sq[0], p = pq[0];
    const float we = wq[0], ee = eq[0];
#pragma unroll
    for (int i = 0; i < PF - 1; i++) {
      sq[i] = sq[i + 1];
      pq[i] = pq[i + 1];
      wq[i] = wq[i + 1];
      eq[i] = eq[i + 1];
    }
    {
      const int rr = clamp_row(r + PF);
      sq[PF - 1] = row4(rr + 1 < rows ? rr + 1 : rows - 1);
      pq[PF - 1] = pow4(rr);
      wq[PF - 1] = west_of(rr);
      eq[PF - 1] = east_of(rr);
    }
    float west = __shfl_up_sync(0xffffffffu, center.w, 1);
    float east = __shfl_down_sync(0xffffffffu, center.x, 1);
    if (west_scalar) west = c0 > 0 ? we : center.x;
    if (east_scalar) east = c0 + 4 < cols ? ee : center.w;
    if (active) {
      float4 out;
      out.x = hs_cell(center.x, north.x, south.x, west, center.y, p.x, k);
      out.y = hs_cell(center.y, north.y, south.y, center.x, center.z, p.y, k);
      out.z = hs_cell(center.z, north.z, south.z, center.y, center.w, p.z, k);
      out.w = hs_cell(center.w, north.w, south.w, center.z, east, p.w, k);
      *reinterpret_cast<float4*>(dst + r * colsl + c0) = out;
    }
    north = center;
    center = south;
  }
}

// Same work split, but the rows in flight live in shared memory instead of
// registers: each lane streams its own float4 of the src/power rows (and the
// strip-edge scalars) D-2 rows ahead of the south row with cp.async into a
// lane-private ring of D slots, so the loads in flight per SM are no longer
// paid for with registers (occupancy) — Little's law at ~6.4 TB/s needs
// ~60 KB in flight per SM.  Every lane reads back only what it copied itself,
// so the ring needs no warp barrier: cp.async.wait_group orders the RAW, and
// a slot is rewritten two iterations after its last read (WAR by program
// order of consumed registers).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int D>
__global__ void __launch_bounds__(128) hotspot_async(const float* __restrict__ src,
                                                     const float* __restrict__ power,
                                                     float* __restrict__ dst, int rows, int cols,
                                                     int r_lo, int r_hi, int c_lo, int c_hi,
                                                     int groups, int bands, HsConst k) {
  static_assert(D >= 3, "ring needs north/centre/south + one row in flight");
  __shared__ __align__(16) float4 ring[4][D][64];  // [warp][slot][src lanes | power lanes]
  __shared__ float edge[4][D][2];                  // [warp][slot][west, east]
  const int lane = threadIdx.x & 31;
  const int wi = threadIdx.x >> 5;
  const int w = blockIdx.x * 4 + wi;
  if (w >= groups * bands) return;  // warp-uniform
  const int band = w / groups, g = w % groups;
  const long long nr = r_hi - r_lo;
  const int r_start = r_lo + (int)(nr * band / bands);
  const int r_end = r_lo + (int)(nr * (band + 1) / bands);
  if (r_start >= r_end) return;
  const int n = r_end - r_start;
  const int c0 = c_lo + g * 128 + lane * 4;
  const bool active = c0 < c_hi;
  const bool west_scalar = lane == 0;
  const bool east_scalar = (lane == 31) || (c0 + 4 >= c_hi);
  const bool west_load = active && west_scalar && c0 > 0;
  const bool east_load = active && east_scalar && c0 + 4 < cols;
  const long long colsl = cols;

  // row sequence q = 0 .. n+1: clamp(r_start - 1 + q); centre rows are 1..n
  auto issue = [&](int q, int s) {
    if (active && q <= n + 1) {
      int r = r_start - 1 + q;
      r = r < 0 ? 0 : (r >= rows ? rows - 1 : r);
      const float* row = src + r * colsl;
      cp_async16(&ring[wi][s][lane], row + c0);
      if (q >= 1 && q <= n) {
        cp_async16(&ring[wi][s][32 + lane], power + r * colsl + c0);
        if (west_load) cp_async4(&edge[wi][s][0], row + c0 - 1);
        if (east_load) cp_async4(&edge[wi][s][1], row + c0 + 4);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int q = 0; q < D - 1; q++) issue(q, q);
  cp_async_wait<D - 3>();
  float4 north = ring[wi][0][lane];
  float4 center = ring[wi][1][lane];
  int s_c = 1;          // slot of the centre row
  int s_i = D - 1;      // slot the next issue writes
  for (int q = 1; q <= n; q++) {
    issue(q + D - 2, s_i);
    s_i = s_i + 1 == D ? 0 : s_i + 1;
    cp_async_wait<D - 3>();
    const int s_s = s_c + 1 == D ? 0 : s_c + 1;
    const float4 south = ring[wi][s_s][lane];
    const float4 p = ring[wi][s_c][32 + lane];
    float west = __shfl_up_sync(0xffffffffu, center.w, 1);
    float east = __shfl_down_sync(0xffffffffu, center.x, 1);
    if (west_scalar) west = c0 > 0 ? edge[wi][s_c][0] : center.x;
    if (east_scalar) east = c0 + 4 < cols ? edge[wi][s_c][1] : center.w;
    if (active) {
      float4 out;
      out.x = hs_cell(center.x, north.x, south.x, west, center.y, p.x, k);
      out.y = hs_cell(center.y, north.y, south.y, center.x, center.z, p.y, k);
      out.z = hs_cell(center.z, north.z, south.z, center.y, center.w, p.z, k);
      out.w = hs_cell(center.w, north.w, south.w, center.z, east, p.w, k);
      *reinterpret_cast<float4*>(dst + (r_start + q - 1) * colsl + c0) = out;
    }
    north = center;
    center = south;
    s_c = s_s;
  }
  cp_async_wait<0>();
}

static int hotspot_pf() {
  static int pf = -1;
  if (pf < 0) {
    const char* e = getenv("BF_HOTSPOT_PF");
    pf = e ? atoi(e) : 1;
    if (pf < 1 || pf > 4) pf = 1;
  }
  return pf;
}

// kernel variant: 0 = register prefetch (hotspot_band<PF>), D >= 3 =
// shared-memory ring of D slots (hotspot_async<D>).  BF_HOTSPOT_RING.
static int hotspot_ring() {
  static int d = -1;
  if (d < 0) {
    const char* e = getenv("BF_HOTSPOT_RING");
    d = e ? atoi(e) : 0;
    if (d != 0 && d != 3 && d != 4 && d != 6 && d != 8) d = 0;
  }
  return d;
}

typedef void (*HsBandFn)(const float*, const float*, float*, int, int, int, int, int, int, int, int,
                         HsConst);
static HsBandFn hotspot_band_fn(int pf) {
  switch (hotspot_ring()) {
    case 3: return hotspot_async<3>;
    case 4: return hotspot_async<4>;
    case 6: return hotspot_async<6>;
    case 8: return hotspot_async<8>;
    default: break;
  }
  switch (pf) {
    case 1: return hotspot_band<1>;
    case 3: return hotspot_band<3>;
    case 4: return hotspot_band<4>;
    default: return hotspot_band<2>;
  }
}

// BF_HOTSPOT_PDL (default 1): band launches carry the programmatic stream
// serialization attribute, so a launch's CTAs are scheduled as the previous
// launch's CTAs retire (launch latency hidden) and wait in-kernel for its
// completion (griddepcontrol.wait) before reading.
static bool hotspot_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_HOTSPOT_PDL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static void hotspot_band_launch(HsBandFn fn, int grid, cudaStream_t stream, const float* src, const float* power,
                                float* dst, int rows, int cols, int r_lo, int r_hi, int c_lo, int c_hi, int groups,
                                int bands, HsConst k) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = hotspot_pdl() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, fn, src, power, dst, rows, cols, r_lo, r_hi, c_lo, c_hi, groups, bands, k);
}

static int hotspot_resident_warps(int num_sms, int pf) {
  return resident_ctas((const void*)hotspot_band_fn(pf), 128, 0) * 4 * num_sms;
}

// Generic path: any geometry or alignment; one thread per cell of the cell
// rectangle, indices evaluated with i32 wrap exactly as the DSL does, every
// access bounds-checked (a trap records the logical block and skips).
__global__ void __launch_bounds__(256) hotspot_cells(const float* src, const float* power,
                                                     float* dst, long long len_src,
                                                     long long len_pow, long long len_dst,
                                                     int rows, int cols, int r_lo, int r_hi,
                                                     int c_lo, int c_hi, HsConst k, KDesc d,
                                                     long long zbase) {
  const long long w = c_hi - c_lo;
  const long long total = w * (long long)(r_hi - r_lo);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = r_lo + (int)(i / w);
    const int c = c_lo + (int)(i % w);
    const int rn = max(r - 1, 0), rs = min(r + 1, rows - 1);
    const int cw = max(c - 1, 0), ce = min(c + 1, cols - 1);
    const int idx = wrap_mad(r, cols, c);
    const int in_ = wrap_mad(rn, cols, c), is_ = wrap_mad(rs, cols, c);
    const int iw = wrap_mad(r, cols, cw), ie = wrap_mad(r, cols, ce);
    if (idx < 0 || idx >= len_src || in_ < 0 || in_ >= len_src || is_ < 0 || is_ >= len_src ||
        iw < 0 || iw >= len_src || ie < 0 || ie >= len_src || idx >= len_pow || idx >= len_dst) {
      const long long blk = zbase + (long long)(r / d.by) * d.gx + c / d.bx;
      record_fault(d, BF_TRAP_OUT_OF_BOUNDS, blk);
      continue;
    }
    dst[idx] = hs_cell(src[idx], src[in_], src[is_], src[iw], src[ie], power[idx], k);
  }
}

// One full-grid step (used by the fused host-loop driver, k_hotspot_fused.cu).
int hotspot_step_full(cudaStream_t stream, int num_sms, const float* src, const float* power,
                      float* dst, int rows, int cols, const double* kc) {
  HsConst k{kc[0], kc[1], kc[2], kc[3], kc[4]};
  if (cols % 4 == 0) {
    const int groups = (cols + 127) / 128;
    const int pf = hotspot_pf();
    const int warps = hotspot_resident_warps(num_sms, pf);
    int bands = std::max(1, warps / groups);
    if (bands > rows) bands = rows;
    const int grid = (groups * bands + 3) / 4;
    hotspot_band_launch(hotspot_band_fn(pf), grid, stream, src, power, dst, rows, cols, 0, rows, 0, cols, groups,
                        bands, k);
  } else {
    KDesc d{};
    int grid = stream_grid((long long)rows * cols, 256, num_sms, 8);
    hotspot_cells<<<grid, 256, 0, stream>>>(src, power, dst, (long long)rows * cols,
                                           (long long)rows * cols, (long long)rows * cols, rows,
                                           cols, 0, rows, 0, cols, k, d, 0);
  }
  return cudaGetLastError() == cudaSuccess ? BF_OK : BF_E_CUDA;
}

static int launch_hotspot(LaunchCtx& ctx) {
  const ArgVal& S = ctx.args[0];
  const ArgVal& P = ctx.args[1];
  const ArgVal& D = ctx.args[2];
  const int rows = ctx.args[3].i32;
  const int cols = ctx.args[4].i32;
  HsConst k{ctx.args[5].f64, ctx.args[6].f64, ctx.args[7].f64, ctx.args[8].f64,
            ctx.args[9].f64};
  if (rows <= 0 || cols <= 0) return BF_OK;
  const long long bx = ctx.block[0], by = ctx.block[1];
  const long long plane = (long long)ctx.grid[0] * ctx.grid[1];
  long long zbase = (ctx.first / plane) * plane;
  const long long need = (long long)rows * cols;
  const bool in_bounds = need <= INT_MAX && S.len >= need && P.len >= need && D.len >= need;
  for (auto& rc : ctx.xy_rects()) {
    long long c_lo = rc.x0 * bx, c_hi = rc.x1 * bx;
    long long r_lo = rc.y0 * by, r_hi = rc.y1 * by;
    if (c_hi > cols) c_hi = cols;
    if (r_hi > rows) r_hi = rows;
    if (c_lo >= c_hi || r_lo >= r_hi) continue;
    // c/r beyond INT_MAX would wrap in the DSL; such launches are rejected
    if (c_hi > INT_MAX || r_hi > INT_MAX) {
      *ctx.error = "hotspot: cell coordinates beyond i32 range";
      return BF_E_UNSUPPORTED;
    }
    const bool aligned = (cols % 4 == 0) && (c_lo % 4 == 0) && (c_hi % 4 == 0);
    if (in_bounds && aligned) {
      const int groups = (int)((c_hi - c_lo + 127) / 128);
      const int pf = hotspot_pf();
      const int warps = hotspot_resident_warps(ctx.num_sms, pf);
      int bands = std::max(1, warps / groups);
      if (bands > r_hi - r_lo) bands = (int)(r_hi - r_lo);
      const int grid = (groups * bands + 3) / 4;
      hotspot_band_launch(hotspot_band_fn(pf), grid, ctx.stream, (const float*)S.ptr, (const float*)P.ptr,
                          (float*)D.ptr, rows, cols, (int)r_lo, (int)r_hi, (int)c_lo, (int)c_hi, groups, bands, k);
    } else {
      long long zb = zbase;
      if (zb + (rc.y0 * ctx.grid[0] + rc.x0) < ctx.first) zb += plane;
      int grid = stream_grid((c_hi - c_lo) * (r_hi - r_lo), 256, ctx.num_sms, 8);
      hotspot_cells<<<grid, 256, 0, ctx.stream>>>(
          (const float*)S.ptr, (const float*)P.ptr, (float*)D.ptr, S.len, P.len, D.len, rows,
          cols, (int)r_lo, (int)r_hi, (int)c_lo, (int)c_hi, k, ctx.desc(), zb);
    }
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_hotspot("hotspot",
                             {{BF_SLOT_HANDLE, BF_F32, "src"},
                              {BF_SLOT_HANDLE, BF_F32, "power"},
                              {BF_SLOT_HANDLE, BF_F32, "dst"},
                              {BF_SLOT_I32, BF_I32, "rows"},
                              {BF_SLOT_I32, BF_I32, "cols"},
                              {BF_SLOT_F32, BF_F32, "sdc"},
                              {BF_SLOT_F32, BF_F32, "rx1"},
                              {BF_SLOT_F32, BF_F32, "ry1"},
                              {BF_SLOT_F32, BF_F32, "rz1"},
                              {BF_SLOT_F32, BF_F32, "amb"}},
                             launch_hotspot);

}  // namespace bf
