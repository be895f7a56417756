// hotspot — paper_2206_07896_b200/kernels/hotspot.kn (Rodinia-style 5-point
// thermal stencil, one iteration per launch, clamped borders).
//
// Semantics (bit-exact with the reference interpreter): temperatures and
// power are f32 in memory; every operator is evaluated in f64 in source order
// (interp.py:58-91) and the result is rounded to f32 once at the store
// (arena.py:111-116).  The f32 scalar params carry doubles (hostprog.py:
// 390-414).  No FMA contraction: dadd/dsub/dmul are the _rn intrinsics.
//
// B200 mapping (fast path, hotspot_rows): persistent CTAs, each streaming
// whole 1024-float row segments down (or, every other launch, up) its band
// through a 6-stage shared-memory ring filled by bulk copies (TMA) from a
// producer warp; 8 consumer warps keep the north / centre rows in registers
// as doubles, so every value is widened to f64 once.  The kernel sits at the
// HBM roofline only because the f64 arithmetic (14 DP ops per cell) and the
// f32<->f64 conversions (quarter-rate XU pipe) are kept to one conversion
// per loaded value; see profiles/r2/hotspot.md.  Algorithmic traffic per
// cell and iteration: 12 B (read src + power, write dst).
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

// The same cell with every operand already widened to f64 (the row
// pipeline keeps rows as doubles across the row loop, so each value is
// converted once, not once per stencil use: F2F runs on the quarter-rate XU
// pipe, which bounds this kernel before HBM does).
__device__ __forceinline__ float hs_cell_d(double tc, double tn, double ts, double tw, double te, double p,
                                           const HsConst& k) {
  const double two_tc = dmul(2.0, tc);
  const double a = dsub(dadd(ts, tn), two_tc);
  const double b = dsub(dadd(te, tw), two_tc);
  const double c = dsub(k.amb, tc);
  double acc = dadd(p, dmul(a, k.ry1));
  acc = dadd(acc, dmul(b, k.rx1));
  acc = dadd(acc, dmul(c, k.rz1));
  const double delta = dmul(k.sdc, acc);
  return __double2float_rn(dadd(tc, delta));
}

struct D4 {
  double x, y, z, w;
};
__device__ __forceinline__ D4 widen4(float4 v) { return D4{(double)v.x, (double)v.y, (double)v.z, (double)v.w}; }

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

// Row-pipeline kernel (default fast path).  The cell rectangle is cut into
// column segments of W = 1024*V floats; a work unit is one (segment, row)
// pair, units are numbered segment-major and every CTA (persistent, one
// resident wave) takes a contiguous run of them: one or two vertical
// sub-bands of its segment, so each CTA streams whole W-float row segments
// (4-8 KB contiguous) down its band instead of 512 B per warp per row.
// A producer warp loads stage q = (src row q with a 4-float halo on each
// side, power row q) by two bulk copies (TMA, cp.async.bulk) into a ring of
// NS stages completing on the stage's mbarrier; 8 consumer warps keep the
// north / centre rows in registers, take the south row and the power row
// from shared memory, west / east neighbours by shuffles (segment edges
// from the halo floats) and store the f32 results straight to HBM.  A stage
// is released (empty barrier, one arrival per consumer warp) once the row
// it centres has been computed.
template <int V, int NS>
struct HsRowsSmem {
  float src[NS][V * 1024 + 8];  // [4 halo | W | 4 halo]
  float pw[NS][V * 1024];
  uint64_t full[NS], empty[NS];
};

template <int V, int NS, int MINB = 1>
__global__ void __launch_bounds__(288, MINB) hotspot_rows(const float* __restrict__ src,
                                                       const float* __restrict__ power,
                                                       float* __restrict__ dst, int rows, int cols,
                                                       int r_lo, int r_hi, int c_lo, int c_hi, int nseg,
                                                       int up, HsConst k) {
  constexpr int W = V * 1024;
  extern __shared__ __align__(128) unsigned char hs_smem[];
  HsRowsSmem<V, NS>& S = *reinterpret_cast<HsRowsSmem<V, NS>*>(hs_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // programmatic dependent launch: wait for the previous grid (and its
  // memory) before the first load, then let the next launch be scheduled
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const long long R = r_hi - r_lo;
  const long long U = R * nseg;
  const long long u_begin = U * blockIdx.x / gridDim.x, u_end = U * (blockIdx.x + 1) / gridDim.x;
  const long long colsl = cols;
  // sub-bands of this CTA's unit run in processing order (`up`: the last
  // one first, rows bottom-up; the stencil is symmetric in north/south, so
  // only the traversal order changes).  From cursor u returns the next
  // cursor and the sub-band's segment and rows [ra, rb).
  auto next_subband = [&](long long u, int& seg, int& ra, int& rb) -> long long {
    if (!up) {
      seg = (int)(u / R);
      const long long ub = min(u_end, (long long)(seg + 1) * R);
      ra = r_lo + (int)(u - (long long)seg * R);
      rb = r_lo + (int)(ub - (long long)seg * R);
      return ub;
    }
    seg = (int)((u - 1) / R);
    const long long ua = max(u_begin, (long long)seg * R);
    ra = r_lo + (int)(ua - (long long)seg * R);
    rb = r_lo + (int)(u - (long long)seg * R);
    return ua;
  };

  if (warp == 8) {  // producer
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    int slot = 0;          // ring cursor
    bool wrapped = false;  // every slot filled once: later stages wait for their slot to be released
    uint32_t phase = 0;    // parity of the empty barrier completion the next wait needs
    for (long long u = up ? u_end : u_begin; up ? u > u_begin : u < u_end;) {
      int seg, ra, rb;
      u = next_subband(u, seg, ra, rb);
      const int c0 = c_lo + seg * W, c1 = min(c0 + W, c_hi);
      const int h0 = max(c0 - 4, 0), h1 = min(c1 + 4, cols);
      const uint32_t sbytes = (uint32_t)(h1 - h0) * 4u, pbytes = (uint32_t)(c1 - c0) * 4u;
      const int soff = 4 - (c0 - h0);
      for (int i = 0; i < rb - ra + 2; i++) {
        const int q = up ? rb - i : ra - 1 + i;
        if (wrapped) mbar_wait_sleep(&S.empty[slot], phase);
        const int r = q < 0 ? 0 : (q >= rows ? rows - 1 : q);
        const bool has_p = q >= ra && q < rb;
        mbar_arrive_expect_tx(&S.full[slot], sbytes + (has_p ? pbytes : 0u));
        bulk_g2s(&S.src[slot][soff], src + r * colsl + h0, sbytes, &S.full[slot], pol);
        if (has_p) bulk_g2s(&S.pw[slot][0], power + r * colsl + c0, pbytes, &S.full[slot], pol);
        if (++slot == NS) {
          slot = 0;
          if (wrapped) phase ^= 1u;
          wrapped = true;
        }
      }
    }
    return;
  }

  // consumers: thread t owns columns x = 4*(t + 256*v) of the segment;
  // north / centre rows stay in registers as doubles, rotating through
  // three register sets (the row loop is unrolled by three so no row is
  // ever copied between registers)
  const int t = threadIdx.x;
  int a_slot = 0;       // next stage to acquire
  uint32_t a_phase = 0;
  auto acquire = [&]() -> int {
    const int sl = a_slot;
    mbar_wait(&S.full[sl], a_phase);
    if (++a_slot == NS) {
      a_slot = 0;
      a_phase ^= 1u;
    }
    return sl;
  };
  auto release = [&](int sl) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[sl]);
  };
  auto load_row = [&](D4 (&d)[V], int sl) {
#pragma unroll
    for (int v = 0; v < V; v++) d[v] = widen4(*reinterpret_cast<const float4*>(&S.src[sl][4 + 4 * (t + 256 * v)]));
  };
  for (long long u = up ? u_end : u_begin; up ? u > u_begin : u < u_end;) {
    int seg, ra, rb;
    u = next_subband(u, seg, ra, rb);
    const int c0 = c_lo + seg * W, c1 = min(c0 + W, c_hi);
    D4 A[V], B[V], C[V];
    int sl = acquire();
    load_row(A, sl);
    release(sl);
    int c_slot = acquire();
    load_row(B, c_slot);
    // one output row: nor / cen in registers, south row `sou` loaded here
    auto row = [&](const D4 (&nor)[V], const D4 (&cen)[V], D4 (&sou)[V], int r) {
      const int s_slot = acquire();
      const float* sc = S.src[c_slot];
      const float* sp = S.pw[c_slot];
      load_row(sou, s_slot);
#pragma unroll
      for (int v = 0; v < V; v++) {
        const int x = 4 * (t + 256 * v);
        const int c = c0 + x;
        const D4 p = widen4(*reinterpret_cast<const float4*>(&sp[x]));
        const D4 cv = cen[v], nv = nor[v], sv = sou[v];
        // strip edges: lane 0 takes its west neighbour, the last lane of a
        // warp (or of the segment) its east one from the halo'd row
        const bool need_w = lane == 0, need_e = lane == 31 || c + 4 >= c1;
        const double wd = (double)sc[4 + x - (c > 0 ? 1 : 0)];
        const double ed = (double)sc[4 + x + (c + 4 < cols ? 4 : 3)];
        double west = __shfl_up_sync(0xffffffffu, cv.w, 1);
        double east = __shfl_down_sync(0xffffffffu, cv.x, 1);
        west = need_w ? wd : west;
        east = need_e ? ed : east;
        if (c < c1) {
          float4 out;
          out.x = hs_cell_d(cv.x, nv.x, sv.x, west, cv.y, p.x, k);
          out.y = hs_cell_d(cv.y, nv.y, sv.y, cv.x, cv.z, p.y, k);
          out.z = hs_cell_d(cv.z, nv.z, sv.z, cv.y, cv.w, p.z, k);
          out.w = hs_cell_d(cv.w, nv.w, sv.w, cv.z, east, p.w, k);
          *reinterpret_cast<float4*>(dst + r * colsl + c) = out;
        }
      }
      release(c_slot);
      c_slot = s_slot;
    };
    const int dr = up ? -1 : 1;
    for (int r = up ? rb - 1 : ra, n = rb - ra;;) {
      if (n-- == 0) break;
      row(A, B, C, r);
      r += dr;
      if (n-- == 0) break;
      row(B, C, A, r);
      r += dr;
      if (n-- == 0) break;
      row(C, A, B, r);
      r += dr;
    }
    release(c_slot);
  }
}

// BF_HOTSPOT_ROWS: 1 (default) = hotspot_rows with 1024-float segments and
// 6 stages (two CTAs per SM); 2 = 2048-float segments, 4 stages; 0 = the
// round-1 warp-strip kernel (hotspot_band).  Measured (8192^2, 100 launches,
// per launch): 125.4 / 126.5 / 139.2 us (profiles/r2/hotspot.md).
static int hotspot_rows_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_HOTSPOT_ROWS");
    v = e ? atoi(e) : 1;
    if (v < 0 || v > 2) v = 1;
  }
  return v;
}

typedef void (*HsRowsFn)(const float*, const float*, float*, int, int, int, int, int, int, int, int, HsConst);

struct HsRowsCfg {
  HsRowsFn fn;
  int width;
  size_t smem;
};

static HsRowsCfg hotspot_rows_cfg(int variant) {
  if (variant == 2) return {hotspot_rows<2, 4, 2>, 2048, sizeof(HsRowsSmem<2, 4>)};
  return {hotspot_rows<1, 6>, 1024, sizeof(HsRowsSmem<1, 6>)};
}

static bool hs_rows_attr_done[64][4];

// BF_HOTSPOT_ALT (default 1): alternate the row traversal direction per launch
static bool hotspot_alternate() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_HOTSPOT_ALT");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static void hotspot_rows_launch(int variant, cudaStream_t stream, int num_sms, const float* src,
                                const float* power, float* dst, int rows, int cols, int r_lo, int r_hi,
                                int c_lo, int c_hi, HsConst k);

typedef void (*HsBandFn)(const float*, const float*, float*, int, int, int, int, int, int, int, int,
                         HsConst);

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

static void hotspot_rows_launch(int variant, cudaStream_t stream, int num_sms, const float* src,
                                const float* power, float* dst, int rows, int cols, int r_lo, int r_hi,
                                int c_lo, int c_hi, HsConst k) {
  const HsRowsCfg cfg = hotspot_rows_cfg(variant);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!hs_rows_attr_done[dev & 63][variant & 3]) {
    cudaFuncSetAttribute((const void*)cfg.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
    hs_rows_attr_done[dev & 63][variant & 3] = true;
  }
  const int nseg = (c_hi - c_lo + cfg.width - 1) / cfg.width;
  const long long units = (long long)(r_hi - r_lo) * nseg;
  long long grid = (long long)num_sms * resident_ctas((const void*)cfg.fn, 288, cfg.smem);
  if (grid > units) grid = units;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(288);
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = hotspot_pdl() ? 1 : 0;
  // alternate the traversal direction launch by launch: a launch then
  // starts on the rows its predecessor wrote last, which are still in L2
  // (loads are evict-first, so L2 holds mostly the freshest stores)
  static int flip[64];
  const int up = hotspot_alternate() ? (flip[dev & 63] ^= 1) : 0;
  cudaLaunchKernelEx(&lc, cfg.fn, src, power, dst, rows, cols, r_lo, r_hi, c_lo, c_hi, nseg, up, k);
}

static int hotspot_resident_warps(int num_sms) {
  return resident_ctas((const void*)hotspot_band<1>, 128, 0) * 4 * num_sms;
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
  if (cols % 4 == 0 && hotspot_rows_variant() > 0) {
    hotspot_rows_launch(hotspot_rows_variant(), stream, num_sms, src, power, dst, rows, cols, 0, rows, 0, cols, k);
  } else if (cols % 4 == 0) {
    const int groups = (cols + 127) / 128;
    const int warps = hotspot_resident_warps(num_sms);
    int bands = std::max(1, warps / groups);
    if (bands > rows) bands = rows;
    const int grid = (groups * bands + 3) / 4;
    hotspot_band_launch(hotspot_band<1>, grid, stream, src, power, dst, rows, cols, 0, rows, 0, cols, groups,
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
    if (in_bounds && aligned && hotspot_rows_variant() > 0) {
      hotspot_rows_launch(hotspot_rows_variant(), ctx.stream, ctx.num_sms, (const float*)S.ptr,
                          (const float*)P.ptr, (float*)D.ptr, rows, cols, (int)r_lo, (int)r_hi, (int)c_lo,
                          (int)c_hi, k);
    } else if (in_bounds && aligned) {
      const int groups = (int)((c_hi - c_lo + 127) / 128);
        const int warps = hotspot_resident_warps(ctx.num_sms);
      int bands = std::max(1, warps / groups);
      if (bands > r_hi - r_lo) bands = (int)(r_hi - r_lo);
      const int grid = (groups * bands + 3) / 4;
      hotspot_band_launch(hotspot_band<1>, grid, ctx.stream, (const float*)S.ptr, (const float*)P.ptr,
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
