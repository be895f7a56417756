// hotspot_run — Rodinia's hotspot host loop (N ping-pong launches of
// kernels/hotspot.kn) fused with temporal blocking (Rodinia's own
// "pyramid" idea, restated for B200).
//
// Each CTA owns a TH x TW output tile and loads the tile plus a T-cell halo
// (src and power) into shared memory once, then advances T iterations
// on-chip: step s recomputes the region shrunk by s cells on every side that
// is not a grid border (a border clamps to itself, so it never shrinks).
// Every intermediate value is rounded to f32 when stored into shared memory,
// exactly as the per-launch kernel rounds at its global store, so the result
// is bit-identical to N launches of hotspot.kn (tests: oracle.hotspot_iterate).
//
// HBM traffic per T iterations: (TH+2T)(TW+2T)*8 B in + TH*TW*4 B out, i.e.
// ~1.9 B per cell-iteration at T=8 instead of 12: the pass becomes
// FP64-bound (13 DP ops + converts per cell-iteration).
#include <climits>
#include <cstdlib>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

struct HsConstF {
  double sdc, rx1, ry1, rz1, amb;
};

__device__ __forceinline__ float hsf_cell(float tcf, float tnf, float tsf, float twf, float tef,
                                          float pf, const HsConstF& k) {
  const double tc = tcf, tn = tnf, ts = tsf, tw = twf, te = tef, p = pf;
  const double two_tc = dmul(2.0, tc);
  const double a = dsub(dadd(ts, tn), two_tc);
  const double b = dsub(dadd(te, tw), two_tc);
  const double c = dsub(k.amb, tc);
  double acc = dadd(p, dmul(a, k.ry1));
  acc = dadd(acc, dmul(b, k.rx1));
  acc = dadd(acc, dmul(c, k.rz1));
  return __double2float_rn(dadd(tc, dmul(k.sdc, acc)));
}

constexpr int kTbH = 64;   // output tile rows
constexpr int kTbW = 128;  // output tile cols

template <int T>
__global__ void __launch_bounds__(512) hotspot_tb(const float* __restrict__ src,
                                                  const float* __restrict__ power,
                                                  float* __restrict__ dst, int rows, int cols,
                                                  HsConstF k, int steps) {
  constexpr int RH = kTbH + 2 * T, RW = kTbW + 2 * T;
  extern __shared__ float sm[];
  float* A = sm;
  float* B = sm + RH * RW;
  float* P = sm + 2 * RH * RW;
  const int r0 = blockIdx.y * kTbH, c0 = blockIdx.x * kTbW;
  const int gr = r0 - T, gc = c0 - T;  // global coords of local (0, 0)
  const int R0 = max(0, r0 - steps), R1 = min(rows, r0 + kTbH + steps);
  const int C0 = max(0, c0 - steps), C1 = min(cols, c0 + kTbW + steps);
  // blockDim = (32, 16): x walks columns (coalesced), y walks rows
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = R0 + ty; r < R1; r += blockDim.y) {
    const long long g = (long long)r * cols;
    float* Ar = A + (r - gr) * RW - gc;
    float* Pr = P + (r - gr) * RW - gc;
    for (int c = C0 + tx; c < C1; c += 32) {
      Ar[c] = __ldg(src + g + c);
      Pr[c] = __ldcs(power + g + c);
    }
  }
  __syncthreads();
  for (int s = 1; s <= steps; s++) {
    const int lo_r = R0 == 0 ? 0 : R0 + s, hi_r = R1 == rows ? rows : R1 - s;
    const int lo_c = C0 == 0 ? 0 : C0 + s, hi_c = C1 == cols ? cols : C1 - s;
    // a thread owns a band of rows and up to NC columns (c = lo_c + tx + 32 j)
    // and slides down its band keeping north/centre/south in registers:
    // NC independent f64 chains per thread, one new shared load per cell for
    // the south row plus west, east and power
    constexpr int NC = (RW + 31) / 32;
    const int nr = hi_r - lo_r;
    const int rb = lo_r + nr * ty / (int)blockDim.y, re = lo_r + nr * (ty + 1) / (int)blockDim.y;
    if (rb < re) {
      float north[NC], center[NC];
      int cj[NC];
#pragma unroll
      for (int j = 0; j < NC; j++) {
        cj[j] = lo_c + tx + 32 * j;
        const int lc = cj[j] < hi_c ? cj[j] : lo_c;  // clamp idle lanes to a valid cell
        const int l = (rb - gr) * RW - gc + lc;
        center[j] = A[l];
        north[j] = rb > 0 ? A[l - RW] : center[j];
      }
      for (int r = rb; r < re; r++) {
        const int lr = (r - gr) * RW - gc;
        const bool has_s = r < rows - 1;
#pragma unroll
        for (int j = 0; j < NC; j++) {
          const int c = cj[j];
          const int lc = c < hi_c ? c : lo_c;
          const int l = lr + lc;
          const float south = has_s ? A[l + RW] : center[j];
          const float west = lc > 0 ? A[l - 1] : center[j];
          const float east = lc < cols - 1 ? A[l + 1] : center[j];
          const float v = hsf_cell(center[j], north[j], south, west, east, P[l], k);
          if (c < hi_c) B[l] = v;
          north[j] = center[j];
          center[j] = south;
        }
      }
    }
    __syncthreads();
    float* t = A;
    A = B;
    B = t;
  }
  {
    const int re = min(rows, r0 + kTbH), ce = min(cols, c0 + kTbW);
    for (int r = r0 + ty; r < re; r += blockDim.y) {
      const float* Ar = A + (r - gr) * RW - gc;
      float* dr = dst + (long long)r * cols;
      for (int c = c0 + tx; c < ce; c += 32) dr[c] = Ar[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Register wavefront (temporal blocking without shared memory).
// A warp owns a strip of 32 lanes x 4 columns (float4 per lane) and a band of
// rows; lanes 0 and 31 are halo, lanes 1..30 the strip's 120 output columns
// (strips overlap by 8 columns).  T time levels advance together down the
// rows: in wave i level 0 takes row i (loaded once from HBM) and level L
// computes row i-L from the last three rows of level L-1, which stay in
// registers as f64 copies of their f32-rounded values (exact), so a cell
// costs 13 f64 ops + 3 converts per level.  West/east neighbours come from
// warp shuffles.  Border rows clamp: level L's "row -1" is its row 0 and its
// "row rows" is row rows-1 (the DSL's max/min clamps).  Invalid columns
// spread one column per level from a strip edge, so T <= 4 keeps lanes 1..30
// exact.  Bit-identical to T launches of hotspot.kn.
// ---------------------------------------------------------------------------
struct D4 {
  double x, y, z, w;
};

__device__ __forceinline__ D4 d4_of(float4 v) {
  return D4{(double)v.x, (double)v.y, (double)v.z, (double)v.w};
}

__device__ __forceinline__ double hs_cell_d(double tc, double tn, double ts, double tw, double te,
                                            double p, const HsConstF& k, float& out) {
  const double two_tc = dmul(2.0, tc);
  const double a = dsub(dadd(ts, tn), two_tc);
  const double b = dsub(dadd(te, tw), two_tc);
  const double c = dsub(k.amb, tc);
  double acc = dadd(p, dmul(a, k.ry1));
  acc = dadd(acc, dmul(b, k.rx1));
  acc = dadd(acc, dmul(c, k.rz1));
  out = __double2float_rn(dadd(tc, dmul(k.sdc, acc)));
  return (double)out;
}

constexpr int kWaveOut = 120;  // output columns per strip

template <int T>
__global__ void __launch_bounds__(128) hotspot_wave(const float* __restrict__ src,
                                                    const float* __restrict__ power,
                                                    float* __restrict__ dst, int rows, int cols,
                                                    HsConstF k, int strips, int bands) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (w >= strips * bands) return;  // warp-uniform
  const int strip = w % strips, band = w / strips;
  const int rs = (int)((long long)rows * band / bands);
  const int re = (int)((long long)rows * (band + 1) / bands);
  if (rs >= re) return;
  const int c0 = strip * kWaveOut;
  const int cl = c0 - 4 + 4 * lane;
  const bool in_grid = cl >= 0 && cl + 3 < cols;
  const bool out_lane = lane >= 1 && lane <= 30 && in_grid;
  const bool left_edge = cl == 0, right_edge = cl + 3 == cols - 1;
  const long long colsl = cols;

  auto load_src = [&](int r) -> float4 {
    r = r < 0 ? 0 : (r > rows - 1 ? rows - 1 : r);
    return in_grid ? __ldg(reinterpret_cast<const float4*>(src + r * colsl + cl))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto load_pow = [&](int r) -> float4 {
    r = r < 0 ? 0 : (r > rows - 1 ? rows - 1 : r);
    return in_grid ? __ldg(reinterpret_cast<const float4*>(power + r * colsl + cl))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  };

  D4 R[T][3];  // R[L] = rows (j-2, j-1, j) of level L, j its newest row
  float4 P[T];  // P[m] = power row i-1-m
#pragma unroll
  for (int L = 0; L < T; L++) {
    R[L][0] = R[L][1] = R[L][2] = D4{0, 0, 0, 0};
    P[L] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int i0 = rs - T, i1 = re - 1 + T;
  // one wave of prefetch: the input and power rows of wave i+1 are in flight
  // while wave i computes
  float4 nxt_src = load_src(i0), nxt_pow = load_pow(i0 - 1);
#pragma unroll 1
  for (int i = i0; i <= i1; i++) {
    const float4 cur_src = nxt_src, cur_pow = nxt_pow;
    nxt_src = load_src(i + 1);
    nxt_pow = load_pow(i);
    // level 0: extended row i of the input (rows clamp at the borders)
    {
      const D4 v = d4_of(cur_src);
      R[0][0] = R[0][1];
      R[0][1] = R[0][2];
      R[0][2] = v;
    }
#pragma unroll
    for (int m = T - 1; m > 0; m--) P[m] = P[m - 1];
    P[0] = cur_pow;
#pragma unroll
    for (int L = 1; L <= T; L++) {
      const int j = i - L;  // row computed at level L in this wave
      D4 nv;
      float4 fo = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j == rows) {
        nv = R[L < T ? L : 0][2];  // ext row rows == row rows-1 (only needed below level T)
      } else {
        const D4 n = R[L - 1][0], c = R[L - 1][1], s = R[L - 1][2];
        double west = __shfl_up_sync(0xffffffffu, c.w, 1);
        double east = __shfl_down_sync(0xffffffffu, c.x, 1);
        if (left_edge) west = c.x;
        if (right_edge) east = c.w;
        const float4 pw = P[L - 1];
        nv.x = hs_cell_d(c.x, n.x, s.x, west, c.y, (double)pw.x, k, fo.x);
        nv.y = hs_cell_d(c.y, n.y, s.y, c.x, c.z, (double)pw.y, k, fo.y);
        nv.z = hs_cell_d(c.z, n.z, s.z, c.y, c.w, (double)pw.z, k, fo.z);
        nv.w = hs_cell_d(c.w, n.w, s.w, c.z, east, (double)pw.w, k, fo.w);
      }
      if (L < T) {
        R[L][0] = R[L][1];
        R[L][1] = R[L][2];
        R[L][2] = nv;
        if (j == 0) R[L][1] = nv;  // ext row -1 of level L is its row 0
      } else if (j >= rs && j < re && out_lane) {
        *reinterpret_cast<float4*>(dst + j * colsl + cl) = fo;
      }
    }
  }
}

template <int T>
static int wave_pass(cudaStream_t stream, int num_sms, const float* a, const float* p, float* b,
                     int rows, int cols, const HsConstF& k) {
  const int per_sm = resident_ctas((const void*)hotspot_wave<T>, 128, 0) * 4;  // warps
  const int strips = (cols + kWaveOut - 1) / kWaveOut;
  int bands = std::max(1, per_sm * num_sms / strips);
  if (bands > rows) bands = rows;
  const int grid = (strips * bands + 3) / 4;
  hotspot_wave<T><<<grid, 128, 0, stream>>>(a, p, b, rows, cols, k, strips, bands);
  return cudaGetLastError() == cudaSuccess ? BF_OK : BF_E_CUDA;
}

static int wave_run(cudaStream_t stream, int num_sms, float* a, float* b, const float* p, int rows,
                    int cols, const HsConstF& k, int iterations, int T, float** result) {
  float* cur = a;
  float* nxt = b;
  for (int done = 0; done < iterations;) {
    const int t = std::min(T, iterations - done);
    int rc;
    switch (t) {
      case 1: rc = wave_pass<1>(stream, num_sms, cur, p, nxt, rows, cols, k); break;
      case 2: rc = wave_pass<2>(stream, num_sms, cur, p, nxt, rows, cols, k); break;
      case 3: rc = wave_pass<3>(stream, num_sms, cur, p, nxt, rows, cols, k); break;
      default: rc = wave_pass<4>(stream, num_sms, cur, p, nxt, rows, cols, k); break;
    }
    if (rc) return rc;
    done += t;
    std::swap(cur, nxt);
  }
  *result = cur;
  return BF_OK;
}

template <int T>
static int run_passes(cudaStream_t stream, float* a, float* b, const float* p, int rows, int cols,
                      const HsConstF& k, int iterations, float** result) {
  constexpr int RH = kTbH + 2 * T, RW = kTbW + 2 * T;
  const size_t smem = (size_t)3 * RH * RW * sizeof(float);
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(hotspot_tb<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  dim3 grid((cols + kTbW - 1) / kTbW, (rows + kTbH - 1) / kTbH);
  float* cur = a;
  float* nxt = b;
  for (int done = 0; done < iterations;) {
    const int steps = std::min(T, iterations - done);
    hotspot_tb<T><<<grid, dim3(32, 16), smem, stream>>>(cur, p, nxt, rows, cols, k, steps);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return BF_E_CUDA;
    done += steps;
    std::swap(cur, nxt);
  }
  *result = cur;
  return BF_OK;
}

}  // namespace bf

// Fused N-iteration hotspot: result of N ping-pong launches of hotspot.kn
// starting from `a`; lands in `a` when N is even and in `b` when N is odd
// (where the per-launch host loop leaves it).  The other buffer is scratch.
extern "C" int bf_hotspot_run_impl(void* stream_v, int num_sms, float* a, float* b,
                                   const float* p, int rows, int cols, const double* kc,
                                   int iterations, int tsteps, char* err, int errcap) {
  using namespace bf;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (rows <= 0 || cols <= 0 || iterations < 0 || (long long)rows * cols > INT_MAX) {
    snprintf(err, errcap, "hotspot_run: bad sizes");
    return BF_E_INVALID;
  }
  if (iterations == 0) return BF_OK;
  HsConstF k{kc[0], kc[1], kc[2], kc[3], kc[4]};
  if (tsteps <= 0) {
    const char* e = getenv("BF_HOTSPOT_T");
    tsteps = e ? atoi(e) : 4;  // register wavefront, 4 levels: fastest in round 1
  }
  float* res = nullptr;
  int rc = BF_OK;
  const char* we = getenv("BF_HOTSPOT_WAVE");
  const bool wave = (we ? atoi(we) : 1) && cols % 4 == 0;
  if (wave && tsteps >= 2 && tsteps <= 4) {
    rc = wave_run(stream, num_sms, a, b, p, rows, cols, k, iterations, tsteps, &res);
  } else if (tsteps == 1) {
    // measured fastest on B200 (round 1): the streaming band kernel per
    // iteration, issued back to back from C++ (no per-launch host work)
    float* cur = a;
    float* nxt = b;
    for (int i = 0; i < iterations && rc == BF_OK; i++) {
      rc = hotspot_step_full(stream, num_sms, cur, p, nxt, rows, cols, kc);
      std::swap(cur, nxt);
    }
    res = cur;
  } else switch (tsteps) {
    case 3:  // wave unavailable (cols % 4 != 0): shared-memory tiles
      rc = run_passes<4>(stream, a, b, p, rows, cols, k, iterations, &res);
      break;
    case 2: rc = run_passes<2>(stream, a, b, p, rows, cols, k, iterations, &res); break;
    case 4: rc = run_passes<4>(stream, a, b, p, rows, cols, k, iterations, &res); break;
    case 12: rc = run_passes<12>(stream, a, b, p, rows, cols, k, iterations, &res); break;
    case 16: rc = run_passes<16>(stream, a, b, p, rows, cols, k, iterations, &res); break;
    default: rc = run_passes<8>(stream, a, b, p, rows, cols, k, iterations, &res); break;
  }
  if (rc) {
    snprintf(err, errcap, "hotspot_run: launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return rc;
  }
  float* want = (iterations % 2 == 0) ? a : b;
  if (res != want) {
    cudaError_t e = cudaMemcpyAsync(want, res, (size_t)rows * cols * sizeof(float),
                                    cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) {
      snprintf(err, errcap, "hotspot_run: %s", cudaGetErrorString(e));
      return BF_E_CUDA;
    }
  }
  return BF_OK;
}
