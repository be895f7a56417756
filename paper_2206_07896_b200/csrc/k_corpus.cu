// The reference corpus kernels other than vecadd (blockfuse/corpus/*.kn):
// reverse, reduce, hist, hist_stride, fir, wreduce.
//
// Each kernel reproduces the reference interpreter's result for the launch
// geometry exactly (executor.py:422-489 lockstep order where the result
// depends on it; integer sums wrap mod 2^32, which makes every integer
// reduction order-free).  Physical CTAs are sized for the B200, not copied
// from the logical geometry: single-block grid-stride kernels (fir,
// hist_stride) are spread over the whole GPU, histograms are privatised per
// lane in shared memory, reductions use warp shuffles.
#include <climits>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

// lowest linear block id of the fetch range whose blockIdx.x is x
__device__ __forceinline__ long long block_of_x(const KDesc& d, long long x) {
  long long x0 = d.first % d.gx;
  return d.first + ((x - x0) % d.gx + d.gx) % d.gx;
}

// Split the fetch range into x-intervals with a uniform copy count: each
// logical block (x, y, z) of the range runs the same body, so an x that
// appears in c rows of the range is executed c times (what matters for
// atomics).  At most three pieces: head row, full rows, tail row.
struct XPiece {
  long long x0, x1, copies;
};

static std::vector<XPiece> x_pieces(const LaunchCtx& ctx) {
  std::vector<XPiece> out;
  long long gx = ctx.grid[0];
  long long b = ctx.first, e = ctx.first + ctx.count;
  long long hx = b % gx;
  if (hx != 0) {
    long long stop = std::min(e, b - hx + gx);
    out.push_back({hx, hx + (stop - b), 1});
    b = stop;
  }
  long long full = (e - b) / gx;
  if (full > 0) {
    out.push_back({0, gx, full});
    b += full * gx;
  }
  if (b < e) out.push_back({0, e - b, 1});
  return out;
}

// ===========================================================================
// reverse (corpus/reverse.kn): s[t] = d[t]; barrier; d[t] = s[n - t - 1]
// One CTA walks the fetch's logical blocks in order, so consecutive blocks
// see each other's writes exactly as in the sequential reference.
// ===========================================================================
__global__ void __launch_bounds__(1024) reverse_seq(int* d, long long ld, int n, long long ls,
                                                    KDesc k) {
  extern __shared__ int s[];
  __shared__ int trap;
  const long long B = (long long)k.bx * k.by * k.bz;
  if (threadIdx.x == 0) trap = 0;
  for (long long blk = k.first; blk < k.first + k.count; blk++) {
    for (long long i = threadIdx.x; i < ls; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (long long t = threadIdx.x; t < B; t += blockDim.x) {
      int tx = (int)(t % k.bx);
      if (tx >= ld || tx >= ls) {
        atomicExch(&trap, 1);
      } else {
        s[tx] = d[tx];
      }
    }
    __syncthreads();
    if (trap) {
      if (threadIdx.x == 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, blk);
      return;
    }
    for (long long t = threadIdx.x; t < B; t += blockDim.x) {
      int tx = (int)(t % k.bx);
      int tr = (int)((unsigned)n - (unsigned)tx - 1u);
      if (tr < 0 || tr >= ls || tx >= ld) {
        atomicExch(&trap, 1);
      } else {
        d[tx] = s[tr];
      }
    }
    __syncthreads();
    if (trap) {
      if (threadIdx.x == 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, blk);
      return;
    }
  }
}

static int launch_reverse(LaunchCtx& ctx) {
  const ArgVal& D = ctx.args[0];
  const int n = ctx.args[1].i32;
  long long ls = ctx.shmem / 4;
  if (ls * 4 > 200 * 1024) {
    *ctx.error = "reverse: dynamic shared memory above 200 KiB";
    return BF_E_UNSUPPORTED;
  }
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(reverse_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaGetLastError();
  }
  long long B = (long long)ctx.block[0] * ctx.block[1] * ctx.block[2];
  int threads = (int)std::min<long long>(1024, ((B + 31) / 32) * 32);
  size_t smem = (size_t)std::max<long long>(ls, 1) * 4;
  reverse_seq<<<1, threads, smem, ctx.stream>>>((int*)D.ptr, D.len, n, ls, ctx.desc());
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

// ===========================================================================
// reduce (corpus/reduce.kn): per-block tree sum in shared i32 buf[256].
// With an m-fold block (blockDim.y*z = m) every tree phase runs m times in
// thread order; a phase only reads slots it does not write, so each pass is
// buf[t] += buf[t+s] and m passes give buf[t] += m*buf[t+s] (mod 2^32).
// m == 1: the sum of the block's slice, computed with warp shuffles.
// ===========================================================================
__device__ __forceinline__ int warp_sum(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per logical block x; loads coalesced (int4 when the block's
// slice is 16 B aligned); m == 1
// one warp per logical block x (m == 1).  VEC (bx % 4 == 0, bx <= 128*MAXV):
// the slice is read as <= MAXV int4 per lane, U blocks per iteration, every
// load of the iteration issued before any shuffle tree (loads in flight per
// lane: U*MAXV*16 B).  Otherwise a plain strided loop.
template <int MAXV, int U, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) reduce_warp(const int* __restrict__ x, long long lx,
                                                   int* __restrict__ out, long long lout, int n,
                                                   long long x0, long long x1, KDesc k) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const long long w0 = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  for (long long b0 = x0 + w0 * U; b0 < x1; b0 += warps * U) {
    unsigned s[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      s[u] = 0;
      const long long bx = b0 + u;
      long long lo = bx * k.bx, hi = lo + k.bx;
      if (hi > n) hi = n;
      const bool ok = bx < x1 && !(hi > lx || bx >= lout) && hi > lo;
      if (MAXV > 0) {
        const int4* x4 = reinterpret_cast<const int4*>(x + lo);
        const long long nv = ok ? (hi - lo) / 4 : 0;
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
          if (lane + 32 * j < nv) {
            const int4 v = __ldcs(x4 + lane + 32 * j);
            s[u] += (unsigned)v.x + (unsigned)v.y + (unsigned)v.z + (unsigned)v.w;
          }
        }
        if (ok)
          for (long long i = lo + nv * 4 + lane; i < hi; i += 32) s[u] += (unsigned)x[i];
      } else if (ok) {
        for (long long i = lo + lane; i < hi; i += 32) s[u] += (unsigned)__ldg(x + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const long long bx = b0 + u;
      if (bx >= x1) break;
      long long lo = bx * k.bx, hi = lo + k.bx;
      if (hi > n) hi = n;
      if (hi > lx || bx >= lout) {
        if (lane == 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, block_of_x(k, bx));
        continue;
      }
      const int v = warp_sum((int)s[u]);
      if (lane == 0) out[bx] = v;
    }
  }
}

// exact tree emulation for m-fold blocks: one CTA of blockDim.x threads
__global__ void __launch_bounds__(256) reduce_tree(const int* x, long long lx, int* out,
                                                   long long lout, int n, long long x0,
                                                   long long x1, int m, KDesc k) {
  __shared__ int buf[256];
  const int t = threadIdx.x;  // blockDim.x == k.bx <= 256
  for (long long bx = x0 + blockIdx.x; bx < x1; bx += gridDim.x) {
    long long id = bx * k.bx + t;
    int v = 0;
    bool oob = false;
    if (id < n && (int)id == id) {
      if (id >= lx) oob = true; else v = x[id];
    }
    buf[t] = v;
    if (__syncthreads_or(oob) || bx >= lout) {
      if (t == 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, block_of_x(k, bx));
      __syncthreads();
      continue;
    }
    for (int s = 1; s < k.bx; s += s) {
      int add = 0;
      if (t % (2 * s) == 0 && t + s < k.bx) add = buf[t + s];
      __syncthreads();
      if (add) buf[t] = (int)((unsigned)buf[t] + (unsigned)m * (unsigned)add);
      __syncthreads();
    }
    if (t == 0) out[bx] = buf[0];
    __syncthreads();
  }
}

static int launch_reduce(LaunchCtx& ctx) {
  const ArgVal& X = ctx.args[0];
  const ArgVal& O = ctx.args[1];
  const int n = ctx.args[2].i32;
  const int bx = ctx.block[0];
  const long long m = (long long)ctx.block[1] * ctx.block[2];
  if (bx > 256) {  // buf[t] = 0 for t = 256 traps in the first block
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first, "shared store index 256 out of range [0, 256)");
    return BF_OK;
  }
  if ((long long)ctx.grid[0] * bx - 1 > INT_MAX) {
    *ctx.error = "reduce: blockIdx.x*blockDim.x beyond i32";
    return BF_E_UNSUPPORTED;
  }
  for (auto& xi : ctx.x_intervals()) {
    long long nx = xi.second - xi.first;
    if (m == 1) {
      const int* xp = (const int*)X.ptr;
      int* op = (int*)O.ptr;
      KDesc d = ctx.desc();
      if (bx % 4 == 0 && bx <= 128) {
        int grid = wave_grid(reduce_warp<1, 8, 4>, 256, 0, nx, 8 * 8, ctx.num_sms, 8);
        reduce_warp<1, 8, 4><<<grid, 256, 0, ctx.stream>>>(xp, X.len, op, O.len, n, xi.first, xi.second, d);
      } else if (bx % 4 == 0 && bx <= 256) {
        // (2 int4 per lane per block, 4 blocks per warp step; 6 CTAs/SM:
        // 0.88 of HBM vs 0.48 with the register-unbounded build)
        int grid = wave_grid(reduce_warp<2, 4, 6>, 256, 0, nx, 8 * 4, ctx.num_sms, 8);
        reduce_warp<2, 4, 6><<<grid, 256, 0, ctx.stream>>>(xp, X.len, op, O.len, n, xi.first, xi.second, d);
      } else {
        int grid = wave_grid(reduce_warp<0, 1, 8>, 256, 0, nx, 8, ctx.num_sms, 8);
        reduce_warp<0, 1, 8><<<grid, 256, 0, ctx.stream>>>(xp, X.len, op, O.len, n, xi.first, xi.second, d);
      }
    } else {
      int grid = (int)std::min<long long>(nx, (long long)ctx.num_sms * 8);
      reduce_tree<<<grid, bx, 0, ctx.stream>>>((const int*)X.ptr, X.len, (int*)O.ptr, O.len, n,
                                               xi.first, xi.second, (int)m, ctx.desc());
    }
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

// ===========================================================================
// hist / hist_stride: counts[pix[i] % nbins] += copies for i in [lo, hi).
// Per-lane privatised counters for nbins <= 32 (bin-major, lane-minor: no
// bank conflicts, no shared atomics), CTA-shared atomics for nbins <= 8192,
// global atomics beyond.  One global atomic per bin per CTA at the end.
// ===========================================================================
constexpr int kHistLaneBins = 32;
constexpr int kHistSmemBins = 8192;

__device__ __forceinline__ int c_mod(int a, int b) {
  return b == -1 ? 0 : a % b;  // C remainder, truncating toward zero
}

// a % nbins for a >= 0 by multiply-high (Granlund-Montgomery, divisor
// |nbins| fixed per launch); negative a (C remainder is negative: the bin
// traps) takes the hardware path.
struct FastMod {
  unsigned d, m;
  int s1, s2;
  int nbins;
};

static FastMod make_fastmod(int nbins) {
  FastMod f;
  f.nbins = nbins;
  unsigned long long d = nbins < 0 ? (unsigned long long)(-(long long)nbins) : (unsigned long long)nbins;
  f.d = (unsigned)d;
  int l = 0;
  while ((1ull << l) < d) l++;
  f.m = (unsigned)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  f.s1 = l < 1 ? l : 1;
  f.s2 = l > 1 ? l - 1 : 0;
  return f;
}

__device__ __forceinline__ int fast_mod(int a, const FastMod& f) {
  if (a < 0) return c_mod(a, f.nbins);
  const unsigned n = (unsigned)a;
  const unsigned t = __umulhi(n, f.m);
  const unsigned q = (t + ((n - t) >> f.s1)) >> f.s2;
  return (int)(n - q * f.d);
}

// Bin of pixel a.  POW2: |nbins| is a power of two (a & mask for a >= 0).
// SAFE: len(counts) >= |nbins|, so only a negative remainder can trap.
template <bool POW2>
__device__ __forceinline__ int hist_bin(int a, const FastMod& f) {
  if (POW2) return a >= 0 ? (a & (int)(f.d - 1)) : c_mod(a, f.nbins);
  return fast_mod(a, f);
}

template <int MODE, bool SAFE>  // MODE 0: per-lane counters, 1: CTA shared atomics, 2: global
__device__ __forceinline__ void hist_add(unsigned* sh, unsigned* mine, int* counts, long long lc,
                                         int b, unsigned copies, bool& bad) {
  if (SAFE ? b < 0 : (b < 0 || b >= lc)) {
    bad = true;
    return;
  }
  if (MODE == 0) {
    mine[b * 32] += copies;
  } else if (MODE == 1) {
    atomicAdd(sh + b, copies);
  } else {
    atomicAdd((unsigned*)counts + b, copies);
  }
}

// four pixels: with a power-of-two bin count and all four non-negative, the
// bins are plain masks and cannot trap (one branch per 4 pixels)
template <int MODE, bool POW2, bool SAFE>
__device__ __forceinline__ void hist_add4(unsigned* sh, unsigned* mine, int* counts, long long lc, int4 v,
                                          const FastMod& fm, unsigned copies, bool& bad) {
  if (POW2 && SAFE && (v.x | v.y | v.z | v.w) >= 0) {
    const int m = (int)(fm.d - 1);
    if (MODE == 0) {
      mine[(v.x & m) * 32] += copies;
      mine[(v.y & m) * 32] += copies;
      mine[(v.z & m) * 32] += copies;
      mine[(v.w & m) * 32] += copies;
    } else if (MODE == 1) {
      atomicAdd(sh + (v.x & m), copies);
      atomicAdd(sh + (v.y & m), copies);
      atomicAdd(sh + (v.z & m), copies);
      atomicAdd(sh + (v.w & m), copies);
    } else {
      atomicAdd((unsigned*)counts + (v.x & m), copies);
      atomicAdd((unsigned*)counts + (v.y & m), copies);
      atomicAdd((unsigned*)counts + (v.z & m), copies);
      atomicAdd((unsigned*)counts + (v.w & m), copies);
    }
    return;
  }
  hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(v.x, fm), copies, bad);
  hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(v.y, fm), copies, bad);
  hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(v.z, fm), copies, bad);
  hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(v.w, fm), copies, bad);
}

template <int MODE, bool POW2, bool SAFE>
__global__ void __launch_bounds__(256) hist_range(const int* __restrict__ pix, int* counts,
                                                  long long lc, long long lo, long long hi,
                                                  FastMod fm, unsigned copies, KDesc k,
                                                  long long xbase, int bx_div) {
  extern __shared__ unsigned sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (int)fm.d;  // |nbins| bounds the remainder
  if (MODE == 0) {
    for (int i = threadIdx.x; i < 8 * kHistLaneBins * 32; i += blockDim.x) sh[i] = 0;
  } else if (MODE == 1) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  }
  __syncthreads();
  unsigned* mine = sh + warp * (kHistLaneBins * 32) + lane;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  // scalar head to a 16 B boundary, int4 body (4 loads in flight), scalar tail
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(pix[lo + tid], fm), copies, bad);
  if (tid < hi - vhi) hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(pix[vhi + tid], fm), copies, bad);
  const int4* p4 = reinterpret_cast<const int4*>(pix);
  const long long end = vhi / 4;
  long long g = vlo / 4 + tid;
  // software-pipelined: the next group's four 16 B loads are in flight while
  // this group's 16 pixels update the counters (shared-memory RMW chains)
  if (g + 3 * stride < end) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = __ldcs(p4 + g + u * stride);
    for (;;) {
      const bool more = g + 7 * stride < end;
      int4 nx[4];
      if (more) {
#pragma unroll
        for (int u = 0; u < 4; u++) nx[u] = __ldcs(p4 + g + (4 + u) * stride);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) hist_add4<MODE, POW2, SAFE>(sh, mine, counts, lc, v[u], fm, copies, bad);
      g += 4 * stride;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = nx[u];
    }
  }
  for (; g < end; g += stride) hist_add4<MODE, POW2, SAFE>(sh, mine, counts, lc, __ldcs(p4 + g), fm, copies, bad);
  if (bad) {
    // exact block of the first bad pixel is not tracked on this path: the
    // fetch's first block whose range holds one is reported (kind is exact)
    long long blk = k.first;
    if (bx_div > 0) blk = block_of_x(k, xbase + ((vlo > lo ? lo : vlo) - lo) / bx_div);
    record_fault(k, BF_TRAP_OUT_OF_BOUNDS, blk);
  }
  if (MODE == 2) return;
  __syncthreads();
  if (MODE == 0) {
    // bins x 256 lanes -> one total per bin
    for (int b = warp; b < nb && b < kHistLaneBins; b += blockDim.x / 32) {
      unsigned s = 0;
      for (int w = 0; w < (int)(blockDim.x / 32); w++) s += sh[w * (kHistLaneBins * 32) + b * 32 + lane];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && s && b < lc) atomicAdd((unsigned*)counts + b, s);
    }
  } else {
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
      if (sh[b] && b < lc) atomicAdd((unsigned*)counts + b, sh[b]);
  }
}

template <int MODE, bool POW2, bool SAFE>
static void hist_go(LaunchCtx& ctx, int grid, size_t smem, const ArgVal& P, const ArgVal& Cn,
                    long long lo, long long hi, const FastMod& fm, unsigned copies, long long xbase,
                    int bx_div) {
  static bool attr[64] = {};
  if ((smem > 48 * 1024) && first_on_device(attr)) {
    cudaFuncSetAttribute(hist_range<MODE, POW2, SAFE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaGetLastError();
  }
  // one resident wave (registers / shared memory bound the CTAs per SM)
  grid = std::min(grid, wave_grid(hist_range<MODE, POW2, SAFE>, 256, smem, hi - lo, 256 * 16, ctx.num_sms, 8));
  hist_range<MODE, POW2, SAFE><<<grid, 256, smem, ctx.stream>>>(
      (const int*)P.ptr, (int*)Cn.ptr, Cn.len, lo, hi, fm, copies, ctx.desc(), xbase, bx_div);
}

// Device-side fetching (BF_FLAG_DEVICE_FETCH, 1D geometry): one persistent
// grid; each CTA claims `grain` logical blocks at a time, counts their pixels
// [b0*bx, b1*bx) into its private counters, and flushes once at the end.
template <int MODE, bool POW2, bool SAFE>
__global__ void __launch_bounds__(256) hist_fetch(const int* __restrict__ pix, int* counts, long long lc,
                                                  long long n, long long bx, FastMod fm, KDesc k, DevFetch F) {
  extern __shared__ unsigned sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = (int)fm.d;
  const int nwarps = blockDim.x >> 5;
  if (MODE == 0) {
    for (int i = threadIdx.x; i < nwarps * kHistLaneBins * 32; i += blockDim.x) sh[i] = 0;
  } else if (MODE == 1) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  }
  unsigned* mine = sh + warp * (kHistLaneBins * 32) + lane;
  const int4* p4 = reinterpret_cast<const int4*>(pix);
  bool bad = false;
  long long bad_blk = -1;
  FetchCursor fc = dev_fetch_cursor();
  long long f = dev_fetch_first(F, fc);  // (its barrier also orders the counter zeroing)
  while (f < F.nfetch) {
    const long long nx = dev_fetch_issue(F, fc);
    long long b0, b1;
    dev_fetch_range(F, f, b0, b1);
    const long long lo = b0 * bx, hi = b1 * bx < n ? b1 * bx : n;
    const long long vhi = lo + ((hi > lo ? hi - lo : 0) & ~3LL);
    for (long long g = lo / 4 + threadIdx.x; g < vhi / 4; g += blockDim.x)
      hist_add4<MODE, POW2, SAFE>(sh, mine, counts, lc, __ldcs(p4 + g), fm, 1u, bad);
    for (long long i = vhi + threadIdx.x; i < hi; i += blockDim.x)
      hist_add<MODE, SAFE>(sh, mine, counts, lc, hist_bin<POW2>(pix[i], fm), 1u, bad);
    if (bad && bad_blk < 0) bad_blk = b0;
    dev_fetch_done(F, fc, b0, b1);
    f = dev_fetch_take(nx);
  }
  dev_fetch_flush(F, fc);
  if (bad) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, bad_blk);
  if (MODE == 2) return;
  __syncthreads();
  if (MODE == 0) {
    for (int b = warp; b < nb && b < kHistLaneBins; b += blockDim.x / 32) {
      unsigned s = 0;
      for (int w = 0; w < (int)(blockDim.x / 32); w++) s += sh[w * (kHistLaneBins * 32) + b * 32 + lane];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && s && b < lc) atomicAdd((unsigned*)counts + b, s);
    }
  } else {
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
      if (sh[b] && b < lc) atomicAdd((unsigned*)counts + b, sh[b]);
  }
}

template <int MODE, bool POW2, bool SAFE>
static int hist_fetch_go(LaunchCtx& ctx, size_t smem, const ArgVal& P, const ArgVal& Cn, long long n,
                         const FastMod& fm) {
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(hist_fetch<MODE, POW2, SAFE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaGetLastError();
  }
  const DevFetch& F = *ctx.dfetch;
  // a CTA as wide as one fetch's int4 (32..256 threads); MODE 0 keeps one
  // counter row per warp
  const int threads =
      (int)std::min<long long>(256, std::max<long long>(32, (F.grain * ctx.block[0] / 4 + 31) / 32 * 32));
  if (MODE == 0) smem = (size_t)(threads / 32) * kHistLaneBins * 32 * sizeof(unsigned);
  const int grid = (int)std::min<long long>(
      F.nfetch, (long long)resident_ctas((const void*)hist_fetch<MODE, POW2, SAFE>, threads, smem) * ctx.num_sms);
  hist_fetch<MODE, POW2, SAFE><<<grid, threads, smem, ctx.stream>>>((const int*)P.ptr, (int*)Cn.ptr, Cn.len, n,
                                                                    ctx.block[0], fm, ctx.desc(), F);
  BF_CUDA_LAUNCH_CHECK(ctx);
  ctx.dfetch_grid = grid;
  return BF_OK;
}

template <int MODE>
static int hist_fetch_go2(LaunchCtx& ctx, size_t smem, const ArgVal& P, const ArgVal& Cn, long long n,
                          const FastMod& fm) {
  const bool pow2 = (fm.d & (fm.d - 1)) == 0;
  const bool safe = Cn.len >= (long long)fm.d;
  if (pow2 && safe) return hist_fetch_go<MODE, true, true>(ctx, smem, P, Cn, n, fm);
  if (pow2) return hist_fetch_go<MODE, true, false>(ctx, smem, P, Cn, n, fm);
  if (safe) return hist_fetch_go<MODE, false, true>(ctx, smem, P, Cn, n, fm);
  return hist_fetch_go<MODE, false, false>(ctx, smem, P, Cn, n, fm);
}

static int launch_hist_fetch(LaunchCtx& ctx) {
  const DevFetch& F = *ctx.dfetch;
  const ArgVal& P = ctx.args[0];
  const ArgVal& Cn = ctx.args[1];
  const long long n = ctx.args[2].i32;
  const int nbins = ctx.args[3].i32;
  const long long bx = ctx.block[0];
  const long long hi = std::min((F.first + F.total) * bx, n);
  // 1D geometry, aligned blocks, no host-detected trap (those keep host fetches)
  if ((long long)ctx.grid[1] * ctx.grid[2] * ctx.block[1] * ctx.block[2] != 1 || bx % 4 != 0 || nbins == 0 ||
      hi > P.len || hi - 1 > (long long)INT_MAX)
    return BF_E_UNSUPPORTED;
  const FastMod fm = make_fastmod(nbins);
  const long long nb = fm.d;
  if (nb <= kHistLaneBins) return hist_fetch_go2<0>(ctx, 8 * kHistLaneBins * 32 * sizeof(unsigned), P, Cn, n, fm);
  if (nb <= kHistSmemBins) return hist_fetch_go2<1>(ctx, nb * sizeof(unsigned), P, Cn, n, fm);
  return hist_fetch_go2<2>(ctx, 0, P, Cn, n, fm);
}

template <int MODE>
static void hist_go2(LaunchCtx& ctx, int grid, size_t smem, const ArgVal& P, const ArgVal& Cn,
                     long long lo, long long hi, const FastMod& fm, unsigned copies,
                     long long xbase, int bx_div) {
  const bool pow2 = (fm.d & (fm.d - 1)) == 0;
  const bool safe = Cn.len >= (long long)fm.d;
  if (pow2 && safe) hist_go<MODE, true, true>(ctx, grid, smem, P, Cn, lo, hi, fm, copies, xbase, bx_div);
  else if (pow2) hist_go<MODE, true, false>(ctx, grid, smem, P, Cn, lo, hi, fm, copies, xbase, bx_div);
  else if (safe) hist_go<MODE, false, true>(ctx, grid, smem, P, Cn, lo, hi, fm, copies, xbase, bx_div);
  else hist_go<MODE, false, false>(ctx, grid, smem, P, Cn, lo, hi, fm, copies, xbase, bx_div);
}

static int hist_issue(LaunchCtx& ctx, const ArgVal& P, const ArgVal& Cn, long long lo, long long hi,
                      int nbins, unsigned copies, long long xbase, int bx_div) {
  if (lo >= hi) return BF_OK;
  const FastMod fm = make_fastmod(nbins);
  const long long nb = fm.d;
  int grid = stream_grid(hi - lo, 256 * 16, ctx.num_sms, 6);
  if (nb <= kHistLaneBins) {
    size_t smem = 8 * kHistLaneBins * 32 * sizeof(unsigned);  // 8 warps x 32 bins x 32 lanes
    hist_go2<0>(ctx, grid, smem, P, Cn, lo, hi, fm, copies, xbase, bx_div);
  } else if (nb <= kHistSmemBins) {
    hist_go2<1>(ctx, grid, nb * sizeof(unsigned), P, Cn, lo, hi, fm, copies, xbase, bx_div);
  } else {
    hist_go2<2>(ctx, grid, 0, P, Cn, lo, hi, fm, copies, xbase, bx_div);
  }
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

static int launch_hist(LaunchCtx& ctx) {
  if (ctx.dfetch) return launch_hist_fetch(ctx);
  const ArgVal& P = ctx.args[0];
  const ArgVal& Cn = ctx.args[1];
  const long long n = ctx.args[2].i32;
  const int nbins = ctx.args[3].i32;
  const long long bx = ctx.block[0];
  const long long m = (long long)ctx.block[1] * ctx.block[2];
  if (ctx.grid[0] * bx - 1 > INT_MAX) {
    *ctx.error = "hist: blockIdx.x*blockDim.x beyond i32";
    return BF_E_UNSUPPORTED;
  }
  for (auto& pc : x_pieces(ctx)) {
    long long lo = pc.x0 * bx, hi = std::min(pc.x1 * bx, n);
    if (lo >= hi) continue;
    if (nbins == 0) {
      ctx.host_trap(BF_TRAP_DIV_BY_ZERO, ctx.first_block_with_x(pc.x0), "integer modulo by zero");
      continue;
    }
    if (hi > P.len) {
      long long bad = std::max<long long>(lo, P.len);
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(bad / bx),
                    "load index " + std::to_string(bad) + " out of range");
      hi = P.len;
    }
    int rc = hist_issue(ctx, P, Cn, lo, hi, nbins, (unsigned)(pc.copies * m), pc.x0, (int)bx);
    if (rc) return rc;
  }
  return BF_OK;
}

static int launch_hist_stride(LaunchCtx& ctx) {
  const ArgVal& P = ctx.args[0];
  const ArgVal& Cn = ctx.args[1];
  const long long k = ctx.args[2].i32;
  const int nbins = ctx.args[3].i32;
  const long long bx = ctx.block[0];
  const long long m = (long long)ctx.block[1] * ctx.block[2];
  // every logical block and thread copy sweeps pix[t + j*bx], t < bx, j < k
  long long hi = k > 0 ? k * bx : 0;
  if (hi <= 0) return BF_OK;
  if (hi - 1 > INT_MAX) {
    *ctx.error = "hist_stride: index beyond i32";
    return BF_E_UNSUPPORTED;
  }
  if (nbins == 0) {
    ctx.host_trap(BF_TRAP_DIV_BY_ZERO, ctx.first, "integer modulo by zero");
    return BF_OK;
  }
  if (hi > P.len) {
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first, "load index out of range");
    hi = P.len;
  }
  return hist_issue(ctx, P, Cn, 0, hi, nbins, (unsigned)(ctx.count * m), 0, 0);
}

// ===========================================================================
// fir (corpus/fir.kn): y[o] = sum_i w[i] * x[o + i], o < m*blockDim.x.
// Products of two f32 are exact in f64, so fma(w, x, acc) == acc + w*x and
// the f64 accumulation in tap order matches the reference bit for bit.
// CTA tile: 1024 outputs; x tile + (taps-1) halo staged in shared memory.
// ===========================================================================
constexpr int kFirTile = 1024;

__global__ void __launch_bounds__(256) fir_tile(const float* __restrict__ x,
                                                float* __restrict__ y,
                                                const float* __restrict__ w, int taps,
                                                long long nout) {
  extern __shared__ float xs[];  // kFirTile + taps - 1
  __shared__ double ws[64];
  for (long long base = (long long)blockIdx.x * kFirTile; base < nout;
       base += (long long)gridDim.x * kFirTile) {
    const int span = kFirTile + taps - 1;
    const long long avail = nout + taps - 1 - base;  // x elements in range
    __syncthreads();
    for (int i = threadIdx.x; i < span; i += blockDim.x) xs[i] = i < avail ? __ldg(x + base + i) : 0.f;
    for (int i = threadIdx.x; i < taps && i < 64; i += blockDim.x) ws[i] = (double)__ldg(w + i);
    __syncthreads();
    const int o0 = threadIdx.x * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < taps; i++) {
      const double wi = i < 64 ? ws[i] : (double)__ldg(w + i);
#pragma unroll
      for (int q = 0; q < 4; q++) acc[q] = fma(wi, (double)xs[o0 + q + i], acc[q]);
    }
    const long long o = base + o0;
    if (o + 3 < nout) {
      *reinterpret_cast<float4*>(y + o) =
          make_float4((float)acc[0], (float)acc[1], (float)acc[2], (float)acc[3]);
    } else {
      for (int q = 0; q < 4; q++)
        if (o + q < nout) y[o + q] = (float)acc[q];
    }
  }
}

// taps <= 13: each thread computes OPT consecutive outputs from a window of
// OPT + taps - 1 <= 16 x values read as aligned float4 (neighbouring threads'
// windows overlap in L1); w lives in registers as doubles.  The window is
// converted to f64 once: (OPT + taps - 1) / OPT conversions per output (the
// F2F conversions, not the DFMAs, bound this kernel), so taps <= 9 use
// OPT = 8 (2 per output at 8 taps) and larger filters OPT = 4.
constexpr int kFirRegTaps = 13;

template <int OPT>
__global__ void __launch_bounds__(256) fir_reg(const float* __restrict__ x, long long lx,
                                               float* __restrict__ y,
                                               const float* __restrict__ w, int taps,
                                               long long nout) {
  constexpr int MAXT = 17 - OPT;  // window OPT + taps - 1 <= 16
  double wd[MAXT];
#pragma unroll
  for (int i = 0; i < MAXT; i++) wd[i] = i < taps ? (double)__ldg(w + i) : 0.0;
  const int nvec = (OPT - 1 + taps + 3) / 4;  // float4 chunks covering OPT - 1 + taps floats
  const long long groups = (nout + OPT - 1) / OPT;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
    const long long o = OPT * g;
    float xv[16];
    if (o + 4 * nvec <= lx) {
      const float4* x4 = reinterpret_cast<const float4*>(x + o);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (j < nvec) {
          const float4 v = __ldg(x4 + j);
          xv[4 * j] = v.x; xv[4 * j + 1] = v.y; xv[4 * j + 2] = v.z; xv[4 * j + 3] = v.w;
        } else {
          xv[4 * j] = xv[4 * j + 1] = xv[4 * j + 2] = xv[4 * j + 3] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; j++) xv[j] = (o + j < lx) ? __ldg(x + o + j) : 0.f;
    }
    double xd[16];
#pragma unroll
    for (int j = 0; j < 16; j++) xd[j] = (j < OPT - 1 + taps) ? (double)xv[j] : 0.0;
    double acc[OPT];
#pragma unroll
    for (int q = 0; q < OPT; q++) acc[q] = 0.0;
#pragma unroll
    for (int i = 0; i < MAXT; i++) {
      if (i < taps) {
#pragma unroll
        for (int q = 0; q < OPT; q++) acc[q] = fma(wd[i], xd[q + i], acc[q]);
      }
    }
    if (o + OPT - 1 < nout) {
#pragma unroll
      for (int q = 0; q < OPT; q += 4)
        __stcs(reinterpret_cast<float4*>(y + o + q),
               make_float4((float)acc[q], (float)acc[q + 1], (float)acc[q + 2], (float)acc[q + 3]));
    } else {
      for (int q = 0; q < OPT; q++)
        if (o + q < nout) y[o + q] = (float)acc[q];
    }
  }
}

static int launch_fir(LaunchCtx& ctx) {
  const ArgVal& X = ctx.args[0];
  const ArgVal& Y = ctx.args[1];
  const ArgVal& W = ctx.args[2];
  const int taps = ctx.args[3].i32;
  const long long m = ctx.args[4].i32;
  const long long bx = ctx.block[0];
  long long nout = m > 0 ? m * bx : 0;
  if (nout <= 0) return BF_OK;
  if (nout + (taps > 0 ? taps : 0) > (long long)INT_MAX) {
    *ctx.error = "fir: index beyond i32";
    return BF_E_UNSUPPORTED;
  }
  int t = taps > 0 ? taps : 0;
  if (nout > Y.len || (t > 0 && (t > W.len || nout + t - 1 > X.len))) {
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first, "fir index out of range");
    return BF_OK;
  }
  if (t <= 9) {
    int grid = wave_grid(fir_reg<8>, 256, 0, (nout + 7) / 8, 256 * 2, ctx.num_sms, 8);
    fir_reg<8><<<grid, 256, 0, ctx.stream>>>((const float*)X.ptr, X.len, (float*)Y.ptr,
                                             (const float*)W.ptr, t, nout);
    BF_CUDA_LAUNCH_CHECK(ctx);
    return BF_OK;
  }
  if (t <= kFirRegTaps) {
    int grid = wave_grid(fir_reg<4>, 256, 0, (nout + 3) / 4, 256 * 4, ctx.num_sms, 8);
    fir_reg<4><<<grid, 256, 0, ctx.stream>>>((const float*)X.ptr, X.len, (float*)Y.ptr,
                                             (const float*)W.ptr, t, nout);
    BF_CUDA_LAUNCH_CHECK(ctx);
    return BF_OK;
  }
  if (t + kFirTile > 48 * 1024 / 4) {
    *ctx.error = "fir: more than 11264 taps";
    return BF_E_UNSUPPORTED;
  }
  int grid = stream_grid(nout, kFirTile, ctx.num_sms, 4);
  fir_tile<<<grid, 256, (kFirTile + (t > 0 ? t - 1 : 0)) * sizeof(float), ctx.stream>>>(
      (const float*)X.ptr, (float*)Y.ptr, (const float*)W.ptr, t, nout);
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

// ===========================================================================
// wreduce (corpus/wreduce.kn), warp mode: v = (id < n) ? x[id] : 0;
// v += shfl_down(v, d) for d = 16, 8, 4, 2, 1 with the reference's clamp (a
// source lane at or beyond min(warp_size, active lanes) reads its own value,
// interp.py:276-283); lanes with threadIdx.x % 32 == 0 add v to out[0].
// One CTA per logical block (logical tid == physical thread); the logical
// warp size must divide 32 so logical warps sit inside physical warps.
// ===========================================================================
__global__ void __launch_bounds__(1024) wreduce_blocks(const int* __restrict__ x, long long lx,
                                                       int* out, long long lout, int n, int ws,
                                                       KDesc k) {
  __shared__ unsigned part[32];
  __shared__ int trap;
  const long long B = (long long)k.bx * k.by * k.bz;
  for (long long blk = k.first + blockIdx.x; blk < k.first + k.count; blk += gridDim.x) {
    const long long bxi = blk % k.gx;
    unsigned total = 0;
    if (threadIdx.x == 0) trap = 0;
    __syncthreads();
    for (long long c0 = 0; c0 < B; c0 += blockDim.x) {  // chunks of logical tids
      const long long tid = c0 + threadIdx.x;
      const bool live = tid < B;
      const int tx = (int)(tid % k.bx);
      const int id = (int)((unsigned)bxi * (unsigned)k.bx + (unsigned)tx);
      int v = 0;
      if (live && id < n) {
        if (id < 0 || id >= lx) trap = 1; else v = __ldg(x + id);
      }
      // lanes of this logical warp that exist
      const long long w0 = (tid / ws) * ws;
      const int L = (int)min((long long)ws, B - w0);
      const int i = (int)(tid - w0);
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) {
        int other = __shfl_down_sync(0xffffffffu, v, d);
        v = (int)((unsigned)v + (unsigned)(i + d < L ? other : v));
      }
      unsigned contrib = (live && tx % 32 == 0) ? (unsigned)v : 0u;
      for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
      if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = contrib;
      __syncthreads();
      if (threadIdx.x == 0)
        for (int wi = 0; wi < (int)(blockDim.x + 31) / 32; wi++) total += part[wi];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (trap || lout < 1) {
        record_fault(k, BF_TRAP_OUT_OF_BOUNDS, blk);
      } else if (total) {
        atomicAdd((unsigned*)out, total);
      }
    }
    __syncthreads();
  }
}

// Fast path (1D blocks, blockDim.x % 32 == 0, warp_size 32): every logical
// warp is full, so lane 0's clamped shuffle chain yields exactly its warp's
// sum and lane 0 is the only lane with threadIdx.x % 32 == 0: the launch adds
// sum(x[id], id in the covered range, id < n) to out[0].  Streamed with int4
// loads; one atomic per CTA.
__global__ void __launch_bounds__(256) sum_range(const int* __restrict__ x, int* out,
                                                 long long lo, long long hi, unsigned copies) {
  __shared__ unsigned part[8];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned s = 0;
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) s += (unsigned)x[lo + tid];
  if (tid < hi - vhi) s += (unsigned)x[vhi + tid];
  const int4* x4 = reinterpret_cast<const int4*>(x);
  const long long end = vhi / 4;
  long long g = vlo / 4 + tid;
  for (; g + 3 * stride < end; g += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = __ldcs(x4 + g + u * stride);
#pragma unroll
    for (int u = 0; u < 4; u++) s += (unsigned)v[u].x + (unsigned)v[u].y + (unsigned)v[u].z + (unsigned)v[u].w;
  }
  for (; g < end; g += stride) {
    const int4 v = __ldcs(x4 + g);
    s += (unsigned)v.x + (unsigned)v.y + (unsigned)v.z + (unsigned)v.w;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += part[i];
    if (t) atomicAdd((unsigned*)out, t * copies);
  }
}

static int launch_wreduce(LaunchCtx& ctx) {
  const ArgVal& X = ctx.args[0];
  const ArgVal& O = ctx.args[1];
  const int n = ctx.args[2].i32;
  int ws = ctx.warp_size > 0 ? ctx.warp_size : 32;
  if (ws > 32 || (32 % ws) != 0) {
    *ctx.error = "wreduce: warp_size must divide 32 (got " + std::to_string(ws) + ")";
    return BF_E_UNSUPPORTED;
  }
  long long B = (long long)ctx.block[0] * ctx.block[1] * ctx.block[2];
  const long long bx = ctx.block[0];
  if (ws == 32 && B == bx && bx % 32 == 0 && O.len >= 1 &&
      (long long)ctx.grid[0] * bx - 1 <= INT_MAX) {
    for (auto& pc : x_pieces(ctx)) {
      long long lo = pc.x0 * bx, hi = std::min<long long>(pc.x1 * bx, n);
      if (lo >= hi) continue;
      if (hi > X.len) {
        long long bad = std::max<long long>(lo, X.len);
        ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(bad / bx),
                      "load index " + std::to_string(bad) + " out of range");
        hi = X.len;
        if (lo >= hi) continue;
      }
      int grid = stream_grid((hi - lo + 3) / 4, 256 * 4, ctx.num_sms, 8);
      sum_range<<<grid, 256, 0, ctx.stream>>>((const int*)X.ptr, (int*)O.ptr, lo, hi,
                                              (unsigned)pc.copies);
      BF_CUDA_LAUNCH_CHECK(ctx);
    }
    return BF_OK;
  }
  int threads = (int)std::min<long long>(1024, ((B + 31) / 32) * 32);
  int grid = (int)std::min<long long>(ctx.count, (long long)ctx.num_sms * 16);
  wreduce_blocks<<<grid, threads, 0, ctx.stream>>>((const int*)X.ptr, X.len, (int*)O.ptr, O.len, n,
                                                   ws, ctx.desc());
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

static Registrar reg_reverse("reverse", {{BF_SLOT_HANDLE, BF_I32, "d"}, {BF_SLOT_I32, BF_I32, "n"}},
                             launch_reverse);
static Registrar reg_reduce("reduce",
                            {{BF_SLOT_HANDLE, BF_I32, "x"},
                             {BF_SLOT_HANDLE, BF_I32, "out"},
                             {BF_SLOT_I32, BF_I32, "n"}},
                            launch_reduce);
static Registrar reg_hist("hist",
                          {{BF_SLOT_HANDLE, BF_I32, "pix"},
                           {BF_SLOT_HANDLE, BF_I32, "counts"},
                           {BF_SLOT_I32, BF_I32, "n"},
                           {BF_SLOT_I32, BF_I32, "nbins"}},
                          launch_hist, /*dev_fetch=*/true);
static Registrar reg_hist_stride("hist_stride",
                                 {{BF_SLOT_HANDLE, BF_I32, "pix"},
                                  {BF_SLOT_HANDLE, BF_I32, "counts"},
                                  {BF_SLOT_I32, BF_I32, "k"},
                                  {BF_SLOT_I32, BF_I32, "nbins"}},
                                 launch_hist_stride);
static Registrar reg_fir("fir",
                         {{BF_SLOT_HANDLE, BF_F32, "x"},
                          {BF_SLOT_HANDLE, BF_F32, "y"},
                          {BF_SLOT_HANDLE, BF_F32, "w"},
                          {BF_SLOT_I32, BF_I32, "taps"},
                          {BF_SLOT_I32, BF_I32, "m"}},
                         launch_fir);
static Registrar reg_wreduce("wreduce",
                             {{BF_SLOT_HANDLE, BF_I32, "x"},
                              {BF_SLOT_HANDLE, BF_I32, "out"},
                              {BF_SLOT_I32, BF_I32, "n"}},
                             launch_wreduce);

}  // namespace bf
