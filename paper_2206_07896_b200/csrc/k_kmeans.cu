// kmeans — paper_2206_07896_b200/kernels/kmeans.kn (Rodinia kmeansPoint plus
// the centroid accumulation).
//
// Membership is bit-exact: the squared distance of point p to centroid c is
// accumulated in f64 in feature order with separately rounded sub/mul/add
// (interp.py:58-91), and the first strictly smaller distance wins (`c == 0 ||
// dist < bestd`), so ties keep the lowest cluster index.  Counts are exact
// (integer atomics).  The f32 sums are accumulated per CTA in shared memory
// and flushed with one global atomic per (cluster, feature): a different
// summation order than the reference's sequential f32 adds, so sums match
// within a stated tolerance only (tests: 1e-4 relative).
//
// B200 mapping: features are feature-major (f[l*npts + p]) so a warp's loads
// of one feature are coalesced; each thread keeps its point's <= 32 features
// in registers; centroids live in shared memory as doubles (broadcast reads).
// Bound: FP64 (3 DP ops per point x cluster x feature), see DESIGN.md.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <climits>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

constexpr int kKmMaxF = 32;

template <bool REG>
__global__ void __launch_bounds__(256) kmeans_assign(const float* __restrict__ f,
                                                     const float* __restrict__ cent,
                                                     int* __restrict__ member, float* sums,
                                                     int* counts, int npts, int nf, int k,
                                                     long long lo, long long hi) {
  extern __shared__ double cs[];  // [kc*nf] centroids, then [kc*nf] f32 sums, [kc] counts
  const int kc = k > 0 ? k : 1;
  float* ssum = reinterpret_cast<float*>(cs + (size_t)kc * nf);
  int* scnt = reinterpret_cast<int*>(ssum + (size_t)kc * nf);
  for (int i = threadIdx.x; i < k * nf; i += blockDim.x) cs[i] = (double)cent[i];
  for (int i = threadIdx.x; i < kc * nf; i += blockDim.x) ssum[i] = 0.f;
  for (int i = threadIdx.x; i < kc; i += blockDim.x) scnt[i] = 0;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < hi; p += stride) {
    float fv[REG ? kKmMaxF : 1];
    if (REG) {
#pragma unroll
      for (int l = 0; l < kKmMaxF; l++)
        if (l < nf) fv[l] = __ldcs(f + (long long)l * npts + p);
    }
    int best = 0;
    double bestd = 0.0;
    for (int c = 0; c < k; c++) {
      const double* cc = cs + c * nf;
      double dist = 0.0;
      if (REG) {
#pragma unroll
        for (int l = 0; l < kKmMaxF; l++) {
          if (l < nf) {
            const double diff = dsub((double)fv[l], cc[l]);
            dist = dadd(dist, dmul(diff, diff));
          }
        }
      } else {
        for (int l = 0; l < nf; l++) {
          const double diff = dsub((double)__ldg(f + (long long)l * npts + p), cc[l]);
          dist = dadd(dist, dmul(diff, diff));
        }
      }
      if (c == 0 || dist < bestd) {
        bestd = dist;
        best = c;
      }
    }
    member[p] = best;
    atomicAdd(scnt + best, 1);
    if (REG) {
#pragma unroll
      for (int l = 0; l < kKmMaxF; l++)
        if (l < nf) atomicAdd(ssum + best * nf + l, fv[l]);
    } else {
      for (int l = 0; l < nf; l++) atomicAdd(ssum + best * nf + l, __ldg(f + (long long)l * npts + p));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kc; i += blockDim.x)
    if (scnt[i]) atomicAdd(counts + i, scnt[i]);
  for (int i = threadIdx.x; i < kc * nf; i += blockDim.x)
    if (ssum[i] != 0.f) atomicAdd(sums + i, ssum[i]);
}

// Fast path (nf <= 32, k*nf <= 1024): membership by an f32 screen with an
// exact f64 re-check of near-ties, sums by a warp transpose.
//
// Screen: for the argmin only s_c = |c|^2 - 2 f.c matters (|f|^2 is common).
// In f32 with FMA, |s_c(f32) - s_c| <= E_c = (nf+4) 2^-22 (2 |f| |c| + |c|^2)
// (dot-product error bound with Cauchy-Schwarz, plus the rounding of |c|^2),
// orders of magnitude above the reference's own f64 rounding.  If the
// screen's argmin i1 satisfies  s_c - E_c > s_i1 + E_i1  for every other c,
// the reference's f64 scan (`c == 0 || dist < bestd`) returns i1 too;
// otherwise (near-ties, exact ties, non-finite values) the point is re-scanned
// with the reference's exact f64 recurrence.  Membership stays bit-exact.
// Sums: each warp transposes its 32 points x nf features through shared
// memory so lane j owns feature j, then adds point q's feature j into its
// private per-warp row for cluster best_q (no atomics, no bank conflicts).
constexpr int kKmWarps = 8;

// NF: compile-time feature count (4, 8, 16 or 32; 0 = dynamic nf <= 32).
// Centroid rows are read as 16 B broadcasts (one LDS.128 per 4 FMAs).
template <int NF>
__global__ void __launch_bounds__(256, 2) kmeans_fast(const float* __restrict__ f,
                                                   const float* __restrict__ cent,
                                                   int* __restrict__ member, float* sums,
                                                   int* counts, int npts, int nf_dyn, int k,
                                                   long long lo, long long hi) {
  const int nf = NF ? NF : nf_dyn;
  constexpr int FM = NF ? NF : 32;  // register array extent
  extern __shared__ float smf[];
  const int kc = k > 0 ? k : 1;
  float* cf = smf;                         // [kc*nf] centroids (f32 as stored)
  float* cA = cf + kc * nf;                // [kc] error slope  (x |f|)
  float* cB = cA + kc;                     // [kc] error offset
  float* cn2 = cB + kc;                    // [kc] |c|^2 in f32
  float* tile = cn2 + kc;                  // [8][32][33] transpose tiles
  float* wsum = tile + kKmWarps * 32 * 33; // [8][kc*nf] per-warp sums
  int* cnt = reinterpret_cast<int*>(wsum + kKmWarps * kc * nf);  // [kc]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k * nf; i += blockDim.x) cf[i] = cent[i];
  for (int i = threadIdx.x; i < kKmWarps * kc * nf; i += blockDim.x) wsum[i] = 0.f;
  for (int i = threadIdx.x; i < kc; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const float errk = (float)(nf + 4) * 2.384185791015625e-7f * 1.01f;  // (nf+4) 2^-22, +1 %
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    float n2 = 0.f;
    for (int l = 0; l < nf; l++) n2 = fmaf(cf[c * nf + l], cf[c * nf + l], n2);
    cn2[c] = n2;
    cA[c] = errk * 2.f * sqrtf(n2) * 1.01f;
    cB[c] = errk * n2 + 1e-30f;
  }
  __syncthreads();
  float* mytile = tile + warp * 32 * 33;
  float* mysum = wsum + warp * kc * nf;
  const long long wstride = (long long)gridDim.x * kKmWarps * 32;
  for (long long base = lo + ((long long)blockIdx.x * kKmWarps + warp) * 32; base < hi; base += wstride) {
    const long long p = base + lane;
    const bool valid = p < hi;
    float fv[FM];
#pragma unroll
    for (int l = 0; l < FM; l++) fv[l] = (valid && l < nf) ? __ldcs(f + (long long)l * npts + p) : 0.f;
    int best = 0;
    if (valid && k > 1) {
      float fn2 = 0.f;
#pragma unroll
      for (int l = 0; l < FM; l++) fn2 = fmaf(fv[l], fv[l], fn2);
      const float fnorm = sqrtf(fn2) * 1.01f;
      float tmin = INFINITY, hi1 = INFINITY, lo1 = INFINITY, lo2 = INFINITY;
      int i1 = 0, lo1i = -1;
      bool finite = fn2 <= 3.0e38f;
      for (int c = 0; c < k; c++) {
        const float* cc = cf + c * nf;
        float dot = 0.f;
        if (NF) {
          const float4* c4 = reinterpret_cast<const float4*>(cc);
#pragma unroll
          for (int l = 0; l < FM / 4; l++) {
            const float4 cv = c4[l];
            dot = fmaf(fv[4 * l], cv.x, dot);
            dot = fmaf(fv[4 * l + 1], cv.y, dot);
            dot = fmaf(fv[4 * l + 2], cv.z, dot);
            dot = fmaf(fv[4 * l + 3], cv.w, dot);
          }
        } else {
#pragma unroll
          for (int l = 0; l < FM; l++)
            if (l < nf) dot = fmaf(fv[l], cc[l], dot);
        }
        const float t = fmaf(-2.f, dot, cn2[c]);
        const float e = fmaf(cA[c], fnorm, cB[c]);
        finite &= fabsf(t) <= 3.0e38f;
        if (t < tmin) {
          tmin = t;
          i1 = c;
          hi1 = t + e;
        }
        const float l_ = t - e;
        if (l_ < lo1) {
          lo2 = lo1;
          lo1 = l_;
          lo1i = c;
        } else if (l_ < lo2) {
          lo2 = l_;
        }
      }
      const float other = lo1i == i1 ? lo2 : lo1;
      best = i1;
      if (!finite || !(other > hi1)) {
        // exact reference recurrence (kernels/kmeans.kn)
        double bestd = 0.0;
        best = 0;
        for (int c = 0; c < k; c++) {
          const float* cc = cf + c * nf;
          double dist = 0.0;
#pragma unroll
          for (int l = 0; l < FM; l++) {
            if (l < nf) {
              const double diff = dsub((double)fv[l], (double)cc[l]);
              dist = dadd(dist, dmul(diff, diff));
            }
          }
          if (c == 0 || dist < bestd) {
            bestd = dist;
            best = c;
          }
        }
      }
    }
    if (valid) {
      member[p] = best;
      atomicAdd(cnt + best, 1);
    }
    // transpose: lane q's features -> row q of the tile
#pragma unroll
    for (int l = 0; l < FM; l++)
      if (l < nf) mytile[lane * 33 + l] = fv[l];
    __syncwarp();
    for (int q = 0; q < 32; q++) {
      const int bq = __shfl_sync(0xffffffffu, best, q);
      const bool vq = base + q < hi;
      if (vq && lane < nf) mysum[bq * nf + lane] += mytile[q * 33 + lane];
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kc * nf; i += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kKmWarps; w++) t += wsum[w * kc * nf + i];
    if (t != 0.f) atomicAdd(sums + i, t);
  }
  for (int i = threadIdx.x; i < kc; i += blockDim.x)
    if (cnt[i]) atomicAdd(counts + i, cnt[i]);
}

// Register-blocked screen (nf in {4, 8, 16, 32}): each thread screens TWO
// points (p and p + 32 of its warp's 64-point tile) against FOUR clusters at
// a time.  Centroids are stored in shared memory transposed in groups of four
// (cg[(g*nf + l)*4 + j] = cent[(4g + j)*nf + l]), so one LDS.128 broadcast
// feeds 8 FFMAs in 8 independent accumulation chains (the one-point,
// one-cluster-at-a-time screen above is a 32-deep dependent FMA chain per
// cluster and 4 FFMAs per LDS).  Each chain is still a sequential f32 dot
// product, so the screen's error bound and the exact f64 fallback are those
// of kmeans_fast; membership stays bit-exact.
struct KmPick {
  float tmin, hi1, lo1, lo2;
  int i1, lo1i;
  bool finite;
  __device__ __forceinline__ void init() {
    tmin = hi1 = lo1 = lo2 = INFINITY;
    i1 = 0;
    lo1i = -1;
    finite = true;
  }
  __device__ __forceinline__ void add(float t, float e, int c) {
    finite &= fabsf(t) <= 3.0e38f;
    if (t < tmin) {
      tmin = t;
      i1 = c;
      hi1 = t + e;
    }
    const float l_ = t - e;
    if (l_ < lo1) {
      lo2 = lo1;
      lo1 = l_;
      lo1i = c;
    } else if (l_ < lo2) {
      lo2 = l_;
    }
  }
  __device__ __forceinline__ bool decided() const {
    const float other = lo1i == i1 ? lo2 : lo1;
    return finite && other > hi1;
  }
};

// exact reference recurrence (kernels/kmeans.kn): f64, feature order, strict '<'
// (rare: re-reads the point's features instead of keeping register arrays
// addressable)
template <int NF>
__device__ __noinline__ int km_exact(const float* __restrict__ f, int npts, long long p,
                                     const float* cf, int k) {
  double bestd = 0.0;
  int best = 0;
  for (int c = 0; c < k; c++) {
    const float* cc = cf + c * NF;
    double dist = 0.0;
    for (int l = 0; l < NF; l++) {
      const double diff = dsub((double)__ldg(f + (long long)l * npts + p), (double)cc[l]);
      dist = dadd(dist, dmul(diff, diff));
    }
    if (c == 0 || dist < bestd) {
      bestd = dist;
      best = c;
    }
  }
  return best;
}

template <int NF>
__device__ __forceinline__ void km_accumulate(float* mytile, float* mysum, const float* fv, int best,
                                              long long base, long long hi, int lane) {
#pragma unroll
  for (int l = 0; l < NF; l++) mytile[lane * 33 + l] = fv[l];
  __syncwarp();
  for (int q = 0; q < 32; q++) {
    const int bq = __shfl_sync(0xffffffffu, best, q);
    if (base + q < hi && lane < NF) mysum[bq * NF + lane] += mytile[q * 33 + lane];
  }
  __syncwarp();
}

template <int NF, int MINB>
__global__ void __launch_bounds__(256, MINB) kmeans_rb(const float* __restrict__ f,
                                                 const float* __restrict__ cent,
                                                 int* __restrict__ member, float* sums, int* counts,
                                                 int npts, int k, long long lo, long long hi) {
  extern __shared__ float smf[];
  const int kc = k > 0 ? k : 1;
  const int kg = (kc + 3) >> 2;              // cluster groups of four
  float* cg = smf;                           // [kg][NF][4] transposed centroids
  float* cf = cg + kg * NF * 4;              // [kc][NF] row-major (exact path)
  float* cA = cf + kc * NF;                  // [4kg] error slope (x |f|)
  float* cB = cA + 4 * kg;                   // [4kg] error offset
  float* cn2 = cB + 4 * kg;                  // [4kg] |c|^2 in f32
  float* tile = cn2 + 4 * kg;                // [8][32][33] transpose tiles
  float* wsum = tile + kKmWarps * 32 * 33;   // [8][kc*NF] per-warp sums
  int* cnt = reinterpret_cast<int*>(wsum + kKmWarps * kc * NF);  // [kc]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kg * 4 * NF; i += blockDim.x) {
    const int j = i & 3, l = (i >> 2) % NF, g = (i >> 2) / NF, c = 4 * g + j;
    cg[i] = c < k ? cent[c * NF + l] : 0.f;
  }
  for (int i = threadIdx.x; i < k * NF; i += blockDim.x) cf[i] = cent[i];
  for (int i = threadIdx.x; i < kKmWarps * kc * NF; i += blockDim.x) wsum[i] = 0.f;
  for (int i = threadIdx.x; i < kc; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const float errk = (float)(NF + 4) * 2.384185791015625e-7f * 1.01f;  // (nf+4) 2^-22, +1 %
  for (int c = threadIdx.x; c < 4 * kg; c += blockDim.x) {
    float n2 = 0.f;
    if (c < k)
      for (int l = 0; l < NF; l++) n2 = fmaf(cf[c * NF + l], cf[c * NF + l], n2);
    cn2[c] = n2;
    cA[c] = errk * 2.f * sqrtf(n2) * 1.01f;
    cB[c] = errk * n2 + 1e-30f;
  }
  __syncthreads();
  float* mytile = tile + warp * 32 * 33;
  float* mysum = wsum + warp * kc * NF;
  const long long wstride = (long long)gridDim.x * kKmWarps * 64;
  for (long long base = lo + ((long long)blockIdx.x * kKmWarps + warp) * 64; base < hi; base += wstride) {
    const long long p0 = base + lane, p1 = p0 + 32;
    const bool v0 = p0 < hi, v1 = p1 < hi;
    float f0[NF], f1[NF];
#pragma unroll
    for (int l = 0; l < NF; l++) {
      f0[l] = v0 ? __ldcs(f + (long long)l * npts + p0) : 0.f;
      f1[l] = v1 ? __ldcs(f + (long long)l * npts + p1) : 0.f;
    }
    int b0 = 0, b1 = 0;
    if (k > 1) {
      float n0 = 0.f, n1 = 0.f;
#pragma unroll
      for (int l = 0; l < NF; l++) {
        n0 = fmaf(f0[l], f0[l], n0);
        n1 = fmaf(f1[l], f1[l], n1);
      }
      KmPick s0, s1;
      s0.init();
      s1.init();
      s0.finite = n0 <= 3.0e38f;
      s1.finite = n1 <= 3.0e38f;
      const float fn0 = sqrtf(n0) * 1.01f, fn1 = sqrtf(n1) * 1.01f;
      for (int g = 0; g < kg; g++) {
        const float4* c4 = reinterpret_cast<const float4*>(cg + g * NF * 4);
        float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int l = 0; l < NF; l++) {
          const float4 cv = c4[l];
          d0[0] = fmaf(f0[l], cv.x, d0[0]);
          d0[1] = fmaf(f0[l], cv.y, d0[1]);
          d0[2] = fmaf(f0[l], cv.z, d0[2]);
          d0[3] = fmaf(f0[l], cv.w, d0[3]);
          d1[0] = fmaf(f1[l], cv.x, d1[0]);
          d1[1] = fmaf(f1[l], cv.y, d1[1]);
          d1[2] = fmaf(f1[l], cv.z, d1[2]);
          d1[3] = fmaf(f1[l], cv.w, d1[3]);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int c = 4 * g + j;
          if (c < k) {
            s0.add(fmaf(-2.f, d0[j], cn2[c]), fmaf(cA[c], fn0, cB[c]), c);
            s1.add(fmaf(-2.f, d1[j], cn2[c]), fmaf(cA[c], fn1, cB[c]), c);
          }
        }
      }
      b0 = s0.i1;
      b1 = s1.i1;
      if (v0 && !s0.decided()) b0 = km_exact<NF>(f, npts, p0, cf, k);
      if (v1 && !s1.decided()) b1 = km_exact<NF>(f, npts, p1, cf, k);
    }
    if (v0) {
      member[p0] = b0;
      atomicAdd(cnt + b0, 1);
    }
    if (v1) {
      member[p1] = b1;
      atomicAdd(cnt + b1, 1);
    }
    km_accumulate<NF>(mytile, mysum, f0, b0, base, hi, lane);
    km_accumulate<NF>(mytile, mysum, f1, b1, base + 32, hi, lane);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kc * NF; i += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kKmWarps; w++) t += wsum[w * kc * NF + i];
    if (t != 0.f) atomicAdd(sums + i, t);
  }
  for (int i = threadIdx.x; i < kc; i += blockDim.x)
    if (cnt[i]) atomicAdd(counts + i, cnt[i]);
}


// ---------------------------------------------------------------------------
// Tensor-core path (nf in {8, 16, 24, 32}, 2 <= k <= 16, npts % 4 == 0).
//
// The assignment is a dense contraction: s[p][c] = |c|^2 - 2 f_p . c_c over a
// 128-point tile x 16 clusters x nf features, and so are the new-centroid
// sums: sums[c][l] = sum_p onehot[p][c] f[p][l].  Both run on the tensor cores
// (mma.sync m16n8k8 TF32, the HMMA path; K = 32 and N = 16 are far too small
// for tcgen05 tiles to pay off) with FP32 accuracy recovered by splitting each
// operand x = hi + lo, hi = x rounded to TF32 (integer add + mask), lo = x - hi
// (exact in f32) truncated to TF32 by a mask (|x - hi - lo| <= 2^-21 |x|):
//   dot ~ hi.hi + hi.lo + lo.hi   (3 MMAs)
// The sums use bf16 pairs on m16n8k16 (x = hi + lo, |x - hi - lo| <= 2^-18 |x|;
// the one-hot is exact): sums = F_hi^T onehot + F_lo^T onehot, 16 points per MMA.
// Screen bound, with S = sum_l |f_l c_l| <= |f||c|: split residue
// (lo.lo plus the two truncated cross terms) <= 5.01 2^-22 S; hi.hi
// accumulates alone over nf/8 <= 4 MMAs of 8 exact products each, every
// product aligned/truncated to >= 24 bits of the running maximum
// (<= 9 2^-23 S per MMA, 18 2^-22 S in all); the cross terms (<= 2^-10 S)
// accumulate in their own registers (negligible error); the final add,
// |c|^2 in f32 (<= 2^-19 |c|^2) and the FMA for s add < 2^-20 (S + |c|^2).
// So |s(tc) - s| < 2^-16.4 S + 2^-18.9 |c|^2, and with cmax = max_c |c| we use
// one bound per point (>= 2.6x slack)
//   E = 2^-16 (2 |f| cmax + cmax^2) (1.03) + 2^-40 |f|^2 + 1e-35,
// where the |f|^2 term covers the reference's own f64 rounding of the full
// distance and the absolute term flushed subnormal products.  Candidates are
// the clusters with s_c <= min(s) + 2E; a single candidate is the answer,
// several are resolved by the reference's exact f64 recurrence evaluated for
// the candidates only (in parallel over the four lanes that hold the point's
// clusters, (distance, lowest index) minimum = the reference's `dist < bestd`
// scan).  Points with a non-finite or huge (|f|^2 > 3e38) norm run the whole
// reference scan on one lane and add their features to the sums on the
// scalar path (0 x NaN inside an MMA would poison every cluster).
// Membership stays bit-exact.
//
// Data movement: a producer warp streams 128-point x nf tiles (nf rows of
// 512 B, one bulk copy each, L2 evict-first) into a 3-stage shared-memory
// ring guarded by full/empty mbarriers; four consumer warps (32 points each)
// read their MMA fragments from the tile (row stride 136 floats: conflict-free
// A fragments).  HBM is read exactly once.
#ifndef KM_TC_WARPS
#define KM_TC_WARPS 4  // consumer warps per CTA (32 points each)
#endif
constexpr int kTcPts = 32 * KM_TC_WARPS;
constexpr int kTcStride = kTcPts + 8;
#ifndef KM_TC_STAGES
#define KM_TC_STAGES 3
#endif
constexpr int kTcStages = KM_TC_STAGES;
constexpr int kTcWarps = KM_TC_WARPS;
#ifndef KM_TC_MINB
#define KM_TC_MINB 3
#endif

// x -> (hi, lo) TF32 pair: hi = round-to-nearest (ties away) TF32 of x,
// lo = (x - hi) truncated to TF32.  Non-finite x only feed rows whose results
// are discarded (non-finite points take the exact path).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi)) & 0xffffe000u;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (x0, x1) -> bf16x2 pairs hi = RN(x), lo = RN(x - hi) (element 0 in the low half)
__device__ __forceinline__ void split_bf16x2(float2 x, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x.x, x.y);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x.x - __low2float(h), x.y - __high2float(h));
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// exact reference recurrence over the point's features in the smem tile
template <int NF>
__device__ __noinline__ int km_exact_tile(const float* T, int col, const float* cf, int k) {
  double bestd = 0.0;
  int best = 0;
  for (int c = 0; c < k; c++) {
    double dist = 0.0;
    for (int l = 0; l < NF; l++) {
      const double diff = dsub((double)T[l * kTcStride + col], (double)cf[c * NF + l]);
      dist = dadd(dist, dmul(diff, diff));
    }
    if (c == 0 || dist < bestd) {
      bestd = dist;
      best = c;
    }
  }
  return best;
}

// exact f64 distance of the point in column `col` to centroid c (reference order)
template <int NF>
__device__ __forceinline__ double km_dist_tile(const float* T, int col, const float* cc) {
  double dist = 0.0;
#pragma unroll 8
  for (int l = 0; l < NF; l++) {
    const double diff = dsub((double)T[l * kTcStride + col], (double)cc[l]);
    dist = dadd(dist, dmul(diff, diff));
  }
  return dist;
}

// f32 distance in the difference form (second-stage screen)
template <int NF>
__device__ __forceinline__ float km_dist_f32(const float* T, int col, const float* cc) {
  float acc = 0.f;
#pragma unroll 8
  for (int l = 0; l < NF; l++) {
    const float d = __fsub_rn(T[l * kTcStride + col], cc[l]);
    acc = fmaf(d, d, acc);
  }
  return acc;
}

template <int NF>
__global__ void __launch_bounds__(32 * (kTcWarps + 1), KM_TC_MINB) kmeans_tc(const float* __restrict__ f,
                                                                   const float* __restrict__ cent,
                                                                   int* __restrict__ member, float* sums,
                                                                   int* counts, int npts, int k,
                                                                   long long lo, long long hi) {
  constexpr int KT = NF / 8;          // feature k-tiles of the distance GEMM
  constexpr int MS = (NF + 15) / 16;  // feature m-tiles of the sums GEMM
  extern __shared__ __align__(16) float smf[];
  float* tiles = smf;                                               // [S][NF][kTcStride]
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + kTcStages * NF * kTcStride);
  uint64_t* empty = full + kTcStages;
  float* cf = reinterpret_cast<float*>(empty + kTcStages);          // [16][NF]
  float* cn2 = cf + 16 * NF;                                        // [16]
  float* ssum = cn2 + 16;                                           // [16][NF]
  int* cnt = reinterpret_cast<int*>(ssum + 16 * NF);                // [16]
  uint4* cfr = reinterpret_cast<uint4*>(cnt + 16);                  // [KT][2][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;

  for (int i = threadIdx.x; i < 16 * NF; i += blockDim.x) {
    cf[i] = i < k * NF ? cent[i] : 0.f;
    ssum[i] = 0.f;
  }
  if (threadIdx.x < 16) cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTcWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const int c = threadIdx.x;
    float n2 = 0.f;
    for (int l = 0; l < NF; l++) n2 = fmaf(cf[c * NF + l], cf[c * NF + l], n2);
    cn2[c] = c < k ? n2 : INFINITY;
  }
  // centroid B fragments (C^T: feature x cluster), split hi/lo, one uint4
  // {b0 hi, b1 hi, b0 lo, b1 lo} per (k-tile, n-tile, lane): one LDS.128 each
  for (int i = threadIdx.x; i < KT * 2 * 32; i += blockDim.x) {
    const int ln = i & 31, nt = (i >> 5) & 1, kt = i >> 6, gg = ln >> 2, tt = ln & 3;
    uint4 v;
    split_tf32(cf[(8 * nt + gg) * NF + 8 * kt + tt], v.x, v.z);
    split_tf32(cf[(8 * nt + gg) * NF + 8 * kt + tt + 4], v.y, v.w);
    cfr[i] = v;
  }
  __syncthreads();

  const long long ntile = (hi - lo + kTcPts - 1) / kTcPts;
  if (warp == kTcWarps) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int n = 0;
      for (long long i = blockIdx.x; i < ntile; i += gridDim.x, n++) {
        const int s = n % kTcStages, use = n / kTcStages;
        if (use > 0) mbar_wait_sleep(&empty[s], (use - 1) & 1);
        const long long p0 = lo + i * kTcPts;
        const uint32_t bytes = (uint32_t)min((long long)kTcPts, hi - p0) * 4u;
        mbar_arrive_expect_tx(&full[s], bytes * NF);
        float* T = tiles + s * NF * kTcStride;
#pragma unroll 1
        for (int l = 0; l < NF; l++) bulk_g2s(T + l * kTcStride, f + (long long)l * npts + p0, bytes, &full[s], pol);
      }
    }
  } else {  // consumers
    // per-lane constants: |c|^2 of the lane's clusters c_j = 8(j>>1) + 2t + (j&1), cmax
    float cn[4];
    float cmax2 = 0.f;
#pragma unroll
    for (int j = 0; j < 4; j++) cn[j] = cn2[8 * (j >> 1) + 2 * t + (j & 1)];
    for (int c = 0; c < k; c++) cmax2 = fmaxf(cmax2, cn2[c]);
    const float cmax = sqrtf(cmax2) * 1.001f;
    const float eA = 1.52587890625e-05f * 1.03f * 2.f * cmax;          // x |f|
    const float eB = 1.52587890625e-05f * 1.03f * cmax * cmax + 1e-35f;
    float acc[MS][2][4];
#pragma unroll
    for (int ms = 0; ms < MS; ms++)
#pragma unroll
      for (int nt = 0; nt < 2; nt++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[ms][nt][j] = 0.f;
    const uint32_t one = __float_as_uint(1.0f);
    int n = 0;
    for (long long i = blockIdx.x; i < ntile; i += gridDim.x, n++) {
      const int s = n % kTcStages;
      mbar_wait(&full[s], (n / kTcStages) & 1);
      const float* T = tiles + s * NF * kTcStride;
      const long long p0 = lo + i * kTcPts;
      const int cntp = (int)min((long long)kTcPts, hi - p0);
#pragma unroll 1
      for (int mt = 0; mt < 2; mt++) {
        const int col = warp * 32 + mt * 16 + g;
        const float* Tc = T + col;
        // ---- distance GEMM: D[16 points x 16 clusters]; hi.hi and the two
        // cross terms accumulate separately (4 independent MMA chains, and
        // the small cross terms never sit in the large accumulator)
        float dh[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        float dl[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        float n0 = 0.f, n1 = 0.f;
#pragma unroll
        for (int kt = 0; kt < KT; kt++) {
          const float x0 = Tc[(8 * kt + t) * kTcStride];
          const float x1 = Tc[(8 * kt + t) * kTcStride + 8];
          const float x2 = Tc[(8 * kt + t + 4) * kTcStride];
          const float x3 = Tc[(8 * kt + t + 4) * kTcStride + 8];
          n0 = fmaf(x0, x0, fmaf(x2, x2, n0));
          n1 = fmaf(x1, x1, fmaf(x3, x3, n1));
          uint32_t ah[4], al[4];
          split_tf32(x0, ah[0], al[0]);
          split_tf32(x1, ah[1], al[1]);
          split_tf32(x2, ah[2], al[2]);
          split_tf32(x3, ah[3], al[3]);
#pragma unroll
          for (int nt = 0; nt < 2; nt++) {
            const uint4 b = cfr[(kt * 2 + nt) * 32 + lane];
            mma_tf32(dl[nt], al, b.x, b.y);
            mma_tf32(dl[nt], ah, b.z, b.w);
            mma_tf32(dh[nt], ah, b.x, b.y);
          }
        }
        n0 += __shfl_xor_sync(0xffffffffu, n0, 1);
        n1 += __shfl_xor_sync(0xffffffffu, n1, 1);
        n0 += __shfl_xor_sync(0xffffffffu, n0, 2);
        n1 += __shfl_xor_sync(0xffffffffu, n1, 2);
        // ---- screen (rows g: r = 0, g+8: r = 1)
        int best[2];
        bool need[2], fin[2], ok[2];
        float tv[2][4], thr[2];
#pragma unroll
        for (int r = 0; r < 2; r++) {
          const float nr = r ? n1 : n0;
          fin[r] = nr <= 3.0e38f;  // false for NaN / inf / huge points
          const float E = fmaf(eA, nr * rsqrtf(nr + 1e-30f) * 1.01f, eB) + 9.2e-13f * nr;  // approx |f| +1 %; 2^-40 |f|^2
          float m = INFINITY;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            tv[r][j] = fmaf(-2.f, dh[j >> 1][2 * r + (j & 1)] + dl[j >> 1][2 * r + (j & 1)], cn[j]);
            m = fminf(m, tv[r][j]);
          }
          m = fminf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fminf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          thr[r] = m + 2.f * E;
          int nc = 0, lowc = 16;
#pragma unroll
          for (int j = 3; j >= 0; j--) {  // descending: lowc ends at the lowest
            const bool cand = tv[r][j] <= thr[r];
            nc += cand;
            const int c = 8 * (j >> 1) + 2 * t + (j & 1);
            if (cand && c < lowc) lowc = c;
          }
          nc += __shfl_xor_sync(0xffffffffu, nc, 1);
          lowc = min(lowc, __shfl_xor_sync(0xffffffffu, lowc, 1));
          nc += __shfl_xor_sync(0xffffffffu, nc, 2);
          lowc = min(lowc, __shfl_xor_sync(0xffffffffu, lowc, 2));
          ok[r] = (r ? col + 8 : col) < cntp;
          best[r] = lowc;
          fin[r] = fin[r] && nc >= 1;  // no candidate: NaN screen (overflowing centroids)
          need[r] = ok[r] && (!fin[r] || nc != 1);
        }
        if (__any_sync(0xffffffffu, need[0] || need[1])) {
#pragma unroll
          for (int r = 0; r < 2; r++) {
            if (!__any_sync(0xffffffffu, need[r])) continue;
            const int cr = col + 8 * r;
            if (!__any_sync(0xffffffffu, need[r] && fin[r])) {
              int e = 0;
              if (t == 0 && need[r]) e = km_exact_tile<NF>(T, cr, cf, k);
              e = __shfl_sync(0xffffffffu, e, lane & ~3);
              if (need[r]) best[r] = e;
              continue;
            }
            // stage 2: the candidates' distances in f32 in the difference
            // form sum (x - c)^2, whose error is relative to the distance
            // itself: |d32 - d| <= (nf + 4) 2^-24 d (+ subnormal slack).
            // A single survivor of that screen is the answer; otherwise the
            // exact f64 recurrence decides among the survivors.
            bool sv[4];
            int nsv = 0;
            {
              float d32[4], u2 = INFINITY;
              const float e2 = (float)(NF + 4) * 5.9604645e-08f * 1.01f;
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const int c = 8 * (j >> 1) + 2 * t + (j & 1);
                sv[j] = need[r] && fin[r] && tv[r][j] <= thr[r];
                d32[j] = sv[j] ? km_dist_f32<NF>(T, cr, cf + c * NF) : INFINITY;
                u2 = fminf(u2, fmaf(d32[j], e2, d32[j]) + 1e-40f);
              }
              u2 = fminf(u2, __shfl_xor_sync(0xffffffffu, u2, 1));
              u2 = fminf(u2, __shfl_xor_sync(0xffffffffu, u2, 2));
              int lowc = 16;
#pragma unroll
              for (int j = 3; j >= 0; j--) {
                sv[j] = sv[j] && fmaf(-d32[j], e2, d32[j]) - 1e-40f <= u2;
                nsv += sv[j];
                if (sv[j]) lowc = 8 * (j >> 1) + 2 * t + (j & 1);
              }
              nsv += __shfl_xor_sync(0xffffffffu, nsv, 1);
              lowc = min(lowc, __shfl_xor_sync(0xffffffffu, lowc, 1));
              nsv += __shfl_xor_sync(0xffffffffu, nsv, 2);
              lowc = min(lowc, __shfl_xor_sync(0xffffffffu, lowc, 2));
              if (need[r] && fin[r] && nsv == 1) {
                best[r] = lowc;
                need[r] = false;
              }
            }
            if (!__any_sync(0xffffffffu, need[r])) continue;
            double bd = INFINITY;
            int bi = 16;
            if (need[r] && fin[r]) {
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const int c = 8 * (j >> 1) + 2 * t + (j & 1);
                if (sv[j]) {
                  const double dist = km_dist_tile<NF>(T, cr, cf + c * NF);
                  if (dist < bd || (dist == bd && c < bi)) {
                    bd = dist;
                    bi = c;
                  }
                }
              }
            }
#pragma unroll
            for (int x = 1; x <= 2; x <<= 1) {
              const double od = __shfl_xor_sync(0xffffffffu, bd, x);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, x);
              if (od < bd || (od == bd && oi < bi)) {
                bd = od;
                bi = oi;
              }
            }
            int e = 0;
            if (t == 0 && need[r] && !fin[r]) e = km_exact_tile<NF>(T, cr, cf, k);
            e = __shfl_sync(0xffffffffu, e, lane & ~3);
            if (need[r]) best[r] = fin[r] ? bi : e;
          }
        }
        if (t == 0) {
#pragma unroll
          for (int r = 0; r < 2; r++)
            if (ok[r]) {
              member[p0 + col + 8 * r] = best[r];
              atomicAdd(cnt + best[r], 1);
              if (!fin[r])  // scalar sums path for non-finite / huge points
                for (int l = 0; l < NF; l++) atomicAdd(ssum + best[r] * NF + l, T[l * kTcStride + col + 8 * r]);
            }
        }
        // ---- sums GEMM: acc[features x clusters] += F^T[features x 16 points] onehot, on
        // bf16 pairs (m16n8k16): x = hi + lo with hi, lo bf16 (|x - hi - lo| <= 2^-18 |x|,
        // far inside the sums tolerance), the one-hot exact in bf16; points that are not
        // valid and finite contribute zeros
        {
          const int bs0 = (ok[0] && fin[0]) ? best[0] : -1;  // point g of the m-tile
          const int bs1 = (ok[1] && fin[1]) ? best[1] : -1;  // point g + 8
          const int qa = __shfl_sync(0xffffffffu, bs0, 8 * t), qb = __shfl_sync(0xffffffffu, bs0, 8 * t + 4);
          const int qc = __shfl_sync(0xffffffffu, bs1, 8 * t), qd = __shfl_sync(0xffffffffu, bs1, 8 * t + 4);
          const float* Tp = T + warp * 32 + mt * 16 + 2 * t;  // points 2t, 2t+1 (and +8) of the m-tile
#pragma unroll
          for (int ms = 0; ms < MS; ms++) {
            const int r0 = 16 * ms + g, r1 = r0 + 8;
            float2 xa = *reinterpret_cast<const float2*>(Tp + r0 * kTcStride);
            float2 xb = *reinterpret_cast<const float2*>(Tp + r0 * kTcStride + 8);
            float2 xc = make_float2(0.f, 0.f), xd = xc;
            if (r1 < NF) {
              xc = *reinterpret_cast<const float2*>(Tp + r1 * kTcStride);
              xd = *reinterpret_cast<const float2*>(Tp + r1 * kTcStride + 8);
            }
            if (qa < 0) xa.x = xc.x = 0.f;
            if (qb < 0) xa.y = xc.y = 0.f;
            if (qc < 0) xb.x = xd.x = 0.f;
            if (qd < 0) xb.y = xd.y = 0.f;
            uint32_t ah[4], al[4];
            split_bf16x2(xa, ah[0], al[0]);
            split_bf16x2(xc, ah[1], al[1]);
            split_bf16x2(xb, ah[2], al[2]);
            split_bf16x2(xd, ah[3], al[3]);
#pragma unroll
            for (int nt = 0; nt < 2; nt++) {
              const int cl = 8 * nt + g;
              const uint32_t b0 = (qa == cl ? 0x3F80u : 0u) | (qb == cl ? 0x3F800000u : 0u);
              const uint32_t b1 = (qc == cl ? 0x3F80u : 0u) | (qd == cl ? 0x3F800000u : 0u);
              mma_bf16(acc[ms][nt], al, b0, b1);
              mma_bf16(acc[ms][nt], ah, b0, b1);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // per-warp sums -> shared
#pragma unroll
    for (int ms = 0; ms < MS; ms++)
#pragma unroll
      for (int nt = 0; nt < 2; nt++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int feat = 16 * ms + g + (j >= 2 ? 8 : 0), c = 8 * nt + 2 * t + (j & 1);
          if (feat < NF && c < k && acc[ms][nt][j] != 0.f) atomicAdd(ssum + c * NF + feat, acc[ms][nt][j]);
        }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * NF; i += blockDim.x)
    if (ssum[i] != 0.f) atomicAdd(sums + i, ssum[i]);
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (cnt[i]) atomicAdd(counts + i, cnt[i]);
}

template <int NF>
static size_t kmeans_tc_smem() {
  return sizeof(float) * kTcStages * NF * kTcStride + sizeof(uint64_t) * 2 * kTcStages +
         sizeof(float) * (16 * NF + 16 + 16 * NF) + sizeof(int) * 16 + sizeof(uint4) * (NF / 8) * 64;
}

// ---------------------------------------------------------------------------
// kmeans_tg: the same screen on the tcgen05 tensor cores (nf = 32, k <= 16).
//
// The fp32 tiles cannot feed tcgen05 as they are: kind::tf32 reads K-major
// operands only (scripts/micro/umma_sw128.cu) and the tiles are feature-major.
// Split into bf16 hi / lo planes instead (x = hi + lo + r, hi = RN_bf16(x),
// lo = RN_bf16(x - hi), |r| <= 2^-16 |x|), the planes ARE legal operands in the
// tiles' own [feature][point] order for both contractions
// (scripts/micro/umma_bf16.cu checks every layout below on the device):
//   distance  D[p][c'] = sum_l F[p][l] B[c'][l], M = 128 points, K = 32:
//             A = the planes read MN-major (SWIZZLE_128B atoms of 8 features x
//             64 points); B = the centroid rows (hi 0..15, lo 16..31, lo2 32..47) K-major.
//             MMA 1: A = F_hi, N = 48 (hi.hi -> cols 0..15, hi.lo -> 16..31,
//             hi.lo2 -> 32..47); MMA 2: A = F_lo, B = [C_hi | C_lo], N = 32,
//             accumulated into cols 16..47.
//   sums      S[r][c] = sum_p P[r][p] onehot[c][p] over a PAIR of tiles:
//             M = 128 rows (tile 2q: 32 hi + 32 lo feature rows, tile 2q+1
//             the same), K = 128 points, N = 32 (the two tiles' one-hots,
//             [cluster][point] K-major, written by the epilogue); A = the
//             same planes read K-major.  The cross blocks (tile 2q rows x tile
//             2q+1 one-hot) are never read.  S lives in TMEM for the whole
//             kernel: 8 MMAs per pair instead of 8 per tile (a tcgen05.mma
//             costs ~45 cycles whatever N <= 64: scripts/micro/umma_rate.cu).
//   Distance and sums MMAs are issued by two warps, so the distances never
//   wait for a screen.
// Screen bound with S = sum_l |f_l c_l| <= |f| cmax.  The centroids are
// split into THREE planes, c = C_hi + C_lo + C_lo2 + r_c (r_c = 0 unless a
// plane is subnormal, measured per launch), the points into two (the split
// is the pipeline's slowest stage), and the distance accumulates F_hi.C_hi,
// F_hi.C_lo + F_lo.C_hi and F_hi.C_lo2 + F_lo.C_lo in three column groups
// (N = 48: 4 MMAs per tile, as with two centroid planes), summed small first.
// Dropped: r_f.c <= 2^-16 S, F_lo.(C_lo2 + r_c) <= 2^-24 S + |f||r_c|; the
// tensor-core accumulation of the exact bf16 products: 2 MMAs of K = 16 into
// the hi.hi columns <= 2 x 17 x 2^-23 S, 8 into the small ones (terms <=
// 2^-7 S) <= 2^-22.9 S; times 2 for s = |c|^2 - 2 f.c, plus 2^-24 |c|^2 (f64
// |c|^2 rounded once) and 2^-22.4 S + 2^-24 |c|^2 (epilogue adds):
// |s(tg) - s| < 2^-14.63 S + 2 |f||r_c| + 2^-23 |c|^2.  Used with (>= 1.5x
// slack; round 2 had 2^-13.17 S with two centroid planes and E = 2^-12 ...,
// which deferred 1.2-2.7 % of the points of the 16M x 32 bench data)
//   E = 2^-14 |f| cmax (1.01) + 2.02 |f| max|r_c| + 2^-21 cmax^2 + 2^-40 |f|^2
//       + 2^-100 cmax + 1e-35
// (the last two: flushed subnormal bf16 inputs / products).  Points with
// several candidates are deferred: no one-hot entry (their tile's planes are
// released without waiting), then the f32 difference-form distance of each
// candidate (the warp's lanes over the features, from global memory: L2
// hits), the exact f64 recurrence if that leaves several, and their features
// added to the sums on the scalar path.  Features with |x| > 3e38 or
// non-finite are zeroed in the planes (0 x NaN would poison every cluster's
// sums); their points (norm not finite) are deferred to the exact scan.
//
// Warp roles (480 threads, one CTA per SM, persistent over the tiles):
//   warps 0-3  split: fp32 tile -> bf16 planes + per-point |f|^2 (features
//              0-15 in warps 0-1, 16-31 in 2-3; two points per thread)
//   warps 4-11 epilogue, two sets of 4 alternating tiles: TMEM lane = point;
//              screen, member, counts, the one-hot tile, deferred re-checks
//   warp 12    producer: one 2D tensor copy {128 points x 32 features} per tile
//   warp 13    distance MMA issuer (one elected lane) and TMEM owner
//   warp 14    sums MMA issuer
// Rings: 5 fp32 tiles (released by the split), 6 plane / one-hot stages (3
// pairs), 6 TMEM accumulators of 48 columns (+ 32 columns of sums): the
// distances run two tiles ahead of the screen, the split further ahead.
namespace tg {
constexpr int kPts = 128;
constexpr int kNF = 32;
#ifndef KM_TG_ST
#define KM_TG_ST 5
#endif
constexpr int kST = KM_TG_ST;  // fp32 tiles (released by the split)
#ifndef KM_TG_SP
#define KM_TG_SP 6
#endif
constexpr int kSP = KM_TG_SP;  // planes / one-hot stages (pairs)
#ifndef KM_TG_SA
#define KM_TG_SA 6
#endif
constexpr int kSA = KM_TG_SA;  // TMEM distance accumulators (32 columns each)
#ifndef KM_TG_SPLIT_SETS
#define KM_TG_SPLIT_SETS 1
#endif
#ifndef KM_TG_EPI_SETS
#define KM_TG_EPI_SETS 2
#endif
constexpr int kSplitSets = KM_TG_SPLIT_SETS;  // split warp sets of 4 (alternating tiles)
constexpr int kEpiSets = KM_TG_EPI_SETS;      // epilogue warp sets of 4 (alternating tiles)
// the measured balance (scripts/ab/km_tg_sets.sh): 2 split sets + 1 epilogue
// set ran 0.60 ms and faulted once in four runs, 2 + 2 spills registers at
// 608 threads (0.70 ms); only 1 + 2 is built and tested
static_assert(kSplitSets == 1 && kEpiSets == 2, "kmeans_tg: untested warp-role balance");
constexpr int kWEpi = 4 * kSplitSets;         // first epilogue warp
constexpr int kWProd = kWEpi + 4 * kEpiSets, kWMma = kWProd + 1, kWSum = kWProd + 2;
constexpr int kThreads = 32 * (kWSum + 1);
constexpr uint32_t kTileB = kNF * kPts * 4;  // 16 KB
constexpr uint32_t kPlaneB = 16384;          // hi + lo planes of a tile
constexpr uint32_t kOneHotB = 4096;
constexpr uint32_t kOffPlanes = kST * kTileB;
constexpr uint32_t kOffOneHot = kOffPlanes + kSP * kPlaneB;
constexpr uint32_t kOffCent = kOffOneHot + kSP * kOneHotB;
constexpr uint32_t kOffNrm = kOffCent + 6144;               // [kSP][2][128] f32
constexpr uint32_t kOffCf = kOffNrm + kSP * 2 * kPts * 4;   // [16][32] f32 centroids
constexpr uint32_t kOffSsx = kOffCf + 16 * kNF * 4;         // [16][32] scalar-path sums
constexpr uint32_t kOffCnt = kOffSsx + 16 * kNF * 4;        // [16] counts
constexpr uint32_t kOffCn = kOffCnt + 16 * 4;               // [16] |c|^2 (f64 sums rounded), [16] |r_c|
constexpr uint32_t kOffBar = kOffCn + 32 * 4;               // mbarriers
constexpr int kNBar = 2 * kST + 3 * kSP + 2 * kSA + 1;
constexpr uint32_t kSmem = kOffBar + kNBar * 8 + 16 + 1024;  // + TMEM slot, + alignment slack
static_assert(kSmem <= 227 * 1024, "kmeans_tg shared memory");
constexpr uint32_t kAccCols = 48;  // hi.hi | hi.lo + lo.hi | hi.lo2 + lo.lo
static_assert(kAccCols * kSA + 32 <= 512, "kmeans_tg TMEM columns");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kSumsCol = kAccCols * kSA;  // 32 columns (M = 128: two stage parities)
static_assert(kSP % 2 == 0, "stages are used in pairs");

// packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100a): two points per instruction
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)), "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
// (lo, hi) -> bf16x2 {lo in bits 0..15, hi in 16..31}, both rounded to nearest even
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// byte offset of (row r, element q) in a SWIZZLE_128B atom of 8 rows x 64 bf16
__device__ __forceinline__ uint32_t sw128(int r, int q) {
  return (uint32_t)(r * 128 + ((((q >> 3) ^ r) & 7) << 4) + (q & 7) * 2);
}
// Stages come in pairs (2q, 2q + 1) laid out so that one M = 128 sums MMA
// reads both tiles' planes: pair buffer = [point half][stage parity][plane
// P][feature group] of 1 KB atoms; stage_planes(b) is the stage's base.
// planes of a tile: plane P (0 hi, 1 lo), feature l, point p (from the stage base)
__device__ __forceinline__ uint32_t plane_off(int P, int l, int p) {
  return (uint32_t)((p >> 6) * 16384 + (P * 4 + (l >> 3)) * 1024) + sw128(l & 7, p & 63);
}
__device__ __forceinline__ uint32_t stage_planes(int b) { return kOffPlanes + (b >> 1) * 32768 + (b & 1) * 8192; }
__device__ __forceinline__ uint32_t cent_off(int R, int l) { return (uint32_t)((R >> 3) * 1024) + sw128(R & 7, l); }
// one-hot pair buffer: [point half][cluster row c' = 16 (b & 1) + c] (K-major, 32 rows)
__device__ __forceinline__ uint32_t onehot_off(int c, int p) {
  return (uint32_t)((p >> 6) * 4096 + (c >> 3) * 1024) + sw128(c & 7, p & 63);
}
__device__ __forceinline__ uint32_t stage_onehot(int b) { return kOffOneHot + (b >> 1) * 8192 + (b & 1) * 2048; }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {  // SWIZZLE_128B, sm100
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool amn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
// MMA helpers are issued by the whole (converged) warp: one elected lane
// executes, so the operands stay warp-uniform (no per-lane issue loop)
// the 4 distance MMAs of a tile + the commit on `bar`, one elected lane, one
// asm block (no per-MMA descriptor arithmetic on the issuing warp):
//   D[0..47]  = F_hi . [C_hi | C_lo | C_lo2]   (K = 32: feature groups 0-1, 2-3)
//   D[16..47] += F_lo . [C_hi | C_lo]
// (each plane is read once per K step: the tile's MMAs are smem-read bound
// together with the TMA writes, the split and the sums)
// aH = the stage's hi-plane descriptor (lo plane +4096 B, second K step
// +2048 B), bC = the centroid descriptor (second K step +32 B)
__device__ __forceinline__ void umma_dist(uint32_t d, uint64_t aH, uint64_t bC, uint32_t id48, uint32_t id32,
                                          uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e, f, t;\n .reg .b64 a1, a2, a3, b1;\n"
      " elect.sync _|e, 0xffffffff;\n setp.eq.u32 f, 1, 0;\n setp.eq.u32 t, 0, 0;\n"
      " add.s64 a1, %1, 128;\n add.s64 a2, %1, 256;\n add.s64 a3, %1, 384;\n add.s64 b1, %2, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, f;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%4], a2, %2, %5, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%4], a3, b1, %5, t;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n}" ::"r"(d),
      "l"(aH), "l"(bC), "r"(id48), "r"(d + 16), "r"(id32), "r"(smem_u32(bar))
      : "memory");
}
// the 8 sums MMAs of a tile pair (two point halves x 4 K steps of 16 points):
// A = the pair's planes (+16384 B per half, +32 B per K step), B = the pair's
// one-hot rows (+4096 B per half, +32 B per K step); `first` clears D
__device__ __forceinline__ void umma_sums(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t first) {
  asm volatile(
      "{\n .reg .pred e, p, t;\n .reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      " elect.sync _|e, 0xffffffff;\n setp.eq.u32 p, %4, 0;\n setp.eq.u32 t, 0, 0;\n"
      " add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      " add.s64 a4, %1, 1024;\n add.s64 a5, %1, 1026;\n add.s64 a6, %1, 1028;\n add.s64 a7, %1, 1030;\n"
      " add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      " add.s64 b4, %2, 256;\n add.s64 b5, %2, 258;\n add.s64 b6, %2, 260;\n add.s64 b7, %2, 262;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, t;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, t;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(first)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// 32 lanes x 32 columns of f32 (thread i <- lane base + i)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}
// columns 16..47 into d, 0..15 into h, one wait
__device__ __forceinline__ void tmem_ld32_16(uint32_t taddr, float (&d)[32], float (&h)[16]) {
  uint32_t r[32], q[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr + 16));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]), "=r"(q[8]),
        "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) d[i] = __uint_as_float(r[i]);
#pragma unroll
  for (int i = 0; i < 16; i++) h[i] = __uint_as_float(q[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// the reference recurrences over a point's features in global memory (rare
// path; the lines were streamed through L2 a few microseconds earlier)
__device__ __noinline__ int exact_g(const float* fp, long long stride, const float* cf, int k) {
  double bestd = 0.0;
  int best = 0;
  for (int c = 0; c < k; c++) {
    double dist = 0.0;
    for (int l = 0; l < kNF; l++) {
      const double diff = dsub((double)fp[l * stride], (double)cf[c * kNF + l]);
      dist = dadd(dist, dmul(diff, diff));
    }
    if (c == 0 || dist < bestd) {
      bestd = dist;
      best = c;
    }
  }
  return best;
}
// the exact f64 recurrence over the clusters of `mask`, ascending, first
// strict minimum (the reference's scan restricted to the survivors)
__device__ __noinline__ int exact_mask_g(const float* fp, long long stride, const float* cf, unsigned mask) {
  double bd = 0.0;
  int bi = -1;
  for (unsigned r = mask; r; r &= r - 1) {
    const int c = __ffs(r) - 1;
    double dist = 0.0;
    for (int l = 0; l < kNF; l++) {
      const double diff = dsub((double)fp[l * stride], (double)cf[c * kNF + l]);
      dist = dadd(dist, dmul(diff, diff));
    }
    if (bi < 0 || dist < bd) {
      bd = dist;
      bi = c;
    }
  }
  return bi;
}
// mbarrier waits of the pipeline roles (default 1: 0.533 -> 0.529 ms,
// scripts/ab/km_tg_wait.sh).  KM_TG_WAIT: 0 = try_wait with a
// 1 ms suspend-time hint everywhere; 1 = the single-thread issuers (producer,
// MMA warps) poll with test_wait; 2 = every role uses try_wait without a
// hint; 3 = the issuers use try_wait without a hint
#ifndef KM_TG_WAIT
#define KM_TG_WAIT 1
#endif
__device__ __forceinline__ void wait_poll(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void wait_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tg_wait_issuer(uint64_t* bar, uint32_t parity) {
  if (KM_TG_WAIT == 1) wait_poll(bar, parity);
  else if (KM_TG_WAIT >= 2) wait_nohint(bar, parity);
  else mbar_wait(bar, parity);
}
__device__ __forceinline__ void tg_wait_worker(uint64_t* bar, uint32_t parity) {
  if (KM_TG_WAIT == 2) wait_nohint(bar, parity);
  else mbar_wait(bar, parity);
}
#ifdef KM_TG_TRACE
// per-tile event times of CTA 0 (ns, %globaltimer): [event][tile]
__device__ unsigned long long g_trace[12][2048];
__device__ __forceinline__ void trace(int ev, int n) {
  if (blockIdx.x == 0 && n < 2048) {
    unsigned long long t;
    t = clock64();
    g_trace[ev][n] = t;
  }
}
#else
__device__ __forceinline__ void trace(int, int) {}
#endif
}  // namespace tg

#ifdef KM_TG_TRACE
extern "C" int bf_debug_tg_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, tg::g_trace, sizeof(tg::g_trace));
}
#endif

__global__ void __launch_bounds__(tg::kThreads, 1) kmeans_tg(const __grid_constant__ CUtensorMap tmap,
                                                            const float* __restrict__ f,
                                                            const float* __restrict__ cent,
                                                            int* __restrict__ member, float* sums, int* counts,
                                                            int npts, int k, long long lo, long long hi) {
  using namespace tg;
  extern __shared__ __align__(16) unsigned char tg_raw[];
  // 1 KB-aligned (SWIZZLE_128B atoms); pointer arithmetic keeps the shared window
  unsigned char* sm = tg_raw + ((1024u - (smem_u32(tg_raw) & 1023u)) & 1023u);
  float* nrm = reinterpret_cast<float*>(sm + kOffNrm);
  float* cf = reinterpret_cast<float*>(sm + kOffCf);
  float* ssx = reinterpret_cast<float*>(sm + kOffSsx);
  int* cnt = reinterpret_cast<int*>(sm + kOffCnt);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBar);
  uint64_t* full_t = bars;                  // [kST] producer -> split (tx bytes)
  uint64_t* empty_t = full_t + kST;         // [kST] epilogue (4 warps) -> producer
  uint64_t* full_p = empty_t + kST;         // [kSP] split (4 warps) -> MMA
  uint64_t* empty_p = full_p + kSP;         // [kSP] sums MMA commit -> split
  uint64_t* oh_full = empty_p + kSP;        // [kSP] epilogue (4 warps) -> MMA
  uint64_t* acc_full = oh_full + kSP;       // [kSA] distance MMA commit -> epilogue
  uint64_t* acc_empty = acc_full + kSA;     // [kSA] epilogue (4 warps) -> MMA
  uint64_t* fin = acc_empty + kSA;          // last sums MMA commit -> epilogue
  uint32_t* tslot = reinterpret_cast<uint32_t*>(fin + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- setup: barriers, TMEM, centroids (f32, and the bf16 hi / lo rows)
  if (tid == 0) {
    for (int s = 0; s < kST; s++) {
      mbar_init(&full_t[s], 1);
      mbar_init(&empty_t[s], 4);
    }
    for (int b = 0; b < kSP; b++) {
      mbar_init(&full_p[b], 4);
      mbar_init(&empty_p[b], 1);
      mbar_init(&oh_full[b], 4);
    }
    for (int a = 0; a < kSA; a++) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (warp == kWMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < 16 * kNF; i += blockDim.x) {
    cf[i] = i < k * kNF ? cent[i] : 0.f;
    ssx[i] = 0.f;
  }
  if (tid < 16) {
    cnt[tid] = 0;
    // |c|^2 as an f64 sum rounded once (error 2^-24 |c|^2), and the norm of
    // the centroid's split residue c - hi - lo - lo2 (exact f32 differences;
    // zero unless a plane is subnormal or overflows), rounded up
    float* cnrm = reinterpret_cast<float*>(sm + kOffCn);
    // (planes below FLT_MIN count as residue: the tensor cores may flush them)
    double n2 = 0.0, r2 = 0.0;
    if (tid < k) {
      for (int l = 0; l < kNF; l++) {
        const float x = cent[tid * kNF + l];
        n2 = fma((double)x, (double)x, n2);
        const float h = __bfloat162float(__float2bfloat16_rn(x));
        const float u = x - h, l1 = __bfloat162float(__float2bfloat16_rn(u));
        const float l2 = __bfloat162float(__float2bfloat16_rn(u - l1));
        const double r = (double)x - (fabsf(h) < FLT_MIN ? 0.0 : (double)h) -
                         (fabsf(l1) < FLT_MIN ? 0.0 : (double)l1) - (fabsf(l2) < FLT_MIN ? 0.0 : (double)l2);
        r2 = fma(r, r, r2);
      }
    }
    cnrm[tid] = tid < k ? (float)n2 : __int_as_float(0x7fffffff);  // NaN: never a candidate
    cnrm[16 + tid] = tid < k ? (r2 == r2 ? (float)sqrt(r2) * 1.001f : INFINITY) : 0.f;  // NaN: screen off
  }
  for (int i = tid; i < 48 * 64; i += blockDim.x) {  // 48 rows x 64 bf16 (features 32..63 zero)
    const int R = i >> 6, q = i & 63, c = R & 15;
    float v = 0.f;
    if (q < kNF && c < k) {  // rows 0..15 hi, 16..31 lo, 32..47 lo2: c = hi + lo + lo2 (+ r_c)
      const float x = cent[c * kNF + q];
      const float h = __bfloat162float(__float2bfloat16_rn(x));
      const float u = x - h;
      v = R < 16 ? h : R < 32 ? u : u - __bfloat162float(__float2bfloat16_rn(u));
    }
    *reinterpret_cast<__nv_bfloat16*>(sm + kOffCent + cent_off(R, q)) = __float2bfloat16_rn(v);
  }
  fence_proxy_async();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const long long ntile = (hi - lo + kPts - 1) / kPts;
  const int nmine = ntile > blockIdx.x ? (int)((ntile - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (warp == kWProd) {  // ---- producer: one 2D tensor copy {128 points x 32 features} per tile
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
      for (int n = 0; n < nmine; n++) {
        const int s = n % kST;
        if (n >= kST) tg_wait_issuer(&empty_t[s], ((n / kST) - 1) & 1);  // wakes on the phase flip (a nanosleep back-off added ~1200 cycles per slot)
        const long long p0 = lo + (blockIdx.x + (long long)n * gridDim.x) * kPts;
        trace(0, n);
        // the box is always written in full (zeros past npts; columns past hi
        // are zeroed by the split)
        mbar_arrive_expect_tx(&full_t[s], kTileB);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm + s * kTileB)),
            "l"(&tmap), "r"((int)p0), "r"(0), "r"(smem_u32(&full_t[s]))
            : "memory");
      }
    }
  } else if (warp == kWMma) {  // ---- distance MMAs (the whole warp; one elected lane issues)
    const uint64_t dC = sdesc(smem_u32(sm + kOffCent), 16, 1024);
    const uint32_t idD48 = idesc(128, 48, true), idD32 = idesc(128, 32, true);
    for (int n = 0; n < nmine; n++) {
      const int b = n % kSP;
      tg_wait_issuer(&full_p[b], (n / kSP) & 1);
      if (lane == 0) trace(8, n);
      const int a = n % kSA;
      if (n >= kSA) tg_wait_issuer(&acc_empty[a], ((n / kSA) - 1) & 1);
      if (lane == 0) trace(9, n);
      __syncwarp();  // elect.sync below needs the converged warp
      tc_after();
      umma_dist(tmem + a * kAccCols, sdesc(smem_u32(sm + stage_planes(b)), 16384, 1024), dC, idD48, idD32,
                &acc_full[a]);
      if (lane == 0) trace(4, n);
      __syncwarp();
    }
  } else if (warp == kWSum) {
    // ---- centroid sums, issued by a second thread so that the distances
    // never wait for a screen: the tile pair (m0, m0 + 1), or a last lone
    // even tile; M = 128 rows = both tiles' hi / lo feature rows, N = 32 =
    // both one-hots (the cross blocks of D are never read).  A pair's
    // distance MMAs completed before its screens began, so the commit on
    // empty_p covers every tensor-core read of the stages.
    const uint32_t idS2 = idesc(128, 32, false), idS1 = idesc(128, 16, false);
    for (int m0 = 0; m0 < nmine; m0 += 2) {
      const int b0 = m0 % kSP;
      const bool pair = m0 + 1 < nmine;
      tg_wait_issuer(&oh_full[b0], (m0 / kSP) & 1);
      if (pair) tg_wait_issuer(&oh_full[b0 + 1], ((m0 + 1) / kSP) & 1);
      if (lane == 0) trace(10, m0 + pair);
      __syncwarp();
      tc_after();
      umma_sums(tmem + kSumsCol, sdesc(smem_u32(sm + stage_planes(b0)), 16, 1024),
                sdesc(smem_u32(sm + stage_onehot(b0)), 16, 1024), pair ? idS2 : idS1, m0 == 0 ? 1u : 0u);
      umma_commit(&empty_p[b0]);
      if (pair) umma_commit(&empty_p[b0 + 1]);
      if (lane == 0) trace(7, m0 + pair);
      __syncwarp();
      if (m0 + 2 >= nmine) umma_commit(fin);
    }
  } else if (warp < kWEpi) {  // ---- split: fp32 tile -> bf16 planes, |f|^2 partials
    const int st = tid & 127, half = st >> 6, pr = st & 63, p = 2 * pr, sset = warp >> 2;
    for (int n = sset; n < nmine; n += kSplitSets) {
      const int s = n % kST, b = n % kSP;
      tg_wait_worker(&full_t[s], (n / kST) & 1);
      if (st == 0) trace(1, n);
      if (n >= kSP) tg_wait_worker(&empty_p[b], ((n / kSP) - 1) & 1);
      if (st == 0) trace(2, n);
      const long long p0 = lo + (blockIdx.x + (long long)n * gridDim.x) * kPts;
      const int cntp = (int)min((long long)kPts, hi - p0);
      const float* T = reinterpret_cast<const float*>(sm + s * kTileB);
      unsigned char* P = sm + stage_planes(b);
      float n0 = 0.f, n1 = 0.f;
      float2 xs[16];
#pragma unroll
      for (int j = 0; j < 16; j++) xs[j] = *reinterpret_cast<const float2*>(T + (16 * half + j) * kPts + p);
      if (cntp < kPts) {  // columns past hi: other ranges' points (or zeros)
        const bool v0 = p < cntp, v1 = p + 1 < cntp;
#pragma unroll
        for (int j = 0; j < 16; j++) {
          xs[j].x = v0 ? xs[j].x : 0.f;
          xs[j].y = v1 ? xs[j].y : 0.f;
        }
      }
      float2 nn = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 16; j++) nn = fma2(xs[j], xs[j], nn);  // = the two scalar fmaf chains
      n0 = nn.x;
      n1 = nn.y;
      // every value of the slot is in registers (the norms consumed them):
      // hand the fp32 slot back to the producer before the conversions
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_t[s]);
      if (st == 0) trace(11, n);
      // finite norms <= 3e38: every |x| <= 2e19, nothing to drop (the common case)
      if (!__all_sync(0xffffffffu, n0 <= 3.0e38f && n1 <= 3.0e38f)) {
#pragma unroll
        for (int j = 0; j < 16; j++) {  // scalar path (and the exact scan: the norm is not finite)
          if (!(fabsf(xs[j].x) <= 3.0e38f)) xs[j].x = 0.f;
          if (!(fabsf(xs[j].y) <= 3.0e38f)) xs[j].y = 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const int l = 16 * half + j;
        const float2 x = xs[j];
        const uint32_t h = bf16x2_rn(x.x, x.y);
        const float2 rr = sub2(x, make_float2(__uint_as_float(h << 16), __uint_as_float(h & 0xffff0000u)));
        const uint32_t r = bf16x2_rn(rr.x, rr.y);
        *reinterpret_cast<uint32_t*>(P + plane_off(0, l, p)) = h;
        *reinterpret_cast<uint32_t*>(P + plane_off(1, l, p)) = r;
      }
      *reinterpret_cast<float2*>(nrm + (b * 2 + half) * kPts + p) = make_float2(n0, n1);
      fence_proxy_async();  // the planes are read by the tensor cores (async proxy)
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_p[b]);
      if (st == 0) trace(3, n);
    }
  } else {  // ---- epilogue: two sets of 4 warps (even / odd tiles); TMEM lanes 32 (warp % 4) + lane
    const int ew = warp & 3, m = 32 * ew + lane, set = (warp - kWEpi) >> 2;
    float cn[16];
    float cmax2 = 0.f, rcmax = 0.f;
    const float* cnrm = reinterpret_cast<const float*>(sm + kOffCn);
#pragma unroll
    for (int c = 0; c < 16; c++) {
      cn[c] = cnrm[c];  // NaN past k: never a candidate, ignored by fminf
      if (c < k) {
        cmax2 = fmaxf(cmax2, cn[c]);
        rcmax = fmaxf(rcmax, cnrm[16 + c]);
      }
    }
    const float cmax = sqrtf(cmax2) * 1.001f;
    // x |f|: 2^-14 cmax (rsqrt approximation + 1 %) + 2 |r_c|
    const float eA = 6.103515625e-05f * 1.01f * cmax + 2.02f * rcmax;
    const float eB = 4.76837158203125e-07f * cmax * cmax + 7.8886e-31f * cmax + 1e-35f;  // 2^-21 cmax^2, 2^-100 cmax
    for (int n = set; n < nmine; n += kEpiSets) {
      const int b = n % kSP;
      const long long p0 = lo + (blockIdx.x + (long long)n * gridDim.x) * kPts;
      const int cntp = (int)min((long long)kPts, hi - p0);
      // full_p as well: orders the split's |f|^2 stores before the loads below
      // (the split cannot complete tile n + kSP before this tile's one-hot exists)
      tg_wait_worker(&full_p[b], (n / kSP) & 1);
      const int a = n % kSA;
      tg_wait_worker(&acc_full[a], (n / kSA) & 1);
      if (m == 0) trace(5, n);
      tc_after();
      float d[32], h[16];  // cols 16..47 (the small terms), 0..15 (hi.hi)
      tmem_ld32_16(tmem + a * kAccCols + ((uint32_t)(32 * ew) << 16), d, h);
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
      const float nr = nrm[(b * 2) * kPts + m] + nrm[(b * 2 + 1) * kPts + m];
      const float E = fmaf(eA, nr * rsqrtf(nr + 1e-30f), eB) + 9.2e-13f * nr;
      float tv[16];
      float mn = INFINITY;
#pragma unroll
      for (int c = 0; c < 16; c++) {
        tv[c] = fmaf(-2.f, h[c] + (d[c] + d[16 + c]), cn[c]);
        mn = fminf(mn, tv[c]);
      }
      const float thr = mn + 2.f * E;
      unsigned cand = 0;
#pragma unroll
      for (int c = 0; c < 16; c++) cand |= (tv[c] <= thr ? 1u : 0u) << c;
      const bool ok = m < cntp;
      const bool fin_ = nr <= 3.0e38f && cand != 0;
      const int best = __ffs(cand) - 1;
      // points whose screen does not decide (several candidates, or a norm
      // that is not finite) are deferred: they get no one-hot entry, so the
      // tile's planes are released before their re-check, and all their
      // features go to the sums on the scalar path
      const bool defer = ok && (!fin_ || (cand & (cand - 1)));
      unsigned char* O = sm + stage_onehot(b);
      {  // zero this warp's 32 one-hot columns (16 rows x 64 B), then set the ones
        const int i0 = 2 * lane;
#pragma unroll
        for (int i = i0; i < i0 + 2; i++) {
          const int c = i >> 2, jj = i & 3;
          *reinterpret_cast<uint4*>(O + onehot_off(c, 32 * ew + 8 * jj)) = make_uint4(0, 0, 0, 0);
        }
      }
      __syncwarp();
      if (ok && !defer) {
        member[p0 + m] = best;
        atomicAdd(cnt + best, 1);
        *reinterpret_cast<unsigned short*>(O + onehot_off(best, m)) = 0x3F80;  // bf16 1.0
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oh_full[b]);
      // deferred points, up to 4 per round, lanes over the features (their
      // loads issued together; the lines went through L2 microseconds ago):
      // the candidates' f32 distances in the difference form (a tree sum,
      // |d32 - d| <= (nf + 4) 2^-24 d in any order); one survivor decides,
      // several (true ties) take the f64 recurrence on the point's lane, as
      // does the full reference scan of a point whose norm is not finite
      const float* fg = f + p0 + 32 * ew;  // the warp's points in global memory
      unsigned dm = __ballot_sync(0xffffffffu, defer);
      while (dm) {
        int srcs[4];
        float xs[4];
        int nq = 0;
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (dm) {
            srcs[q] = __ffs(dm) - 1;
            dm &= dm - 1;
            xs[q] = __ldg(fg + (long long)lane * npts + srcs[q]);
            nq = q + 1;
          }
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (q >= nq) break;
          const int src = srcs[q];
          const float x = xs[q];
          const unsigned cs = __shfl_sync(0xffffffffu, cand, src);
          const bool sfin = __shfl_sync(0xffffffffu, fin_ ? 1 : 0, src) != 0;
          int pick = 0;
          if (sfin) {
            const float e2 = (float)(kNF + 4) * 5.9604645e-08f * 1.01f;
            float myd = INFINITY, u2 = INFINITY;
            for (unsigned r = cs; r; r &= r - 1) {
              const int c = __ffs(r) - 1;
              const float dl = __fsub_rn(x, cf[c * kNF + lane]);
              float v = __fmul_rn(dl, dl);
#pragma unroll
              for (int o = 16; o >= 1; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
              if (lane == c) myd = v;
              u2 = fminf(u2, fmaf(v, e2, v) + 1e-40f);
            }
            const unsigned sv =
                __ballot_sync(0xffffffffu, ((cs >> lane) & 1) && !(fmaf(-myd, e2, myd) - 1e-40f > u2));
            if (lane == src) pick = (sv & (sv - 1)) ? exact_mask_g(fg + lane, npts, cf, sv) : __ffs(sv) - 1;
          } else if (lane == src) {
            pick = exact_g(fg + lane, npts, cf, k);
          }
          pick = __shfl_sync(0xffffffffu, pick, src);
          if (lane == src) {
            member[p0 + 32 * ew + src] = pick;
            atomicAdd(cnt + pick, 1);
          }
          atomicAdd(ssx + pick * kNF + lane, x);  // feature `lane` of the point (NaN / inf included)
        }
      }
      if (m == 0) trace(6, n);
        }
    if (nmine > 0 && set == 0) {  // the sums accumulator: lane r = 64 parity + 32 P + feature
      mbar_wait(fin, 0);
      tc_after();
      float v[16];
      // rows 0..63 (even stages) x cols 0..15, rows 64..127 (odd stages) x cols 16..31
      tmem_ld16(tmem + kSumsCol + (ew >= 2 ? 16u : 0u) + ((uint32_t)(32 * ew) << 16), v);
      if (ew < 2 || nmine >= 2) {  // odd-stage rows exist (and were initialised) only with two tiles
#pragma unroll
        for (int c = 0; c < 16; c++)
          if (c < k && v[c] != 0.f) atomicAdd(sums + c * kNF + lane, v[c]);
      }
    }
  }
  tc_before();
  __syncthreads();
  for (int i = tid; i < k * kNF; i += blockDim.x)
    if (ssx[i] != 0.f) atomicAdd(sums + i, ssx[i]);
  for (int i = tid; i < k; i += blockDim.x)
    if (cnt[i]) atomicAdd(counts + i, cnt[i]);
  if (warp == kWMma) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// 2D tensor map over the feature-major points: dims {npts, 32}, box {128, 32}
static bool kmeans_tile_map(CUtensorMap* m, const void* f, long long npts) {
  static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!enc || npts > INT_MAX || ((uintptr_t)f & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)npts, (cuuint64_t)tg::kNF};
  cuuint64_t strides[1] = {(cuuint64_t)npts * 4};
  cuuint32_t box[2] = {(cuuint32_t)tg::kPts, (cuuint32_t)tg::kNF}, es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(f), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int kmeans_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_KMEANS_V");
    v = e ? atoi(e) : 5;  // 5: kmeans_tg (nf = 32, else as 4); 4: kmeans_tc; 2/3: kmeans_rb; 1: kmeans_fast
  }
  return v;
}

static int launch_kmeans(LaunchCtx& ctx) {
  const ArgVal& F = ctx.args[0];
  const ArgVal& Ce = ctx.args[1];
  const ArgVal& M = ctx.args[2];
  const ArgVal& S = ctx.args[3];
  const ArgVal& Cn = ctx.args[4];
  const long long npts = ctx.args[5].i32;
  const int nf = ctx.args[6].i32 > 0 ? ctx.args[6].i32 : 0;
  const int k = ctx.args[7].i32;
  const long long bx = ctx.block[0];
  const long long m = (long long)ctx.block[1] * ctx.block[2];
  if (m != 1 || ctx.grid[1] * (long long)ctx.grid[2] != 1) {
    // duplicated threads would add the same point several times; only the
    // 1D geometry is implemented
    *ctx.error = "kmeans: only 1D grids/blocks are supported";
    return BF_E_UNSUPPORTED;
  }
  const int kc = k > 0 ? k : 1;
  if ((long long)nf * npts > INT_MAX || (long long)kc * nf > 4096) {
    *ctx.error = "kmeans: nf*npts beyond i32 or k*nf above 4096";
    return BF_E_UNSUPPORTED;
  }
  for (auto& xi : ctx.x_intervals()) {
    long long lo = xi.first * bx, hi = std::min(xi.second * bx, npts);
    if (lo >= hi) continue;
    bool ok = (long long)nf * npts <= F.len && (long long)(k > 0 ? k : 0) * nf <= Ce.len &&
              hi <= M.len && (long long)kc * nf <= S.len && kc <= Cn.len;
    if (!ok) {
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(xi.first), "kmeans index out of range");
      continue;
    }
    CUtensorMap tmap;
    if (kmeans_variant() >= 5 && nf == 32 && k >= 2 && k <= 16 && npts % 4 == 0 && lo % 4 == 0 && hi - lo >= 4 &&
        kmeans_tile_map(&tmap, F.ptr, npts)) {
      const long long main_hi = lo + (hi - lo) / 4 * 4;
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        cudaFuncSetAttribute(kmeans_tg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tg::kSmem);
        cudaGetLastError();
      }
      const int grid = stream_grid(main_hi - lo, tg::kPts, ctx.num_sms, 1);
      kmeans_tg<<<grid, tg::kThreads, tg::kSmem, ctx.stream>>>(tmap, (const float*)F.ptr, (const float*)Ce.ptr,
                                                               (int*)M.ptr, (float*)S.ptr, (int*)Cn.ptr, (int)npts,
                                                               k, lo, main_hi);
      BF_CUDA_LAUNCH_CHECK(ctx);
      if (main_hi == hi) continue;
      lo = main_hi;  // < 4 trailing points: register-blocked path below
    }
    if (kmeans_variant() >= 4 && (nf == 32 || nf == 16 || nf == 24 || nf == 8) && k >= 2 && k <= 16 &&
        npts % 4 == 0 && lo % 4 == 0 && hi - lo >= 4) {
      const long long main_hi = lo + (hi - lo) / 4 * 4;
      auto fn = nf == 32 ? kmeans_tc<32> : nf == 24 ? kmeans_tc<24> : nf == 16 ? kmeans_tc<16> : kmeans_tc<8>;
      const size_t smem = nf == 32 ? kmeans_tc_smem<32>() : nf == 24 ? kmeans_tc_smem<24>()
                        : nf == 16 ? kmeans_tc_smem<16>() : kmeans_tc_smem<8>();
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        cudaFuncSetAttribute(kmeans_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kmeans_tc_smem<32>());
        cudaFuncSetAttribute(kmeans_tc<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kmeans_tc_smem<24>());
        cudaFuncSetAttribute(kmeans_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kmeans_tc_smem<16>());
        cudaFuncSetAttribute(kmeans_tc<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kmeans_tc_smem<8>());
        cudaGetLastError();
      }
      const int grid = stream_grid(main_hi - lo, kTcPts, ctx.num_sms, KM_TC_MINB);
      fn<<<grid, 32 * (kTcWarps + 1), smem, ctx.stream>>>((const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr,
                                                          (float*)S.ptr, (int*)Cn.ptr, (int)npts, k, lo, main_hi);
      BF_CUDA_LAUNCH_CHECK(ctx);
      if (main_hi == hi) continue;
      lo = main_hi;  // < 4 trailing points: register-blocked path below
    }
    if (kmeans_variant() >= 2 && (nf == 32 || nf == 16 || nf == 8 || nf == 4) && kc * nf <= 1024) {
      const int kg = (kc + 3) / 4;
      size_t smem = sizeof(float) * ((size_t)kg * 4 * nf + (size_t)kc * nf + 12 * kg +
                                     kKmWarps * 32 * 33 + (size_t)kKmWarps * kc * nf) +
                    sizeof(int) * kc;
      const bool one = kmeans_variant() == 3;
      auto fn = nf == 32 ? (one ? kmeans_rb<32, 1> : kmeans_rb<32, 2>) : nf == 16 ? kmeans_rb<16, 2>
              : nf == 8 ? kmeans_rb<8, 2> : kmeans_rb<4, 2>;
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        for (auto g : {kmeans_rb<32, 1>, kmeans_rb<32, 2>, kmeans_rb<16, 2>, kmeans_rb<8, 2>, kmeans_rb<4, 2>})
          cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        cudaGetLastError();
      }
      int grid = stream_grid(hi - lo, 256 * 2, ctx.num_sms, 2);
      fn<<<grid, 256, smem, ctx.stream>>>((const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr,
                                          (float*)S.ptr, (int*)Cn.ptr, (int)npts, k, lo, hi);
      BF_CUDA_LAUNCH_CHECK(ctx);
      continue;
    }
    if (nf <= kKmMaxF && kc * nf <= 1024) {
      size_t smem = sizeof(float) * ((size_t)kc * nf + 3 * kc + kKmWarps * 32 * 33 +
                                     (size_t)kKmWarps * kc * nf) + sizeof(int) * kc;
      auto fn = nf == 32 ? kmeans_fast<32> : nf == 16 ? kmeans_fast<16> : nf == 8 ? kmeans_fast<8>
              : nf == 4 ? kmeans_fast<4> : kmeans_fast<0>;
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        for (auto g : {kmeans_fast<32>, kmeans_fast<16>, kmeans_fast<8>, kmeans_fast<4>, kmeans_fast<0>})
          cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaGetLastError();
      }
      int grid = stream_grid(hi - lo, 256 * 4, ctx.num_sms, 4);
      fn<<<grid, 256, smem, ctx.stream>>>((const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr,
                                          (float*)S.ptr, (int*)Cn.ptr, (int)npts, nf, k, lo, hi);
      BF_CUDA_LAUNCH_CHECK(ctx);
      continue;
    }
    size_t smem = (size_t)kc * nf * (sizeof(double) + sizeof(float)) + kc * sizeof(int);
    int grid = stream_grid(hi - lo, 256 * 4, ctx.num_sms, 4);
    if (nf <= kKmMaxF) {
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        cudaFuncSetAttribute(kmeans_assign<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      }
      kmeans_assign<true><<<grid, 256, smem, ctx.stream>>>(
          (const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr, (float*)S.ptr, (int*)Cn.ptr,
          (int)npts, nf, k, lo, hi);
    } else {
      static bool attr[64] = {};
      if (first_on_device(attr)) {
        cudaFuncSetAttribute(kmeans_assign<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      }
      kmeans_assign<false><<<grid, 256, smem, ctx.stream>>>(
          (const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr, (float*)S.ptr, (int*)Cn.ptr,
          (int)npts, nf, k, lo, hi);
    }
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_kmeans("kmeans",
                            {{BF_SLOT_HANDLE, BF_F32, "f"},
                             {BF_SLOT_HANDLE, BF_F32, "cent"},
                             {BF_SLOT_HANDLE, BF_I32, "member"},
                             {BF_SLOT_HANDLE, BF_F32, "sums"},
                             {BF_SLOT_HANDLE, BF_I32, "counts"},
                             {BF_SLOT_I32, BF_I32, "npts"},
                             {BF_SLOT_I32, BF_I32, "nf"},
                             {BF_SLOT_I32, BF_I32, "k"}},
                            launch_kmeans);

}  // namespace bf

// ---- Rodinia kmeans host loop, device part (cluster.kmeans_iterate) -------
// After an assignment launch (and, across ranks, the all-reduce of sums and
// counts): new centroid = sums / counts in f32 where the count is non-zero
// (kmeans_clustering.c: clusters[i][j] = new_centers[i][j] /
// new_centers_len[i]), sums and counts cleared for the next pass, and the
// number of points in [p_lo, p_hi) whose membership changed since the
// previous pass (Rodinia's delta), with prev := member.
namespace bf {
__global__ void kmeans_centroids(float* cent, float* sums, int* counts, int nf, int k) {
  for (int i = threadIdx.x; i < k * nf; i += blockDim.x) {
    const int c = i / nf, n = counts[c];
    if (n > 0) cent[i] = __fdiv_rn(sums[i], (float)n);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * nf; i += blockDim.x) sums[i] = 0.f;
  for (int i = threadIdx.x; i < k; i += blockDim.x) counts[i] = 0;
}

__global__ void __launch_bounds__(256) kmeans_delta(const int* __restrict__ member, int* prev, long long lo,
                                                    long long hi, unsigned long long* delta) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned c = 0;
  // 16 B vectors over the 4-aligned middle (two in flight per thread), prev
  // rewritten only where a membership changed; scalar head and tail
  const long long a0 = (lo + 3) & ~3LL, a1 = hi & ~3LL;
  if (a0 < a1) {
    const int4* m4 = reinterpret_cast<const int4*>(member + a0);
    int4* p4 = reinterpret_cast<int4*>(prev + a0);
    const long long nv4 = (a1 - a0) / 4;
    for (long long i = tid; i < nv4; i += 2 * stride) {
      const bool two = i + stride < nv4;
      const int4 m = __ldcs(m4 + i), q = p4[i];
      int4 m2 = make_int4(0, 0, 0, 0), q2 = m2;
      if (two) {
        m2 = __ldcs(m4 + i + stride);
        q2 = p4[i + stride];
      }
      const unsigned d = (m.x != q.x) + (m.y != q.y) + (m.z != q.z) + (m.w != q.w);
      const unsigned d2 = (m2.x != q2.x) + (m2.y != q2.y) + (m2.z != q2.z) + (m2.w != q2.w);
      if (d) p4[i] = m;
      if (d2) p4[i + stride] = m2;
      c += d + d2;
    }
  }
  for (long long p = lo + tid; p < hi && p < a0; p += stride) {
    const int m = member[p];
    c += m != prev[p];
    prev[p] = m;
  }
  for (long long p = (a1 > a0 ? a1 : a0) + tid; p < hi; p += stride) {
    const int m = member[p];
    c += m != prev[p];
    prev[p] = m;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned wsum[8];  // one atomic per CTA, not per warp (a single hot address)
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += wsum[w];
    if (t) atomicAdd(delta, t);
  }
}
}  // namespace bf

namespace bf {
struct KmUpdateScratch : StreamScratch {
  unsigned long long* d = nullptr;  // device delta counter
  unsigned long long* h = nullptr;  // pinned read-back
  void release() {
    if (d) cudaFree(d);
    if (h) cudaFreeHost(h);
    d = h = nullptr;
  }
  ~KmUpdateScratch() override { release(); }
};
}  // namespace bf

extern "C" int bf_kmeans_update_impl(void* stream_v, int num_sms, float* cent, float* sums, int* counts, int nf,
                                     int k, const int* member, int* prev, long long p_lo, long long p_hi,
                                     long long* delta, char* err, int errcap) {
  using namespace bf;
  cudaStream_t stream = (cudaStream_t)stream_v;
  // the delta counter and its pinned read-back, keyed by the stream (several
  // runtimes or host threads never share them)
  KmUpdateScratch& S = scratch_for<KmUpdateScratch>(stream, SCRATCH_KM_UPDATE);
  if (!S.d) {
    if (cudaMalloc((void**)&S.d, 8) != cudaSuccess || cudaMallocHost((void**)&S.h, 8) != cudaSuccess) {
      snprintf(err, errcap, "kmeans_update: scratch allocation failed");
      cudaGetLastError();
      S.release();
      return BF_E_CUDA;
    }
  }
  unsigned long long* d = S.d;
  unsigned long long* h = S.h;
  kmeans_centroids<<<1, 512, 0, stream>>>(cent, sums, counts, nf, k);
  cudaMemsetAsync(d, 0, 8, stream);
  if (p_hi > p_lo) {
    const int grid = wave_grid(kmeans_delta, 256, 0, (p_hi - p_lo + 7) / 8, 256, num_sms, 8);
    kmeans_delta<<<grid, 256, 0, stream>>>(member, prev, p_lo, p_hi, d);
  }
  cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, stream);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "kmeans_update: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  *delta = (long long)*h;
  return BF_OK;
}
