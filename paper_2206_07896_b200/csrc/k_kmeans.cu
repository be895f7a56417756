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
#include <cuda_bf16.h>

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

static int kmeans_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_KMEANS_V");
    v = e ? atoi(e) : 4;  // 4: kmeans_tc; 2/3: kmeans_rb; 1: kmeans_fast
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

extern "C" int bf_kmeans_update_impl(void* stream_v, int num_sms, float* cent, float* sums, int* counts, int nf,
                                     int k, const int* member, int* prev, long long p_lo, long long p_hi,
                                     long long* delta, char* err, int errcap) {
  using namespace bf;
  cudaStream_t stream = (cudaStream_t)stream_v;
  static unsigned long long* dd[64] = {};  // per-device scratch counter + pinned read-back
  static unsigned long long* hh[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  unsigned long long*& d = dd[dev & 63];
  unsigned long long*& h = hh[dev & 63];
  if (!d) {
    if (cudaMalloc((void**)&d, 8) != cudaSuccess || cudaMallocHost((void**)&h, 8) != cudaSuccess) {
      snprintf(err, errcap, "kmeans_update: scratch allocation failed");
      cudaGetLastError();
      d = nullptr;
      return BF_E_CUDA;
    }
  }
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
