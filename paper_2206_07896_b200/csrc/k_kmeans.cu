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
    if (nf <= kKmMaxF && kc * nf <= 1024) {
      size_t smem = sizeof(float) * ((size_t)kc * nf + 3 * kc + kKmWarps * 32 * 33 +
                                     (size_t)kKmWarps * kc * nf) + sizeof(int) * kc;
      auto fn = nf == 32 ? kmeans_fast<32> : nf == 16 ? kmeans_fast<16> : nf == 8 ? kmeans_fast<8>
              : nf == 4 ? kmeans_fast<4> : kmeans_fast<0>;
      static bool attr = false;
      if (!attr) {
        for (auto g : {kmeans_fast<32>, kmeans_fast<16>, kmeans_fast<8>, kmeans_fast<4>, kmeans_fast<0>})
          cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaGetLastError();
        attr = true;
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
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(kmeans_assign<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr = true;
      }
      kmeans_assign<true><<<grid, 256, smem, ctx.stream>>>(
          (const float*)F.ptr, (const float*)Ce.ptr, (int*)M.ptr, (float*)S.ptr, (int*)Cn.ptr,
          (int)npts, nf, k, lo, hi);
    } else {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(kmeans_assign<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr = true;
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
