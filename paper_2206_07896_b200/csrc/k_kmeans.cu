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
