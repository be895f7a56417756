// kmeans_t5 — the kmeans assignment (kernels/kmeans.kn, Rodinia kmeansPoint
// plus the centroid accumulation) as a warp-specialised tcgen05 pipeline
// (nf == 32, 2 <= k <= 16, npts % 4 == 0).  Same results as kmeans_tc
// (k_kmeans.cu): membership and counts bit-exact (the tensor-core screen with
// its proven error bound, the reference's exact f64 recurrence for near-ties
// and non-finite points), sums within the stated tolerance.
//
// Per 128-point tile (thread p of the four epilogue warps <-> point p <->
// TMEM lane p), stage s of a 2-deep ring:
//   TMA     one warp loads the tile with four 2D tensor-map boxes
//           {32 points, 32 features}, SWIZZLE_128B: raw[block][feature][32
//           points] (feature-major global layout -> an MN-major operand);
//   split   thread p reads its 32 features (conflict-free swizzled LDS),
//           writes lo = x - trunc_tf32(x) as its own K-major SW128 row (eight
//           16 B stores) and |x|^2 for the screen bound;
//   dist    one thread issues D_hh = raw B_hi, D_x = raw B_lo + lo B_hi
//           (M = 128 points, N = 16 clusters, K = 32, kind::tf32: the tensor
//           core truncates raw to TF32, lo restores it) into TMEM buffer
//           t & 1 (double-buffered: the MMAs of tile t+1 run while tile t is
//           screened);
//   screen  tcgen05.ld gives thread p its 2 x 16 cluster values; the bound
//           and the candidate rule are kmeans_tc's (k_kmeans.cu header);
//           several candidates or a non-finite point: the exact f64
//           recurrence over the candidates, features from the raw tile;
//   sums    thread p writes its one-hot column (K-major SW128 [cluster][point]),
//           and one thread accumulates S[l][c] += raw^T onehot + lo^T onehot
//           (the raw tile read K-major, the lo tile read MN-major: M = the 32
//           feature rows, K = points) into a TMEM accumulator kept for the
//           whole kernel; the commit releases the stage to the TMA warp.
// Counts by warp ballots; points outside the task range or non-finite have
// their raw column / lo row zeroed before the sums MMA (0 x NaN would poison
// every cluster) and non-finite ones add their features on a scalar path.
// HBM is read exactly once (128 B per point) plus 4 B per point written.
// Descriptor layouts: scripts/micro/umma_sw128.cu (probed on the device).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstring>
#include <mutex>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

namespace {

constexpr int kT5Stages = 2;
constexpr int kT5Pts = 128;
constexpr int kT5Raw = 16384;   // [4 blocks][32 features][128 B]
constexpr int kT5Lo = 16384;    // [128 points][128 B]
constexpr int kT5Oh = 8192;     // [4 blocks][16 clusters][128 B]
constexpr int kT5Stage = kT5Raw + kT5Lo + kT5Oh;

__device__ __forceinline__ uint64_t t5_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t t5_idesc(bool a_mn, bool b_mn) {  // kind::tf32, f32 accumulate, M 128, N 16
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void t5_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void t5_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void t5_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void t5_tma2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// byte offset of (feature l, point q of a 32-point block) in a raw block
__device__ __forceinline__ int t5_raw_off(int l, int q) { return l * 128 + ((((q >> 2) ^ (l & 7))) << 4) + (q & 3) * 4; }

}  // namespace

__global__ void __launch_bounds__(192, 2) kmeans_t5(const __grid_constant__ CUtensorMap tmap,
                                                    const float* __restrict__ f, const float* __restrict__ cent,
                                                    int* __restrict__ member, float* sums, int* counts, int npts,
                                                    int k, long long lo, long long hi) {
  constexpr int NF = 32;
  extern __shared__ __align__(1024) unsigned char t5raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(t5raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* stages = sm;                                               // kT5Stages x kT5Stage
  uint32_t* Bhi = reinterpret_cast<uint32_t*>(sm + kT5Stages * kT5Stage);  // 2 KB
  uint32_t* Blo = Bhi + 512;                                                // 2 KB
  // 16 KB of slack after the B tiles: the M = 128 sums operands read past
  // their 32 feature rows (those accumulator rows are discarded)
  float* cf = reinterpret_cast<float*>(Blo + 512 + 4096);  // [16][32]
  float* cn2 = cf + 16 * NF;                                // [16]
  float* ssum = cn2 + 16;                                   // [16][32] scalar-path sums
  int* cnt = reinterpret_cast<int*>(ssum + 16 * NF);        // [16]
  uint64_t* full = reinterpret_cast<uint64_t*>(cnt + 16);
  uint64_t* lo_ready = full + kT5Stages;
  uint64_t* oh_ready = lo_ready + kT5Stages;
  uint64_t* empty = oh_ready + kT5Stages;
  uint64_t* dist_done = empty + kT5Stages;  // [2]
  uint64_t* sums_done = dist_done + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sums_done + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 16 * NF; i += blockDim.x) {
    cf[i] = i < k * NF ? cent[i] : 0.f;
    ssum[i] = 0.f;
  }
  if (tid < 16) cnt[tid] = 0;
  if (tid == 0) {
    for (int s = 0; s < kT5Stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&lo_ready[s], 128);
      mbar_init(&oh_ready[s], 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&dist_done[0], 1);
    mbar_init(&dist_done[1], 1);
    mbar_init(sums_done, 1);
    fence_barrier_init();
  }
  if (warp == 5) {  // TMEM: D_hh / D_x of buffer b at 32b / 32b+16, sums at 64
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid < 16) {
    float n2 = 0.f;
    for (int l = 0; l < NF; l++) n2 = fmaf(cf[tid * NF + l], cf[tid * NF + l], n2);
    cn2[tid] = tid < k ? n2 : INFINITY;
  }
  // centroid operands, K-major SWIZZLE_NONE: (c, l) at (c%8)*16 + (c/8)*128 + (l/4)*256 + (l%4)*4 bytes;
  // hi = RN_tf32(c), lo = trunc_tf32(c - hi)
  for (int i = tid; i < 16 * NF; i += blockDim.x) {
    const int c = i / NF, l = i % NF;
    const float x = cf[i];
    const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    const uint32_t lw = __float_as_uint(x - __uint_as_float(h)) & 0xffffe000u;
    const int w = ((c & 7) * 16 + (c >> 3) * 128 + (l >> 2) * 256) / 4 + (l & 3);
    Bhi[w] = h;
    Blo[w] = lw;
  }
  fence_proxy_async();
  t5_fence_before();
  __syncthreads();
  t5_fence_after();
  const uint32_t tbase = *tmem_slot;
  const long long ntile = (hi - lo + kT5Pts - 1) / kT5Pts;
  int my_tiles = 0;
  if ((long long)blockIdx.x < ntile) my_tiles = (int)((ntile - 1 - blockIdx.x) / gridDim.x) + 1;

  if (warp == 4) {  // ---- TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int n = 0; n < my_tiles; n++) {
        const int s = n % kT5Stages;
        if (n >= kT5Stages) mbar_wait_sleep(&empty[s], ((n / kT5Stages) - 1) & 1);
        const long long p0 = lo + ((long long)blockIdx.x + (long long)n * gridDim.x) * kT5Pts;
        unsigned char* raw = stages + s * kT5Stage;
        mbar_arrive_expect_tx(&full[s], kT5Raw);
#pragma unroll
        for (int b = 0; b < 4; b++) t5_tma2d(raw + b * 4096, &tmap, (int)(p0 + 32 * b), 0, &full[s], pol);
      }
    }
  } else if (warp == 5) {  // ---- MMA issuer
    if (lane == 0) {
      const uint32_t sBhi = smem_u32(Bhi), sBlo = smem_u32(Blo);
      const uint32_t id_mn = t5_idesc(true, false), id_k = t5_idesc(false, false);
      auto dist = [&](int n) {
        const int s = n % kT5Stages, b = n & 1;
        mbar_wait(&lo_ready[s], (n / kT5Stages) & 1);
        t5_fence_after();
        const uint32_t sraw = smem_u32(stages + s * kT5Stage), slo = sraw + kT5Raw;
        const uint32_t dh = tbase + 32 * b, dx = dh + 16;
#pragma unroll
        for (int kt = 0; kt < NF / 8; kt++) {
          const uint64_t ar = t5_desc(sraw + kt * 1024, 4096, 1024, 2);  // MN-major SW128
          const uint64_t al = t5_desc(slo + kt * 32, 16, 1024, 2);       // K-major SW128
          const uint64_t bh = t5_desc(sBhi + kt * 512, 256, 128, 0), bl = t5_desc(sBlo + kt * 512, 256, 128, 0);
          t5_mma(dh, ar, bh, id_mn, kt > 0);
          t5_mma(dx, ar, bl, id_mn, kt > 0);
          t5_mma(dx, al, bh, id_k, 1u);
        }
        t5_commit(&dist_done[b]);
      };
      auto sums = [&](int n) {
        const int s = n % kT5Stages;
        mbar_wait(&oh_ready[s], (n / kT5Stages) & 1);
        t5_fence_after();
        const uint32_t sraw = smem_u32(stages + s * kT5Stage), slo = sraw + kT5Raw, soh = slo + kT5Lo;
#pragma unroll
        for (int b = 0; b < 4; b++)
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            const uint64_t ar = t5_desc(sraw + b * 4096 + kk * 32, 16, 1024, 2);     // raw read K-major
            const uint64_t al = t5_desc(slo + b * 4096 + kk * 1024, 4096, 1024, 2);  // lo read MN-major
            const uint64_t bo = t5_desc(soh + b * 2048 + kk * 32, 16, 1024, 2);
            t5_mma(tbase + 64, ar, bo, id_k, (n > 0 || b > 0 || kk > 0) ? 1u : 0u);
            t5_mma(tbase + 64, al, bo, id_mn, 1u);
          }
        t5_commit(&empty[s]);
        if (n == my_tiles - 1) t5_commit(sums_done);
      };
      if (my_tiles > 0) dist(0);
      for (int n = 0; n < my_tiles; n++) {
        if (n + 1 < my_tiles) dist(n + 1);
        sums(n);
      }
    }
  } else {  // ---- epilogue: thread p <-> point p <-> TMEM lane p
    const int p = tid, blk = p >> 5, q = p & 31;
    float cmax2 = 0.f;
    for (int c = 0; c < k; c++) cmax2 = fmaxf(cmax2, cn2[c]);
    const float cmax = sqrtf(cmax2) * 1.001f;
    const float eA = 1.52587890625e-05f * 1.03f * 2.f * cmax;
    const float eB = 1.52587890625e-05f * 1.03f * cmax * cmax + 1e-35f;
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    const int lorow = (p >> 3) * 1024 + (p & 7) * 128;  // byte offset of point p's lo row
    float fn2_cur = 0.f, fn2_next = 0.f;
    bool ok_cur = false, ok_next = false;  // finite, in range
    auto split = [&](int n) {
      const int s = n % kT5Stages;
      const long long p0 = lo + ((long long)blockIdx.x + (long long)n * gridDim.x) * kT5Pts;
      const bool valid = p0 + p < hi;
      mbar_wait(&full[s], (n / kT5Stages) & 1);
      unsigned char* raw = stages + s * kT5Stage + blk * 4096;
      unsigned char* lot = stages + s * kT5Stage + kT5Raw + lorow;
      float n2 = 0.f;
#pragma unroll
      for (int j = 0; j < NF / 4; j++) {
        float x[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          x[u] = *reinterpret_cast<const float*>(raw + t5_raw_off(4 * j + u, q));
          r[u] = x[u] - __uint_as_float(__float_as_uint(x[u]) & 0xffffe000u);
          n2 = fmaf(x[u], x[u], n2);
        }
        *reinterpret_cast<float4*>(lot + ((j ^ (p & 7)) << 4)) = make_float4(r[0], r[1], r[2], r[3]);
      }
      const bool ok = valid && n2 <= 3.0e38f;
      if (!ok) {  // outside the range or non-finite / huge: zero the operands (exact path)
#pragma unroll
        for (int l = 0; l < NF; l++) *reinterpret_cast<float*>(raw + t5_raw_off(l, q)) = 0.f;
#pragma unroll
        for (int j = 0; j < NF / 4; j++)
          *reinterpret_cast<float4*>(lot + ((j ^ (p & 7)) << 4)) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      fn2_next = n2;
      ok_next = ok;
      fence_proxy_async();
      mbar_arrive(&lo_ready[s]);
    };
    if (my_tiles > 0) split(0);
    for (int n = 0; n < my_tiles; n++) {
      const int s = n % kT5Stages, b = n & 1;
      fn2_cur = fn2_next;
      ok_cur = ok_next;
      if (n + 1 < my_tiles) split(n + 1);  // the next tile's MMAs overlap this screen
      const long long p0 = lo + ((long long)blockIdx.x + (long long)n * gridDim.x) * kT5Pts;
      const bool valid = p0 + p < hi;
      mbar_wait(&dist_done[b], (n >> 1) & 1);
      t5_fence_after();
      float dh[16], dx[16];
      t5_ld16(tbase + 32 * b + lane_off, dh);
      t5_ld16(tbase + 32 * b + 16 + lane_off, dx);
      const float fn2 = fn2_cur;
      const float E = fmaf(eA, fn2 * rsqrtf(fn2 + 1e-30f) * 1.01f, eB) + 9.2e-13f * fn2;
      float tv[16];
      float m = INFINITY;
#pragma unroll
      for (int c = 0; c < 16; c++) {
        tv[c] = fmaf(-2.f, dh[c] + dx[c], cn2[c]);
        m = fminf(m, tv[c]);
      }
      const float thr = m + 2.f * E;
      unsigned cm = 0;
#pragma unroll
      for (int c = 0; c < 16; c++) cm |= (tv[c] <= thr ? 1u : 0u) << c;
      const int nc = __popc(cm);
      int best = cm ? __ffs(cm) - 1 : 0;
      const bool fin = ok_cur && nc >= 1;
      const unsigned char* raw = stages + s * kT5Stage + blk * 4096;
      if (valid && (!fin || nc > 1)) {
        // the reference's exact recurrence over the candidates (all clusters
        // when the screen is not usable); features from the raw tile, or from
        // global memory when the point's column was zeroed
        double bd = 0.0;
        int bi = 0;
        bool first = true;
        const unsigned cand = fin ? cm : ((1u << k) - 1u);
        for (unsigned r = cand; r; r &= r - 1) {
          const int c = __ffs(r) - 1;
          double dist = 0.0;
          for (int l = 0; l < NF; l++) {
            const float xv = ok_cur ? *reinterpret_cast<const float*>(raw + t5_raw_off(l, q))
                                    : f[(long long)l * npts + p0 + p];
            const double diff = dsub((double)xv, (double)cf[c * NF + l]);
            dist = dadd(dist, dmul(diff, diff));
          }
          if (first || dist < bd) {
            bd = dist;
            bi = c;
            first = false;
          }
        }
        best = bi;
      }
      if (valid) {
        member[p0 + p] = best;
        if (!ok_cur)
          for (int l = 0; l < NF; l++) atomicAdd(ssum + best * NF + l, f[(long long)l * npts + p0 + p]);
      }
      // counts by ballots (one shared atomic per cluster present in the warp)
      for (int c = 0; c < k; c++) {
        const unsigned bal = __ballot_sync(0xffffffffu, valid && best == c);
        if (lane == 0 && bal) atomicAdd(cnt + c, __popc(bal));
      }
      // one-hot column of point p: [cluster c][point q] K-major SW128, block blk
      unsigned char* oh = stages + s * kT5Stage + kT5Raw + kT5Lo + blk * 2048;
      const int sel = (valid && ok_cur) ? best : -1;
#pragma unroll
      for (int c = 0; c < 16; c++)
        *reinterpret_cast<float*>(oh + (c >> 3) * 1024 + (c & 7) * 128 + (((q >> 2) ^ (c & 7)) << 4) + (q & 3) * 4) =
            c == sel ? 1.f : 0.f;
      fence_proxy_async();
      t5_fence_before();
      mbar_arrive(&oh_ready[s]);
    }
  }
  // ---- drain: the sums accumulator (lanes 0-31 = features) and counts
  if (warp < 4 && my_tiles > 0) {
    mbar_wait(sums_done, 0);
    t5_fence_after();
    if (warp == 0) {
      float v[16];
      t5_ld16(tbase + 64, v);
      for (int c = 0; c < k; c++) {
        const float x = v[c] + ssum[c * NF + lane];
        if (x != 0.f) atomicAdd(sums + c * NF + lane, x);
      }
    }
  }
  t5_fence_before();
  __syncthreads();
  if (warp == 5) {
    t5_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
  }
  if (my_tiles == 0) return;
  for (int i = tid; i < k; i += blockDim.x)
    if (cnt[i]) atomicAdd(counts + i, cnt[i]);
}

static size_t kmeans_t5_smem() {
  return 1024 + kT5Stages * kT5Stage + 4096 + 16384 + sizeof(float) * (16 * 32 + 16 + 16 * 32) + sizeof(int) * 16 +
         sizeof(uint64_t) * (4 * kT5Stages + 3) + 16;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 t5_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

int launch_kmeans_t5(LaunchCtx& ctx, const float* f, const float* cent, int* member, float* sums, int* counts,
                     int npts, int nf, int k, long long lo, long long hi) {
  if (nf != 32 || k < 2 || k > 16 || npts % 4 != 0 || hi <= lo) return BF_E_UNSUPPORTED;
  auto enc = t5_encoder();
  if (!enc) return BF_E_UNSUPPORTED;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)npts, (cuuint64_t)nf};
  cuuint64_t strides[1] = {(cuuint64_t)npts * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(f), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return BF_E_UNSUPPORTED;
  const size_t smem = kmeans_t5_smem();
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(kmeans_t5, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kmeans_t5, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaGetLastError();
  }
  const long long ntile = (hi - lo + kT5Pts - 1) / kT5Pts;
  const int grid = (int)std::min<long long>(ntile, (long long)ctx.num_sms * 2);
  kmeans_t5<<<grid, 192, smem, ctx.stream>>>(tm, f, cent, member, sums, counts, npts, k, lo, hi);
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

}  // namespace bf
