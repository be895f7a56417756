// backprop — paper_2206_07896_b200/kernels/backprop.kn (Rodinia backprop's
// device kernels bpnn_layerforward_CUDA and bpnn_adjust_weights_cuda).
//
// Geometry: Rodinia's 16 x 16 blocks on a 1 x (in/16) grid with hid = 16
// (the kernel's tile is 16 wide, so Rodinia requires hid == 16); logical
// block `by` owns weight rows 16by+1 .. 16by+16, columns 1..16, i.e. the
// 272 contiguous floats w[272by + 17 .. 272by + 288] of the row-major
// [(in+1) x 17] matrix.  Other geometries return BF_E_UNSUPPORTED (loud; the
// lockstep semantics of duplicated threads are not reproduced here).
//
// layerforward, bit-exact: one thread per (block, column) keeps the column's
// 16 products in registers (the DSL stores each product into the f32 shared
// tile: f64 product of two f32 rounded once == f32 multiply) and replays
// Rodinia's in-place tree (strides 1, 2, 4, 8; f32 adds, exact the same way),
// writes every row's final tile value back over the weights and the column
// total to partial[16by + column].  Two logical blocks per warp; the 16 row
// loads of a lane are all in flight together; the misaligned 68 B row pitch
// is absorbed by L1 (each block's 1088 B region is read once from HBM).
// Bytes per input unit (row): 64 read + 64 written + 4 input + 4 partial/16.
//
// adjust_weights, bit-exact: w += (0.3*delta[x])*ly[y] + 0.3*oldw and
// oldw = the same update, in f64 with separately rounded operators (no FMA
// contraction), one f32 rounding per store; the bias row (row 0) by block 0.
// Bytes per element: 16 (w and oldw read and written) + ly per row.
#include <algorithm>
#include <climits>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

constexpr int kBpHid = 16;

// Both kernels stream the contiguous region of their logical blocks: blocks
// [b0, b1) own the floats [272 b0 + 17, 272 b1 + 17) of w (rows 16 b0 + 1 ..
// 16 b1, all 17 columns).  A region offset of 17 (mod 4) means the interior
// is moved with 16 B vector accesses and at most 3 + 1 edge floats singly.
constexpr int kBpChunk = 16;                 // logical blocks per CTA step (forward)
constexpr int kBpChunkF = 272 * kBpChunk;    // floats per chunk

// forward: the region of kBpChunk blocks moves through a two-buffer
// shared-memory ring: the aligned interior comes in by one bulk copy (TMA,
// completing on the buffer's mbarrier) issued a step ahead, the <= 3 + 1 edge
// floats by plain loads; one thread per (block, column) replays the tree in
// shared memory (conflict-free: 17-float pitch) and the interior goes back by
// one bulk store (column 0, the bias weights, is rewritten unchanged: it lies
// inside the CTA's own rows).
struct BpChunk {
  long long c0, g0, g1, a0, a1;
  int nblk;
  __device__ BpChunk(long long c, long long b1) {
    c0 = c;
    nblk = (int)min((long long)kBpChunk, b1 - c);
    g0 = 272 * c0 + 17;
    g1 = 272 * (c0 + nblk) + 17;
    a0 = (g0 + 3) & ~3LL;
    a1 = g1 & ~3LL;
  }
};

// three buffers: the load of chunk n+1 goes into the buffer whose bulk store
// left two chunks ago, so it waits for at most the older of the two stores
// in flight (wait_group.read 1) instead of the last one
constexpr int kBpStages = 3;

__global__ void __launch_bounds__(256) bp_forward(const float* __restrict__ input, float* __restrict__ w,
                                                  float* __restrict__ partial, long long b0, long long b1) {
  extern __shared__ __align__(16) float bp_dyn[];
  float (*sm)[kBpChunkF + 8] = reinterpret_cast<float (*)[kBpChunkF + 8]>(bp_dyn);
  __shared__ __align__(8) uint64_t full[kBpStages];
  const long long cstride = (long long)gridDim.x * kBpChunk;
  const long long first = b0 + (long long)blockIdx.x * kBpChunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBpStages; i++) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](long long c, int buf) {  // thread 0
    const BpChunk k(c, b1);
    const uint32_t bytes = (uint32_t)((k.a1 - k.a0) * 4);
    mbar_arrive_expect_tx(&full[buf], bytes);
    bulk_g2s(sm[buf] + 4, w + k.a0, bytes, &full[buf], policy_evict_first());
  };
  if (threadIdx.x == 0 && first < b1) issue(first, 0);
  int n = 0;
  for (long long c0 = first; c0 < b1; c0 += cstride, n++) {
    const int buf = n % kBpStages;
    const BpChunk k(c0, b1);
    if (threadIdx.x == 0 && c0 + cstride < b1) {
      bulk_wait_read<1>();  // the store of chunk n-2 (the target buffer) has left shared memory
      issue(c0 + cstride, (n + 1) % kBpStages);
    }
    float* Sa = sm[buf] + 4;             // a0 -> 16 B aligned
    const int sh = (int)(k.a0 - k.g0);   // 0..3 leading edge floats
    float* Sg = Sa - sh;                 // g0
    if (threadIdx.x < sh) Sg[threadIdx.x] = w[k.g0 + threadIdx.x];
    if (threadIdx.x < (int)(k.g1 - k.a1)) Sa[(k.a1 - k.a0) + threadIdx.x] = w[k.a1 + threadIdx.x];
    const int blk = threadIdx.x >> 4, col = threadIdx.x & 15;
    const bool on = blk < k.nblk;  // whole warps stay converged for the shuffles
    const long long by = c0 + blk;
    const float node_mine = on ? __ldg(input + 16 * by + col + 1) : 0.f;
    mbar_wait(&full[buf], (n / kBpStages) & 1);
    __syncthreads();  // edge floats visible
    float* T = Sg + 272 * blk + col + 1;  // row 0 of the block, this column
    float p[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const float nd = __shfl_sync(0xffffffffu, node_mine, (threadIdx.x & 16) | r);
      p[r] = on ? __fmul_rn(T[17 * r], nd) : 0.f;
    }
    // Rodinia's tree: wm[ty] += wm[ty + s] for ty % 2s == 0, s = 1, 2, 4, 8
#pragma unroll
    for (int s2 = 1; s2 < 16; s2 *= 2)
#pragma unroll
      for (int r = 0; r < 16; r += 2 * s2) p[r] = __fadd_rn(p[r], p[r + s2]);
    if (on) {
#pragma unroll
      for (int r = 0; r < 16; r++) T[17 * r] = p[r];
      partial[16 * by + col] = p[0];
    }
    fence_proxy_async();  // tile writes before the bulk store (async proxy)
    __syncthreads();
    if (threadIdx.x < sh) w[k.g0 + threadIdx.x] = Sg[threadIdx.x];
    if (threadIdx.x < (int)(k.g1 - k.a1)) w[k.a1 + threadIdx.x] = Sa[(k.a1 - k.a0) + threadIdx.x];
    if (threadIdx.x == 0) {
      bulk_s2g(w + k.a0, Sa, (uint32_t)((k.a1 - k.a0) * 4));
      bulk_commit();
    }
    __syncthreads();  // edge reads done before the buffer is refilled
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
}

// adjust: elementwise over the region; element g = 17 row + col (col != 0):
// ix = g, iy = row, delta index = col (DSL: index, iy = 16by+ty+1, ix = tx+1).
__device__ __forceinline__ float bp_upd(float wv, float& ov, double cx, double l) {
  const double s = dadd(dmul(cx, l), dmul(0.3, (double)ov));
  ov = __double2float_rn(s);
  return __double2float_rn(dadd((double)wv, s));
}

// adjust: the same two-buffer bulk-copy ring over the w and oldw regions of
// kBpChunkA blocks; every element of the region is updated in shared memory
// (column 0 is left as loaded) and both regions go back by bulk stores.
constexpr int kBpChunkA = 8;
constexpr int kBpChunkAF = 272 * kBpChunkA;

__global__ void __launch_bounds__(256) bp_adjust(const float* __restrict__ delta, const float* __restrict__ ly,
                                                 float* __restrict__ w, float* __restrict__ oldw, long long b0,
                                                 long long b1, bool bias) {
  extern __shared__ __align__(16) float bp_dyn[];
  float (*sw)[kBpChunkAF + 8] = reinterpret_cast<float (*)[kBpChunkAF + 8]>(bp_dyn);
  float (*so)[kBpChunkAF + 8] = sw + kBpStages;
  __shared__ __align__(8) uint64_t full[kBpStages];
  static_assert(kBpChunkA * 16 * 2 == 256, "two threads per weight row");
  double cx[8];  // 0.3 * delta[col] of this thread's eight columns
#pragma unroll
  for (int j = 0; j < 8; j++) cx[j] = dmul(0.3, (double)__ldg(delta + 1 + 8 * (threadIdx.x & 1) + j));
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBpStages; i++) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const long long cstride = (long long)gridDim.x * kBpChunkA;
  const long long first = b0 + (long long)blockIdx.x * kBpChunkA;
  auto region = [&](long long c, long long& g0, long long& g1, long long& a0, long long& a1) {
    const long long nb = min((long long)kBpChunkA, b1 - c);
    g0 = 272 * c + 17;
    g1 = 272 * (c + nb) + 17;
    a0 = (g0 + 3) & ~3LL;
    a1 = g1 & ~3LL;
  };
  auto issue = [&](long long c, int buf) {  // thread 0
    long long g0, g1, a0, a1;
    region(c, g0, g1, a0, a1);
    const uint32_t bytes = (uint32_t)((a1 - a0) * 4);
    const uint64_t pol = policy_evict_first();
    mbar_arrive_expect_tx(&full[buf], 2 * bytes);
    bulk_g2s(sw[buf] + 4, w + a0, bytes, &full[buf], pol);
    bulk_g2s(so[buf] + 4, oldw + a0, bytes, &full[buf], pol);
  };
  if (threadIdx.x == 0 && first < b1) issue(first, 0);
  int n = 0;
  for (long long c0 = first; c0 < b1; c0 += cstride, n++) {
    const int buf = n % kBpStages;
    if (threadIdx.x == 0 && c0 + cstride < b1) {
      bulk_wait_read<1>();
      issue(c0 + cstride, (n + 1) % kBpStages);
    }
    long long g0, g1, a0, a1;
    region(c0, g0, g1, a0, a1);
    const int sh = (int)(a0 - g0), tl = (int)(g1 - a1);
    float* W = sw[buf] + 4 - sh;  // g0
    float* O = so[buf] + 4 - sh;
    const int len = (int)(g1 - g0);
    if (threadIdx.x < sh) {
      W[threadIdx.x] = w[g0 + threadIdx.x];
      O[threadIdx.x] = oldw[g0 + threadIdx.x];
    }
    if (threadIdx.x < tl) {
      W[len - tl + threadIdx.x] = w[a1 + threadIdx.x];
      O[len - tl + threadIdx.x] = oldw[a1 + threadIdx.x];
    }
    mbar_wait(&full[buf], (n / kBpStages) & 1);
    __syncthreads();
    // two threads per row (columns 1-8 and 9-16): ly[row] is read and
    // converted once per 8 elements, 0.3*delta[col] stays in registers.
    // Row r of the region = weight row 16 c0 + 1 + r; element (r, col) is
    // region index 17 r + col.
    {
      const int r = threadIdx.x >> 1, cb = 1 + 8 * (threadIdx.x & 1);
      if (r < len / 17) {
        const double l = (double)__ldg(ly + 16 * c0 + 1 + r);
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int i = 17 * r + cb + j;
          const double sv = dadd(dmul(cx[j], l), dmul(0.3, (double)O[i]));
          O[i] = __double2float_rn(sv);
          W[i] = __double2float_rn(dadd((double)W[i], sv));
        }
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x < sh) {
      w[g0 + threadIdx.x] = W[threadIdx.x];
      oldw[g0 + threadIdx.x] = O[threadIdx.x];
    }
    if (threadIdx.x < tl) {
      w[a1 + threadIdx.x] = W[len - tl + threadIdx.x];
      oldw[a1 + threadIdx.x] = O[len - tl + threadIdx.x];
    }
    if (threadIdx.x == 0) {
      bulk_s2g(w + a0, sw[buf] + 4, (uint32_t)((a1 - a0) * 4));
      bulk_s2g(oldw + a0, so[buf] + 4, (uint32_t)((a1 - a0) * 4));
      bulk_commit();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
  if (bias && blockIdx.x == 0 && threadIdx.x < 16) {  // row 0 (bias), block 0's ty == 0 threads
    const int x = threadIdx.x + 1;
    const double o = (double)oldw[x];
    const double sv = dadd(dmul(0.3, (double)delta[x]), dmul(0.3, o));
    w[x] = __double2float_rn(dadd((double)w[x], sv));
    oldw[x] = __double2float_rn(sv);
  }
}

// Common geometry check; returns false (and sets the error) when unsupported.
static bool bp_geometry(LaunchCtx& ctx, int hid, const char* what) {
  if (ctx.block[0] != 16 || ctx.block[1] != 16 || ctx.block[2] != 1 || ctx.grid[0] != 1 || ctx.grid[2] != 1 ||
      hid != kBpHid) {
    *ctx.error = std::string(what) + ": only Rodinia's geometry (block 16x16x1, grid 1 x n x 1, hid = 16)";
    return false;
  }
  return true;
}

// Lowest block index >= b0 with an affine index beyond `len` (index = a*by + c,
// a > 0), or b1 when none; also catches the i32 wrap of the DSL's index.
static long long first_bad(long long b0, long long b1, long long a, long long c, long long len) {
  long long lim = std::min(len, (long long)INT_MAX + 1);  // index must be < lim
  if (c >= lim) return b0;
  long long bad = (lim - c + a - 1) / a;  // smallest by with a*by + c >= lim
  return std::max(b0, std::min(b1, bad));
}

static int launch_bp_forward(LaunchCtx& ctx) {
  const ArgVal& In = ctx.args[0];
  const ArgVal& W = ctx.args[1];
  const ArgVal& P = ctx.args[2];
  const int hid = ctx.args[3].i32;
  if (!bp_geometry(ctx, hid, "bpnn_layerforward")) return BF_E_UNSUPPORTED;
  long long b0 = ctx.first, b1 = ctx.first + ctx.count;
  // section order: input[16by+ty+1] (max 16by+16), w[index] (max 272by+288),
  // then (after the write-back) partial[16by+ty] (max 16by+15)
  long long bad = std::min({first_bad(b0, b1, 16, 16, In.len), first_bad(b0, b1, 272, 288, W.len),
                            first_bad(b0, b1, 16, 15, P.len)});
  if (bad < b1) {
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, bad, "bpnn_layerforward index out of range");
    b1 = bad;
  }
  if (b0 >= b1) return BF_OK;
  const size_t smem = sizeof(float) * kBpStages * (kBpChunkF + 8);
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(bp_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaGetLastError();
  }
  const int per_sm = resident_ctas((const void*)bp_forward, 256, smem);
  const int grid = stream_grid(b1 - b0, kBpChunk, ctx.num_sms, per_sm);
  bp_forward<<<grid, 256, smem, ctx.stream>>>((const float*)In.ptr, (float*)W.ptr, (float*)P.ptr, b0, b1);
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

static int launch_bp_adjust(LaunchCtx& ctx) {
  const ArgVal& D = ctx.args[0];
  const int hid = ctx.args[1].i32;
  const ArgVal& L = ctx.args[2];
  const ArgVal& W = ctx.args[4];
  const ArgVal& O = ctx.args[5];
  if (!bp_geometry(ctx, hid, "bpnn_adjust_weights")) return BF_E_UNSUPPORTED;
  long long b0 = ctx.first, b1 = ctx.first + ctx.count;
  // first thread of a block touches w/oldw[index], delta[1..16], ly[16by+1..16]
  long long bad = std::min({first_bad(b0, b1, 272, 288, W.len), first_bad(b0, b1, 272, 288, O.len),
                            first_bad(b0, b1, 16, 16, L.len)});
  if (D.len < kBpHid + 1) bad = b0;  // delta[tx + 1] of every block
  if (bad < b1) {
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, bad, "bpnn_adjust_weights index out of range");
    b1 = bad;
  }
  if (b0 >= b1) return BF_OK;
  const bool bias = b0 == 0;
  const size_t smem = sizeof(float) * 2 * kBpStages * (kBpChunkAF + 8);
  static bool attr[64] = {};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(bp_adjust, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaGetLastError();
  }
  const int per_sm = resident_ctas((const void*)bp_adjust, 256, smem);
  const int grid = stream_grid(b1 - b0, kBpChunkA, ctx.num_sms, per_sm);
  bp_adjust<<<grid, 256, smem, ctx.stream>>>((const float*)D.ptr, (const float*)L.ptr, (float*)W.ptr,
                                             (float*)O.ptr, b0, b1, bias);
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

static Registrar reg_bp_forward("bpnn_layerforward",
                                {{BF_SLOT_HANDLE, BF_F32, "input"},
                                 {BF_SLOT_HANDLE, BF_F32, "w"},
                                 {BF_SLOT_HANDLE, BF_F32, "partial"},
                                 {BF_SLOT_I32, BF_I32, "hid"}},
                                launch_bp_forward);

static Registrar reg_bp_adjust("bpnn_adjust_weights",
                               {{BF_SLOT_HANDLE, BF_F32, "delta"},
                                {BF_SLOT_I32, BF_I32, "hid"},
                                {BF_SLOT_HANDLE, BF_F32, "ly"},
                                {BF_SLOT_I32, BF_I32, "inn"},
                                {BF_SLOT_HANDLE, BF_F32, "w"},
                                {BF_SLOT_HANDLE, BF_F32, "oldw"}},
                               launch_bp_adjust);

}  // namespace bf
