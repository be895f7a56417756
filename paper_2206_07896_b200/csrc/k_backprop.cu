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

// blocks [b0, b1): warp w handles blocks 2w, 2w+1 of its grid-stride step
__global__ void __launch_bounds__(256) bp_forward(const float* __restrict__ input, float* __restrict__ w,
                                                  float* __restrict__ partial, long long b0, long long b1) {
  const int lane = threadIdx.x & 31;
  const int col = lane & 15, half = lane >> 4;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long pair = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);; pair += warps) {
    const long long by = b0 + 2 * pair + half;
    if (b0 + 2 * pair >= b1) break;
    const bool on = by < b1;
    // input node of row `col` of this lane's block, shuffled to the column lanes
    const float node_mine = on ? __ldg(input + 16 * by + col + 1) : 0.f;
    float p[16];
    const long long base = 272 * by + 17 + col + 1;  // row 0 of the block, this column
#pragma unroll
    for (int r = 0; r < 16; r++) p[r] = on ? __ldcs(w + base + 17 * r) : 0.f;
#pragma unroll
    for (int r = 0; r < 16; r++) p[r] = __fmul_rn(p[r], __shfl_sync(0xffffffffu, node_mine, (lane & 16) | r));
    // Rodinia's tree: wm[ty] += wm[ty + s] for ty % 2s == 0, s = 1, 2, 4, 8
#pragma unroll
    for (int s = 1; s < 16; s *= 2)
#pragma unroll
      for (int r = 0; r < 16; r += 2 * s) p[r] = __fadd_rn(p[r], p[r + s]);
    if (on) {
#pragma unroll
      for (int r = 0; r < 16; r++) __stcs(w + base + 17 * r, p[r]);
      partial[16 * by + col] = p[0];
    }
  }
}

__global__ void __launch_bounds__(256) bp_adjust(const float* __restrict__ delta, const float* __restrict__ ly,
                                                 float* __restrict__ w, float* __restrict__ oldw, long long b0,
                                                 long long b1, bool bias) {
  // element e of the range = (block, row, col): 256 per block
  const long long n = (b1 - b0) * 256;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int col = threadIdx.x & 15;  // blockDim.x % 16 == 0 and stride % 16 == 0
  const double cx = dmul(0.3, (double)__ldg(delta + col + 1));
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const long long by = b0 + (e >> 8);
    const int ty = (int)((e >> 4) & 15);
    const long long ix = 272 * by + 17 * ty + col + 18;
    const double l = (double)__ldg(ly + 16 * by + ty + 1);
    const double o = (double)__ldcs(oldw + ix);
    const double wv = (double)__ldcs(w + ix);
    const double s = dadd(dmul(cx, l), dmul(0.3, o));
    __stcs(w + ix, __double2float_rn(dadd(wv, s)));
    __stcs(oldw + ix, __double2float_rn(s));
  }
  if (bias && blockIdx.x == 0 && threadIdx.x < 16) {  // row 0 (bias), block 0's ty == 0 threads
    const int x = threadIdx.x + 1;
    const double o = (double)oldw[x];
    const double s = dadd(dmul(0.3, (double)delta[x]), dmul(0.3, o));
    w[x] = __double2float_rn(dadd((double)w[x], s));
    oldw[x] = __double2float_rn(s);
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
  const int grid = stream_grid((b1 - b0 + 1) / 2, 8, ctx.num_sms, 8);
  bp_forward<<<grid, 256, 0, ctx.stream>>>((const float*)In.ptr, (float*)W.ptr, (float*)P.ptr, b0, b1);
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
  const int grid = stream_grid((b1 - b0) * 256, 256 * 4, ctx.num_sms, 8);
  bp_adjust<<<grid, 256, 0, ctx.stream>>>((const float*)D.ptr, (const float*)L.ptr, (float*)W.ptr, (float*)O.ptr,
                                          b0, b1, bias);
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
