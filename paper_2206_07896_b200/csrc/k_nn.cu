// nn — paper_2206_07896_b200/kernels/nn.kn (Rodinia nn "euclid").
//
// d[id] = sqrt((ll[2id] - x)^2 + (ll[2id+1] - y)^2) for id < n, evaluated in
// f64 operator by operator (interp.py:58-91, 147-150: math.sqrt is the
// correctly rounded IEEE sqrt == __dsqrt_rn) and rounded to f32 at the store.
// Records are {lat, lng} f32 pairs (array of structs, as Rodinia's LatLong).
//
// B200 mapping: 4 records per thread step = two 16 B loads + one 16 B store,
// streaming cache hints; 12 B per record.  Bound: HBM (f64 sqrt is a handful
// of DFMA per record, well under the FP64 roof at this intensity).
#include <climits>
#include <cstdlib>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

// RN_f32(RN_f64(sqrt(s))) without the ~30-op f64 sqrt sequence.
// f = sqrtf((float)s) is within one f32 ulp of the answer.  The f32
// midpoints m = f +- ulp/2 have <= 25 significant bits, so m*m is exact in
// f64 and s - m*m (an FMA) has the sign of sqrt(s) - m.  Pick the neighbour
// whose rounding interval holds sqrt(s); then emulate the double rounding:
// if RN_f64(sqrt(s)) == m exactly (|s - m*m| <= m * ulp64(m)), the f32
// rounding of m is a tie and goes to the even neighbour.  Values outside
// [2^-60, 2^60] (and s <= 0, NaN) take the exact f64 path.
// midpoints of the f32 rounding interval of f (f positive normal), exact in
// f64: f +- half an f32 ulp (a quarter below a power of two)
__device__ __forceinline__ void f32_midpoints(float f, double& mh, double& ml) {
  const int fb = __float_as_int(f);
  const long long e = (fb >> 23) & 0xff;  // biased f32 exponent
  const double hu = __longlong_as_double((e - 127 - 24 + 1023) << 52);  // ulp/2
  const double fd = (double)f;
  mh = fd + hu;
  ml = fd - ((fb & 0x7fffff) ? hu : 0.5 * hu);
}

__device__ __forceinline__ float sqrt_f64_to_f32(double s) {
  if (!(s >= 0x1p-60 && s <= 0x1p60)) return __double2float_rn(__dsqrt_rn(s));
  float f = sqrtf(__double2float_rn(s));  // within one f32 ulp of the answer
  double mh, ml;
  f32_midpoints(f, mh, ml);
  double eh = fma(-mh, mh, s), el = fma(-ml, ml, s);  // exact near the answer
  if (eh > 0.0 || el < 0.0) {  // sqrt(s) lies in a neighbour's interval
    f = __int_as_float(__float_as_int(f) + (eh > 0.0 ? 1 : -1));
    f32_midpoints(f, mh, ml);
    eh = fma(-mh, mh, s);
    el = fma(-ml, ml, s);
  }
  // double rounding: RN64(sqrt(s)) == m exactly iff sqrt(s) is within half
  // an f64 ulp of m, i.e. -m*u < s - m^2 <= m*u with u = ulp64(m) (f64 ties
  // go to m: it has <= 25 significant bits); then the f32 rounding of m is a
  // tie and goes to the even neighbour
  // m * ulp64(m): add ulp64's exponent to m's (exact, integer pipe)
  auto times_ulp = [](double m) {
    const long long b = __double_as_longlong(m);
    const long long e = (b >> 52) & 0x7ff;
    return __longlong_as_double(b + ((e - 1075) << 52));
  };
  const double th = times_ulp(mh), tl = times_ulp(ml);
  const bool even = (__float_as_int(f) & 1) == 0;
  if (eh > -th && eh <= th) return even ? f : __int_as_float(__float_as_int(f) + 1);
  if (el > -tl && el <= tl) return even ? f : __int_as_float(__float_as_int(f) - 1);
  return f;
}

template <bool EMU>
__device__ __forceinline__ float nn_dist(float lat, float lng, double x, double y) {
  const double a = dsub((double)lat, x);
  const double b = dsub((double)lng, y);
  const double s = dadd(dmul(a, a), dmul(b, b));
  return EMU ? sqrt_f64_to_f32(s) : __double2float_rn(__dsqrt_rn(s));
}

template <bool EMU>
__global__ void __launch_bounds__(256) nn_stream(const float* __restrict__ ll,
                                                 float* __restrict__ d, long long lo, long long hi,
                                                 double x, double y) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long vlo = (lo + 3) & ~3LL;
  if (vlo > hi) vlo = hi;
  long long vhi = hi & ~3LL;
  if (vhi < vlo) vhi = vlo;
  if (tid < vlo - lo) d[lo + tid] = nn_dist<EMU>(ll[2 * (lo + tid)], ll[2 * (lo + tid) + 1], x, y);
  if (tid < hi - vhi) d[vhi + tid] = nn_dist<EMU>(ll[2 * (vhi + tid)], ll[2 * (vhi + tid) + 1], x, y);
  const float4* l4 = reinterpret_cast<const float4*>(ll);
  float4* d4 = reinterpret_cast<float4*>(d);
  long long g = vlo / 4 + tid;
  const long long end = vhi / 4;
  // 4 x 16 B loads per step, software-pipelined: the next step's loads are
  // in flight while this step's eight f64 distances (DSQRT) are computed
  if (g + stride < end) {
    float4 p0 = __ldcs(l4 + 2 * g), q0 = __ldcs(l4 + 2 * g + 1);
    float4 p1 = __ldcs(l4 + 2 * (g + stride)), q1 = __ldcs(l4 + 2 * (g + stride) + 1);
    for (;;) {
      const long long gn = g + 2 * stride;
      const bool more = gn + stride < end;
      float4 np0, nq0, np1, nq1;
      if (more) {
        np0 = __ldcs(l4 + 2 * gn);
        nq0 = __ldcs(l4 + 2 * gn + 1);
        np1 = __ldcs(l4 + 2 * (gn + stride));
        nq1 = __ldcs(l4 + 2 * (gn + stride) + 1);
      }
      __stcs(d4 + g, make_float4(nn_dist<EMU>(p0.x, p0.y, x, y), nn_dist<EMU>(p0.z, p0.w, x, y),
                                 nn_dist<EMU>(q0.x, q0.y, x, y), nn_dist<EMU>(q0.z, q0.w, x, y)));
      __stcs(d4 + g + stride, make_float4(nn_dist<EMU>(p1.x, p1.y, x, y), nn_dist<EMU>(p1.z, p1.w, x, y),
                                          nn_dist<EMU>(q1.x, q1.y, x, y), nn_dist<EMU>(q1.z, q1.w, x, y)));
      g = gn;
      if (!more) break;
      p0 = np0;
      q0 = nq0;
      p1 = np1;
      q1 = nq1;
    }
  }
  if (g < end) {
    const float4 p = __ldcs(l4 + 2 * g), q = __ldcs(l4 + 2 * g + 1);
    __stcs(d4 + g, make_float4(nn_dist<EMU>(p.x, p.y, x, y), nn_dist<EMU>(p.z, p.w, x, y),
                               nn_dist<EMU>(q.x, q.y, x, y), nn_dist<EMU>(q.z, q.w, x, y)));
  }
}

static int launch_nn(LaunchCtx& ctx) {
  const ArgVal& L = ctx.args[0];
  const ArgVal& D = ctx.args[1];
  const long long n = ctx.args[2].i32;
  const double x = ctx.args[3].f64, y = ctx.args[4].f64;
  const long long bx = ctx.block[0];
  for (auto& xi : ctx.x_intervals()) {
    long long lo = xi.first * bx, hi = std::min(xi.second * bx, n);
    if (lo >= hi) continue;
    if (2 * (hi - 1) + 1 > (long long)INT_MAX) {
      // 2*id wraps to a negative i32 index in the DSL: the load traps
      long long bad = ((long long)INT_MAX + 1) / 2;
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(std::max(lo, bad) / bx),
                    "record index 2*id beyond i32");
      hi = std::max(lo, bad);
    }
    long long safe = std::min(L.len / 2, D.len);
    if (hi > safe) {
      long long bad = std::max(lo, safe);
      ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, ctx.first_block_with_x(bad / bx),
                    "load index " + std::to_string(bad) + " out of range");
      hi = bad;
    }
    if (lo >= hi) continue;
    static int emu = -1;
    if (emu < 0) {
      const char* e = getenv("BF_NN_SQRT_EMU");
      emu = e ? atoi(e) : 0;
    }
    const int grid = emu ? wave_grid(nn_stream<true>, 256, 0, (hi - lo + 3) / 4, 256, ctx.num_sms, 8)
                         : wave_grid(nn_stream<false>, 256, 0, (hi - lo + 3) / 4, 256, ctx.num_sms, 8);
    if (emu)
      nn_stream<true><<<grid, 256, 0, ctx.stream>>>((const float*)L.ptr, (float*)D.ptr, lo, hi, x, y);
    else
      nn_stream<false><<<grid, 256, 0, ctx.stream>>>((const float*)L.ptr, (float*)D.ptr, lo, hi, x, y);
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_nn("nn",
                        {{BF_SLOT_HANDLE, BF_F32, "ll"},
                         {BF_SLOT_HANDLE, BF_F32, "d"},
                         {BF_SLOT_I32, BF_I32, "n"},
                         {BF_SLOT_F32, BF_F32, "x"},
                         {BF_SLOT_F32, BF_F32, "y"}},
                        launch_nn);

// ---------------------------------------------------------------------------
// nn_topk — paper_2206_07896_b200/kernels/nn_topk.kn (Rodinia nn's selection
// of the k nearest records).  The DSL kernel's k passes each pick the least
// record after the previous pick in (distance, index) order, NaN distances
// last: that is the first k entries of a stable sort of d.  On the device the
// order is a 64-bit key (monotone f32 key << 32 | index; NaN -> all ones,
// -0.0 -> +0.0, which compare equal in the DSL), so picks are unique.
//
// One pass over d (4 B per record): every thread keeps the K smallest keys
// of its grid-stride share in registers (sorted; a key is inserted by one
// compare-exchange sweep, and the fast reject compares only the high word),
// each CTA merges its threads' lists into its k smallest (k rounds of a
// block-wide min; the owner pops), writes them to scratch, and the last CTA
// to finish (ticket) merges the grid's candidates the same way and writes
// idx / dist (dist re-read from d, so a -0.0 keeps its sign).  k > 32 runs
// in rounds of 32 picks, each round taking keys above the previous round's
// last pick (kept on the device).
__device__ __forceinline__ unsigned long long topk_key(float v, unsigned i) {
  unsigned b = __float_as_uint(v);
  if (v != v) b = 0xffffffffu;  // NaN after every number
  else {
    if (v == 0.0f) b = 0u;  // -0.0 == +0.0
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  return ((unsigned long long)b << 32) | i;
}

// high word of topk_key for a non-NaN value, and its inverse
__device__ __forceinline__ unsigned topk_hi(float v) {
  unsigned b = v == 0.0f ? 0u : __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float topk_from_hi(unsigned hb) {
  return __uint_as_float((hb & 0x80000000u) ? (hb & 0x7fffffffu) : ~hb);
}

template <int K>
struct TopList {
  unsigned long long l[K];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < K; j++) l[j] = ~0ull;
  }
  __device__ __forceinline__ void insert(unsigned long long key) {
    if (key >= l[K - 1]) return;
#pragma unroll
    for (int j = 0; j < K; j++) {  // sorted insert as one min/max sweep
      const unsigned long long lo = key < l[j] ? key : l[j];
      key = key < l[j] ? l[j] : key;
      l[j] = lo;
    }
  }
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int j = 0; j < K - 1; j++) l[j] = l[j + 1];
    l[K - 1] = ~0ull;
  }
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// The `cnt` smallest keys of the union of the block's lists -> out[0..cnt)
// (every thread of the block calls it; out may be shared or global).
template <int K>
__device__ void block_merge(TopList<K>& t, int cnt, unsigned long long* out) {
  __shared__ unsigned long long wmin[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int r = 0; r < cnt; r++) {
    const unsigned long long m = warp_min_u64(t.l[0]);
    if (lane == 0) wmin[warp] = m;
    __syncthreads();
    unsigned long long bm = wmin[0];
    for (int w = 1; w < nw; w++) bm = wmin[w] < bm ? wmin[w] : bm;
    if (bm != ~0ull && t.l[0] == bm) t.pop();  // keys are unique: one owner
    if (threadIdx.x == 0) out[r] = bm;
    __syncthreads();
  }
}

struct TopkArgs {
  const float* d;
  long long n;
  int* idx;
  float* dist;
  int base;                  // first output slot of this round
  int cnt;                   // picks this round (<= K)
  int kw_idx, kw_dist;       // slots [0, kw) of idx / dist may be written
  unsigned long long* cand;  // [gridDim.x][K] scratch
  unsigned* ticket;
  unsigned long long* lo;    // keys must exceed *lo (the previous round's last pick)
};

// Scan: one producer warp streams 16 KB chunks of d into a shared-memory ring
// with bulk copies (TMA, 1D); eight consumer warps test them (a thread owns
// four float4 of each chunk).  Many bytes stay in flight with few threads, so
// the scan runs at the DRAM rate although its per-value work is light.
constexpr int kTkChunk = 4096;  // floats per chunk
constexpr int kTkStages = 4;
constexpr int kTkThreads = 288;  // 8 consumer warps + 1 producer warp

template <int K>
__global__ void __launch_bounds__(kTkThreads) nn_topk_pass(TopkArgs a) {
  extern __shared__ __align__(128) float tk_ring[];  // kTkStages x kTkChunk
  __shared__ uint64_t tk_full[kTkStages], tk_empty[kTkStages];
  __shared__ unsigned s_thr;
  const unsigned long long lo = *a.lo;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TopList<K> t;
  t.init();
  // fast reject on the raw float: v > tf cannot enter (a value such that some
  // thread of the CTA holds K keys at or below it); NaN tf rejects nothing
  float tf = __uint_as_float(0x7fffffffu);
  if (threadIdx.x == 0) {
    s_thr = 0xffffffffu;
    for (int s = 0; s < kTkStages; s++) {
      mbar_init(&tk_full[s], 1);
      mbar_init(&tk_empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  auto offer = [&](float v, long long i) {
    if (v > tf) return;
    const unsigned long long key = topk_key(v, (unsigned)i);
    if (key >= t.l[K - 1] || key <= lo) return;
    t.insert(key);
    const unsigned hb = (unsigned)(t.l[K - 1] >> 32);
    // fminf keeps a tighter (shared) bound; NaN (list not full) never wins
    tf = fminf(tf, hb == 0xffffffffu ? __uint_as_float(0x7fffffffu) : topk_from_hi(hb));
  };
  const long long n4 = a.n >> 2;            // whole float4 of d; the last n & 3 values below
  const long long nchunk = (4 * n4 + kTkChunk - 1) / kTkChunk;
  if (warp == 8) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int j = 0;
      for (long long c = blockIdx.x; c < nchunk; c += gridDim.x, j++) {
        const int st = j % kTkStages;
        if (j >= kTkStages) mbar_wait(&tk_empty[st], ((j / kTkStages) - 1) & 1);
        const long long f0 = c * kTkChunk;
        const uint32_t bytes = (uint32_t)(min((long long)kTkChunk, 4 * n4 - f0) * 4);
        mbar_arrive_expect_tx(&tk_full[st], bytes);
        bulk_g2s(tk_ring + st * kTkChunk, a.d + f0, bytes, &tk_full[st], pol);
      }
    }
  } else {  // consumers
    int j = 0;
    for (long long c = blockIdx.x; c < nchunk; c += gridDim.x, j++) {
      const int st = j % kTkStages;
      mbar_wait(&tk_full[st], (j / kTkStages) & 1);
      const long long f0 = c * kTkChunk;
      const int cnt4 = (int)(min((long long)kTkChunk, 4 * n4 - f0) >> 2);
      const float4* r4 = reinterpret_cast<const float4*>(tk_ring + st * kTkChunk);
      float4 v[4];
      float m[4];
      if (cnt4 == kTkChunk / 4) {  // every chunk but the last: no bounds, no padding values
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = r4[threadIdx.x + 256 * u];
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int q = threadIdx.x + 256 * u;
          v[u] = q < cnt4 ? r4[q] : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) m[u] = fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w));
      __syncwarp();
      if (lane == 0) mbar_arrive(&tk_empty[st]);  // the values are in registers
      // warp-uniform branches (votes): the insert code is skipped, not
      // if-converted into predicated straight-line code
      if (__any_sync(0xffffffffu, !(fminf(fminf(m[0], m[1]), fminf(m[2], m[3])) > tf))) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int q = threadIdx.x + 256 * u;
          const bool pass = q < cnt4 && !(m[u] > tf);
          if (__any_sync(0xffffffffu, pass) && pass) {
            const long long i = f0 + 4ll * q;
            offer(v[u].x, i);
            offer(v[u].y, i + 1);
            offer(v[u].z, i + 2);
            offer(v[u].w, i + 3);
          }
        }
      }
      // the smallest bound over the warp, then over the CTA (order keys
      // min-combined in shared memory; 0xffffffff: none yet), every second
      // chunk (the exchange is a fifth of the per-chunk instructions and the
      // scan is issue-bound: ncu issue-active 61 %)
      if (j & 1) continue;
#pragma unroll
      for (int o = 16; o; o >>= 1) tf = fminf(tf, __shfl_xor_sync(0xffffffffu, tf, o));
      if (K <= 8 && (j & 3) == 2) {
        // every fourth chunk, a tighter bound: the cnt-th smallest of the
        // warp's lane-best values (cnt lanes each hold a key at or below it,
        // and only the round's cnt <= K smallest keys are wanted), by cnt
        // rounds of a warp minimum that retires one lane each
        const unsigned hb0 = (unsigned)(t.l[0] >> 32);
        float x = hb0 == 0xffffffffu ? INFINITY : topk_from_hi(hb0);
        float kth = INFINITY;
#pragma unroll 1
        for (int r = 0; r < a.cnt; r++) {
          float m = x;
#pragma unroll
          for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
          kth = m;
          const unsigned who = __ballot_sync(0xffffffffu, x == m);
          if (lane == __ffs(who) - 1) x = INFINITY;
        }
        if (kth < INFINITY) tf = fminf(tf, kth);
      }
      if (lane == 0 && tf == tf) atomicMin(&s_thr, topk_hi(tf));
      __syncwarp();
      const unsigned ct = *(volatile unsigned*)&s_thr;
      if (ct != 0xffffffffu) tf = fminf(tf, topk_from_hi(ct));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (int)(a.n & 3)) offer(a.d[4 * n4 + threadIdx.x], 4 * n4 + threadIdx.x);
  block_merge<K>(t, a.cnt, a.cand + (long long)blockIdx.x * K);
  // last CTA merges every CTA's candidates
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  t.init();
  const long long total = (long long)gridDim.x * K;
  for (long long j = threadIdx.x; j < total; j += blockDim.x) {
    const long long c = j / K, r = j % K;
    if (r < a.cnt) t.insert(__ldcg(a.cand + c * K + r));
  }
  __shared__ unsigned long long fin[K];
  block_merge<K>(t, a.cnt, fin);
  if (threadIdx.x == 0) {
    unsigned long long lastkey = ~0ull;
    for (int r = 0; r < a.cnt; r++) {
      const int slot = a.base + r;
      const unsigned long long key = fin[r];
      const int i = key == ~0ull ? -1 : (int)(key & 0xffffffffu);
      if (slot < a.kw_idx) a.idx[slot] = i;
      if (i >= 0 && slot < a.kw_dist) a.dist[slot] = a.d[i];
      if (i >= 0) lastkey = key;
    }
    // the next round starts after this round's last pick (all of them when
    // the records ran out)
    *a.lo = fin[a.cnt - 1] == ~0ull ? ~0ull : lastkey;
    *a.ticket = 0;
  }
}

// a round with no records left: the remaining slots get -1
__global__ void nn_topk_fill(int* idx, int from, int to) {
  for (int j = from + threadIdx.x; j < to; j += blockDim.x) idx[j] = -1;
}

struct TopkScratch : StreamScratch {
  unsigned long long* cand = nullptr;
  unsigned* ticket = nullptr;
  unsigned long long* lo = nullptr;
  long long cap = 0;
  ~TopkScratch() override {
    cudaFree(cand);
    cudaFree(ticket);
    cudaFree(lo);
  }
};

static int launch_nn_topk(LaunchCtx& ctx) {
  const ArgVal& D = ctx.args[0];
  const ArgVal& I = ctx.args[1];
  const ArgVal& O = ctx.args[2];
  const long long n = std::max(0, ctx.args[3].i32);
  const long long k = ctx.args[4].i32;
  // only logical blocks with blockIdx.x == 0 select (thread 0 of each; all
  // of them write the same values): one selection if the fetch holds one
  bool any = false;
  for (auto& xi : ctx.x_intervals())
    if (xi.first == 0) any = true;
  if (!any || k <= 0) return BF_OK;
  const long long blk = ctx.first_block_with_x(0);
  const long long ld = D.len, li = I.len, lo_ = O.len;
  if (n > ld) {  // pass 0 reads d[len(d)]
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, blk, "nn_topk: n beyond len(d)");
    return BF_OK;
  }
  // pass j writes idx[j], then dist[j] when a record was picked (j < n)
  long long kw_idx = k, kw_dist = std::min(k, n);
  long long jt = LLONG_MAX;
  if (k > li) jt = li;
  if (std::min(k, n) > lo_) jt = std::min(jt, lo_);
  if (jt != LLONG_MAX) {
    ctx.host_trap(BF_TRAP_OUT_OF_BOUNDS, blk, "nn_topk: output index out of range");
    kw_idx = std::min(kw_idx, jt < li ? jt + 1 : jt);  // idx[jt] is written before dist[jt] traps
    kw_idx = std::min(kw_idx, li);
    kw_dist = std::min(kw_dist, jt);
  }
  const bool small = k <= 8;
  const int K = small ? 8 : 32;
  const size_t tk_smem = sizeof(float) * kTkStages * kTkChunk;
  static bool tk_attr[64] = {};
  if (first_on_device(tk_attr)) {
    cudaFuncSetAttribute(nn_topk_pass<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tk_smem);
    cudaFuncSetAttribute(nn_topk_pass<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tk_smem);
    cudaGetLastError();
  }
  const int grid = small ? wave_grid(nn_topk_pass<8>, kTkThreads, tk_smem, std::max(1LL, n / kTkChunk), 1,
                                     ctx.num_sms, 3)
                         : wave_grid(nn_topk_pass<32>, kTkThreads, tk_smem, std::max(1LL, n / kTkChunk), 1,
                                     ctx.num_sms, 2);
  TopkScratch& S = scratch_for<TopkScratch>(ctx.stream, SCRATCH_NN_TOPK);
  if (S.cap < (long long)grid * K) {
    cudaStreamSynchronize(ctx.stream);
    cudaFree(S.cand);
    S.cand = nullptr;
    S.cap = 0;
    if (cudaMalloc((void**)&S.cand, (size_t)grid * K * 8) != cudaSuccess) {
      cudaGetLastError();
      *ctx.error = "nn_topk: scratch allocation failed";
      return BF_E_CUDA;
    }
    S.cap = (long long)grid * K;
  }
  if (!S.ticket) {
    if (cudaMalloc((void**)&S.ticket, 4) != cudaSuccess || cudaMalloc((void**)&S.lo, 8) != cudaSuccess) {
      cudaGetLastError();
      *ctx.error = "nn_topk: scratch allocation failed";
      return BF_E_CUDA;
    }
    cudaMemsetAsync(S.ticket, 0, 4, ctx.stream);
  }
  cudaMemsetAsync(S.lo, 0, 8, ctx.stream);  // every key exceeds 0
  for (long long base = 0; base < k; base += K) {
    TopkArgs a{(const float*)D.ptr, n, (int*)I.ptr, (float*)O.ptr, (int)base, (int)std::min<long long>(K, k - base),
               (int)kw_idx, (int)kw_dist, S.cand, S.ticket, S.lo};
    if (base >= n) {  // no records left: -1 for the rest
      const int to = (int)std::min(k, kw_idx);
      if (base < to) nn_topk_fill<<<1, 256, 0, ctx.stream>>>((int*)I.ptr, (int)base, to);
      BF_CUDA_LAUNCH_CHECK(ctx);
      break;
    }
    if (small) nn_topk_pass<8><<<grid, kTkThreads, tk_smem, ctx.stream>>>(a);
    else nn_topk_pass<32><<<grid, kTkThreads, tk_smem, ctx.stream>>>(a);
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

static Registrar reg_nn_topk("nn_topk",
                             {{BF_SLOT_HANDLE, BF_F32, "d"},
                              {BF_SLOT_HANDLE, BF_I32, "idx"},
                              {BF_SLOT_HANDLE, BF_F32, "dist"},
                              {BF_SLOT_I32, BF_I32, "n"},
                              {BF_SLOT_I32, BF_I32, "k"}},
                             launch_nn_topk);

}  // namespace bf
