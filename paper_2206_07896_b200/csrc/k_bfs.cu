// bfs — paper_2206_07896_b200/kernels/bfs.kn: one level-synchronous step of a
// top-down BFS over a CSR graph (Rodinia bfs, one launch per level).
//
// For u < nv with lvl[u] == cur: every out-neighbour v with lvl[v] == -1 gets
// lvl[v] = cur + 1 and changed[0] = 1.  All writers of lvl[v] write the same
// value and a vertex discovered in this launch has cur+1 != cur, so the
// result is independent of the order the device visits vertices in — it is
// exactly the reference's sequential result (executor.py:422-489).
//
// B200 mapping: one thread per vertex scan (coalesced lvl reads), the CSR row
// pair read once, neighbour levels read through L2.  This is the per-launch
// semantics the reference API exposes; the whole-traversal driver with a
// frontier queue is bfs_levels (k_bfs_driver).
#include <climits>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

__device__ __forceinline__ long long bfs_block_of_x(const KDesc& d, long long x) {
  long long x0 = d.first % d.gx;
  return d.first + ((x - x0) % d.gx + d.gx) % d.gx;
}

// Expand frontier vertex u: edges in chunks of 8 with all col loads, then all
// lvl loads, in flight together (random reads dominate this kernel).
__device__ __forceinline__ bool bfs_expand(const int* __restrict__ row, long long lr,
                                           const int* __restrict__ col, long long lcol, int* lvl,
                                           long long ll, long long u, int cur, bool& bad) {
  if (u + 1 >= lr) {
    bad = true;
    return false;
  }
  const int e0 = __ldg(row + u), e1 = __ldg(row + u + 1);
  bool any = false;
  for (int e = e0; e < e1; e += 8) {
    int v[8], lv[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      v[i] = -1;
      if (e + i < e1) {
        if (e + i < 0 || e + i >= lcol) bad = true; else v[i] = __ldg(col + e + i);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
      lv[i] = 0;
      if (e + i < e1 && e + i >= 0 && e + i < lcol) {
        if (v[i] < 0 || v[i] >= ll) bad = true; else lv[i] = lvl[v[i]];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (lv[i] == -1 && e + i < e1 && v[i] >= 0 && v[i] < ll) {
        lvl[v[i]] = (int)((unsigned)cur + 1u);
        any = true;
      }
    }
    if (bad) break;
  }
  return any;
}

// One thread per 4 consecutive vertices: the frontier test reads lvl as int4.
__global__ void __launch_bounds__(256) bfs_step(const int* __restrict__ row, long long lr,
                                                const int* __restrict__ col, long long lcol,
                                                int* lvl, long long ll, int* changed,
                                                long long lch, long long lo, long long hi, int cur,
                                                int bx, KDesc k) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool any = false, bad = false;
  long long bad_u = -1;
  const bool vec = (lo % 4 == 0) && hi <= ll;
  const long long groups = (hi - lo + 3) / 4;
  for (long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += stride) {
    const long long u0 = lo + 4 * gi;
    int l4[4];
    if (vec && u0 + 3 < hi) {
      const int4 t = *reinterpret_cast<const int4*>(lvl + u0);
      l4[0] = t.x; l4[1] = t.y; l4[2] = t.z; l4[3] = t.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const long long u = u0 + q;
        l4[q] = (u < hi && u < ll) ? lvl[u] : INT_MIN;
        if (u < hi && u >= ll && bad_u < 0) bad_u = u;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const long long u = u0 + q;
      if (u < hi && l4[q] == cur) {
        bool b = false;
        any |= bfs_expand(row, lr, col, lcol, lvl, ll, u, cur, b);
        if (b && bad_u < 0) bad_u = u;
      }
    }
  }
  if (bad_u >= 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, bfs_block_of_x(k, bad_u / bx));
  (void)bad;
  if (__syncthreads_or(any) && threadIdx.x == 0) {
    if (lch < 1) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, k.first);
    else changed[0] = 1;
  }
}

// CTA-wide queue append: every thread contributes c items and gets its first
// slot; one atomicAdd per CTA (the counter is a single hot address: per-warp
// atomics serialise at the L2 on the largest levels).  Must be called by all
// threads of the CTA (CTA-uniform loops).
__device__ __forceinline__ int cta_append(int c, int* counter, int* extra_total = nullptr, int extra = 0) {
  __shared__ int wtot[32], wext[32];
  __shared__ int cbase;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int ex = extra;
  for (int o = 16; o > 0; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
  if (lane == 31) {
    wtot[warp] = incl;
    wext[warp] = ex;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0, et = 0;
    for (int w = 0; w < nw; w++) {
      const int t = wtot[w];
      wtot[w] = run;
      run += t;
      et += wext[w];
    }
    cbase = run ? atomicAdd(counter, run) : 0;
    if (extra_total && et) atomicAdd(extra_total, et);
  }
  __syncthreads();
  const int base = cbase + wtot[warp] + incl - c;
  __syncthreads();  // wtot / cbase are rewritten by the next call
  return base;
}

// Two-phase level step (a launch whose fetch covers the whole grid):
//   scan    one pass over lvl[0, ll) builds an "unvisited" bitmap (lvl == -1,
//           8 MB at 2^26 vertices, L2-resident) and appends the frontier
//           (lvl == cur, u in [lo, hi)) to a queue;
//   expand  frontier vertices relax their out-edges against the bitmap; the
//           first thread to clear a target's bit (atomicAnd) writes
//           lvl[v] = cur + 1 once.
// Same result as bfs_step (frontier = lvl == cur at launch start, targets =
// lvl == -1 at launch start, every write is cur + 1), but the per-edge test is
// an L2 hit instead of a random DRAM read of the 256 MB lvl array.
__global__ void __launch_bounds__(256) bfs_scan(const int* __restrict__ lvl, long long ll, unsigned* unv,
                                                long long words, int* q, int* qn, long long lo, long long hi,
                                                int cur) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long w0 = (long long)blockIdx.x * blockDim.x; w0 < words; w0 += stride) {  // CTA-uniform
    const long long w = w0 + threadIdx.x;
    unsigned um = 0, fm = 0;
    if (w < words) {
      const long long v0 = w * 32;
      if (v0 + 32 <= ll) {
        const int4* l4 = reinterpret_cast<const int4*>(lvl + v0);
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const int4 x = __ldcs(l4 + j);
          um |= (x.x == -1 ? 1u : 0u) << (4 * j) | (x.y == -1 ? 1u : 0u) << (4 * j + 1) |
                (x.z == -1 ? 1u : 0u) << (4 * j + 2) | (x.w == -1 ? 1u : 0u) << (4 * j + 3);
          fm |= (x.x == cur ? 1u : 0u) << (4 * j) | (x.y == cur ? 1u : 0u) << (4 * j + 1) |
                (x.z == cur ? 1u : 0u) << (4 * j + 2) | (x.w == cur ? 1u : 0u) << (4 * j + 3);
        }
      } else {
        for (int j = 0; j < 32 && v0 + j < ll; j++) {
          const int x = lvl[v0 + j];
          um |= (x == -1 ? 1u : 0u) << j;
          fm |= (x == cur ? 1u : 0u) << j;
        }
      }
      unv[w] = um;
      // frontier restricted to the fetch's vertices [lo, hi)
      if (v0 < lo) fm &= lo - v0 >= 32 ? 0u : (0xffffffffu << (lo - v0));
      if (v0 + 32 > hi) fm &= hi <= v0 ? 0u : (0xffffffffu >> (v0 + 32 - hi));
    }
    int pos = cta_append(__popc(fm), qn);
    for (; fm; fm &= fm - 1) q[pos++] = (int)(w * 32 + __ffs(fm) - 1);
  }
}

// bfs_scan with one int4 of lvl per thread (fully coalesced loads), the
// bitmap words assembled by 8-lane OR reductions, the unvisited set written
// twice (unv, mutated by the relax, and unv0, the launch-start snapshot the
// deferred lvl writes diff against), and the frontier staged in shared memory
// and appended as one contiguous queue run per CTA iteration.
__global__ void __launch_bounds__(256) bfs_scan2(const int* __restrict__ lvl, long long ll, unsigned* unv,
                                                 unsigned* unv0, int* q, int* qn, long long lo, long long hi,
                                                 int cur) {
  constexpr int J = 8;  // quads per thread per iteration (8 x 16 B loads in flight)
  __shared__ int stage[256 * 4 * J];
  __shared__ int wtot[8];
  __shared__ int cbase, ctot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long quads = ((ll + 31) / 32) * 8;  // whole words
  const long long stride = (long long)gridDim.x * blockDim.x * J;
  int uc = 0;  // unvisited vertices seen by this thread (qn[1]: the relax's probe choice)
  for (long long t0 = (long long)blockIdx.x * blockDim.x * J; t0 < quads; t0 += stride) {  // CTA-uniform
    int4 x[J];
#pragma unroll
    for (int j = 0; j < J; j++) {
      const long long t = t0 + j * 256 + threadIdx.x;
      x[j] = make_int4(0, 0, 0, 0);
      if (t * 4 + 4 <= ll) x[j] = __ldcs(reinterpret_cast<const int4*>(lvl + t * 4));
    }
    unsigned fm[J];
    int c = 0;
#pragma unroll
    for (int j = 0; j < J; j++) {
      const long long t = t0 + j * 256 + threadIdx.x;
      const long long v0 = t * 4;
      unsigned um = 0, f = 0;
      if (t < quads) {
        if (v0 + 4 <= ll) {
          um = (x[j].x == -1) | (x[j].y == -1) << 1 | (x[j].z == -1) << 2 | (x[j].w == -1) << 3;
          f = (x[j].x == cur) | (x[j].y == cur) << 1 | (x[j].z == cur) << 2 | (x[j].w == cur) << 3;
        } else {
          for (int e = 0; e < 4 && v0 + e < ll; e++) {
            const int y = lvl[v0 + e];
            um |= (unsigned)(y == -1) << e;
            f |= (unsigned)(y == cur) << e;
          }
        }
        // frontier restricted to the fetch's vertices [lo, hi)
        if (v0 < lo || v0 + 4 > hi)
          for (int e = 0; e < 4; e++)
            if (v0 + e < lo || v0 + e >= hi) f &= ~(1u << e);
      }
      unsigned word = um << (4 * (lane & 7));
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      word |= __shfl_xor_sync(0xffffffffu, word, 4);
      if ((lane & 7) == 0 && t < quads) {
        unv[t >> 3] = word;
        unv0[t >> 3] = word;
      }
      fm[j] = f;
      c += __popc(f);
      uc += __popc(um);
    }
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < 8; w++) {
        const int y = wtot[w];
        wtot[w] = run;
        run += y;
      }
      ctot = run;
      cbase = run ? atomicAdd(qn, run) : 0;
    }
    __syncthreads();
    const int tot = ctot;
    if (tot) {  // CTA-uniform
      int pos = wtot[warp] + incl - c;
#pragma unroll
      for (int j = 0; j < J; j++) {
        const long long v0 = (t0 + j * 256 + threadIdx.x) * 4;
        for (unsigned f = fm[j]; f; f &= f - 1) stage[pos++] = (int)(v0 + __ffs(f) - 1);
      }
      __syncthreads();
      const int base = cbase;
      for (int j = threadIdx.x; j < tot; j += blockDim.x) q[base + j] = stage[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) uc += __shfl_xor_sync(0xffffffffu, uc, o);
  if (lane == 0 && uc) atomicAdd(qn + 1, uc);
}

__global__ void __launch_bounds__(256) bfs_relax(const int* __restrict__ row, long long lr,
                                                 const int* __restrict__ col, long long lcol, int* lvl,
                                                 long long ll, unsigned* unv, const int* __restrict__ q,
                                                 const int* qn, int* changed, long long lch, int cur, int bx,
                                                 KDesc k) {
  const int n = *qn;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool any = false;
  long long bad_u = -1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int u = __ldg(q + i);
    if ((long long)u + 1 >= lr) {
      if (bad_u < 0) bad_u = u;
      continue;
    }
    const int e0 = __ldg(row + u), e1 = __ldg(row + u + 1);
    for (int e = e0; e < e1; e += 8) {
      int v[8];
      unsigned wv[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        v[j] = -1;
        if (e + j < e1) {
          if (e + j < 0 || e + j >= lcol) bad_u = bad_u < 0 ? u : bad_u;
          else v[j] = __ldg(col + e + j);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; j++) {
        wv[j] = 0u;
        if (e + j < e1 && e + j >= 0 && e + j < lcol) {
          if (v[j] < 0 || v[j] >= ll) bad_u = bad_u < 0 ? u : bad_u;
          else wv[j] = __ldcg(unv + (v[j] >> 5));
        }
      }
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const unsigned bit = 1u << (v[j] & 31);
        if (wv[j] & bit) {
          const unsigned old = atomicAnd(unv + (v[j] >> 5), ~bit);
          if (old & bit) {
            lvl[v[j]] = (int)((unsigned)cur + 1u);
            any = true;
          }
        }
      }
      if (bad_u >= 0) break;
    }
  }
  if (bad_u >= 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, bfs_block_of_x(k, bad_u / bx));
  if (__syncthreads_or(any) && threadIdx.x == 0) {
    if (lch < 1) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, k.first);
    else changed[0] = 1;
  }
}

// Relax step with whole-adjacency vector loads and no claiming atomics:
// every thread that finds a target still unvisited writes lvl[v] = cur + 1
// (all writers of a vertex write the same value) and clears the bit with a
// RED, so no thread waits on an atomic round trip.  V frontier vertices per
// thread, eight edges per step (two 16 B loads when aligned).  Same lvl and
// changed flag as bfs_relax; faults as bfs_relax (kind and vertex).
template <int V>
__global__ void __launch_bounds__(256) bfs_relax_v(const int* __restrict__ row, long long lr,
                                                   const int* __restrict__ col, long long lcol, int* lvl,
                                                   long long ll, unsigned* unv, const int* __restrict__ q,
                                                   const int* qn, int* changed, long long lch, int cur, int bx,
                                                   KDesc k, int defer_min) {
  const int n = *qn;
  const bool DEFER = n >= defer_min;  // big frontier: bfs_apply writes lvl
  // with deferred writes a RED on an already visited target changes nothing,
  // so while most vertices are unvisited (qn[1], counted by bfs_scan2) the
  // bitmap probe before it is skipped: one L2 operation per edge, not two
  const bool probe = !DEFER || defer_min == INT_MAX || 2ll * qn[1] <= ll;
  const long long stride = (long long)gridDim.x * blockDim.x * V;
  bool any = false;
  long long bad_u = -1;
  const int nxt = (int)((unsigned)cur + 1u);
  for (long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * V; i0 < n; i0 += stride) {
    int e0[V], e1[V], uu[V];
#pragma unroll
    for (int a = 0; a < V; a++) {
      e0[a] = e1[a] = 0;
      uu[a] = 0;
      if (i0 + a < n) {
        const int u = __ldg(q + i0 + a);
        uu[a] = u;
        if ((long long)u + 1 >= lr) {
          if (bad_u < 0) bad_u = u;
          continue;
        }
        e0[a] = __ldg(row + u);
        e1[a] = __ldg(row + u + 1);
        if (e1[a] > e0[a] && (e0[a] < 0 || e1[a] > lcol)) {  // edge index outside col
          if (bad_u < 0) bad_u = u;
          e1[a] = e0[a];
        }
      }
    }
    int maxd = 0;
#pragma unroll
    for (int a = 0; a < V; a++) maxd = max(maxd, e1[a] - e0[a]);
    for (int j = 0; j < maxd; j += 8) {
      int v[V][8];
#pragma unroll
      for (int a = 0; a < V; a++) {
        const int b = e0[a] + j;
        if (b + 8 <= e1[a] && (b & 3) == 0) {
          const int4 x = __ldg(reinterpret_cast<const int4*>(col + b));
          const int4 y = __ldg(reinterpret_cast<const int4*>(col + b + 4));
          v[a][0] = x.x; v[a][1] = x.y; v[a][2] = x.z; v[a][3] = x.w;
          v[a][4] = y.x; v[a][5] = y.y; v[a][6] = y.z; v[a][7] = y.w;
        } else {
#pragma unroll
          for (int t = 0; t < 8; t++) v[a][t] = b + t < e1[a] ? __ldg(col + b + t) : -1;
        }
      }
      unsigned w[V][8];
#pragma unroll
      for (int a = 0; a < V; a++)
#pragma unroll
        for (int t = 0; t < 8; t++) {
          w[a][t] = 0u;
          if (e0[a] + j + t < e1[a]) {
            if (v[a][t] < 0 || v[a][t] >= ll) {
              if (bad_u < 0) bad_u = uu[a];
            } else {
              w[a][t] = probe ? __ldcg(unv + (v[a][t] >> 5)) : 0xffffffffu;
            }
          }
        }
#pragma unroll
      for (int a = 0; a < V; a++)
#pragma unroll
        for (int t = 0; t < 8; t++) {
          const unsigned bit = 1u << (v[a][t] & 31);
          if (w[a][t] & bit) {
            if (!DEFER) lvl[v[a][t]] = nxt;
            atomicAnd(unv + (v[a][t] >> 5), ~bit);  // result unused: RED
            any = true;
          }
        }
    }
  }
  if (bad_u >= 0) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, bfs_block_of_x(k, bad_u / bx));
  if (DEFER) return;  // bfs_apply writes lvl and the changed flag
  if (__syncthreads_or(any) && threadIdx.x == 0) {
    if (lch < 1) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, k.first);
    else changed[0] = 1;
  }
}

// Deferred level writes of the relax step: the vertices claimed in this
// launch are unv0 & ~unv (unvisited at the start, cleared by the relax); one
// thread per 4 vertices rewrites their int4 of lvl only where a claim falls
// (read-merge-write of whole 16 B pieces, all 4 claimed: plain store), so the
// big levels write lvl in full sectors instead of one scattered 4 B store per
// claimed vertex (a partial-sector read-modify-write in DRAM).
__global__ void __launch_bounds__(256) bfs_apply(const unsigned* __restrict__ unv0, const unsigned* unv, int* lvl,
                                                 long long ll, int cur, int* changed, long long lch, KDesc k,
                                                 const int* qn, int defer_min) {
  if (*qn < defer_min) return;  // the relax wrote lvl itself
  const long long quads = (ll + 3) / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int nxt = (int)((unsigned)cur + 1u);
  bool any = false;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < quads; t += stride) {
    const long long w = t >> 3;
    const unsigned m = ((unv0[w] & ~__ldcg(unv + w)) >> (4 * (t & 7))) & 0xFu;
    if (!m) continue;
    any = true;
    const long long v0 = t * 4;
    if (v0 + 4 <= ll) {
      int4* p = reinterpret_cast<int4*>(lvl + v0);
      int4 x = m == 0xFu ? make_int4(nxt, nxt, nxt, nxt) : *p;
      if (m & 1u) x.x = nxt;
      if (m & 2u) x.y = nxt;
      if (m & 4u) x.z = nxt;
      if (m & 8u) x.w = nxt;
      *p = x;
    } else {
      for (int j = 0; j < 4; j++)
        if (m & (1u << j)) lvl[v0 + j] = nxt;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) {
    if (lch < 1) record_fault(k, BF_TRAP_OUT_OF_BOUNDS, k.first);
    else changed[0] = 1;
  }
}

// per-stream scratch of the two-phase step (grow-only)
struct BfsStepScratch : StreamScratch {
  long long cap_words = 0, cap_q = 0;
  unsigned* unv = nullptr;
  unsigned* unv0 = nullptr;  // unvisited set at the launch start (deferred lvl writes)
  int* q = nullptr;
  int* qn = nullptr;
  void release() {
    cudaFree(unv);
    cudaFree(unv0);
    cudaFree(q);
    cudaFree(qn);
    unv = unv0 = nullptr;
    q = qn = nullptr;
    cap_words = cap_q = 0;
  }
  ~BfsStepScratch() override { release(); }
};

static int launch_bfs_two_phase(LaunchCtx& ctx, const ArgVal& R, const ArgVal& Co, const ArgVal& L,
                                const ArgVal& Ch, long long lo, long long hi, int cur, long long bx) {
  // keyed by the fetch's stream: fetches on other worker streams may run
  // concurrently and have their own; growing orders against this stream only
  BfsStepScratch& S = scratch_for<BfsStepScratch>(ctx.stream, SCRATCH_BFS_STEP);
  const long long ll = L.len, words = (ll + 31) / 32, nq = hi - lo;
  if (S.cap_words < words || S.cap_q < nq || !S.qn) {
    cudaStreamSynchronize(ctx.stream);
    S.release();
    if (cudaMalloc((void**)&S.unv, words * 4) != cudaSuccess || cudaMalloc((void**)&S.unv0, words * 4) != cudaSuccess ||
        cudaMalloc((void**)&S.q, nq * 4) != cudaSuccess ||
        cudaMalloc((void**)&S.qn, 8) != cudaSuccess) {
      *ctx.error = "bfs: scratch allocation failed";
      cudaGetLastError();
      return BF_E_CUDA;
    }
    S.cap_words = words;
    S.cap_q = nq;
  }
  // BF_BFS_RELAX: 3 (default) = bfs_scan2 + bfs_relax_v<2> with the big
  // levels' lvl writes deferred to bfs_apply; 2 = bfs_scan + bfs_relax_v<2>;
  // 0 = bfs_scan + bfs_relax (claiming atomics)
  static int relax_v = -1, defer_div = -1;
  if (relax_v < 0) {
    const char* e = getenv("BF_BFS_RELAX");
    relax_v = e ? atoi(e) : 3;
    const char* d = getenv("BF_BFS_DEFER_DIV");  // frontier >= len(lvl) / div: deferred writes
    defer_div = d ? std::max(1, atoi(d)) : 64;
  }
  cudaMemsetAsync(S.qn, 0, 8, ctx.stream);  // [0] frontier, [1] unvisited
  if (relax_v == 3) {
    const int defer_min = (int)std::max(1LL, ll / defer_div);
    const int g1 = wave_grid(bfs_scan2, 256, 0, words * 8, 256 * 8, ctx.num_sms, 8);
    bfs_scan2<<<g1, 256, 0, ctx.stream>>>((const int*)L.ptr, ll, S.unv, S.unv0, S.q, S.qn, lo, hi, cur);
    BF_CUDA_LAUNCH_CHECK(ctx);
    const int g2 = wave_grid(bfs_relax_v<2>, 256, 0, (nq + 1) / 2, 256, ctx.num_sms, 8);
    bfs_relax_v<2><<<g2, 256, 0, ctx.stream>>>((const int*)R.ptr, R.len, (const int*)Co.ptr, Co.len, (int*)L.ptr,
                                               ll, S.unv, S.q, S.qn, (int*)Ch.ptr, Ch.len, cur, (int)bx, ctx.desc(),
                                               defer_min);
    BF_CUDA_LAUNCH_CHECK(ctx);
    const int g3 = wave_grid(bfs_apply, 256, 0, (ll + 3) / 4, 256, ctx.num_sms, 8);
    bfs_apply<<<g3, 256, 0, ctx.stream>>>(S.unv0, S.unv, (int*)L.ptr, ll, cur, (int*)Ch.ptr, Ch.len, ctx.desc(),
                                          S.qn, defer_min);
    BF_CUDA_LAUNCH_CHECK(ctx);
    return BF_OK;
  }
  const int g1 = wave_grid(bfs_scan, 256, 0, words, 256, ctx.num_sms, 8);
  bfs_scan<<<g1, 256, 0, ctx.stream>>>((const int*)L.ptr, ll, S.unv, words, S.q, S.qn, lo, hi, cur);
  BF_CUDA_LAUNCH_CHECK(ctx);
  if (relax_v > 0) {
    const int g2 = wave_grid(bfs_relax_v<2>, 256, 0, (nq + 1) / 2, 256, ctx.num_sms, 8);
    bfs_relax_v<2><<<g2, 256, 0, ctx.stream>>>((const int*)R.ptr, R.len, (const int*)Co.ptr, Co.len, (int*)L.ptr,
                                               ll, S.unv, S.q, S.qn, (int*)Ch.ptr, Ch.len, cur, (int)bx, ctx.desc(),
                                               INT_MAX);
  } else {
    const int g2 = wave_grid(bfs_relax, 256, 0, nq, 256, ctx.num_sms, 8);
    bfs_relax<<<g2, 256, 0, ctx.stream>>>((const int*)R.ptr, R.len, (const int*)Co.ptr, Co.len, (int*)L.ptr, ll,
                                          S.unv, S.q, S.qn, (int*)Ch.ptr, Ch.len, cur, (int)bx, ctx.desc());
  }
  BF_CUDA_LAUNCH_CHECK(ctx);
  return BF_OK;
}

static int launch_bfs(LaunchCtx& ctx) {
  const ArgVal& R = ctx.args[0];
  const ArgVal& Co = ctx.args[1];
  const ArgVal& L = ctx.args[2];
  const ArgVal& Ch = ctx.args[3];
  const long long nv = ctx.args[4].i32;
  const int cur = ctx.args[5].i32;
  const long long bx = ctx.block[0];
  if ((long long)ctx.grid[1] * ctx.grid[2] * ctx.block[1] * ctx.block[2] != 1) {
    // duplicated vertex threads are harmless here (idempotent), but keep the
    // geometry contract uniform with the other graph kernels
    *ctx.error = "bfs: only 1D grids/blocks are supported";
    return BF_E_UNSUPPORTED;
  }
  if ((long long)ctx.grid[0] * bx - 1 > INT_MAX) {
    *ctx.error = "bfs: vertex id beyond i32";
    return BF_E_UNSUPPORTED;
  }
  static int step_v = -1;
  if (step_v < 0) {
    const char* e = getenv("BF_BFS_STEP_V");
    step_v = e ? atoi(e) : 2;
  }
  const bool whole = ctx.first == 0 && ctx.count == (long long)ctx.grid[0];
  for (auto& xi : ctx.x_intervals()) {
    long long lo = xi.first * bx, hi = std::min(xi.second * bx, nv);
    if (lo >= hi) continue;
    if (step_v == 2 && whole && hi <= L.len) {
      // the fetch covers the whole grid: one lvl pass builds the visited bitmap
      int rc = launch_bfs_two_phase(ctx, R, Co, L, Ch, lo, hi, cur, bx);
      if (rc) return rc;
      continue;
    }
    int grid = wave_grid(bfs_step, 256, 0, (hi - lo + 3) / 4, 256, ctx.num_sms, 8);
    bfs_step<<<grid, 256, 0, ctx.stream>>>((const int*)R.ptr, R.len, (const int*)Co.ptr, Co.len,
                                           (int*)L.ptr, L.len, (int*)Ch.ptr, Ch.len, lo, hi, cur,
                                           (int)bx, ctx.desc());
    BF_CUDA_LAUNCH_CHECK(ctx);
  }
  return BF_OK;
}

// ===========================================================================
// Fused traversal (the Rodinia host loop, on the device): bf_bfs_levels.
// Level-synchronous, direction-optimizing (Beamer's top-down / bottom-up
// switch) over two nv-bit bitmaps (8 MB each at 2^26 vertices, L2-resident):
//   top-down expand:  for u in frontier, v in out(u): if v's bit in `now` is
//            clear, set it (fire-and-forget red.or);
//   compact: next frontier = bits in `now` not in `prev` (a sweep over the
//            bitmap, not over lvl[]), prev |= now; ids appended as one
//            contiguous run per CTA, level bytes merged per 32 B sector;
//   bottom-up step (bf_bfs_levels_do, with the transposed graph): every
//            unvisited vertex scans its in-edges until one comes from the
//            frontier bitmap; the step writes the next frontier's bitmap,
//            queue and level bytes itself (no separate compaction).
// BFS levels are unique, so the direction never changes a level: same levels
// as repeated `bfs` launches.  The choice is made on the device from exact
// counts (frontier size, visited count) by the first kernel of each level,
// so the pipelined host loop never waits for it.
// ===========================================================================

// Level-counter block of the pipelined loop (4 ints per level, rotating over
// three levels): [0] frontier size, [1] frontier bitmap F of this level
// written (the bottom-up step may run), [2] CSR error flag, [3] direction
// chosen for this level (1: bottom-up).  Bottom-up when F exists and
// |F| * alpha16 >= 16 * unvisited.
__device__ __forceinline__ bool bfs_pick_bottom_up(const int* B, const int* vis, long long nv, int alpha16) {
  if (!vis || !B[1]) return false;
  const long long unvisited = nv - 1 - (long long)*vis;
  return (long long)B[0] * alpha16 >= 16 * unvisited;
}

// Expansion with whole-adjacency vector loads: two frontier vertices per
// thread, eight edges per vertex per step; an 8-edge chunk starting at a
// multiple of 4 is fetched as two 16 B loads (the full 32 B sector at once,
// default caching), anything else edge by edge.  All 16 targets' bitmap
// words are loaded before any RED is issued.
constexpr int kBfsV2 = 2;

template <bool TEST, int V = kBfsV2>
__global__ void __launch_bounds__(256) bfs_expand_v(const int* __restrict__ row,
                                                    const int* __restrict__ col, long long ne,
                                                    unsigned* now, long long nv,
                                                    const int* __restrict__ q, int* sizes,
                                                    int* zero_p, int* hist, const int* vis = nullptr,
                                                    int alpha16 = 0, const unsigned* __restrict__ fin = nullptr,
                                                    const int* visc = nullptr, int probe_mode = 1) {
  const int qn = sizes[0];
  // probe the target's bitmap word before the RED: always (1), never (0), or
  // once more than half of the vertices are visited (2; visc: visited count)
  const bool probe = TEST && (probe_mode == 1 || (probe_mode == 2 && visc && 2ll * *visc > nv));
  const bool bottom_up = bfs_pick_bottom_up(sizes, vis, nv, alpha16);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // pipelined loop: next-next level's block, qn record, direction
    if (zero_p) {
      zero_p[0] = 0;
      zero_p[1] = 0;
      zero_p[3] = 0;
    }
    if (hist) *(volatile int*)hist = qn;
    if (vis) sizes[3] = bottom_up;
  }
  if (bottom_up) return;  // bfs_bottom_up expands this level
  if (fin && sizes[1] == 2) {  // a bottom-up level left this frontier as a bitmap only
    const long long words = (nv + 31) / 32;
    const long long gstride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gstride) {
      for (unsigned f = __ldg(fin + i); f; f &= f - 1) {
        const int u = (int)(i * 32 + __ffs(f) - 1);
        int e0 = __ldg(row + u), e1 = __ldg(row + u + 1);
        if (e0 < 0 || e1 > ne || e1 < e0) {
          sizes[2] = 1;
          continue;
        }
        for (int b = e0; b < e1; b += 8) {
          int v[8];
          unsigned wv[8];
#pragma unroll
          for (int t = 0; t < 8; t++) v[t] = b + t < e1 ? __ldg(col + b + t) : -1;
#pragma unroll
          for (int t = 0; t < 8; t++) {
            wv[t] = 0xffffffffu;
            if (v[t] >= nv) sizes[2] = 1;
            else if (v[t] >= 0) wv[t] = __ldcg(now + (v[t] >> 5));
          }
#pragma unroll
          for (int t = 0; t < 8; t++)
            if (v[t] >= 0 && v[t] < nv && !(wv[t] & (1u << (v[t] & 31)))) atomicOr(now + (v[t] >> 5), 1u << (v[t] & 31));
        }
      }
    }
    return;
  }
  const long long stride = (long long)gridDim.x * blockDim.x * V;
  for (long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * V; i0 < qn; i0 += stride) {
    int e0[V], e1[V];
#pragma unroll
    for (int a = 0; a < V; a++) {
      e0[a] = e1[a] = 0;
      if (i0 + a < qn) {
        const int u = __ldg(q + i0 + a);
        const int2 rr = (u & 1) ? make_int2(__ldg(row + u), __ldg(row + u + 1))
                                : __ldg(reinterpret_cast<const int2*>(row + u));
        e0[a] = rr.x;
        e1[a] = rr.y;
        if (e0[a] < 0 || e1[a] > ne || e1[a] < e0[a]) {
          sizes[2] = 1;
          e1[a] = e0[a];
        }
      }
    }
    int maxd = 0;
#pragma unroll
    for (int a = 0; a < V; a++) maxd = max(maxd, e1[a] - e0[a]);
    for (int j = 0; j < maxd; j += 8) {
      int v[V][8];
#pragma unroll
      for (int a = 0; a < V; a++) {
        const int b = e0[a] + j;
        if (b + 8 <= e1[a] && (b & 3) == 0) {
          const int4 x = __ldg(reinterpret_cast<const int4*>(col + b));
          const int4 y = __ldg(reinterpret_cast<const int4*>(col + b + 4));
          v[a][0] = x.x; v[a][1] = x.y; v[a][2] = x.z; v[a][3] = x.w;
          v[a][4] = y.x; v[a][5] = y.y; v[a][6] = y.z; v[a][7] = y.w;
        } else {
#pragma unroll
          for (int t = 0; t < 8; t++) v[a][t] = b + t < e1[a] ? __ldg(col + b + t) : -1;
        }
      }
      unsigned w[V][8];
#pragma unroll
      for (int a = 0; a < V; a++)
#pragma unroll
        for (int t = 0; t < 8; t++) {
          w[a][t] = 0xffffffffu;
          if (v[a][t] >= 0) {
            if (v[a][t] >= nv) sizes[2] = 1;
            else w[a][t] = probe ? __ldcg(now + (v[a][t] >> 5)) : 0u;
          }
        }
#pragma unroll
      for (int a = 0; a < V; a++)
#pragma unroll
        for (int t = 0; t < 8; t++) {
          const unsigned bit = 1u << (v[a][t] & 31);
          if (v[a][t] >= 0 && v[a][t] < nv && !(w[a][t] & bit)) atomicOr(now + (v[a][t] >> 5), bit);
        }
    }
  }
}

// Compaction with coalesced writes (depth + 1 < 255): the CTA's new
// vertices are staged in shared memory and leave as one contiguous queue run,
// and a word's 32 level bytes (one 32 B sector of lv8) are merged in
// registers and stored as two 16 B vectors instead of one byte store per new
// vertex.  Same queue contents and order as bfs_compact8.
__device__ __forceinline__ unsigned lv8_merge(unsigned x, unsigned fresh, int sh, unsigned lb) {
  const unsigned m4 = (fresh >> sh) & 0xFu;
  const unsigned bm = ((m4 * 0x00204081u) & 0x01010101u) * 0xFFu;  // bit j -> byte j
  return (x & ~bm) | (lb & bm);
}

__global__ void __launch_bounds__(256) bfs_compact8s(unsigned* now, unsigned* prev, long long words,
                                                     int* nq, const int* qn_p, int* out_cnt,
                                                     unsigned char* lv8, int* lvl, int depth,
                                                     unsigned* fout = nullptr, int* vis = nullptr) {
  // qn_p / out_cnt: this and the next level's counter blocks (bfs_pick_bottom_up);
  // fout: the next level's frontier bitmap, every word written (bottom-up may
  // expand it); vis: running count of visited vertices
  __shared__ int stage[256 * 32];
  __shared__ int wtot[8];
  __shared__ int cbase, ctot;
  if (qn_p[0] == 0 || qn_p[3]) return;  // nothing was expanded, or the bottom-up step ran
  if (fout && blockIdx.x == 0 && threadIdx.x == 0) out_cnt[1] = 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool bytes = depth + 1 < 255;
  const unsigned lb = (unsigned)(depth + 1) * 0x01010101u;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // the next iteration's bitmap words are loaded one iteration ahead, and an
  // iteration whose 256 words hold no new vertex (most of them on small
  // levels) costs one barrier
  unsigned cn = 0, cp = 0;
  {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < words) {
      cn = __ldcg(now + i);
      cp = prev[i];
    }
  }
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < words; i0 += stride) {  // CTA-uniform
    const long long i = i0 + threadIdx.x;
    const unsigned nw = cn, pw = cp;
    if (i + stride < words) {
      cn = __ldcg(now + i + stride);
      cp = prev[i + stride];
    }
    unsigned fresh = i < words ? nw & ~pw : 0u;
    if (fout && i < words) fout[i] = fresh;
    if (!__syncthreads_or(fresh != 0)) continue;
    if (i < words) {
      if (fresh && !bytes) {  // levels beyond a byte: lvl written directly
        prev[i] = nw;
        for (unsigned f = fresh; f; f &= f - 1) lvl[i * 32 + __ffs(f) - 1] = depth + 1;
      } else if (fresh) {
        prev[i] = nw;
        uint4* p = reinterpret_cast<uint4*>(lv8 + i * 32);
        uint4 a = p[0], b = p[1];
        a.x = lv8_merge(a.x, fresh, 0, lb);
        a.y = lv8_merge(a.y, fresh, 4, lb);
        a.z = lv8_merge(a.z, fresh, 8, lb);
        a.w = lv8_merge(a.w, fresh, 12, lb);
        b.x = lv8_merge(b.x, fresh, 16, lb);
        b.y = lv8_merge(b.y, fresh, 20, lb);
        b.z = lv8_merge(b.z, fresh, 24, lb);
        b.w = lv8_merge(b.w, fresh, 28, lb);
        p[0] = a;
        p[1] = b;
      }
    }
    const int c = __popc(fresh);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < 8; w++) {
        const int t = wtot[w];
        wtot[w] = run;
        run += t;
      }
      ctot = run;
      cbase = run ? atomicAdd(out_cnt, run) : 0;
      if (run && vis) atomicAdd(vis, run);
    }
    __syncthreads();
    int pos = wtot[warp] + incl - c;
    for (unsigned f = fresh; f; f &= f - 1) stage[pos++] = (int)(i * 32 + __ffs(f) - 1);
    __syncthreads();
    const int tot = ctot, base = cbase;
    for (int j = threadIdx.x; j < tot; j += blockDim.x) nq[base + j] = stage[j];
    __syncthreads();
  }
}

// lvl[v] from the level bytes (0xFF: unvisited, or a level >= 255 already in lvl)
__global__ void __launch_bounds__(256) bfs_finish(const unsigned char* __restrict__ lv8, int* lvl, long long nv,
                                                  bool deep) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const uchar4* b4 = reinterpret_cast<const uchar4*>(lv8);
  int4* l4 = reinterpret_cast<int4*>(lvl);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv / 4; i += stride) {
    const uchar4 b = b4[i];
    int4 o = deep ? l4[i] : make_int4(-1, -1, -1, -1);
    if (b.x != 0xFF) o.x = b.x;
    if (b.y != 0xFF) o.y = b.y;
    if (b.z != 0xFF) o.z = b.z;
    if (b.w != 0xFF) o.w = b.w;
    __stcs(l4 + i, o);
  }
  for (long long i = nv / 4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    const unsigned char b = lv8[i];
    lvl[i] = b != 0xFF ? (int)b : (deep ? lvl[i] : -1);
  }
}

__global__ void __launch_bounds__(256) bfs_init8(unsigned char* lv8, unsigned* now, unsigned* prev,
                                                 long long nv, long long words, int src, int* q0, int* sizes) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  uint4* b16 = reinterpret_cast<uint4*>(lv8);
  for (long long i = t; i < nv / 16; i += stride) b16[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
  for (long long i = nv / 16 * 16 + t; i < nv; i += stride) lv8[i] = 0xFF;
  for (long long i = t; i < words; i += stride) {
    now[i] = 0u;
    prev[i] = 0u;
  }
  if (t == 0) {
    sizes[0] = 1;
    sizes[1] = 0;
    sizes[2] = 0;
    q0[0] = src;
  }
}

__global__ void bfs_seed8(unsigned char* lv8, unsigned* now, unsigned* prev, int src) {
  lv8[src] = 0;
  now[src >> 5] = 1u << (src & 31);
  prev[src >> 5] = 1u << (src & 31);
}

__global__ void __launch_bounds__(256) bfs_fill_m1(int* lvl, long long nv) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) lvl[i] = -1;
}

// ---- sharded traversal (one process per GPU, parallel.bfs_levels_sharded) --
// Every rank keeps the whole visited bitmap and the level bytes; it expands
// only the frontier vertices of its own range [vlo, vhi); after the ranks'
// bitmaps are OR-merged (an all-gather of the nv-bit `now`), the compaction
// sees the same fresh set on every rank: all ranks record the same levels,
// each enqueues only its own fresh vertices, and the global fresh count (the
// loop condition) agrees without another collective.
__global__ void __launch_bounds__(256) bfs_merge_or(unsigned* now, const unsigned* __restrict__ g,
                                                    long long words, int world) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) {
    unsigned v = now[i];
    for (int r = 0; r < world; r++) v |= __ldcs(g + (long long)r * words + i);
    now[i] = v;
  }
}

// one rank's slice of the visited bitmap after an all-to-all: recv holds the
// world ranks' copies of words [first, first + count) back to back
__global__ void __launch_bounds__(256) bfs_merge_slice(unsigned* now, const unsigned* __restrict__ recv,
                                                       long long count, int world) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    unsigned v = 0;
    for (int r = 0; r < world; r++) v |= __ldcs(recv + (long long)r * count + i);
    now[i] = v;
  }
}

// sizes: [0] own queue length, [1] next own queue length, [2] CSR error, [3] global fresh
__global__ void __launch_bounds__(256) bfs_compact_sh(unsigned* now, unsigned* prev, long long words, int* nq,
                                                      int* sizes, unsigned char* lv8, int* lvl, int depth,
                                                      long long vlo, long long vhi) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const bool bytes = depth + 1 < 255;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < words; i0 += stride) {  // CTA-uniform
    const long long i = i0 + threadIdx.x;
    unsigned fresh = 0, own = 0;
    if (i < words) {
      const unsigned nw = __ldcg(now + i);
      fresh = nw & ~prev[i];
      if (fresh) prev[i] = nw;
      // bits of word i inside [vlo, vhi)
      const long long b0 = i * 32;
      unsigned m = 0xffffffffu;
      if (b0 < vlo) m = vlo - b0 >= 32 ? 0u : (m << (vlo - b0));
      if (b0 + 32 > vhi) m &= vhi <= b0 ? 0u : (0xffffffffu >> (b0 + 32 - vhi));
      own = fresh & m;
    }
    int pos = cta_append(__popc(own), sizes + 1, sizes + 3, __popc(fresh));
    if (fresh && bytes) {  // the word's 32 level bytes: one merged 32 B sector store
      const unsigned lb = (unsigned)(depth + 1) * 0x01010101u;
      uint4* p = reinterpret_cast<uint4*>(lv8 + i * 32);
      uint4 a = p[0], c = p[1];
      a.x = lv8_merge(a.x, fresh, 0, lb);
      a.y = lv8_merge(a.y, fresh, 4, lb);
      a.z = lv8_merge(a.z, fresh, 8, lb);
      a.w = lv8_merge(a.w, fresh, 12, lb);
      c.x = lv8_merge(c.x, fresh, 16, lb);
      c.y = lv8_merge(c.y, fresh, 20, lb);
      c.z = lv8_merge(c.z, fresh, 24, lb);
      c.w = lv8_merge(c.w, fresh, 28, lb);
      p[0] = a;
      p[1] = c;
    }
    while (fresh) {
      const int b = __ffs(fresh) - 1;
      const int v = (int)(i * 32 + b);
      if (own >> b & 1) nq[pos++] = v;
      if (!bytes) lvl[v] = depth + 1;
      fresh &= fresh - 1;
    }
  }
}

// ---- bottom-up step (direction-optimizing traversal) ------------------------
// A warp owns a chunk of 32 bitmap words (1024 vertices) at a time: one
// coalesced load of the words, a warp scan of their unvisited counts, then
// the chunk's unvisited vertices are dealt to the lanes by rank (rank ->
// word by a shuffle binary search, -> bit by __fns), two per lane in flight,
// each scanning its in-edges four at a time until one comes from the
// frontier bitmap F.  Hits are OR-ed into the warp's 32 new-bit words in
// shared memory; then lane j writes word j of the chunk: now/prev, the next
// frontier bitmap Fn (every word), and the word's 32 level bytes as one
// merged sector.  No CTA barriers and no queue: a top-down level that
// follows a bottom-up one reads its frontier from Fn (block flag [1] = 2),
// and the new-vertex count leaves with one atomic per CTA at the end.
__device__ __forceinline__ int bu_rank_to_vertex(int r, int T, int incl, int c, unsigned un, long long ch) {
  // smallest lane j with incl_j > r (all lanes take part in every shuffle)
  int j = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int x = __shfl_sync(0xffffffffu, incl, j + step - 1);
    if (x <= r) j += step;
  }
  const int ex = __shfl_sync(0xffffffffu, incl - c, j);
  const unsigned wj = __shfl_sync(0xffffffffu, un, j);
  if (r >= T) return -1;
  const int bit = (int)__fns(wj, 0, r - ex + 1);
  return (int)((ch * 32 + j) * 32 + bit);
}

__global__ void __launch_bounds__(256) bfs_bottom_up(const int* __restrict__ crow, const int* __restrict__ ccol,
                                                     long long ncc, unsigned* now, unsigned* prev, long long words,
                                                     long long nv, const unsigned* __restrict__ F, unsigned* Fn,
                                                     int* B, int* Bn, int* vis, unsigned char* lv8, int* lvl,
                                                     int depth) {
  __shared__ unsigned fr[8][32];
  __shared__ int cnt_s[8];
  if (!B[3]) return;  // top-down level
  if (blockIdx.x == 0 && threadIdx.x == 0) Bn[1] = 2;  // F written, no queue
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool bytes = depth + 1 < 255;
  const unsigned lb = (unsigned)(depth + 1) * 0x01010101u;
  const int tail = (int)(nv & 31);
  const long long nchunks = (words + 31) / 32;
  int count = 0;
  for (long long ch = (long long)blockIdx.x * 8 + warp; ch < nchunks; ch += (long long)gridDim.x * 8) {
    const long long i = ch * 32 + lane;
    const unsigned w = i < words ? now[i] : ~0u;
    unsigned un = ~w;
    if (i == words - 1 && tail) un &= (1u << tail) - 1u;
    const int c = __popc(un);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int T = __shfl_sync(0xffffffffu, incl, 31);
    if (T == 0) {
      if (i < words) Fn[i] = 0u;
      continue;
    }
    fr[warp][lane] = 0u;
    __syncwarp();
    for (int r0 = 0; r0 < T; r0 += 64) {
      const int v0 = bu_rank_to_vertex(r0 + lane, T, incl, c, un, ch);
      const int v1 = bu_rank_to_vertex(r0 + 32 + lane, T, incl, c, un, ch);
      int a0 = 0, a1 = 0, b0 = 0, b1 = 0;
      if (v0 >= 0) {
        a0 = __ldg(crow + v0);
        a1 = __ldg(crow + v0 + 1);
      }
      if (v1 >= 0) {
        b0 = __ldg(crow + v1);
        b1 = __ldg(crow + v1 + 1);
      }
      if (a0 < 0 || a1 > ncc || a1 < a0) {
        B[2] = 1;
        a1 = a0;
      }
      if (b0 < 0 || b1 > ncc || b1 < b0) {
        B[2] = 1;
        b1 = b0;
      }
      bool h0 = false, h1 = false;
      while (a0 < a1 || b0 < b1) {
        int u[8];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          u[k] = a0 + k < a1 ? __ldg(ccol + a0 + k) : -1;
          u[4 + k] = b0 + k < b1 ? __ldg(ccol + b0 + k) : -1;
        }
        unsigned fw[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
          fw[k] = 0u;
          if (u[k] >= 0) {
            if (u[k] >= nv) B[2] = 1;
            else fw[k] = __ldg(F + (u[k] >> 5)) & (1u << (u[k] & 31));
          }
        }
        const bool x0 = (fw[0] | fw[1] | fw[2] | fw[3]) != 0u;
        const bool x1 = (fw[4] | fw[5] | fw[6] | fw[7]) != 0u;
        h0 |= x0;
        h1 |= x1;
        a0 = x0 ? a1 : a0 + 4;
        b0 = x1 ? b1 : b0 + 4;
      }
      if (h0) atomicOr(&fr[warp][(v0 >> 5) - (int)(ch * 32)], 1u << (v0 & 31));
      if (h1) atomicOr(&fr[warp][(v1 >> 5) - (int)(ch * 32)], 1u << (v1 & 31));
    }
    __syncwarp();
    const unsigned fresh = fr[warp][lane];
    if (i < words) {
      Fn[i] = fresh;
      if (fresh) {
        now[i] = w | fresh;
        prev[i] = w | fresh;
        if (bytes) {
          uint4* p = reinterpret_cast<uint4*>(lv8 + i * 32);
          uint4 a = p[0], b = p[1];
          a.x = lv8_merge(a.x, fresh, 0, lb);
          a.y = lv8_merge(a.y, fresh, 4, lb);
          a.z = lv8_merge(a.z, fresh, 8, lb);
          a.w = lv8_merge(a.w, fresh, 12, lb);
          b.x = lv8_merge(b.x, fresh, 16, lb);
          b.y = lv8_merge(b.y, fresh, 20, lb);
          b.z = lv8_merge(b.z, fresh, 24, lb);
          b.w = lv8_merge(b.w, fresh, 28, lb);
          p[0] = a;
          p[1] = b;
        } else {
          for (unsigned f = fresh; f; f &= f - 1) lvl[i * 32 + __ffs(f) - 1] = depth + 1;
        }
      }
    }
    count += __popc(fresh);
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
  if (lane == 0) cnt_s[warp] = count;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int k = 0; k < 8; k++) tot += cnt_s[k];
    if (tot) {
      atomicAdd(Bn, tot);
      atomicAdd(vis, tot);
    }
  }
}

// ---- graph transpose (in-edge CSR for the bottom-up step) --------------------
// A stable radix sort of the (target, source) pairs by target: ccol is the
// sorted sources (so every in-list is in ascending source order:
// deterministic), crow[v] the first sorted position with target >= v.
// Edges are [row[0], row[nv]); a malformed row or an out-of-range target
// sets err.
__global__ void __launch_bounds__(256) bfs_tr_pairs(const int* __restrict__ row, const int* __restrict__ col,
                                                    long long nv, int e_base, int e_end, unsigned* key, int* srcv,
                                                    int* err) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < nv; u += stride) {
    const int e0 = __ldg(row + u), e1 = __ldg(row + u + 1);
    if (e1 < e0 || e0 < e_base || e1 > e_end) {
      *err = 1;
      continue;
    }
    for (int e = e0; e < e1; e++) {
      const int v = __ldg(col + e);
      if (v < 0 || v >= nv) *err = 1;
      key[e - e_base] = (unsigned)v;
      srcv[e - e_base] = (int)u;
    }
  }
}

// crow[v] = first i with key[i] >= v (key sorted), crow[nv] = n
__global__ void __launch_bounds__(256) bfs_tr_offsets(const unsigned* __restrict__ key, long long n, long long nv,
                                                      int* crow) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
    const long long lo = i == 0 ? 0 : (long long)__ldg(key + i - 1) + 1;
    const long long hi = i == n ? nv : (long long)__ldg(key + i);
    for (long long v = lo; v <= hi && v <= nv; v++) crow[v] = (int)i;
  }
}

}  // namespace bf

// In-edge CSR (crow: nv + 1, ccol: the edge count) of the CSR graph (row,
// col); BF_E_FAULT when row is malformed or a target is out of range.
extern "C" int bf_bfs_transpose_impl(void* stream_v, int num_sms, const int* row, long long lr, const int* col,
                                     long long lcol, int nv, int* crow, long long lcrow, int* ccol, long long lccol,
                                     char* err, int errcap) {
  using namespace bf;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (nv <= 0 || lr < (long long)nv + 1 || lcrow < (long long)nv + 1) {
    snprintf(err, errcap, "bfs_transpose: bad sizes (nv=%d len(row)=%lld len(crow)=%lld)", nv, lr, lcrow);
    return BF_E_INVALID;
  }
  int h[2] = {0, 0};
  cudaError_t e = cudaMemcpyAsync(&h[0], row, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h[1], row + nv, 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e == cudaSuccess && (h[0] < 0 || h[1] < h[0] || h[1] > lcol)) {
    snprintf(err, errcap, "bfs_transpose: CSR index out of range");
    e = cudaErrorInvalidValue;
  }
  const long long n = (long long)h[1] - h[0];
  if (e == cudaSuccess && n > lccol) {
    snprintf(err, errcap, "bfs_transpose: %lld edges do not fit len(ccol)=%lld", n, lccol);
    e = cudaErrorInvalidValue;
  }
  int end_bit = 1;
  while (end_bit < 32 && (1ll << end_bit) < (long long)nv) end_bit++;
  unsigned *key = nullptr, *key_out = nullptr;
  int *srcv = nullptr, *flag = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  if (e == cudaSuccess) e = cudaMalloc((void**)&flag, 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&key, (size_t)std::max(n, 1LL) * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&key_out, (size_t)std::max(n, 1LL) * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&srcv, (size_t)std::max(n, 1LL) * 4);
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key_out, srcv, ccol, (int)n, 0, end_bit, stream);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 16));
  if (e == cudaSuccess) {
    int f = 0;
    const int g = stream_grid(nv, 256, num_sms, 8);
    cudaMemsetAsync(flag, 0, 4, stream);
    bfs_tr_pairs<<<g, 256, 0, stream>>>(row, col, nv, h[0], h[1], key, srcv, flag);
    e = cudaMemcpyAsync(&f, flag, 4, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e == cudaSuccess && f) {
      snprintf(err, errcap, "bfs_transpose: CSR index out of range");
      e = cudaErrorInvalidValue;
    }
    if (e == cudaSuccess && n > 0)
      e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_out, srcv, ccol, (int)n, 0, end_bit, stream);
    if (e == cudaSuccess) {
      bfs_tr_offsets<<<stream_grid(n + 1, 256, num_sms, 8), 256, 0, stream>>>(key_out, n, nv, crow);
      e = cudaStreamSynchronize(stream);
    }
  }
  cudaFree(tmp);
  cudaFree(key);
  cudaFree(key_out);
  cudaFree(srcv);
  cudaFree(flag);
  if (e != cudaSuccess) {
    const bool fault = e == cudaErrorInvalidValue && err[0];
    if (!err[0]) snprintf(err, errcap, "bfs_transpose: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return fault ? BF_E_FAULT : BF_E_CUDA;
  }
  return BF_OK;
}

// crow/ccol null: top-down only (bf_bfs_levels); else direction-optimizing
// (bf_bfs_levels_do) over the in-edge CSR made by bf_bfs_transpose.
extern "C" int bf_bfs_levels_impl(void* stream_v, int num_sms, const int* row, long long lr, const int* col,
                                  long long lcol, const int* crow, long long lcrow, const int* ccol, long long lccol,
                                  int* lvl, long long ll, int nv, int src, int* depth_out, char* err, int errcap) {
  using namespace bf;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (nv <= 0 || src < 0 || src >= nv || lr < (long long)nv + 1 || ll < nv ||
      (crow && lcrow < (long long)nv + 1)) {
    snprintf(err, errcap, "bfs_levels: bad sizes (nv=%d src=%d len(row)=%lld len(lvl)=%lld)", nv, src, lr, ll);
    return BF_E_INVALID;
  }
  const long long words = ((long long)nv + 31) / 32;
  // scratch (bitmaps, frontier queues and bitmaps, counters) per stream, grow-only:
  // a traversal does no allocation after the first
  struct Scratch : StreamScratch {
    std::mutex busy;  // a traversal is a synchronous host loop: one caller at a time per stream
    long long cap_v = 0;
    unsigned *now = nullptr, *prev = nullptr, *fb[2] = {nullptr, nullptr};
    int *qa = nullptr, *qb = nullptr;
    unsigned char* lv8 = nullptr;
    int* ctr = nullptr;  // 3 rotating level blocks of 4 ints, [12] visited count
    int *hist = nullptr, *hist_d = nullptr;  // host-mapped frontier sizes
    cudaEvent_t evx[4] = {};
    void release() {
      cudaFree(now);
      cudaFree(prev);
      cudaFree(fb[0]);
      cudaFree(fb[1]);
      cudaFree(qa);
      cudaFree(qb);
      cudaFree(lv8);
      now = prev = fb[0] = fb[1] = nullptr;
      qa = qb = nullptr;
      lv8 = nullptr;
      cap_v = 0;
    }
    ~Scratch() override {
      release();
      cudaFree(ctr);
      if (hist) cudaFreeHost(hist);
      for (auto& ev : evx)
        if (ev) cudaEventDestroy(ev);
    }
  };
  Scratch& S = scratch_for<Scratch>(stream, SCRATCH_BFS_LEVELS);
  std::lock_guard<std::mutex> busy(S.busy);
  cudaError_t e = cudaSuccess;
  if (S.cap_v < nv) {
    cudaStreamSynchronize(stream);
    S.release();
    e = cudaMalloc((void**)&S.now, words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.prev, words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.fb[0], words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.fb[1], words * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.qa, (size_t)nv * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.qb, (size_t)nv * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&S.lv8, (size_t)words * 32 + 16);  // whole sectors
    if (e == cudaSuccess) S.cap_v = nv;
  }
  if (e == cudaSuccess && !S.ctr) e = cudaMalloc((void**)&S.ctr, 16 * sizeof(int));
  if (e == cudaSuccess && !S.hist) {
    e = cudaHostAlloc((void**)&S.hist, 64 * sizeof(int), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&S.hist_d, S.hist, 0);
    for (int i = 0; i < 4 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&S.evx[i], cudaEventDisableTiming);
  }
  // BF_BFS_DO=0 keeps a direction-optimizing call top-down (A/B); BF_BFS_ALPHA16:
  // bottom-up when 16 * |frontier| * alpha16 / 16 >= unvisited
  static int do_on = -1, alpha16 = 32, probe_mode = 2;
  if (do_on < 0) {
    const char* pe = getenv("BF_BFS_PROBE");
    if (pe) probe_mode = atoi(pe);
    const char* de = getenv("BF_BFS_DO");
    do_on = de ? atoi(de) : 1;
    const char* ae = getenv("BF_BFS_ALPHA16");
    if (ae) alpha16 = std::max(1, atoi(ae));
  }
  const bool dir = crow && ccol && do_on;
  bool deep = false;
  int depth = 0;
  if (e == cudaSuccess) {
    unsigned *now = S.now, *prev = S.prev;
    unsigned char* lv8 = S.lv8;
    int* vis = S.ctr + 12;
    const int g = stream_grid(nv, 256 * 4, num_sms, 8);
    const int xgrid = wave_grid(bfs_expand_v<true>, 256, 0, ((long long)nv + 1) / 2, 256, num_sms, 8);
    const int sgrid = wave_grid(bfs_compact8s, 256, 0, words, 256, num_sms, 8);
    const int bgrid = wave_grid(bfs_bottom_up, 256, 0, (words + 31) / 32, 8, num_sms, 8);
    // Pipelined: the host enqueues level d + 2 as soon as level d + 1's
    // expansion has recorded its frontier size (host-mapped), so the device
    // never waits for a host round trip between levels.  Level L uses
    // counter block ctr[4(L%3)] (its frontier), appends into ctr[4((L+1)%3)],
    // and its expansion clears ctr[4((L+2)%3)] (consumed by level L - 1).
    // Bottom-up steps are armed (the previous compaction writes the frontier
    // bitmap and the step is launched; the device still picks) while the
    // last known frontier could reach the switch point within two levels.
    long long seen = 1;  // vertices in the frontiers whose sizes the host has read
    bool armed = false;
    auto arm = [&](long long f_last) {
      const long long unvisited = (long long)nv - seen;
      return dir && f_last * 256LL * alpha16 >= 16 * unvisited;
    };
    bool armed_next = false;  // compaction L wrote F_{L+1}
    auto enqueue = [&](int L) {
      int* B = S.ctr + 4 * (L % 3);
      int* Bn = S.ctr + 4 * ((L + 1) % 3);
      int* Bz = S.ctr + 4 * ((L + 2) % 3);
      int* qL = (L & 1) ? S.qb : S.qa;
      int* nqL = (L & 1) ? S.qa : S.qb;
      if (L + 1 >= 255 && !deep) {  // levels beyond a byte: lvl written directly from here on
        bfs_fill_m1<<<g, 256, 0, stream>>>(lvl, nv);
        deep = true;
      }
      const bool bu = armed_next;  // F_L exists: the bottom-up step may run
      armed_next = armed;
      bfs_expand_v<true><<<xgrid, 256, 0, stream>>>(row, col, lcol, now, nv, qL, B, Bz, S.hist_d + (L & 63),
                                                     bu ? vis : nullptr, alpha16, dir ? S.fb[L & 1] : nullptr,
                                                     vis, probe_mode);
      cudaEventRecord(S.evx[L & 3], stream);
      if (bu)
        bfs_bottom_up<<<bgrid, 256, 0, stream>>>(crow, ccol, lccol, now, prev, words, nv, S.fb[L & 1],
                                                  S.fb[(L + 1) & 1], B, Bn, vis, lv8, lvl, L);
      bfs_compact8s<<<sgrid, 256, 0, stream>>>(now, prev, words, nqL, B, Bn, lv8, lvl, L,
                                               armed_next ? S.fb[(L + 1) & 1] : nullptr, vis);
    };
    cudaMemsetAsync(S.ctr, 0, 16 * sizeof(int), stream);
    bfs_init8<<<g, 256, 0, stream>>>(lv8, now, prev, nv, words, src, S.qa, S.ctr);
    bfs_seed8<<<1, 1, 0, stream>>>(lv8, now, prev, src);
    enqueue(0);
    enqueue(1);
    for (int d = 0;; d++) {
      e = cudaEventSynchronize(S.evx[(d + 1) & 3]);
      if (e != cudaSuccess) break;
      const int qn1 = ((volatile int*)S.hist)[(d + 1) & 63];
      if (qn1 == 0) {
        depth = d + 1;
        break;
      }
      seen += qn1;
      armed = arm(qn1);
      enqueue(d + 2);
    }
    if (e == cudaSuccess) {
      int c[12];
      cudaMemcpyAsync(c, S.ctr, sizeof(c), cudaMemcpyDeviceToHost, stream);
      e = cudaStreamSynchronize(stream);
      if (e == cudaSuccess && (c[2] | c[6] | c[10])) {
        snprintf(err, errcap, "bfs_levels: CSR index out of range");
        e = cudaErrorInvalidValue;
      }
    }
    if (e == cudaSuccess) bfs_finish<<<g, 256, 0, stream>>>(lv8, lvl, nv, deep);
  }
  cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    if (!err[0]) snprintf(err, errcap, "bfs_levels: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorInvalidValue ? BF_E_FAULT : BF_E_CUDA;
  }
  *depth_out = depth;
  return BF_OK;
}


// ---- sharded traversal state (bf_bfs_* in include/bfgpu.h) ----------------
struct BfsShard {
  int nv = 0;
  long long words = 0, vlo = 0, vhi = 0;
  unsigned *now = nullptr, *prev = nullptr;
  int *qa = nullptr, *qb = nullptr, *sizes = nullptr, *hs = nullptr, *lvl_tmp = nullptr;
  unsigned char* lv8 = nullptr;
  int depth = 0, qn = 0;
  bool deep = false;
  int* q = nullptr;
  int* nq = nullptr;
};

extern "C" int bf_bfs_shard_destroy_impl(void* p);

extern "C" int bf_bfs_shard_create_impl(int nv, void** out, char* err, int errcap) {
  using namespace bf;
  if (nv <= 0) {
    snprintf(err, errcap, "bfs shard: nv must be > 0");
    return BF_E_INVALID;
  }
  BfsShard* s = new BfsShard();
  s->nv = nv;
  s->words = ((long long)nv + 31) / 32;
  // `now` carries 64 zero words of padding so an exchange can treat it as
  // world x ceil(words / world) words for any world <= 64 (parallel.py)
  cudaError_t e = cudaMalloc((void**)&s->now, (s->words + 64) * 4);
  if (e == cudaSuccess) e = cudaMemset(s->now, 0, (s->words + 64) * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->prev, s->words * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->qa, (size_t)nv * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->qb, (size_t)nv * 4);
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->lv8, (size_t)s->words * 32 + 16);  // whole sectors
  if (e == cudaSuccess) e = cudaMalloc((void**)&s->sizes, 16);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&s->hs, 16);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    cudaGetLastError();
    bf_bfs_shard_destroy_impl(s);
    return BF_E_CUDA;
  }
  *out = s;
  return BF_OK;
}

extern "C" int bf_bfs_shard_destroy_impl(void* p) {
  BfsShard* s = (BfsShard*)p;
  if (!s) return BF_OK;
  cudaFree(s->now);
  cudaFree(s->prev);
  cudaFree(s->qa);
  cudaFree(s->qb);
  cudaFree(s->lv8);
  cudaFree(s->sizes);
  if (s->hs) cudaFreeHost(s->hs);
  delete s;
  return BF_OK;
}

extern "C" int bf_bfs_shard_bitmap_impl(void* p, void** ptr, long long* words) {
  BfsShard* s = (BfsShard*)p;
  *ptr = s->now;
  *words = s->words;
  return BF_OK;
}

extern "C" int bf_bfs_shard_begin_impl(void* p, void* stream_v, int num_sms, int src, long long vlo, long long vhi,
                                       char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (src < 0 || src >= s->nv || vlo < 0 || vhi < vlo || vhi > s->nv) {
    snprintf(err, errcap, "bfs shard: bad source or vertex range");
    return BF_E_INVALID;
  }
  s->vlo = vlo;
  s->vhi = vhi;
  s->depth = 0;
  s->deep = false;
  s->q = s->qa;
  s->nq = s->qb;
  const int g = stream_grid(s->nv, 256 * 4, num_sms, 8);
  bfs_init8<<<g, 256, 0, stream>>>(s->lv8, s->now, s->prev, s->nv, s->words, src, s->qa, s->sizes);
  bfs_seed8<<<1, 1, 0, stream>>>(s->lv8, s->now, s->prev, src);
  s->qn = (src >= vlo && src < vhi) ? 1 : 0;
  s->hs[0] = s->qn;
  s->hs[1] = 0;
  s->hs[2] = 0;
  s->hs[3] = 0;
  cudaMemcpyAsync(s->sizes, s->hs, 16, cudaMemcpyHostToDevice, stream);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  return BF_OK;
}

extern "C" int bf_bfs_shard_expand_impl(void* p, void* stream_v, int num_sms, const int* row, long long lr,
                                        const int* col, long long lcol, char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (lr < (long long)s->nv + 1) {
    snprintf(err, errcap, "bfs shard: row shorter than nv + 1");
    return BF_E_INVALID;
  }
  if (s->qn > 0) {
    const int grid = stream_grid((s->qn + kBfsV2 - 1) / kBfsV2, 256, num_sms, 8);
    bfs_expand_v<true><<<grid, 256, 0, stream>>>(row, col, lcol, s->now, s->nv, s->q, s->sizes, nullptr, nullptr);
  }
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  return BF_OK;
}

extern "C" int bf_bfs_shard_merge_impl(void* p, void* stream_v, int num_sms, const void* gathered, int world,
                                       char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  const int grid = stream_grid(s->words, 256, num_sms, 8);
  bfs_merge_or<<<grid, 256, 0, stream>>>(s->now, (const unsigned*)gathered, s->words, world);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  return BF_OK;
}

extern "C" int bf_bfs_shard_merge_slice_impl(void* p, void* stream_v, int num_sms, const void* recv, int world,
                                             long long first, long long count, char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (first < 0 || count < 0 || first + count > s->words + 64) {
    snprintf(err, errcap, "bfs shard: slice outside the bitmap");
    return BF_E_INVALID;
  }
  if (count > 0) {
    const int grid = stream_grid(count, 256, num_sms, 8);
    bfs_merge_slice<<<grid, 256, 0, stream>>>(s->now + first, (const unsigned*)recv, count, world);
  }
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  return BF_OK;
}

extern "C" int bf_bfs_shard_compact_impl(void* p, void* stream_v, int num_sms, int* lvl, long long ll,
                                         long long* fresh, char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (ll < s->nv) {
    snprintf(err, errcap, "bfs shard: lvl shorter than nv");
    return BF_E_INVALID;
  }
  if (s->depth + 1 >= 255 && !s->deep) {
    const int g = stream_grid(s->nv, 256 * 4, num_sms, 8);
    bfs_fill_m1<<<g, 256, 0, stream>>>(lvl, s->nv);
    s->deep = true;
  }
  const int cgrid = stream_grid(s->words, 256, num_sms, 8);
  bfs_compact_sh<<<cgrid, 256, 0, stream>>>(s->now, s->prev, s->words, s->nq, s->sizes, s->lv8, lvl, s->depth,
                                             s->vlo, s->vhi);
  cudaMemcpyAsync(s->hs, s->sizes, 16, cudaMemcpyDeviceToHost, stream);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  if (s->hs[2]) {
    snprintf(err, errcap, "bfs_levels: CSR index out of range");
    return BF_E_FAULT;
  }
  *fresh = s->hs[3];
  s->depth++;
  s->qn = s->hs[1];
  s->hs[0] = s->qn;
  s->hs[1] = 0;
  s->hs[3] = 0;
  cudaMemcpyAsync(s->sizes, s->hs, 16, cudaMemcpyHostToDevice, stream);
  int* t = s->q;
  s->q = s->nq;
  s->nq = t;
  return BF_OK;
}

extern "C" int bf_bfs_shard_finish_impl(void* p, void* stream_v, int num_sms, int* lvl, long long ll, int* depth,
                                        char* err, int errcap) {
  using namespace bf;
  BfsShard* s = (BfsShard*)p;
  cudaStream_t stream = (cudaStream_t)stream_v;
  if (ll < s->nv) {
    snprintf(err, errcap, "bfs shard: lvl shorter than nv");
    return BF_E_INVALID;
  }
  const int g = stream_grid(s->nv, 256 * 4, num_sms, 8);
  bfs_finish<<<g, 256, 0, stream>>>(s->lv8, lvl, s->nv, s->deep);
  cudaError_t e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    snprintf(err, errcap, "bfs shard: %s", cudaGetErrorString(e));
    return BF_E_CUDA;
  }
  *depth = s->depth;
  return BF_OK;
}

namespace bf {

static Registrar reg_bfs("bfs",
                         {{BF_SLOT_HANDLE, BF_I32, "row"},
                          {BF_SLOT_HANDLE, BF_I32, "col"},
                          {BF_SLOT_HANDLE, BF_I32, "lvl"},
                          {BF_SLOT_HANDLE, BF_I32, "changed"},
                          {BF_SLOT_I32, BF_I32, "nv"},
                          {BF_SLOT_I32, BF_I32, "cur"}},
                         launch_bfs);

}  // namespace bf
