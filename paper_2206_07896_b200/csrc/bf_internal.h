// Host-side internals of libbfgpu.so shared by the runtime and the kernel
// launchers.  Nothing here crosses the C ABI (include/bfgpu.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bfgpu.h"

namespace bf {

struct DevFault;
struct KDesc;

// One resolved kernel argument (an ArgSlot after unpack_args, executor.py:48-75).
struct ArgVal {
  int32_t kind;     // bf_slot_kind
  int32_t scalar;   // element type for handles
  void* ptr;        // device pointer for handles
  int64_t len;      // element count for handles
  uint32_t handle;
  int32_t i32;
  int64_t i64;
  double f64;       // f32 and f64 slots
};

// Host-detected trap, raised at the next synchronize (runtime.py:335-343).
struct HostTrap {
  int kind = BF_TRAP_NONE;
  long long block = 0;
  std::string message;
};

// Device-side block fetching (BF_FLAG_DEVICE_FETCH): one persistent launch
// per task whose CTAs claim `grain` logical blocks at a time from the
// worker's claim counters (runtime.py:175-201 on the GPU).
// The fetches are split into kFetchSubs contiguous sub-ranges, each with its
// own claim counter (CTA b starts on sub-range b % kFetchSubs and moves on
// when one is drained), so the claims of fine grains do not serialise on one
// address.  The runtime zeroes the worker's counters before each
// device-fetched launch (stream-ordered).  (Measured: 8 counters with one
// atomic per claim beat 32 counters with a plain-load drain check, which
// puts two round trips on every claim.)
constexpr int kFetchSubs = 8;
struct DevFetch {
  unsigned long long* cursor;  // the worker's kFetchSubs claim counters (zero at launch)
  unsigned long long* stats;   // per worker slot: [2w] successful claims, [2w+1] blocks executed
  int slots;                   // worker slots (pool size): CTA b accounts to slot b % slots
  long long nfetch, grain;     // fetches of the task, blocks per fetch
  long long first, total;      // the task's logical blocks [first, first + total)
  int* executed;               // KernelTask.executed indexed by absolute block (nullable)
};

// Everything a launcher needs to issue one fetched block range.
struct LaunchCtx {
  const char* name;
  int grid[3];
  int block[3];
  long long first, count;    // logical block range of this fetch
  int64_t shmem;             // dynamic shared bytes (Runtime.launch shmem_bytes)
  int warp_size;             // MpmdKernel.warp_size (0 if not warp mode)
  const ArgVal* args;
  int nargs;
  cudaStream_t stream;
  int num_sms;
  int* executed;             // device, per task (nullable)
  DevFault* fault;           // device fault word of the runtime
  unsigned long long task;
  HostTrap* trap;            // host-side trap sink (first wins)
  std::string* error;        // BF_E_UNSUPPORTED / BF_E_CUDA message sink
  const void* user = nullptr;  // KernelEntry::user (JIT kernels)
  // device-side fetching: the whole task in one persistent launch.  A
  // launcher that cannot (geometry, a host-detected trap) returns
  // BF_E_UNSUPPORTED without launching anything, and the runtime falls back
  // to host-issued fetches; otherwise it sets dfetch_grid to its CTA count.
  const DevFetch* dfetch = nullptr;
  int dfetch_grid = 0;

  KDesc desc() const;
  // Record a trap detected on the host before launching (e.g. an affine
  // index range that leaves a buffer); first one wins.
  void host_trap(int kind, long long blk, const std::string& msg) const;
  // Lowest linear block id in [first, first+count) whose x coordinate is x.
  long long first_block_with_x(long long x) const;
  // Distinct blockIdx.x values of the fetch range as half-open intervals
  // (at most two; y/z copies of the same x are folded together).
  std::vector<std::pair<long long, long long>> x_intervals() const;
  // The fetch range as rectangles of (blockIdx.x, blockIdx.y) in block
  // units, z copies folded: {x0, x1, y0, y1} half-open.
  struct Rect { long long x0, x1, y0, y1; };
  std::vector<Rect> xy_rects() const;
};

typedef int (*LauncherFn)(LaunchCtx& ctx);

struct ParamSpec {
  int32_t kind;    // bf_slot_kind
  int32_t scalar;  // element bf_scalar for handles
  const char* name;
};

struct KernelEntry {
  const char* name;
  std::vector<ParamSpec> params;
  LauncherFn launch;
  const void* user = nullptr;
  bool has_fp = false;     // expected MpmdKernel body fingerprint (bf_kernel_set_fingerprint)
  uint8_t fp[32] = {0};
  bool dev_fetch = false;  // the launcher handles LaunchCtx::dfetch
};

// Registry (static registrars in each k_*.cu file, plus JIT kernels added at
// run time; a deque keeps entry addresses stable).
std::deque<KernelEntry>& registry();
const KernelEntry* find_kernel(const char* name);

struct Registrar {
  Registrar(const char* name, std::vector<ParamSpec> params, LauncherFn fn, bool dev_fetch = false) {
    registry().push_back(KernelEntry{name, std::move(params), fn, nullptr});
    registry().back().dev_fetch = dev_fetch;
  }
};

// Grid sizing for streaming kernels: a multiple of the SM count, capped by
// the work available.
inline int stream_grid(long long work_items, int items_per_cta, int num_sms,
                       int ctas_per_sm) {
  long long need = (work_items + items_per_cta - 1) / items_per_cta;
  long long cap = (long long)num_sms * ctas_per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// True the first time it is called for the current device with this flag
// array (function attributes such as the dynamic shared-memory limit are set
// per device).
inline bool first_on_device(bool (&done)[64]) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63]) return false;
  done[dev & 63] = true;
  return true;
}

// CTAs of `fn` resident per SM at this block size / dynamic smem (cached).
// Grid-stride kernels size their grid with it: a grid larger than one
// resident wave leaves a partial second wave (a tail) on every launch.
int resident_ctas(const void* fn, int threads, size_t smem);

// stream_grid capped at one resident wave of `fn`
template <typename F>
inline int wave_grid(F fn, int threads, size_t smem, long long work_items, int items_per_cta, int num_sms,
                     int ctas_per_sm) {
  const int r = resident_ctas((const void*)fn, threads, smem);
  return stream_grid(work_items, items_per_cta, num_sms, r < ctas_per_sm ? r : ctas_per_sm);
}

// Per-stream device scratch.  Kernels that keep scratch across the launches
// of one fetch (the bfs level step, the fused traversal) key it by the
// stream the fetch runs on, so concurrent fetches on different worker
// streams (pool_size > 1) or runtimes never share it; growing it only has
// to order against that stream.  The runtime releases a stream's scratch
// when it destroys the stream (bf_runtime_destroy).
struct StreamScratch {
  virtual ~StreamScratch() {}
};
std::mutex& stream_scratch_mutex();
std::unique_ptr<StreamScratch>& stream_scratch_slot(cudaStream_t s, int kind);
void release_stream_scratch(cudaStream_t s);

template <class T>
T& scratch_for(cudaStream_t s, int kind) {
  std::lock_guard<std::mutex> lk(stream_scratch_mutex());
  std::unique_ptr<StreamScratch>& slot = stream_scratch_slot(s, kind);
  if (!slot) slot.reset(new T());
  return *static_cast<T*>(slot.get());
}
enum { SCRATCH_BFS_STEP = 1, SCRATCH_BFS_LEVELS = 2, SCRATCH_NN_TOPK = 3, SCRATCH_KM_UPDATE = 4 };

// full-grid hotspot step with the streaming band kernel (k_hotspot.cu)
int hotspot_step_full(cudaStream_t stream, int num_sms, const float* src, const float* power,
                      float* dst, int rows, int cols, const double* kc);

#define BF_CUDA_LAUNCH_CHECK(ctx)                                   \
  do {                                                              \
    cudaError_t e_ = cudaGetLastError();                            \
    if (e_ != cudaSuccess) {                                        \
      *(ctx).error = std::string("launch failed: ") + cudaGetErrorString(e_); \
      return BF_E_CUDA;                                             \
    }                                                               \
  } while (0)

}  // namespace bf
