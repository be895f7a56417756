// libbfgpu.so — the launch runtime and memory shim behind include/bfgpu.h.
//
// Reference: /root/reference/pkg/src/blockfuse/runtime.py (Runtime, TaskQueue,
// KernelTask, RuntimeCounters, resolve_grain) and arena.py (DeviceArena).
//
// B200 mapping
//   * DeviceArena  -> handle table over cudaMalloc'd HBM buffers (zero-filled),
//                     pinned staging for host copies; frees are deferred to the
//                     next quiescence point so a free can never race a kernel.
//   * TaskQueue    -> the same FIFO/cursor protocol, run by the host dispatcher.
//   * pool workers -> `pool_size` in-order CUDA streams on the arena's device;
//                     each fetched range of `grain` logical blocks becomes one
//                     grid launch on the next worker stream (round robin).
//   * hold_blocks  -> fetched ranges are kept on the host and issued, in
//                     launch order, at the next synchronize: no block runs
//                     before it, and nothing occupies the device meanwhile
//                     (copies and JIT module loads proceed).
//   * traps        -> a device fault word (first wins) plus host-detected traps,
//                     surfaced at synchronize as BF_E_FAULT.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "bf_internal.h"
#include "common.cuh"

// ---- occupancy cache ----------------------------------------------------------
namespace bf {
static std::map<std::pair<cudaStream_t, int>, std::unique_ptr<StreamScratch>>& scratch_map() {
  static std::map<std::pair<cudaStream_t, int>, std::unique_ptr<StreamScratch>> m;
  return m;
}
std::mutex& stream_scratch_mutex() {
  static std::mutex mu;
  return mu;
}
std::unique_ptr<StreamScratch>& stream_scratch_slot(cudaStream_t s, int kind) {
  return scratch_map()[std::make_pair(s, kind)];
}
void release_stream_scratch(cudaStream_t s) {
  std::vector<std::unique_ptr<StreamScratch>> dead;
  {
    std::lock_guard<std::mutex> lk(stream_scratch_mutex());
    auto& m = scratch_map();
    for (auto it = m.begin(); it != m.end();) {
      if (it->first.first == s) {
        dead.push_back(std::move(it->second));
        it = m.erase(it);
      } else {
        ++it;
      }
    }
  }
  dead.clear();  // destructors free the device memory outside the lock
}

int resident_ctas(const void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(fn, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 1;
  }
  cache[key] = n;
  return n;
}
}  // namespace bf


namespace bf {

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(BF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                  \
  do {                                            \
    cudaError_t e__ = (call);                     \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

static const int kScalarSize[4] = {4, 8, 4, 8};

// ---------------------------------------------------------------------------
// registry
// ---------------------------------------------------------------------------

std::deque<KernelEntry>& registry() {
  static std::deque<KernelEntry> r;
  return r;
}

const KernelEntry* find_kernel(const char* name) {
  for (auto& k : registry())
    if (std::strcmp(k.name, name) == 0) return &k;
  return nullptr;
}

KDesc LaunchCtx::desc() const {
  KDesc d;
  d.gx = grid[0]; d.gy = grid[1]; d.gz = grid[2];
  d.bx = block[0]; d.by = block[1]; d.bz = block[2];
  d.first = first; d.count = count;
  d.executed = executed;
  d.fault = fault;
  d.task = task;
  return d;
}

void LaunchCtx::host_trap(int kind, long long blk, const std::string& msg) const {
  if (trap->kind == BF_TRAP_NONE) {
    trap->kind = kind;
    trap->block = blk;
    trap->message = msg;
  }
}

long long LaunchCtx::first_block_with_x(long long x) const {
  long long gx = grid[0];
  long long x0 = first % gx;
  long long delta = (x - x0 + gx) % gx;
  return first + delta;
}

std::vector<std::pair<long long, long long>> LaunchCtx::x_intervals() const {
  std::vector<std::pair<long long, long long>> out;
  long long gx = grid[0];
  if (count >= gx) {
    out.push_back({0, gx});
    return out;
  }
  long long x0 = first % gx;
  if (x0 + count <= gx) {
    out.push_back({x0, x0 + count});
  } else {
    out.push_back({0, x0 + count - gx});
    out.push_back({x0, gx});
  }
  return out;
}

std::vector<LaunchCtx::Rect> LaunchCtx::xy_rects() const {
  std::vector<Rect> out;
  long long gx = grid[0], gy = grid[1];
  long long plane = gx * gy;
  if (count >= plane) {
    out.push_back({0, gx, 0, gy});
    return out;
  }
  // at most two segments (the range crosses at most one z boundary)
  long long s = first % plane;
  std::vector<std::pair<long long, long long>> segs;
  if (s + count <= plane) {
    segs.push_back({s, s + count});
  } else {
    segs.push_back({s, plane});
    segs.push_back({0, s + count - plane});
  }
  for (auto& sg : segs) {
    long long p0 = sg.first, p1 = sg.second;  // [p0, p1) within the plane
    long long y0 = p0 / gx, x0 = p0 % gx;
    long long yl = (p1 - 1) / gx, xl = (p1 - 1) % gx;  // last block
    if (y0 == yl) {
      out.push_back({x0, xl + 1, y0, y0 + 1});
      continue;
    }
    long long full_lo = y0, full_hi = yl + 1;
    if (x0 > 0) {
      out.push_back({x0, gx, y0, y0 + 1});
      full_lo = y0 + 1;
    }
    if (xl < gx - 1) {
      out.push_back({0, xl + 1, yl, yl + 1});
      full_hi = yl;
    }
    if (full_hi > full_lo) out.push_back({0, gx, full_lo, full_hi});
  }
  return out;
}

__global__ void mark_kernel(int* executed, long long first, long long count) {
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = first + (long long)blockIdx.x * blockDim.x + threadIdx.x; b < first + count;
       b += stride)
    atomicAdd(executed + b, 1);
}

// ---------------------------------------------------------------------------
// arena
// ---------------------------------------------------------------------------

struct Buffer {
  int32_t scalar;
  int64_t length;
  void* ptr;
  uint32_t parent = 0;  // != 0: an element-range view of that buffer (owns no memory)
  int32_t views = 0;    // live views of this buffer
};

}  // namespace bf

struct bf_arena {
  int device = 0;
  uint32_t next_handle = 1;
  std::map<uint32_t, bf::Buffer> buffers;
  std::vector<void*> zombies;     // freed buffers awaiting a quiescence point
  // host<->device copies: uploads/fills/copies on copy_stream, downloads on
  // d2h_stream with their own staging, so a download issued from one host
  // thread overlaps an upload from another (both PCIe directions busy).
  cudaStream_t copy_stream = nullptr;
  cudaStream_t d2h_stream = nullptr;
  void* staging[2] = {nullptr, nullptr};
  void* dl_staging[2] = {nullptr, nullptr};
  size_t staging_bytes = 0;
  cudaEvent_t staging_ev[2] = {nullptr, nullptr};
  cudaEvent_t dl_ev[2] = {nullptr, nullptr};
  std::mutex mu;  // buffers map + staging allocation
  int live_runtimes = 0;
  bool destroy_pending = false;  // destroyed while runtimes still reference it
};

namespace bf {

static int set_device(int dev) {
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return BF_OK;
}

static Buffer* lookup(bf_arena* a, uint32_t h) {
  std::lock_guard<std::mutex> g(a->mu);
  auto it = a->buffers.find(h);
  return it == a->buffers.end() ? nullptr : &it->second;
}

static void release_zombies(bf_arena* a) {
  for (void* p : a->zombies) cudaFree(p);
  a->zombies.clear();
}

static const size_t kStagingChunk = 32u << 20;  // 32 MiB double-buffered staging

static int ensure_staging(bf_arena* a, bool download) {
  std::lock_guard<std::mutex> g(a->mu);
  void** st = download ? a->dl_staging : a->staging;
  cudaEvent_t* ev = download ? a->dl_ev : a->staging_ev;
  if (st[0]) return BF_OK;
  for (int i = 0; i < 2; i++) {
    CK(cudaHostAlloc(&st[i], kStagingChunk, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  }
  a->staging_bytes = kStagingChunk;
  return BF_OK;
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

}  // namespace bf

// ---------------------------------------------------------------------------
// task queue (TaskQueue, runtime.py:146-205)
// ---------------------------------------------------------------------------

struct bf_queue {
  struct Entry {
    uint64_t tag;
    int64_t total;
    int64_t grain;
    int64_t cursor = 0;
    int64_t fetches = 0;
  };
  std::mutex mu;
  std::deque<Entry> tasks;
  std::map<uint64_t, std::pair<int64_t, int64_t>> retired;  // tag -> (fetches, cursor)
  bool closed = false;
  int64_t fetch_count = 0;
  int64_t queue_waits = 0;
};

// ---------------------------------------------------------------------------
// runtime
// ---------------------------------------------------------------------------

namespace bf {

struct Fetch {
  const KernelEntry* ke = nullptr;
  std::shared_ptr<std::vector<ArgVal>> args;
  HostTrap pre;
  uint64_t task = 0;
  int worker = 0;
  long long first = 0, count = 0;
  int grid[3], block[3];
  int64_t shmem = 0;
  int warp_size = 0;
};

struct FetchRecord {
  uint64_t task;
  int worker;
  long long first, count;
  bool device = false;  // a device-fetched task (counters come from the device)
  cudaEvent_t done;  // shared by the fetches a lazy cover event covers (event_refs)
};

struct TaskRec {
  std::string kernel;
  int64_t total = 0;
  int64_t grain = 0;
  int64_t fetches = 0;
  int64_t cursor = 0;
  int64_t completed = 0;        // blocks of retired fetches
  int64_t base = 0;             // first logical block (bf_launch_range)
  int* executed_dev = nullptr;  // BF_FLAG_INSTRUMENT
  std::vector<std::pair<long long, long long>> done_ranges;
};

__global__ void delay_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace bf

struct bf_runtime {
  bf_arena* arena = nullptr;
  int device = 0;
  int pool = 1;
  uint32_t flags = 0;
  double block_delay = 0.0;
  std::mt19937_64 rng;
  int num_sms = 148;
  bool shut_down = false;
  std::vector<cudaStream_t> streams;
  bool holding = false;          // hold_blocks: launches wait on the host
  bf::DevFault* fault_dev = nullptr;
  bf::DevFault* fault_host = nullptr;  // pinned copy, fetched only after the flag is seen
  int* fault_flag = nullptr;           // host-mapped: a kernel's first fault sets it
  bf::HostTrap trap;             // first trap (host- or device-detected)
  uint64_t trap_task = 0;
  std::string trap_kernel;
  bf_queue queue;
  std::map<uint64_t, bf::TaskRec> tasks;
  std::deque<bf::FetchRecord> inflight;
  std::deque<bf::Fetch> deferred;  // held launches (hold_blocks)
  std::vector<cudaEvent_t> event_pool;
  std::map<cudaEvent_t, int> event_refs;  // fetch records still pointing at each in-use event
  uint64_t next_task = 1;
  uint64_t rr = 0;               // round-robin worker cursor
  // device-side fetching (BF_FLAG_DEVICE_FETCH): per worker a claim counter,
  // per worker slot (claims, blocks executed); host copy of the counters' bases
  unsigned long long* dfetch_dev = nullptr;  // [pool][kFetchSubs] counters, then [pool][2] stats
  bool dfetch_used = false;
  // counters
  int64_t blocks_executed = 0;
  int64_t syncs = 0;
  std::vector<int64_t> busy;
};

namespace bf {

static cudaEvent_t get_event(bf_runtime* rt) {
  if (!rt->event_pool.empty()) {
    cudaEvent_t e = rt->event_pool.back();
    rt->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

static int fetch_event_mode() {
  // BF_FETCH_EVENTS: 1 = an event after every fetch; 2 (default) = lazy: no
  // stream operation between launches, a query covers every worker's
  // untracked tail with one event (stream order: when it completes, so did
  // every fetch before it), so task.remaining still falls without a
  // synchronize; 0 = untracked until the next synchronize
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("BF_FETCH_EVENTS");
    m = e ? atoi(e) : 2;
  }
  return m;
}

// A fetch record retires: its event returns to the pool when no other
// record still points at it (a lazy cover event is shared by every fetch it
// covers, and they may retire out of order across workers).
static void drop_event_ref(bf_runtime* rt, cudaEvent_t ev) {
  auto it = rt->event_refs.find(ev);
  if (it == rt->event_refs.end() || --it->second <= 0) {
    if (it != rt->event_refs.end()) rt->event_refs.erase(it);
    rt->event_pool.push_back(ev);
  }
}

// lazy mode: one event per worker stream covers its fetches without one
static void cover_untracked(bf_runtime* rt) {
  for (size_t w = 0; w < rt->streams.size(); w++) {
    FetchRecord* last = nullptr;
    for (auto& f : rt->inflight)
      if (f.worker == (int)w && !f.done) last = &f;
    if (!last) continue;
    cudaEvent_t ev = get_event(rt);
    if (cudaEventRecord(ev, rt->streams[w]) != cudaSuccess) {
      cudaGetLastError();
      rt->event_pool.push_back(ev);
      continue;
    }
    int n = 0;
    for (auto& f : rt->inflight)
      if (f.worker == (int)w && !f.done) {
        f.done = ev;
        n++;
      }
    rt->event_refs[ev] = n;  // back to the pool once the last of them retires
  }
}

// Retire completed fetches (all of them when `wait`).
static int retire(bf_runtime* rt, bool wait) {
  if (!wait && fetch_event_mode() == 2) cover_untracked(rt);
  while (!rt->inflight.empty()) {
    FetchRecord& f = rt->inflight.front();
    if (!f.done) {
      // untracked fetch (fetch events off): complete only once the workers
      // were synchronized
      if (!wait) return BF_OK;
    } else if (wait) {
      cudaError_t e = cudaEventSynchronize(f.done);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    } else {
      cudaError_t e = cudaEventQuery(f.done);
      if (e == cudaErrorNotReady) {
        // fetches on other workers may have finished; keep FIFO simple and
        // scan the rest without blocking
        for (auto it = rt->inflight.begin() + 1; it != rt->inflight.end();) {
          if (it->done && cudaEventQuery(it->done) == cudaSuccess) {
            TaskRec& t = rt->tasks[it->task];
            t.completed += it->count;
            t.done_ranges.push_back({it->first, it->count});
            if (!it->device) {  // device-fetched: busy / executed counted on the device
              rt->blocks_executed += it->count;
              rt->busy[it->worker] += it->count;
            }
            drop_event_ref(rt, it->done);
            it = rt->inflight.erase(it);
          } else {
            cudaGetLastError();
            ++it;
          }
        }
        return BF_OK;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventQuery");
    }
    TaskRec& t = rt->tasks[f.task];
    t.completed += f.count;
    t.done_ranges.push_back({f.first, f.count});
    if (!f.device) {
      rt->blocks_executed += f.count;
      rt->busy[f.worker] += f.count;
    }
    if (f.done) drop_event_ref(rt, f.done);
    rt->inflight.pop_front();
  }
  return BF_OK;
}

static int issue_fetch(bf_runtime* rt, Fetch& f);

// Release a hold: issue every deferred fetch in launch order.
static int open_gate(bf_runtime* rt) {
  rt->holding = false;
  while (!rt->deferred.empty()) {
    Fetch f = std::move(rt->deferred.front());
    rt->deferred.pop_front();
    int rc = issue_fetch(rt, f);
    if (rc) return rc;
  }
  return BF_OK;
}

static int sync_workers(bf_runtime* rt) {
  int rc = open_gate(rt);
  if (rc) return rc;
  for (auto s : rt->streams) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  }
  return retire(rt, true);
}

// sync_workers plus the device fault record.  A fault also sets a
// host-mapped flag (record_fault), so the common no-fault synchronize is one
// stream synchronize per worker; the record is copied only when the flag is
// set (the first fault stays in it: later syncs re-raise it).
static int sync_workers_fault(bf_runtime* rt) {
  int rc = open_gate(rt);
  if (rc) return rc;
  for (size_t i = 0; i < rt->streams.size(); i++) {
    cudaError_t e = cudaStreamSynchronize(rt->streams[i]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  }
  if (*(volatile int*)rt->fault_flag && rt->fault_host->kind == BF_TRAP_NONE) {
    int* keep = rt->fault_host->host_flag;
    cudaError_t e = cudaMemcpy(rt->fault_host, rt->fault_dev, sizeof(DevFault), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy fault record");
    rt->fault_host->host_flag = keep;
  }
  return retire(rt, true);
}

static void absorb_device_fault(bf_runtime* rt) {
  const DevFault f = *rt->fault_host;  // fetched by sync_workers_fault
  if (f.kind != BF_TRAP_NONE && rt->trap.kind == BF_TRAP_NONE) {
    rt->trap.kind = f.kind;
    rt->trap.block = f.block;
    auto it = rt->tasks.find(f.task);
    rt->trap_task = f.task;
    rt->trap_kernel = it == rt->tasks.end() ? "?" : it->second.kernel;
    static const char* names[] = {"", "index out of range", "division by zero",
                                  "type fault", "non-uniform trip"};
    rt->trap.message = std::string(names[f.kind < 5 ? f.kind : 0]) + " (device)";
  }
}

static void fill_fault(bf_runtime* rt, bf_fault* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->kind = rt->trap.kind;
  out->block_id = rt->trap.block;
  out->task_id = rt->trap_task;
  std::snprintf(out->kernel, sizeof(out->kernel), "%s", rt->trap_kernel.c_str());
  std::snprintf(out->message, sizeof(out->message), "%s", rt->trap.message.c_str());
}

}  // namespace bf

using namespace bf;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int bf_abi_version(void) { return BFGPU_ABI_VERSION; }

const char* bf_last_error(void) { return g_last_error.c_str(); }

int bf_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(BF_E_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *count = n;
  return BF_OK;
}

// ---- arena ---------------------------------------------------------------

int bf_arena_create(int32_t device, bf_arena** out) {
  if (!out) return fail(BF_E_INVALID, "null out");
  int rc = set_device(device);
  if (rc) return rc;
  auto* a = new bf_arena();
  a->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&a->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->d2h_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    if (a->copy_stream) cudaStreamDestroy(a->copy_stream);
    delete a;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *out = a;
  return BF_OK;
}

static void arena_free(bf_arena* a);

int bf_arena_destroy(bf_arena* a) {
  if (!a) return BF_OK;
  if (a->live_runtimes > 0) {
    // a runtime still points at this arena: free it with the last runtime
    a->destroy_pending = true;
    return BF_OK;
  }
  arena_free(a);
  return BF_OK;
}

static void arena_free(bf_arena* a) {
  set_device(a->device);
  cudaDeviceSynchronize();
  for (auto& kv : a->buffers)
    if (!kv.second.parent) cudaFree(kv.second.ptr);
  release_zombies(a);
  for (int i = 0; i < 2; i++) {
    if (a->staging[i]) cudaFreeHost(a->staging[i]);
    if (a->staging_ev[i]) cudaEventDestroy(a->staging_ev[i]);
    if (a->dl_staging[i]) cudaFreeHost(a->dl_staging[i]);
    if (a->dl_ev[i]) cudaEventDestroy(a->dl_ev[i]);
  }
  if (a->copy_stream) cudaStreamDestroy(a->copy_stream);
  if (a->d2h_stream) cudaStreamDestroy(a->d2h_stream);
  delete a;
}

int bf_alloc(bf_arena* a, int32_t scalar, int64_t length, uint32_t* handle) {
  if (!a || !handle) return fail(BF_E_INVALID, "null argument");
  if (scalar < 0 || scalar > 3) return fail(BF_E_INVALID, "bad scalar type");
  if (length < 0) return fail(BF_E_INVALID, "negative buffer length " + std::to_string(length));
  int rc = set_device(a->device);
  if (rc) return rc;
  size_t bytes = (size_t)length * kScalarSize[scalar];
  void* p = nullptr;
  // always allocate at least one 512 B line so every handle has a distinct,
  // 16 B-aligned pointer and vector loads past a ragged tail stay mapped
  size_t alloc = ((bytes + 511) / 512) * 512;
  if (alloc == 0) alloc = 512;
  CK(cudaMalloc(&p, alloc));
  CK(cudaMemsetAsync(p, 0, alloc, a->copy_stream));
  CK(cudaStreamSynchronize(a->copy_stream));
  std::lock_guard<std::mutex> g(a->mu);
  uint32_t h = a->next_handle++;
  a->buffers[h] = Buffer{scalar, length, p};
  *handle = h;
  return BF_OK;
}

int bf_free(bf_arena* a, uint32_t h) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  {
    std::lock_guard<std::mutex> g(a->mu);
    auto it = a->buffers.find(h);
    if (it == a->buffers.end())
      return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
    if (it->second.views > 0)
      return fail(BF_E_INVALID, "buffer " + std::to_string(h) + " still has " +
                                    std::to_string(it->second.views) + " live view(s)");
    if (it->second.parent) {  // a view: the parent keeps the memory
      auto p = a->buffers.find(it->second.parent);
      if (p != a->buffers.end()) p->second.views--;
      a->buffers.erase(it);
      return BF_OK;
    }
    a->zombies.push_back(it->second.ptr);
    a->buffers.erase(it);
  }
  if (a->live_runtimes == 0) {
    set_device(a->device);
    cudaDeviceSynchronize();
    release_zombies(a);
  }
  return BF_OK;
}

int bf_view(bf_arena* a, uint32_t h, int64_t first, int64_t length, uint32_t* handle) {
  if (!a || !handle) return fail(BF_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(a->mu);
  auto it = a->buffers.find(h);
  if (it == a->buffers.end()) return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
  Buffer& b = it->second;
  if (first < 0 || length < 0 || first + length > b.length)
    return fail(BF_E_INVALID, "view [" + std::to_string(first) + ", " + std::to_string(first + length) +
                                  ") outside buffer of " + std::to_string(b.length) + " elements");
  const int64_t off = first * kScalarSize[b.scalar];
  if (off % 16)
    return fail(BF_E_INVALID, "view offset of " + std::to_string(off) + " bytes is not 16 B aligned");
  const uint32_t root = b.parent ? b.parent : h;
  uint32_t v = a->next_handle++;
  a->buffers[v] = Buffer{b.scalar, length, (char*)b.ptr + off, root, 0};
  a->buffers[root].views++;
  *handle = v;
  return BF_OK;
}

int bf_buffer_info(bf_arena* a, uint32_t h, int32_t* scalar, int64_t* length,
                   uint64_t* device_ptr) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  Buffer* b = lookup(a, h);
  if (!b) return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
  if (scalar) *scalar = b->scalar;
  if (length) *length = b->length;
  if (device_ptr) *device_ptr = (uint64_t)(uintptr_t)b->ptr;
  return BF_OK;
}

static int check_range(Buffer* b, int64_t nbytes, int64_t offset) {
  int64_t cap = b->length * kScalarSize[b->scalar];
  if (nbytes < 0 || offset < 0 || offset + nbytes > cap)
    return fail(BF_E_INVALID, "byte range [" + std::to_string(offset) + ", " +
                                  std::to_string(offset + nbytes) + ") outside buffer of " +
                                  std::to_string(cap) + " bytes");
  return BF_OK;
}

int bf_upload(bf_arena* a, uint32_t h, const void* src, int64_t nbytes, int64_t offset) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  Buffer* b = lookup(a, h);
  if (!b) return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
  int rc = check_range(b, nbytes, offset);
  if (rc) return rc;
  if (nbytes == 0) return BF_OK;
  rc = set_device(a->device);
  if (rc) return rc;
  char* dst = (char*)b->ptr + offset;
  if (is_pinned(src)) {
    CK(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyHostToDevice, a->copy_stream));
    CK(cudaStreamSynchronize(a->copy_stream));
    return BF_OK;
  }
  rc = ensure_staging(a, false);
  if (rc) return rc;
  // double-buffered: memcpy into staging[i] while staging[i^1] is in flight
  int64_t done = 0;
  int i = 0;
  while (done < nbytes) {
    int64_t n = std::min<int64_t>(nbytes - done, (int64_t)a->staging_bytes);
    CK(cudaEventSynchronize(a->staging_ev[i]));
    std::memcpy(a->staging[i], (const char*)src + done, n);
    CK(cudaMemcpyAsync(dst + done, a->staging[i], n, cudaMemcpyHostToDevice, a->copy_stream));
    CK(cudaEventRecord(a->staging_ev[i], a->copy_stream));
    done += n;
    i ^= 1;
  }
  CK(cudaStreamSynchronize(a->copy_stream));
  return BF_OK;
}

int bf_download(bf_arena* a, uint32_t h, void* dstp, int64_t nbytes, int64_t offset) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  Buffer* b = lookup(a, h);
  if (!b) return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
  int rc = check_range(b, nbytes, offset);
  if (rc) return rc;
  if (nbytes == 0) return BF_OK;
  rc = set_device(a->device);
  if (rc) return rc;
  const char* src = (const char*)b->ptr + offset;
  if (is_pinned(dstp)) {
    CK(cudaMemcpyAsync(dstp, src, nbytes, cudaMemcpyDeviceToHost, a->d2h_stream));
    CK(cudaStreamSynchronize(a->d2h_stream));
    return BF_OK;
  }
  rc = ensure_staging(a, true);
  if (rc) return rc;
  // pipeline: D2H chunk k+1 in flight while chunk k is memcpy'd out
  int64_t chunk = (int64_t)a->staging_bytes;
  int64_t nchunks = (nbytes + chunk - 1) / chunk;
  for (int64_t k = 0; k < nchunks; k++) {
    int i = (int)(k & 1);
    int64_t off = k * chunk;
    int64_t n = std::min<int64_t>(nbytes - off, chunk);
    CK(cudaMemcpyAsync(a->dl_staging[i], src + off, n, cudaMemcpyDeviceToHost, a->d2h_stream));
    CK(cudaEventRecord(a->dl_ev[i], a->d2h_stream));
    if (k > 0) {
      int j = i ^ 1;
      int64_t poff = (k - 1) * chunk;
      int64_t pn = std::min<int64_t>(nbytes - poff, chunk);
      CK(cudaEventSynchronize(a->dl_ev[j]));
      std::memcpy((char*)dstp + poff, a->dl_staging[j], pn);
    }
  }
  {
    int64_t k = nchunks - 1;
    int i = (int)(k & 1);
    int64_t off = k * chunk;
    int64_t n = std::min<int64_t>(nbytes - off, chunk);
    CK(cudaEventSynchronize(a->dl_ev[i]));
    std::memcpy((char*)dstp + off, a->dl_staging[i], n);
  }
  return BF_OK;
}

int bf_fill32(bf_arena* a, uint32_t h, uint32_t pattern, int64_t offset, int64_t nbytes) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  Buffer* b = lookup(a, h);
  if (!b) return fail(BF_E_DANGLING, "dangling buffer handle " + std::to_string(h));
  int rc = check_range(b, nbytes, offset);
  if (rc) return rc;
  if ((offset | nbytes) & 3) return fail(BF_E_INVALID, "fill32 needs 4-byte alignment");
  if (nbytes == 0) return BF_OK;
  rc = set_device(a->device);
  if (rc) return rc;
  char* p = (char*)b->ptr + offset;
  if (pattern == 0 || pattern == 0xffffffffu) {
    CK(cudaMemsetAsync(p, pattern & 0xff, nbytes, a->copy_stream));
  } else {
    // cudaMemset2D trick is byte-wise; use the driver-free path: a pinned
    // pattern chunk replicated by copies.
    std::vector<uint32_t> pat((size_t)std::min<int64_t>(nbytes / 4, 1 << 20), pattern);
    int64_t chunk = (int64_t)pat.size() * 4;
    for (int64_t off = 0; off < nbytes; off += chunk) {
      int64_t n = std::min(chunk, nbytes - off);
      CK(cudaMemcpyAsync(p + off, pat.data(), n, cudaMemcpyHostToDevice, a->copy_stream));
    }
  }
  CK(cudaStreamSynchronize(a->copy_stream));
  return BF_OK;
}

int bf_copy(bf_arena* a, uint32_t dst, int64_t dst_offset, uint32_t src, int64_t src_offset,
            int64_t nbytes) {
  if (!a) return fail(BF_E_INVALID, "null arena");
  Buffer* d = lookup(a, dst);
  Buffer* s = lookup(a, src);
  if (!d || !s) return fail(BF_E_DANGLING, "dangling buffer handle");
  int rc = check_range(d, nbytes, dst_offset);
  if (rc) return rc;
  rc = check_range(s, nbytes, src_offset);
  if (rc) return rc;
  if (nbytes == 0) return BF_OK;
  rc = set_device(a->device);
  if (rc) return rc;
  CK(cudaMemcpyAsync((char*)d->ptr + dst_offset, (char*)s->ptr + src_offset, nbytes,
                     cudaMemcpyDeviceToDevice, a->copy_stream));
  CK(cudaStreamSynchronize(a->copy_stream));
  return BF_OK;
}

// ---- task queue ------------------------------------------------------------

int bf_queue_create(bf_queue** out) {
  if (!out) return fail(BF_E_INVALID, "null out");
  *out = new bf_queue();
  return BF_OK;
}

int bf_queue_destroy(bf_queue* q) {
  delete q;
  return BF_OK;
}

int bf_queue_push(bf_queue* q, uint64_t tag, int64_t total, int64_t grain) {
  if (!q) return fail(BF_E_INVALID, "null queue");
  std::lock_guard<std::mutex> g(q->mu);
  if (q->closed) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  if (total < 1 || grain < 1) return fail(BF_E_INVALID, "total and grain must be >= 1");
  bf_queue::Entry e;
  e.tag = tag;
  e.total = total;
  e.grain = grain;
  q->tasks.push_back(e);
  return BF_OK;
}

int bf_queue_fetch(bf_queue* q, int32_t* got, uint64_t* tag, int64_t* first, int64_t* count) {
  if (!q || !got) return fail(BF_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(q->mu);
  if (q->tasks.empty()) {
    *got = 0;
    return BF_OK;
  }
  bf_queue::Entry& t = q->tasks.front();
  int64_t f = t.cursor;
  int64_t c = std::min(t.grain, t.total - f);
  t.cursor = f + c;
  t.fetches += 1;
  q->fetch_count += 1;
  *got = 1;
  if (tag) *tag = t.tag;
  if (first) *first = f;
  if (count) *count = c;
  if (t.cursor == t.total) {
    q->retired[t.tag] = {t.fetches, t.cursor};
    q->tasks.pop_front();
  }
  return BF_OK;
}

int bf_queue_close(bf_queue* q) {
  if (!q) return fail(BF_E_INVALID, "null queue");
  std::lock_guard<std::mutex> g(q->mu);
  q->closed = true;
  return BF_OK;
}

int bf_queue_is_empty(bf_queue* q, int32_t* empty) {
  if (!q || !empty) return fail(BF_E_INVALID, "null argument");
  std::lock_guard<std::mutex> g(q->mu);
  *empty = q->tasks.empty() ? 1 : 0;
  return BF_OK;
}

int bf_queue_task(bf_queue* q, uint64_t tag, int64_t* fetches, int64_t* cursor) {
  if (!q) return fail(BF_E_INVALID, "null queue");
  std::lock_guard<std::mutex> g(q->mu);
  for (auto& t : q->tasks)
    if (t.tag == tag) {
      if (fetches) *fetches = t.fetches;
      if (cursor) *cursor = t.cursor;
      return BF_OK;
    }
  auto it = q->retired.find(tag);
  if (it == q->retired.end()) return fail(BF_E_INVALID, "unknown task tag");
  if (fetches) *fetches = it->second.first;
  if (cursor) *cursor = it->second.second;
  return BF_OK;
}

int bf_queue_counters(bf_queue* q, int64_t* fetch_count, int64_t* queue_waits) {
  if (!q) return fail(BF_E_INVALID, "null queue");
  std::lock_guard<std::mutex> g(q->mu);
  if (fetch_count) *fetch_count = q->fetch_count;
  if (queue_waits) *queue_waits = q->queue_waits;
  return BF_OK;
}

// ---- grain -----------------------------------------------------------------

int bf_resolve_grain(int32_t policy, int64_t fixed_grain, int64_t grid_size, int64_t pool_size,
                     int32_t has_atomics, int64_t estimate, int64_t light_threshold,
                     int64_t* grain) {
  if (!grain) return fail(BF_E_INVALID, "null out");
  if (grid_size < 1 || pool_size < 1)
    return fail(BF_E_INVALID, "grid_size and pool_size must be >= 1");
  int64_t average = (grid_size + pool_size - 1) / pool_size;
  int64_t g;
  if (policy == BF_POLICY_AVERAGE) {
    g = average;
  } else if (policy == BF_POLICY_FIXED) {
    if (fixed_grain < 1) return fail(BF_E_INVALID, "grain must be >= 1");
    g = std::min(fixed_grain, grid_size);
  } else if (policy == BF_POLICY_AUTO) {
    g = average;
    if (has_atomics > 0) {
      g = std::min(2 * average, grid_size);
    } else if (has_atomics == 0 && estimate >= 0 && estimate < light_threshold) {
      g = std::min(std::max(average, grid_size / 2), grid_size);
    }
  } else {
    return fail(BF_E_INVALID, "unknown policy");
  }
  *grain = std::max<int64_t>(g, 1);
  return BF_OK;
}

// ---- runtime ---------------------------------------------------------------

int bf_runtime_create(bf_arena* a, int32_t pool_size, uint32_t flags, double block_delay,
                      uint64_t seed, bf_runtime** out) {
  if (!a || !out) return fail(BF_E_INVALID, "null argument");
  if (pool_size < 1)
    return fail(BF_E_INVALID, "pool size must be >= 1, got " + std::to_string(pool_size));
  int rc = set_device(a->device);
  if (rc) return rc;
  auto* rt = new bf_runtime();
  rt->arena = a;
  rt->device = a->device;
  rt->pool = pool_size;
  rt->flags = flags;
  rt->block_delay = block_delay;
  rt->rng.seed(seed);
  rt->busy.assign(pool_size, 0);
  cudaDeviceGetAttribute(&rt->num_sms, cudaDevAttrMultiProcessorCount, a->device);
  for (int i = 0; i < pool_size; i++) {
    cudaStream_t s;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      for (auto x : rt->streams) cudaStreamDestroy(x);
      delete rt;
      return cuda_fail(e, "cudaStreamCreate");
    }
    rt->streams.push_back(s);
  }
  rt->holding = (flags & BF_FLAG_HOLD_BLOCKS) != 0;
  if (cudaMalloc(&rt->fault_dev, sizeof(DevFault)) != cudaSuccess ||
      cudaMallocHost(&rt->fault_host, sizeof(DevFault)) != cudaSuccess ||
      cudaHostAlloc((void**)&rt->fault_flag, sizeof(int), cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return fail(BF_E_CUDA, "fault word allocation failed");
  }
  {
    int* flag_dev = nullptr;
    *rt->fault_flag = 0;
    std::memset(rt->fault_host, 0, sizeof(DevFault));
    if (cudaHostGetDevicePointer((void**)&flag_dev, rt->fault_flag, 0) != cudaSuccess) {
      cudaGetLastError();
      return fail(BF_E_CUDA, "fault flag mapping failed");
    }
    rt->fault_host->host_flag = flag_dev;
    if (cudaMemcpy(rt->fault_dev, rt->fault_host, sizeof(DevFault), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      return fail(BF_E_CUDA, "fault word initialisation failed");
    }
  }
  if (flags & BF_FLAG_DEVICE_FETCH) {
    const size_t nctr = (size_t)pool_size * (kFetchSubs + 2);
    if (cudaMalloc((void**)&rt->dfetch_dev, sizeof(unsigned long long) * nctr) != cudaSuccess ||
        cudaMemset(rt->dfetch_dev, 0, sizeof(unsigned long long) * nctr) != cudaSuccess) {
      cudaGetLastError();
      return fail(BF_E_CUDA, "device fetch counters allocation failed");
    }
  }
  a->live_runtimes++;
  *out = rt;
  return BF_OK;
}

int bf_shutdown(bf_runtime* rt) {
  if (!rt) return fail(BF_E_INVALID, "null runtime");
  if (rt->shut_down) return BF_OK;
  rt->shut_down = true;
  set_device(rt->device);
  bf_queue_close(&rt->queue);
  int rc = sync_workers_fault(rt);
  if (rc == BF_OK) absorb_device_fault(rt);
  return rc;
}

int bf_runtime_destroy(bf_runtime* rt) {
  if (!rt) return BF_OK;
  bf_shutdown(rt);
  set_device(rt->device);
  for (auto s : rt->streams) {
    release_stream_scratch(s);
    cudaStreamDestroy(s);
  }
  for (auto e : rt->event_pool) cudaEventDestroy(e);
  for (auto& kv : rt->tasks)
    if (kv.second.executed_dev) cudaFree(kv.second.executed_dev);
  if (rt->fault_dev) cudaFree(rt->fault_dev);
  if (rt->dfetch_dev) cudaFree(rt->dfetch_dev);
  if (rt->fault_host) cudaFreeHost(rt->fault_host);
  if (rt->fault_flag) cudaFreeHost(rt->fault_flag);
  bf_arena* a = rt->arena;
  a->live_runtimes--;
  if (a->live_runtimes == 0) {
    release_zombies(a);
    if (a->destroy_pending) arena_free(a);
  }
  delete rt;
  return BF_OK;
}

}  // extern "C"

namespace bf {
// One fetched block range, issued as one grid launch on a worker stream.
static int issue_fetch(bf_runtime* rt, Fetch& f) {
  cudaStream_t s = rt->streams[f.worker];
  TaskRec& tr = rt->tasks[f.task];
  if (rt->block_delay > 0.0) {
    std::uniform_real_distribution<double> u(0.0, rt->block_delay);
    delay_kernel<<<1, 1, 0, s>>>((unsigned long long)(u(rt->rng) * 1e9));
  }
  if (f.pre.kind != BF_TRAP_NONE) {
    // reference: the trap aborts the worker's range (runtime.py:335-343)
    if (rt->trap.kind == BF_TRAP_NONE) {
      rt->trap = f.pre;
      rt->trap.block = f.first;  // absolute block id
      rt->trap_task = f.task;
      rt->trap_kernel = tr.kernel;
    }
  } else {
    LaunchCtx ctx;
    ctx.name = f.ke->name;
    for (int i = 0; i < 3; i++) {
      ctx.grid[i] = f.grid[i];
      ctx.block[i] = f.block[i];
    }
    ctx.first = f.first;
    ctx.count = f.count;
    ctx.shmem = f.shmem;
    ctx.warp_size = f.warp_size;
    ctx.args = f.args->data();
    ctx.nargs = (int)f.args->size();
    ctx.stream = s;
    ctx.num_sms = rt->num_sms;
    ctx.executed = tr.executed_dev;
    ctx.fault = rt->fault_dev;
    ctx.task = f.task;
    HostTrap ht;
    std::string err;
    ctx.trap = &ht;
    ctx.error = &err;
    ctx.user = f.ke->user;
    int lrc = f.ke->launch(ctx);
    if (lrc != BF_OK) return fail(lrc, std::string(f.ke->name) + ": " + err);
    if (tr.executed_dev) {
      int g = (int)std::min<long long>((f.count + 255) / 256, 1184);
      mark_kernel<<<g, 256, 0, s>>>(tr.executed_dev - tr.base, f.first, f.count);
    }
    if (ht.kind != BF_TRAP_NONE && rt->trap.kind == BF_TRAP_NONE) {
      rt->trap = ht;
      rt->trap_task = f.task;
      rt->trap_kernel = tr.kernel;
    }
  }
  FetchRecord fr;
  fr.task = f.task;
  fr.worker = f.worker;
  fr.first = f.first;
  fr.count = f.count;
  // completion tracking (fetch_event_mode): an event after the fetch only in
  // mode 1; by default a query covers the untracked tail lazily
  fr.done = nullptr;
  if (fetch_event_mode() == 1) {
    fr.done = get_event(rt);
    CK(cudaEventRecord(fr.done, s));
  }
  rt->inflight.push_back(fr);
  return BF_OK;
}
}  // namespace bf

extern "C" {

static int launch_impl(bf_runtime* rt, const char* kernel, const int32_t grid[3],
                       const int32_t block[3], int64_t shmem_bytes, const bf_slot* slots,
                       int32_t nslots, int32_t warp_size, int64_t range_first,
                       int64_t range_count, int64_t grain, uint64_t* task_id) {
  if (!rt || !kernel || !grid || !block) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  for (int i = 0; i < 3; i++)
    if (grid[i] < 1 || block[i] < 1) return fail(BF_E_INVALID, "dim3 components must be >= 1");
  int64_t gtotal = (int64_t)grid[0] * grid[1] * grid[2];
  int64_t bsize = (int64_t)block[0] * block[1] * block[2];
  if (gtotal > 2147483647LL || bsize > 2147483647LL)
    return fail(BF_E_INVALID, "dim3 product overflows i32");
  if (range_count < 0) {
    range_first = 0;
    range_count = gtotal;
  }
  if (range_first < 0 || range_count < 1 || range_first + range_count > gtotal)
    return fail(BF_E_INVALID, "block range outside the grid");
  const int64_t total = range_count;  // blocks of this task
  if (grain < 1) return fail(BF_E_INVALID, "grain must be >= 1");
  if (grain > total) grain = total;
  const KernelEntry* ke = find_kernel(kernel);
  if (!ke)
    return fail(BF_E_UNKNOWN_KERNEL,
                std::string("no sm_100a kernel registered for '") + kernel + "'");
  int rc = set_device(rt->device);
  if (rc) return rc;

  uint64_t id = rt->next_task++;
  TaskRec& tr = rt->tasks[id];
  tr.kernel = kernel;
  tr.total = total;
  tr.base = range_first;
  tr.grain = grain;
  if (task_id) *task_id = id;

  // unpack_args (executor.py:48-75): positional kind check; in the reference
  // a mismatch traps inside the worker and surfaces at sync as RuntimeFault.
  std::vector<ArgVal> args(ke->params.size());
  HostTrap pre;
  if ((size_t)nslots != ke->params.size()) {
    pre.kind = BF_TRAP_TYPE_FAULT;
    pre.message = "expected " + std::to_string(ke->params.size()) + " arguments, got " +
                  std::to_string(nslots);
  } else {
    for (size_t i = 0; i < ke->params.size() && pre.kind == BF_TRAP_NONE; i++) {
      const ParamSpec& p = ke->params[i];
      const bf_slot& s = slots[i];
      ArgVal& v = args[i];
      v.kind = s.kind;
      if (p.kind == BF_SLOT_HANDLE) {
        if (s.kind != BF_SLOT_HANDLE) {
          pre.kind = BF_TRAP_TYPE_FAULT;
          pre.message = std::string("param '") + p.name + "' needs a buffer handle";
          break;
        }
        Buffer* b = lookup(rt->arena, s.v.handle);
        if (!b) {
          pre.kind = BF_TRAP_OUT_OF_BOUNDS;
          pre.message = "dangling buffer handle " + std::to_string(s.v.handle);
          break;
        }
        if (b->scalar != p.scalar) {
          pre.kind = BF_TRAP_TYPE_FAULT;
          pre.message = std::string("param '") + p.name + "' wants a buffer of a different scalar type";
          break;
        }
        v.scalar = b->scalar;
        v.ptr = b->ptr;
        v.len = b->length;
        v.handle = s.v.handle;
      } else {
        if (s.kind != p.kind) {
          pre.kind = BF_TRAP_TYPE_FAULT;
          pre.message = std::string("param '") + p.name + "' has the wrong scalar kind";
          break;
        }
        v.i32 = s.v.i32;
        v.i64 = s.v.i64;
        v.f64 = s.v.f64;
      }
    }
  }

  if ((rt->flags & BF_FLAG_INSTRUMENT) && total > 0) {
    CK(cudaMalloc((void**)&tr.executed_dev, total * sizeof(int)));
    CK(cudaMemsetAsync(tr.executed_dev, 0, total * sizeof(int), rt->streams[0]));
    CK(cudaStreamSynchronize(rt->streams[0]));
  }

  // device-side fetching: the task's fetches are claimed by the CTAs of one
  // persistent launch on the next worker stream
  if (rt->dfetch_dev && ke->dev_fetch && !rt->holding && rt->block_delay <= 0.0 && pre.kind == BF_TRAP_NONE) {
    const int w = (int)(rt->rr % (uint64_t)rt->pool);
    const int64_t nfetch = (total + grain - 1) / grain;
    DevFetch df;
    df.cursor = rt->dfetch_dev + (size_t)w * kFetchSubs;
    df.stats = rt->dfetch_dev + (size_t)rt->pool * kFetchSubs;
    df.slots = rt->pool;
    df.nfetch = nfetch;
    df.grain = grain;
    df.first = range_first;
    df.total = total;
    df.executed = tr.executed_dev ? tr.executed_dev - tr.base : nullptr;
    LaunchCtx ctx;
    ctx.name = ke->name;
    for (int i = 0; i < 3; i++) {
      ctx.grid[i] = grid[i];
      ctx.block[i] = block[i];
    }
    ctx.first = range_first;
    ctx.count = total;
    ctx.shmem = shmem_bytes;
    ctx.warp_size = warp_size;
    ctx.args = args.data();
    ctx.nargs = (int)args.size();
    ctx.stream = rt->streams[w];
    ctx.num_sms = rt->num_sms;
    ctx.executed = tr.executed_dev;
    ctx.fault = rt->fault_dev;
    ctx.task = id;
    HostTrap ht;
    std::string err;
    ctx.trap = &ht;
    ctx.error = &err;
    ctx.user = ke->user;
    ctx.dfetch = &df;
    // the worker's claim counters start at zero (ordered before the launch
    // on its stream; the previous launch on this stream is done with them)
    CK(cudaMemsetAsync(df.cursor, 0, sizeof(unsigned long long) * kFetchSubs, ctx.stream));
    int lrc = ke->launch(ctx);
    if (lrc == BF_OK && ctx.dfetch_grid > 0 && ht.kind == BF_TRAP_NONE) {
      rt->rr++;
      rt->dfetch_used = true;
      tr.fetches = nfetch;
      tr.cursor = total;
      FetchRecord fr;
      fr.task = id;
      fr.worker = w;
      fr.first = range_first;
      fr.count = total;
      fr.device = true;
      fr.done = nullptr;
      if (fetch_event_mode() == 1) {
        fr.done = get_event(rt);
        CK(cudaEventRecord(fr.done, ctx.stream));
      }
      rt->inflight.push_back(fr);
      return BF_OK;
    }
    if (lrc != BF_OK && lrc != BF_E_UNSUPPORTED) return fail(lrc, std::string(ke->name) + ": " + err);
    if (ctx.dfetch_grid > 0) return fail(BF_E_INVALID, std::string(ke->name) + ": device-fetch launcher trapped after launching");
    // not this time (geometry, a trap the host detects): host-issued fetches
  }

  // push + dispatch: the host dispatcher plays the pool's fetch loop
  rc = bf_queue_push(&rt->queue, id, total, grain);
  if (rc) return rc;
  auto shared_args = std::make_shared<std::vector<ArgVal>>(std::move(args));
  for (;;) {
    int32_t got = 0;
    uint64_t tag;
    int64_t first, count;
    bf_queue_fetch(&rt->queue, &got, &tag, &first, &count);
    if (!got) break;
    tr.fetches += 1;
    tr.cursor = first + count;
    Fetch f;
    f.ke = ke;
    f.args = shared_args;
    f.pre = pre;
    f.task = id;
    f.worker = (int)(rt->rr++ % (uint64_t)rt->pool);
    f.first = range_first + first;  // absolute logical block ids
    f.count = count;
    for (int k = 0; k < 3; k++) {
      f.grid[k] = grid[k];
      f.block[k] = block[k];
    }
    f.shmem = shmem_bytes;
    f.warp_size = warp_size;
    if (rt->holding) {
      // hold_blocks: nothing reaches the device before the next synchronize
      // (runtime.py:219-222, 311); launches stay queued on the host
      rt->deferred.push_back(std::move(f));
    } else {
      rc = issue_fetch(rt, f);
      if (rc) return rc;
    }
  }
  return BF_OK;
}

int bf_launch(bf_runtime* rt, const char* kernel, const int32_t grid[3], const int32_t block[3],
              int64_t shmem_bytes, const bf_slot* slots, int32_t nslots, int32_t warp_size,
              int64_t grain, uint64_t* task_id) {
  return launch_impl(rt, kernel, grid, block, shmem_bytes, slots, nslots, warp_size, 0, -1, grain,
                     task_id);
}

int bf_launch_described(bf_runtime* rt, const bf_launch_desc* d, uint64_t* task_id) {
  if (!d || !d->kernel) return fail(BF_E_INVALID, "null launch descriptor");
  if (d->fingerprint) {
    const KernelEntry* ke = find_kernel(d->kernel);
    if (ke && ke->has_fp && std::memcmp(ke->fp, d->fingerprint, 32) != 0)
      return fail(BF_E_UNKNOWN_KERNEL, std::string("kernel '") + d->kernel +
                                           "': body fingerprint differs from the registered sm_100a kernel");
  }
  return launch_impl(rt, d->kernel, d->grid, d->block, d->shmem_bytes, d->slots, d->nslots, d->warp_size,
                     d->count < 0 ? 0 : d->first, d->count, d->grain, task_id);
}

int bf_kernel_set_fingerprint(const char* kernel, const uint8_t fingerprint[32]) {
  if (!kernel || !fingerprint) return fail(BF_E_INVALID, "null argument");
  for (auto& k : registry())
    if (std::strcmp(k.name, kernel) == 0) {
      std::memcpy(k.fp, fingerprint, 32);
      k.has_fp = true;
      return BF_OK;
    }
  return fail(BF_E_UNKNOWN_KERNEL, std::string("no sm_100a kernel registered for '") + kernel + "'");
}

int bf_launch_range(bf_runtime* rt, const char* kernel, const int32_t grid[3],
                    const int32_t block[3], int64_t shmem_bytes, const bf_slot* slots,
                    int32_t nslots, int32_t warp_size, int64_t first, int64_t count,
                    int64_t grain, uint64_t* task_id) {
  return launch_impl(rt, kernel, grid, block, shmem_bytes, slots, nslots, warp_size, first, count,
                     grain, task_id);
}

int bf_synchronize(bf_runtime* rt, bf_fault* fault) {
  if (!rt) return fail(BF_E_INVALID, "null runtime");
  int rc = set_device(rt->device);
  if (rc) return rc;
  rc = sync_workers_fault(rt);
  if (rc) return rc;
  rt->syncs += 1;
  absorb_device_fault(rt);
  if (rt->arena->live_runtimes <= 1) release_zombies(rt->arena);
  if (rt->flags & BF_FLAG_HOLD_BLOCKS) {
    // the reference re-arms only on hold_new_blocks(); nothing to do here
  }
  if (rt->trap.kind != BF_TRAP_NONE) {
    fill_fault(rt, fault);
    return fail(BF_E_FAULT, "block " + std::to_string(rt->trap.block) + ": [" +
                                std::to_string(rt->trap.kind) + "] " + rt->trap.message);
  }
  if (fault) std::memset(fault, 0, sizeof(*fault));
  return BF_OK;
}

int bf_hold_new_blocks(bf_runtime* rt) {
  if (!rt) return fail(BF_E_INVALID, "null runtime");
  rt->holding = true;
  return BF_OK;
}

int bf_task_get(bf_runtime* rt, uint64_t task_id, bf_task_info* out) {
  if (!rt || !out) return fail(BF_E_INVALID, "null argument");
  auto it = rt->tasks.find(task_id);
  if (it == rt->tasks.end()) return fail(BF_E_INVALID, "unknown task");
  retire(rt, false);
  const TaskRec& t = it->second;
  out->total_blocks = t.total;
  out->block_per_fetch = t.grain;
  out->curr_block_id = t.cursor;
  out->fetches = t.fetches;
  out->remaining = t.total - t.completed;
  return BF_OK;
}

int bf_task_executed(bf_runtime* rt, uint64_t task_id, int32_t* executed, int64_t n) {
  if (!rt || !executed) return fail(BF_E_INVALID, "null argument");
  auto it = rt->tasks.find(task_id);
  if (it == rt->tasks.end()) return fail(BF_E_INVALID, "unknown task");
  TaskRec& t = it->second;
  if (n != t.total) return fail(BF_E_INVALID, "executed[] length mismatch");
  set_device(rt->device);
  if (t.executed_dev) {
    // device-observed counts are only meaningful once the fetches drained;
    // the copy is ordered after every worker's work
    for (auto s : rt->streams) {
      if (rt->holding) break;  // held: nothing has run yet
      CK(cudaStreamSynchronize(s));
    }
    if (rt->holding) {
      std::memset(executed, 0, n * sizeof(int32_t));
      return BF_OK;
    }
    CK(cudaMemcpy(executed, t.executed_dev, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    return BF_OK;
  }
  retire(rt, false);
  std::memset(executed, 0, n * sizeof(int32_t));
  for (auto& r : t.done_ranges)
    for (long long b = r.first; b < r.first + r.second; b++) executed[b - t.base] += 1;
  return BF_OK;
}

int bf_counters_get(bf_runtime* rt, bf_counters* out, int64_t* busy, int32_t n) {
  if (!rt || !out) return fail(BF_E_INVALID, "null argument");
  retire(rt, false);
  int64_t fc = 0, qw = 0;
  bf_queue_counters(&rt->queue, &fc, &qw);
  out->fetch_count = fc;
  out->queue_waits = qw;
  out->blocks_executed = rt->blocks_executed;
  out->syncs = rt->syncs;
  out->pool_size = rt->pool;
  if (busy)
    for (int i = 0; i < n && i < rt->pool; i++) busy[i] = rt->busy[i];
  if (rt->dfetch_used) {
    // device-fetched launches: claims and blocks counted by the CTAs (only
    // their retired launches count, as for host fetches: read once drained)
    bool drained = true;
    for (auto& f : rt->inflight)
      if (f.device) drained = false;
    if (drained) {
      std::vector<unsigned long long> st(2 * rt->pool);
      set_device(rt->device);
      CK(cudaMemcpy(st.data(), rt->dfetch_dev + (size_t)rt->pool * kFetchSubs, st.size() * sizeof(unsigned long long),
                    cudaMemcpyDeviceToHost));
      for (int i = 0; i < rt->pool; i++) {
        out->fetch_count += (int64_t)st[2 * i];
        out->blocks_executed += (int64_t)st[2 * i + 1];
        if (busy && i < n) busy[i] += (int64_t)st[2 * i + 1];
      }
    }
  }
  return BF_OK;
}

int bf_worker_stream(bf_runtime* rt, int32_t worker, void** stream) {
  if (!rt || !stream) return fail(BF_E_INVALID, "null argument");
  if (worker < 0 || worker >= rt->pool) return fail(BF_E_INVALID, "worker out of range");
  *stream = (void*)rt->streams[worker];
  return BF_OK;
}

// ---- host-program drivers ---------------------------------------------------

int bf_bfs_levels_impl(void* stream, int num_sms, const int* row, long long lr, const int* col, long long lcol,
                       const int* crow, long long lcrow, const int* ccol, long long lccol, int* lvl, long long ll,
                       int nv, int src, int* depth_out, char* err, int errcap);
int bf_bfs_transpose_impl(void* stream, int num_sms, const int* row, long long lr, const int* col, long long lcol,
                          int nv, int* crow, long long lcrow, int* ccol, long long lccol, char* err, int errcap);

static int bfs_levels_common(bf_runtime* rt, uint32_t row, uint32_t col, const uint32_t* crow, const uint32_t* ccol,
                             uint32_t lvl, int32_t nv, int32_t source, int32_t* depth) {
  if (!rt || !depth) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  Buffer* R = lookup(rt->arena, row);
  Buffer* C = lookup(rt->arena, col);
  Buffer* L = lookup(rt->arena, lvl);
  Buffer* CR = crow ? lookup(rt->arena, *crow) : nullptr;
  Buffer* CC = ccol ? lookup(rt->arena, *ccol) : nullptr;
  if (!R || !C || !L || (crow && !CR) || (ccol && !CC)) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (R->scalar != BF_I32 || C->scalar != BF_I32 || L->scalar != BF_I32 || (CR && CR->scalar != BF_I32) ||
      (CC && CC->scalar != BF_I32))
    return fail(BF_E_TYPEFAULT, "bfs_levels: row, col, lvl (and the transposed graph) must be i32 buffers");
  int rc = set_device(rt->device);
  if (rc) return rc;
  rc = sync_workers(rt);
  if (rc) return rc;
  char err[256] = {0};
  rc = bf_bfs_levels_impl((void*)rt->streams[0], rt->num_sms, (const int*)R->ptr, R->length, (const int*)C->ptr,
                          C->length, CR ? (const int*)CR->ptr : nullptr, CR ? CR->length : 0,
                          CC ? (const int*)CC->ptr : nullptr, CC ? CC->length : 0, (int*)L->ptr, L->length, nv,
                          source, depth, err, sizeof(err));
  if (rc) return fail(rc, err);
  return BF_OK;
}

int bf_bfs_levels(bf_runtime* rt, uint32_t row, uint32_t col, uint32_t lvl, int32_t nv, int32_t source,
                  int32_t* depth) {
  return bfs_levels_common(rt, row, col, nullptr, nullptr, lvl, nv, source, depth);
}

int bf_bfs_levels_do(bf_runtime* rt, uint32_t row, uint32_t col, uint32_t crow, uint32_t ccol, uint32_t lvl,
                     int32_t nv, int32_t source, int32_t* depth) {
  return bfs_levels_common(rt, row, col, &crow, &ccol, lvl, nv, source, depth);
}

int bf_bfs_transpose(bf_runtime* rt, uint32_t row, uint32_t col, int32_t nv, uint32_t crow, uint32_t ccol) {
  if (!rt) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  Buffer* R = lookup(rt->arena, row);
  Buffer* C = lookup(rt->arena, col);
  Buffer* CR = lookup(rt->arena, crow);
  Buffer* CC = lookup(rt->arena, ccol);
  if (!R || !C || !CR || !CC) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (R->scalar != BF_I32 || C->scalar != BF_I32 || CR->scalar != BF_I32 || CC->scalar != BF_I32)
    return fail(BF_E_TYPEFAULT, "bfs_transpose: row, col, crow and ccol must be i32 buffers");
  int rc = set_device(rt->device);
  if (rc) return rc;
  rc = sync_workers(rt);
  if (rc) return rc;
  char err[256] = {0};
  rc = bf_bfs_transpose_impl((void*)rt->streams[0], rt->num_sms, (const int*)R->ptr, R->length,
                             (const int*)C->ptr, C->length, nv, (int*)CR->ptr, CR->length, (int*)CC->ptr,
                             CC->length, err, sizeof(err));
  if (rc) return fail(rc, err);
  return BF_OK;
}

// ---- sharded BFS traversal (parallel.bfs_levels_sharded) --------------------
extern "C" {
int bf_bfs_shard_create_impl(int nv, void** out, char* err, int errcap);
int bf_bfs_shard_destroy_impl(void* p);
int bf_bfs_shard_bitmap_impl(void* p, void** ptr, long long* words);
int bf_bfs_shard_begin_impl(void* p, void* stream, int num_sms, int src, long long vlo, long long vhi, char* err,
                            int errcap);
int bf_bfs_shard_expand_impl(void* p, void* stream, int num_sms, const int* row, long long lr, const int* col,
                             long long lcol, char* err, int errcap);
int bf_bfs_shard_merge_impl(void* p, void* stream, int num_sms, const void* gathered, int world, char* err,
                            int errcap);
int bf_bfs_shard_merge_slice_impl(void* p, void* stream, int num_sms, const void* recv, int world, long long first,
                                  long long count, char* err, int errcap);
int bf_bfs_shard_compact_impl(void* p, void* stream, int num_sms, int* lvl, long long ll, long long* fresh,
                              char* err, int errcap);
int bf_bfs_shard_finish_impl(void* p, void* stream, int num_sms, int* lvl, long long ll, int* depth, char* err,
                             int errcap);
}

struct bf_bfs_shard {
  bf_runtime* rt;
  void* impl;
};

#define BFS_SHARD_PRE(s)                                                   \
  if (!(s) || !(s)->rt) return fail(BF_E_INVALID, "null bfs shard");      \
  if ((s)->rt->shut_down) return fail(BF_E_SHUTDOWN, "runtime shut down"); \
  {                                                                        \
    int rc_ = set_device((s)->rt->device);                                 \
    if (rc_) return rc_;                                                   \
  }

int bf_bfs_shard_create(bf_runtime* rt, int32_t nv, bf_bfs_shard** out) {
  if (!rt || !out) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "runtime shut down");
  int rc = set_device(rt->device);
  if (rc) return rc;
  char err[256] = {0};
  void* impl = nullptr;
  rc = bf_bfs_shard_create_impl(nv, &impl, err, sizeof(err));
  if (rc) return fail(rc, err);
  *out = new bf_bfs_shard{rt, impl};
  return BF_OK;
}

int bf_bfs_shard_destroy(bf_bfs_shard* s) {
  if (!s) return BF_OK;
  if (s->rt) set_device(s->rt->device);
  bf_bfs_shard_destroy_impl(s->impl);
  delete s;
  return BF_OK;
}

int bf_bfs_shard_bitmap(bf_bfs_shard* s, void** dev_ptr, int64_t* words) {
  if (!s || !dev_ptr || !words) return fail(BF_E_INVALID, "null argument");
  long long w = 0;
  bf_bfs_shard_bitmap_impl(s->impl, dev_ptr, &w);
  *words = w;
  return BF_OK;
}

int bf_bfs_shard_begin(bf_bfs_shard* s, int32_t source, int64_t vlo, int64_t vhi) {
  BFS_SHARD_PRE(s);
  int rc = sync_workers(s->rt);
  if (rc) return rc;
  char err[256] = {0};
  rc = bf_bfs_shard_begin_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, source, vlo, vhi, err,
                               sizeof(err));
  return rc ? fail(rc, err) : BF_OK;
}

int bf_bfs_shard_expand(bf_bfs_shard* s, uint32_t row, uint32_t col) {
  BFS_SHARD_PRE(s);
  Buffer* R = lookup(s->rt->arena, row);
  Buffer* C = lookup(s->rt->arena, col);
  if (!R || !C) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (R->scalar != BF_I32 || C->scalar != BF_I32) return fail(BF_E_TYPEFAULT, "row and col must be i32 buffers");
  char err[256] = {0};
  int rc = bf_bfs_shard_expand_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, (const int*)R->ptr,
                                    R->length, (const int*)C->ptr, C->length, err, sizeof(err));
  return rc ? fail(rc, err) : BF_OK;
}

int bf_bfs_shard_merge(bf_bfs_shard* s, const void* gathered, int32_t world) {
  BFS_SHARD_PRE(s);
  if (!gathered || world < 1) return fail(BF_E_INVALID, "bad gathered bitmaps");
  char err[256] = {0};
  int rc = bf_bfs_shard_merge_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, gathered, world, err,
                                   sizeof(err));
  return rc ? fail(rc, err) : BF_OK;
}

int bf_bfs_shard_merge_slice(bf_bfs_shard* s, const void* recv, int32_t world, int64_t first, int64_t count) {
  BFS_SHARD_PRE(s);
  if (!recv || world < 1) return fail(BF_E_INVALID, "bad received slices");
  char err[256] = {0};
  int rc = bf_bfs_shard_merge_slice_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, recv, world, first,
                                         count, err, sizeof(err));
  return rc ? fail(rc, err) : BF_OK;
}

int bf_bfs_shard_compact(bf_bfs_shard* s, uint32_t lvl, int64_t* fresh) {
  BFS_SHARD_PRE(s);
  if (!fresh) return fail(BF_E_INVALID, "null argument");
  Buffer* L = lookup(s->rt->arena, lvl);
  if (!L) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (L->scalar != BF_I32) return fail(BF_E_TYPEFAULT, "lvl must be an i32 buffer");
  char err[256] = {0};
  long long f = 0;
  int rc = bf_bfs_shard_compact_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, (int*)L->ptr, L->length,
                                     &f, err, sizeof(err));
  *fresh = f;
  return rc ? fail(rc, err) : BF_OK;
}

int bf_bfs_shard_finish(bf_bfs_shard* s, uint32_t lvl, int32_t* depth) {
  BFS_SHARD_PRE(s);
  if (!depth) return fail(BF_E_INVALID, "null argument");
  Buffer* L = lookup(s->rt->arena, lvl);
  if (!L) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (L->scalar != BF_I32) return fail(BF_E_TYPEFAULT, "lvl must be an i32 buffer");
  char err[256] = {0};
  int rc = bf_bfs_shard_finish_impl(s->impl, (void*)s->rt->streams[0], s->rt->num_sms, (int*)L->ptr, L->length,
                                    depth, err, sizeof(err));
  return rc ? fail(rc, err) : BF_OK;
}

int bf_hotspot_run_impl(void* stream, int num_sms, float* a, float* b, const float* p, int rows,
                        int cols, const double* kc, int iterations, int tsteps, char* err,
                        int errcap);

int bf_hotspot_run(bf_runtime* rt, uint32_t a, uint32_t power, uint32_t b, int32_t rows,
                   int32_t cols, const double params[5], int32_t iterations, int32_t tsteps) {
  if (!rt || !params) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  Buffer* A = lookup(rt->arena, a);
  Buffer* P = lookup(rt->arena, power);
  Buffer* B = lookup(rt->arena, b);
  if (!A || !P || !B) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (A->scalar != BF_F32 || P->scalar != BF_F32 || B->scalar != BF_F32)
    return fail(BF_E_TYPEFAULT, "hotspot_run: buffers must be f32");
  long long need = (long long)rows * cols;
  if (rows <= 0 || cols <= 0 || A->length < need || P->length < need || B->length < need)
    return fail(BF_E_INVALID, "hotspot_run: buffers shorter than rows*cols");
  if (a == b || a == power || b == power)
    return fail(BF_E_INVALID, "hotspot_run: src, power and dst must be distinct buffers");
  int rc = set_device(rt->device);
  if (rc) return rc;
  // order after every worker's queued work
  for (int w = 1; w < rt->pool; w++) {
    cudaEvent_t ev = get_event(rt);
    cudaEventRecord(ev, rt->streams[w]);
    cudaStreamWaitEvent(rt->streams[0], ev, 0);
    rt->event_pool.push_back(ev);
  }
  char err[256] = {0};
  rc = bf_hotspot_run_impl((void*)rt->streams[0], rt->num_sms, (float*)A->ptr, (float*)B->ptr,
                           (const float*)P->ptr, rows, cols, params, iterations, tsteps, err,
                           sizeof(err));
  if (rc) return fail(rc, err);
  return BF_OK;
}

int bf_kmeans_update_impl(void* stream, int num_sms, float* cent, float* sums, int* counts, int nf, int k,
                          const int* member, int* prev, long long p_lo, long long p_hi, long long* delta,
                          char* err, int errcap);

int bf_kmeans_update(bf_runtime* rt, uint32_t cent, uint32_t sums, uint32_t counts, int32_t nf, int32_t k,
                     uint32_t member, uint32_t prev_member, int64_t p_lo, int64_t p_hi, int64_t* delta) {
  if (!rt || !delta) return fail(BF_E_INVALID, "null argument");
  if (rt->shut_down) return fail(BF_E_SHUTDOWN, "launch after shutdown");
  Buffer* Ce = lookup(rt->arena, cent);
  Buffer* S = lookup(rt->arena, sums);
  Buffer* Cn = lookup(rt->arena, counts);
  Buffer* M = lookup(rt->arena, member);
  Buffer* P = lookup(rt->arena, prev_member);
  if (!Ce || !S || !Cn || !M || !P) return fail(BF_E_DANGLING, "dangling buffer handle");
  if (Ce->scalar != BF_F32 || S->scalar != BF_F32 || Cn->scalar != BF_I32 || M->scalar != BF_I32 ||
      P->scalar != BF_I32)
    return fail(BF_E_TYPEFAULT, "kmeans_update: cent/sums f32, counts/member/prev i32");
  if (nf <= 0 || k <= 0 || Ce->length < (long long)k * nf || S->length < (long long)k * nf || Cn->length < k ||
      p_lo < 0 || p_hi < p_lo || M->length < p_hi || P->length < p_hi)
    return fail(BF_E_INVALID, "kmeans_update: buffer shorter than k*nf / k / point range");
  int rc = set_device(rt->device);
  if (rc) return rc;
  rc = sync_workers(rt);
  if (rc) return rc;
  char err[256] = {0};
  long long d = 0;
  rc = bf_kmeans_update_impl((void*)rt->streams[0], rt->num_sms, (float*)Ce->ptr, (float*)S->ptr, (int*)Cn->ptr,
                             nf, k, (const int*)M->ptr, (int*)P->ptr, p_lo, p_hi, &d, err, sizeof(err));
  if (rc) return fail(rc, err);
  *delta = d;
  return BF_OK;
}

// ---- JIT kernels ---------------------------------------------------------------

int bf_jit_register_impl(const char* key, const char* source, const char* entry, int32_t nparams,
                         const int32_t* kinds, const int32_t* scalars, int32_t dyn_scalar,
                         char* log, int32_t logcap);

int bf_jit_register(const char* key, const char* source, const char* entry, int32_t nparams,
                    const int32_t* kinds, const int32_t* scalars, int32_t dyn_scalar) {
  if (!key || !source || !entry || nparams < 0 || (nparams > 0 && (!kinds || !scalars)))
    return fail(BF_E_INVALID, "null argument");
  std::vector<char> log(16384, 0);
  int rc = bf_jit_register_impl(key, source, entry, nparams, kinds, scalars, dyn_scalar,
                                log.data(), (int32_t)log.size());
  if (rc) return fail(rc, log.data());
  return BF_OK;
}

// ---- registry --------------------------------------------------------------

int bf_kernel_count(int32_t* count) {
  if (!count) return fail(BF_E_INVALID, "null out");
  *count = (int32_t)registry().size();
  return BF_OK;
}

int bf_kernel_info(int32_t index, char* name, int32_t name_cap, int32_t* nparams, int32_t* kinds,
                   int32_t* scalars, int32_t cap) {
  if (index < 0 || index >= (int32_t)registry().size()) return fail(BF_E_INVALID, "bad index");
  const KernelEntry& k = registry()[index];
  if (name && name_cap > 0) std::snprintf(name, name_cap, "%s", k.name);
  if (nparams) *nparams = (int32_t)k.params.size();
  for (int i = 0; i < (int)k.params.size() && i < cap; i++) {
    if (kinds) kinds[i] = k.params[i].kind;
    if (scalars) scalars[i] = k.params[i].scalar;
  }
  return BF_OK;
}

}  // extern "C"
