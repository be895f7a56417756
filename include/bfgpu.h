/*
 * bfgpu.h — C ABI of the B200-native launch runtime (libbfgpu.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `blockfuse` (arXiv 2206.07896, CuPBoP restated in Python).  Every entry point
 * replaces one reference interface; the citation on each declaration names it
 * (paths relative to /root/reference/pkg/src/blockfuse/).  Plain C types only:
 * no torch, no C++ types cross this boundary, and no C++ exception escapes it.
 *
 * Conventions
 *   - Every function returns an int status (BF_OK == 0).  On failure the
 *     thread-local message is available from bf_last_error().
 *   - Buffers are addressed by handles (uint32) that start at 1 and are never
 *     reused within an arena (arena.py:69-84).  The library owns all device
 *     memory; host pointers are borrowed for the duration of the call only.
 *   - f32 scalar kernel arguments travel as double (the reference boxes a
 *     Python float into an f32 slot without rounding, hostprog.py:390-414,
 *     executor.py:42-75); kernels evaluate float math in f64 and round to f32
 *     only at stores (interp.py:58-99, arena.py:44-45).
 *   - Launch is asynchronous; bf_synchronize is the quiescence point and the
 *     place where device traps surface (runtime.py:255-278).
 */
#ifndef BFGPU_H_
#define BFGPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFGPU_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------ */
enum bf_status {
  BF_OK = 0,
  BF_E_INVALID = 1,         /* bad argument (ValueError in the reference)          */
  BF_E_SHUTDOWN = 2,        /* launch after shutdown -> PoolShutdown (runtime.py:28,258) */
  BF_E_TYPEFAULT = 3,       /* slot/param mismatch -> Trap(TypeFault) (executor.py:56-74) */
  BF_E_UNKNOWN_KERNEL = 4,  /* no sm_100a kernel registered under that name         */
  BF_E_CUDA = 5,            /* CUDA runtime error                                    */
  BF_E_DANGLING = 6,        /* unknown / freed handle -> Trap(OutOfBounds) (arena.py:86-90) */
  BF_E_FAULT = 7,           /* a launched kernel trapped -> RuntimeFault (runtime.py:32-38) */
  BF_E_UNSUPPORTED = 8      /* geometry/feature outside what the kernel supports     */
};

/* ---- scalar and slot kinds (syntax.py:12-17, executor.py:42-46) ---------- */
enum bf_scalar { BF_I32 = 0, BF_I64 = 1, BF_F32 = 2, BF_F64 = 3 };
enum bf_slot_kind {
  BF_SLOT_I32 = 0, BF_SLOT_I64 = 1, BF_SLOT_F32 = 2, BF_SLOT_F64 = 3,
  BF_SLOT_HANDLE = 4
};

/* One packed kernel argument (the reference's ArgSlot, executor.py:42-46).
 * F32 and F64 slots both carry a double.  16 bytes, 8-byte aligned. */
typedef struct bf_slot {
  int32_t kind;     /* enum bf_slot_kind */
  int32_t _pad;
  union {
    int32_t i32;
    int64_t i64;
    double f64;     /* used for both BF_SLOT_F32 and BF_SLOT_F64 */
    uint32_t handle;
  } v;
} bf_slot;

/* ---- traps (arena.py:24-36) --------------------------------------------- */
enum bf_trap_kind {
  BF_TRAP_NONE = 0,
  BF_TRAP_OUT_OF_BOUNDS = 1,
  BF_TRAP_DIV_BY_ZERO = 2,
  BF_TRAP_TYPE_FAULT = 3,
  BF_TRAP_NON_UNIFORM_TRIP = 4
};

/* The first fault recorded since the runtime was created (runtime.py:340-341
 * keeps the first; later syncs re-raise it, runtime.py:276-278). */
typedef struct bf_fault {
  int32_t kind;        /* enum bf_trap_kind */
  int32_t _pad;
  int64_t block_id;    /* linear logical block id that trapped */
  uint64_t task_id;    /* task that trapped */
  char kernel[32];
  char message[160];
} bf_fault;

/* Per-launch record (KernelTask, runtime.py:108-125). */
typedef struct bf_task_info {
  int64_t total_blocks;     /* totalBlocks */
  int64_t block_per_fetch;  /* grain */
  int64_t curr_block_id;    /* queue cursor (== total once fully fetched) */
  int64_t fetches;
  int64_t remaining;        /* blocks not yet known complete on the device */
} bf_task_info;

/* RuntimeCounters (runtime.py:128-143); busy_blocks is returned separately. */
typedef struct bf_counters {
  int64_t fetch_count;
  int64_t blocks_executed;
  int64_t syncs;
  int64_t queue_waits;
  int32_t pool_size;
  int32_t _pad;
} bf_counters;

/* Fetch policies (runtime.py:45-65). */
enum bf_policy { BF_POLICY_AVERAGE = 0, BF_POLICY_FIXED = 1, BF_POLICY_AUTO = 2 };

/* Runtime creation flags. */
#define BF_FLAG_HOLD_BLOCKS 0x1u  /* gate every block until the next sync (runtime.py:219-222) */
#define BF_FLAG_INSTRUMENT  0x2u  /* device-side per-block executed[] counters (runtime.py:121,345) */
/* Device-side block fetching: a launch whose kernel supports it is ONE
 * persistent grid whose CTAs claim block_per_fetch logical blocks at a time
 * from a device claim counter (the paper's block fetching, runtime.py:175-201,
 * 305-350, done by the GPU's own CTAs instead of host-issued launches);
 * fetch counts, busy blocks and executed[] come from the device.  Other
 * kernels (and held or delayed launches) keep host-issued fetches. */
#define BF_FLAG_DEVICE_FETCH 0x4u

typedef struct bf_arena bf_arena;
typedef struct bf_runtime bf_runtime;
typedef struct bf_queue bf_queue;

/* ---- library ------------------------------------------------------------- */
int bf_abi_version(void);
const char *bf_last_error(void);
int bf_device_count(int32_t *count);

/* ---- memory shim: DeviceArena (arena.py:66-152) -------------------------- */
/* DeviceArena.__init__ (arena.py:68-73); buffers live in `device`'s HBM. */
int bf_arena_create(int32_t device, bf_arena **out);
int bf_arena_destroy(bf_arena *arena);
/* DeviceArena.alloc (arena.py:75-84): zero-filled, handle never reused. */
int bf_alloc(bf_arena *arena, int32_t scalar, int64_t length, uint32_t *handle);
/* DeviceArena.free (arena.py:86-87); orders after launches in flight. */
int bf_free(bf_arena *arena, uint32_t handle);
/* An element-range view [first, first + length) of a buffer under a new
 * handle (no copy; the reference has no views — this is the multi-GPU
 * partitioner's way to hand one rank's element range of a grid-stride
 * launch to the unchanged kernel, parallel.py).  The offset must be 16 B
 * aligned; the parent cannot be freed while views of it are live. */
int bf_view(bf_arena *arena, uint32_t handle, int64_t first, int64_t length, uint32_t *view);
/* DeviceArena.scalar_type / length (arena.py:95-99) plus the device pointer. */
int bf_buffer_info(bf_arena *arena, uint32_t handle, int32_t *scalar,
                   int64_t *length, uint64_t *device_ptr);
/* DeviceArena.fill / from_bytes (arena.py:126-152): raw little-endian bytes
 * written at byte `offset`; returns after the copy completed (host buffer may
 * be reused).  Ordered after every launch previously issued on the arena. */
int bf_upload(bf_arena *arena, uint32_t handle, const void *src, int64_t nbytes,
              int64_t offset);
/* DeviceArena.to_bytes / to_list (arena.py:122-134): raw bytes at `offset`,
 * ordered after every launch previously issued on the arena. */
int bf_download(bf_arena *arena, uint32_t handle, void *dst, int64_t nbytes,
                int64_t offset);
/* Fill `nbytes` at `offset` with a repeated 4-byte pattern (device memset). */
int bf_fill32(bf_arena *arena, uint32_t handle, uint32_t pattern, int64_t offset,
              int64_t nbytes);
/* Copy between two buffers of the same arena (device to device). */
int bf_copy(bf_arena *arena, uint32_t dst, int64_t dst_offset, uint32_t src,
            int64_t src_offset, int64_t nbytes);

/* ---- task queue (TaskQueue, runtime.py:146-205) -------------------------- */
/* A standalone FIFO of block ranges; the runtime drives one internally.  The
 * standalone form exists so the fetch protocol can be tested without a GPU
 * (test_runtime.py:33-111 drives TaskQueue with dummy tasks). */
int bf_queue_create(bf_queue **out);
int bf_queue_destroy(bf_queue *q);
/* TaskQueue.push (runtime.py:159-168); BF_E_SHUTDOWN after close. */
int bf_queue_push(bf_queue *q, uint64_t task_tag, int64_t total_blocks,
                  int64_t block_per_fetch);
/* TaskQueue.fetch (runtime.py:175-201), non-blocking form: *got = 0 when the
 * queue is empty (or closed); else the claimed range of the front task. */
int bf_queue_fetch(bf_queue *q, int32_t *got, uint64_t *task_tag, int64_t *first,
                   int64_t *count);
int bf_queue_close(bf_queue *q);
int bf_queue_is_empty(bf_queue *q, int32_t *empty);
/* Per-task fetch count and cursor of a task still known to the queue. */
int bf_queue_task(bf_queue *q, uint64_t task_tag, int64_t *fetches,
                  int64_t *curr_block_id);
int bf_queue_counters(bf_queue *q, int64_t *fetch_count, int64_t *queue_waits);

/* ---- grain resolution (resolve_grain, runtime.py:78-101) ---------------- */
int bf_resolve_grain(int32_t policy, int64_t fixed_grain, int64_t grid_size,
                     int64_t pool_size, int32_t has_atomics,
                     int64_t static_instruction_estimate,
                     int64_t light_kernel_threshold, int64_t *grain);

/* ---- launch runtime (Runtime, runtime.py:208-350) ----------------------- */
/* Runtime.__init__ (runtime.py:225-251): `pool_size` workers, each an
 * in-order CUDA stream on the arena's device (the pool threads of the
 * reference).  Workers are created once and destroyed once. */
int bf_runtime_create(bf_arena *arena, int32_t pool_size, uint32_t flags,
                      double block_delay, uint64_t seed, bf_runtime **out);
/* Runtime.shutdown (runtime.py:288-295): idempotent; waits for the device. */
int bf_shutdown(bf_runtime *rt);
int bf_runtime_destroy(bf_runtime *rt);
/* Runtime.launch (runtime.py:255-267).  Non-blocking: pushes the task, the
 * dispatcher fetches `grain`-block ranges off the queue and issues each range
 * as one grid launch on the next worker stream.  `kernel` names a registered
 * sm_100a kernel (the MpmdKernel.name dispatch key, transform.py:109).
 * `warp_size` is MpmdKernel.warp_size for warp-mode kernels (0 otherwise).
 * Errors: BF_E_SHUTDOWN, BF_E_TYPEFAULT, BF_E_UNKNOWN_KERNEL, BF_E_INVALID. */
int bf_launch(bf_runtime *rt, const char *kernel, const int32_t grid[3],
              const int32_t block[3], int64_t shmem_bytes, const bf_slot *slots,
              int32_t nslots, int32_t warp_size, int64_t grain, uint64_t *task_id);
/* One worker's share of a launch: only logical blocks [first, first+count)
 * of the grid run (the fetched range of runtime.py:175-201 handed to this
 * process — ranks of a multi-GPU job are the workers, parallel.py).  The
 * task has `count` blocks; executed[] is indexed relative to `first`. */
int bf_launch_range(bf_runtime *rt, const char *kernel, const int32_t grid[3],
                    const int32_t block[3], int64_t shmem_bytes, const bf_slot *slots,
                    int32_t nslots, int32_t warp_size, int64_t first, int64_t count,
                    int64_t grain, uint64_t *task_id);
/* Runtime.launch / launch_range through one descriptor (the Python binding
 * keeps one per (routine, geometry, PackedArgs) and passes a single pointer:
 * a 10-argument foreign call costs more than the launch itself).
 * `fingerprint` (nullable) is the sha256 of the routine's MpmdKernel.to_dict()
 * (routines.fingerprint_of); when the kernel has a registered fingerprint
 * (bf_kernel_set_fingerprint) a mismatch fails with BF_E_UNKNOWN_KERNEL, so
 * a caller cannot run the hand-written kernel for a different body under a
 * registered name.  count < 0 launches the whole grid. */
typedef struct bf_launch_desc {
  const char *kernel;
  const uint8_t *fingerprint;  /* 32 bytes or NULL */
  int32_t grid[3];
  int32_t block[3];
  int64_t shmem_bytes;
  const bf_slot *slots;
  int32_t nslots;
  int32_t warp_size;
  int64_t first;
  int64_t count;
  int64_t grain;
} bf_launch_desc;
int bf_launch_described(bf_runtime *rt, const bf_launch_desc *desc, uint64_t *task_id);
/* Register the expected body fingerprint of a hand-written kernel
 * (paper_2206_07896_b200/fingerprints.json, made from the reference's own
 * transform() by oracle/gen_golden.py). */
int bf_kernel_set_fingerprint(const char *kernel, const uint8_t fingerprint[32]);
/* Runtime.device_synchronize (runtime.py:269-278): releases a hold, waits for
 * every worker, increments syncs, and returns BF_E_FAULT with *fault filled
 * if any launch trapped (now or earlier). */
int bf_synchronize(bf_runtime *rt, bf_fault *fault);
/* Runtime.hold_new_blocks (runtime.py:284-286). */
int bf_hold_new_blocks(bf_runtime *rt);
/* KernelTask fields (runtime.py:108-125). */
int bf_task_get(bf_runtime *rt, uint64_t task_id, bf_task_info *out);
/* KernelTask.executed: per-block run counts (needs BF_FLAG_INSTRUMENT for
 * device-observed counts; otherwise the dispatcher's completed ranges). */
int bf_task_executed(bf_runtime *rt, uint64_t task_id, int32_t *executed,
                     int64_t n);
/* Runtime.counters (runtime.py:128-143); busy_blocks has pool_size entries. */
int bf_counters_get(bf_runtime *rt, bf_counters *out, int64_t *busy_blocks,
                    int32_t n);
/* The CUDA stream (cudaStream_t) of worker `worker`, for event timing and for
 * ordering collectives with launches. */
int bf_worker_stream(bf_runtime *rt, int32_t worker, void **stream);

/* ---- host-program drivers --------------------------------------------------- */
/* Whole BFS traversal from `source` over the CSR graph in buffers (row, col)
 * (Rodinia's bfs host loop fused on the device; kernels/bfs.kn is the
 * per-level step).  Writes lvl[v] = hop distance from source, -1 when
 * unreachable — exactly the levels of launching `bfs` with cur = 0, 1, ...
 * until `changed` stays 0 after lvl = -1 except lvl[source] = 0.  *depth =
 * max level + 1.  Runs on worker 0's stream after draining every worker;
 * returns when done.  BF_E_FAULT when the CSR indexes out of range. */
int bf_bfs_levels(bf_runtime *rt, uint32_t row, uint32_t col, uint32_t lvl,
                  int32_t nv, int32_t source, int32_t *depth);

/* In-edge CSR of the graph (row, col) for the bottom-up steps: crow
 * (nv + 1 entries) and ccol (at least row[nv] entries), i32 arena buffers;
 * ccol[crow[v] .. crow[v+1]) holds the sources u of the edges u -> v in an
 * unspecified order.  Built once per graph (a GPU counting sort).  BF_E_FAULT
 * when row is malformed or a target is out of range.  No reference
 * counterpart: the bottom-up direction needs the in-edges. */
int bf_bfs_transpose(bf_runtime *rt, uint32_t row, uint32_t col, int32_t nv,
                     uint32_t crow, uint32_t ccol);
/* bf_bfs_levels, direction-optimizing: levels whose frontier is large run
 * bottom-up over (crow, ccol) from bf_bfs_transpose (each unvisited vertex
 * looks for a frontier in-neighbour).  Same levels as bf_bfs_levels (BFS
 * levels are unique); (crow, ccol) must be the transpose of (row, col). */
int bf_bfs_levels_do(bf_runtime *rt, uint32_t row, uint32_t col, uint32_t crow,
                     uint32_t ccol, uint32_t lvl, int32_t nv, int32_t source,
                     int32_t *depth);

/* One pass of Rodinia's kmeans host loop after an assignment launch of
 * kernels/kmeans.kn (kmeans_clustering.c's do/while): cent[c][l] =
 * sums[c][l] / counts[c] in f32 for clusters with members (others keep
 * their centroid), sums and counts zeroed for the next pass, and *delta =
 * number of points p in [p_lo, p_hi) with member[p] != prev_member[p]
 * (Rodinia's delta), after which prev_member = member on that range.  With
 * several ranks the caller all-reduces sums and counts before and delta
 * after (cluster.kmeans_iterate).  Runs on worker 0's stream after draining
 * every worker; returns when done. */
int bf_kmeans_update(bf_runtime *rt, uint32_t cent, uint32_t sums, uint32_t counts,
                     int32_t nf, int32_t k, uint32_t member, uint32_t prev_member,
                     int64_t p_lo, int64_t p_hi, int64_t *delta);

/* Sharded BFS traversal, one process per GPU (parallel.bfs_levels_sharded;
 * SURVEY §8e "bfs: per-level frontier exchange").  A shard keeps the whole
 * nv-bit visited bitmap and per-vertex level bytes on its device and expands
 * only the frontier vertices of its own range [vlo, vhi).  Per level the host
 * calls expand, all-gathers every rank's bitmap (world x words uint32 in
 * rank order, e.g. torch.distributed.all_gather_into_tensor over NCCL) and
 * passes it to merge (OR), then compact, which returns the number of vertices
 * discovered in the level — the same on every rank, so the loop ends together
 * (stop at 0).  finish writes lvl (identical on every rank; exactly the
 * levels of bf_bfs_levels).  All calls run on worker 0's stream and return
 * when their work is done (merge only enqueues). */
typedef struct bf_bfs_shard bf_bfs_shard;
int bf_bfs_shard_create(bf_runtime *rt, int32_t nv, bf_bfs_shard **out);
int bf_bfs_shard_destroy(bf_bfs_shard *s);
/* device pointer and length (uint32 words) of the shard's visited bitmap */
int bf_bfs_shard_bitmap(bf_bfs_shard *s, void **dev_ptr, int64_t *words);
int bf_bfs_shard_begin(bf_bfs_shard *s, int32_t source, int64_t vlo, int64_t vhi);
int bf_bfs_shard_expand(bf_bfs_shard *s, uint32_t row, uint32_t col);
int bf_bfs_shard_merge(bf_bfs_shard *s, const void *gathered_dev, int32_t world);
/* One rank's bitmap slice after an all-to-all of the world bitmaps:
 * now[first + i] = OR over r < world of recv[r * count + i] (the visited
 * bitmap has 64 zero words of padding past `words`). */
int bf_bfs_shard_merge_slice(bf_bfs_shard *s, const void *recv_dev, int32_t world, int64_t first,
                             int64_t count);
int bf_bfs_shard_compact(bf_bfs_shard *s, uint32_t lvl, int64_t *fresh);
int bf_bfs_shard_finish(bf_bfs_shard *s, uint32_t lvl, int32_t *depth);

/* Rodinia's hotspot host loop fused: the result of `iterations` ping-pong
 * launches of `hotspot` (kernels/hotspot.kn) starting from buffer `a`, with
 * `b` as the other buffer — bit-identical.  tsteps = 1: one streaming pass
 * per iteration; 2..4: register-wavefront temporal blocking (`tsteps`
 * iterations per pass through HBM); 8/12/16: shared-memory tiles; 0 =
 * default (4, the fastest on B200 in round 1).  The result
 * lands where the launch loop leaves it: `a` for even, `b` for odd
 * `iterations`; the other buffer is scratch.  params = {step/Cap, 1/Rx,
 * 1/Ry, 1/Rz, ambient} as doubles.  Asynchronous on worker 0's stream,
 * ordered after everything already launched on the runtime. */
int bf_hotspot_run(bf_runtime *rt, uint32_t a, uint32_t power, uint32_t b,
                   int32_t rows, int32_t cols, const double params[5],
                   int32_t iterations, int32_t tsteps);

/* ---- JIT kernels ---------------------------------------- */
/* Compile CUDA `source` (generated from a reference MpmdKernel by
 * paper_2206_07896_b200/codegen.py) with NVRTC for sm_100a and register its
 * extern "C" `entry` under `key`; bf_launch(key, ...) then runs it through
 * the same fetch protocol as a hand-written kernel.  kinds/scalars as in
 * bf_kernel_info; dyn_scalar is the bf_scalar of the extern shared array, or
 * -1.  Idempotent per key; BF_E_INVALID carries the NVRTC log. */
int bf_jit_register(const char *key, const char *source, const char *entry,
                    int32_t nparams, const int32_t *kinds, const int32_t *scalars,
                    int32_t dyn_scalar);

/* ---- kernel registry ---------------------------------------------------- */
int bf_kernel_count(int32_t *count);
/* Name and parameter signature of registered kernel `index`: kinds[i] is a
 * bf_slot_kind; for handle params scalars[i] is the element bf_scalar. */
int bf_kernel_info(int32_t index, char *name, int32_t name_cap, int32_t *nparams,
                   int32_t *kinds, int32_t *scalars, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* BFGPU_H_ */
