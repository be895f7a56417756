// JIT path for kernels without a hand-written implementation (SURVEY §8f
// row 2): CUDA source generated from the reference's MpmdKernel AST
// (paper_2206_07896_b200/codegen.py) is compiled with NVRTC for sm_100a,
// loaded with cudaLibraryLoadData and registered under a fingerprint key, so
// Runtime.launch dispatches it exactly like a registered kernel (same fetch
// protocol, worker streams, fault word and counters).
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "bf_internal.h"
#include "common.cuh"

namespace bf {

// must match PRELUDE in codegen.py
struct BfJitGeom {
  int gx, gy, gz, bx, by, bz;
  long long first, count;
  long long dyn_elems;
  int* fault;
  unsigned long long task;
  int warp_size;
  unsigned long long* dcur;
  unsigned long long* dstats;
  int* dexec;
  long long nfetch, grain;
  int dslots;
};

struct JitInfo {
  std::string key;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  int nwords = 2;
  int dyn_elem_size = 0;  // element size of the extern shared array (0: none)
  int max_dyn_set = 48 * 1024;
};

static std::vector<std::unique_ptr<JitInfo>>& jit_infos() {
  static std::vector<std::unique_ptr<JitInfo>> v;
  return v;
}

static int jit_launch(LaunchCtx& ctx) {
  const JitInfo* ji = static_cast<const JitInfo*>(ctx.user);
  const long long B = (long long)ctx.block[0] * ctx.block[1] * ctx.block[2];
  if (B > 1024) {
    *ctx.error = "jit kernel: blocks above 1024 threads are not supported";
    return BF_E_UNSUPPORTED;
  }
  std::vector<long long> w((size_t)ji->nwords, 0);
  for (int i = 0; i < ctx.nargs; i++) {
    const ArgVal& a = ctx.args[i];
    if (a.kind == BF_SLOT_HANDLE) {
      w[2 * i] = (long long)(uintptr_t)a.ptr;
      w[2 * i + 1] = a.len;
    } else if (a.kind == BF_SLOT_I32) {
      w[2 * i] = a.i32;
    } else if (a.kind == BF_SLOT_I64) {
      w[2 * i] = a.i64;
    } else {
      long long bits;
      std::memcpy(&bits, &a.f64, 8);
      w[2 * i] = bits;
    }
  }
  BfJitGeom g;
  g.gx = ctx.grid[0]; g.gy = ctx.grid[1]; g.gz = ctx.grid[2];
  g.bx = ctx.block[0]; g.by = ctx.block[1]; g.bz = ctx.block[2];
  g.first = ctx.first;
  g.count = ctx.count;
  g.dyn_elems = ji->dyn_elem_size ? ctx.shmem / ji->dyn_elem_size : 0;
  g.fault = reinterpret_cast<int*>(ctx.fault);
  g.task = ctx.task;
  g.warp_size = ctx.warp_size;
  size_t smem = ji->dyn_elem_size ? (size_t)(g.dyn_elems * ji->dyn_elem_size) : 0;
  if (smem > 200 * 1024) {
    *ctx.error = "jit kernel: dynamic shared memory above 200 KiB";
    return BF_E_UNSUPPORTED;
  }
  if ((int)smem > ji->max_dyn_set) {
    cudaFuncSetAttribute((const void*)ji->kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    const_cast<JitInfo*>(ji)->max_dyn_set = 200 * 1024;
  }
  g.dcur = nullptr;
  g.dstats = nullptr;
  g.dexec = nullptr;
  g.nfetch = g.grain = 0;
  g.dslots = 1;
  int grid = (int)std::min<long long>(ctx.count, (long long)ctx.num_sms * 8);
  if (ctx.dfetch) {  // persistent grid claiming the task's fetches (codegen.py)
    const DevFetch& F = *ctx.dfetch;
    g.dcur = F.cursor;
    g.dstats = F.stats;
    g.dexec = F.executed;
    static_assert(kFetchSubs == 8, "codegen.py's bf_claim splits the fetches into 8 sub-ranges");
    g.nfetch = F.nfetch;
    g.grain = F.grain;
    g.dslots = F.slots;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)ji->kern, (int)B, smem) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    grid = (int)std::min<long long>(F.nfetch, (long long)per_sm * ctx.num_sms);
  }
  void* params[2] = {w.data(), &g};
  cudaError_t e = cudaLaunchKernel((const void*)ji->kern, dim3(grid), dim3((unsigned)B), params,
                                   smem, ctx.stream);
  if (e != cudaSuccess) {
    *ctx.error = std::string("jit launch failed: ") + cudaGetErrorString(e);
    return BF_E_CUDA;
  }
  if (ctx.dfetch) ctx.dfetch_grid = grid;
  return BF_OK;
}

}  // namespace bf

using namespace bf;

extern "C" int bf_jit_register_impl(const char* key, const char* source, const char* entry,
                                    int32_t nparams, const int32_t* kinds, const int32_t* scalars,
                                    int32_t dyn_scalar, char* log, int32_t logcap) {
  if (find_kernel(key)) return BF_OK;  // already registered in this process
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source, "bfjit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    snprintf(log, logcap, "nvrtcCreateProgram failed");
    return BF_E_INVALID;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17",
                        "-default-device", "-lineinfo"};
  nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string l(n, '\0');
    nvrtcGetProgramLog(prog, &l[0]);
    snprintf(log, logcap, "NVRTC: %s: %s", nvrtcGetErrorString(r), l.c_str());
    nvrtcDestroyProgram(&prog);
    return BF_E_INVALID;
  }
  size_t cubin_size = 0;
  nvrtcGetCUBINSize(prog, &cubin_size);
  std::vector<char> cubin(cubin_size);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);

  auto ji = std::make_unique<JitInfo>();
  ji->key = key;
  cudaError_t e = cudaLibraryLoadData(&ji->lib, cubin.data(), nullptr, nullptr, 0, nullptr,
                                      nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&ji->kern, ji->lib, entry);
  if (e != cudaSuccess) {
    snprintf(log, logcap, "loading the JIT module failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return BF_E_CUDA;
  }
  ji->nwords = nparams > 0 ? 2 * nparams : 2;
  ji->dyn_elem_size = dyn_scalar < 0 ? 0 : (dyn_scalar == BF_I64 || dyn_scalar == BF_F64 ? 8 : 4);
  std::vector<ParamSpec> params;
  for (int i = 0; i < nparams; i++) params.push_back(ParamSpec{kinds[i], scalars[i], "p"});
  JitInfo* raw = ji.get();
  jit_infos().push_back(std::move(ji));
  registry().push_back(KernelEntry{raw->key.c_str(), std::move(params), jit_launch, raw});
  registry().back().dev_fetch = true;
  return BF_OK;
}
