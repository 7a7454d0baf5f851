// CUDA driver entry points, resolved from libcuda.so.1 at first use so the
// library (and its planning half) loads on machines without a GPU driver.
#pragma once

#include <cuda.h>
#include <dlfcn.h>

#include <stdexcept>
#include <string>

namespace stitch {
namespace exec {

struct CudaApi {
#define STITCH_CU_FN(name) decltype(&::name) name = nullptr;
  STITCH_CU_FN(cuInit)
  STITCH_CU_FN(cuDeviceGet)
  STITCH_CU_FN(cuDeviceGetAttribute)
  STITCH_CU_FN(cuCtxGetCurrent)
  STITCH_CU_FN(cuCtxSetCurrent)
  STITCH_CU_FN(cuDevicePrimaryCtxRetain)
  STITCH_CU_FN(cuDevicePrimaryCtxRelease)
  STITCH_CU_FN(cuCtxPushCurrent)
  STITCH_CU_FN(cuCtxPopCurrent)
  STITCH_CU_FN(cuModuleLoadData)
  STITCH_CU_FN(cuModuleUnload)
  STITCH_CU_FN(cuModuleGetFunction)
  STITCH_CU_FN(cuFuncSetAttribute)
  STITCH_CU_FN(cuFuncGetAttribute)
  STITCH_CU_FN(cuOccupancyMaxActiveBlocksPerMultiprocessor)
  STITCH_CU_FN(cuLaunchKernelEx)
  STITCH_CU_FN(cuMemAlloc)
  STITCH_CU_FN(cuMemFree)
  STITCH_CU_FN(cuMemsetD8Async)
  STITCH_CU_FN(cuMemcpyHtoDAsync)
  STITCH_CU_FN(cuMemcpyDtoHAsync)
  STITCH_CU_FN(cuMemcpyDtoDAsync)
  STITCH_CU_FN(cuStreamSynchronize)
  STITCH_CU_FN(cuStreamCreate)
  STITCH_CU_FN(cuCtxGetStreamPriorityRange)
  STITCH_CU_FN(cuStreamDestroy)
  STITCH_CU_FN(cuStreamWaitEvent)
  STITCH_CU_FN(cuEventCreate)
  STITCH_CU_FN(cuEventDestroy)
  STITCH_CU_FN(cuEventRecord)
  STITCH_CU_FN(cuEventSynchronize)
  STITCH_CU_FN(cuEventElapsedTime)
  STITCH_CU_FN(cuStreamBeginCapture)
  STITCH_CU_FN(cuStreamEndCapture)
  STITCH_CU_FN(cuGraphInstantiate)
  STITCH_CU_FN(cuGraphLaunch)
  STITCH_CU_FN(cuGraphExecDestroy)
  STITCH_CU_FN(cuGraphDestroy)
  STITCH_CU_FN(cuGetErrorString)
  STITCH_CU_FN(cuTensorMapEncodeTiled)
#undef STITCH_CU_FN

  static CudaApi& get() {
    static CudaApi api = load();
    return api;
  }

 private:
  static CudaApi load() {
    CudaApi a;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) throw std::runtime_error(std::string("stitched executor needs the CUDA driver: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) throw std::runtime_error(std::string("libcuda.so.1 lacks ") + n);
      return p;
    };
#define STITCH_CU_LOAD(field, symbol) a.field = reinterpret_cast<decltype(a.field)>(sym(symbol));
    STITCH_CU_LOAD(cuInit, "cuInit")
    STITCH_CU_LOAD(cuDeviceGet, "cuDeviceGet")
    STITCH_CU_LOAD(cuDeviceGetAttribute, "cuDeviceGetAttribute")
    STITCH_CU_LOAD(cuCtxGetCurrent, "cuCtxGetCurrent")
    STITCH_CU_LOAD(cuCtxSetCurrent, "cuCtxSetCurrent")
    STITCH_CU_LOAD(cuDevicePrimaryCtxRetain, "cuDevicePrimaryCtxRetain")
    STITCH_CU_LOAD(cuDevicePrimaryCtxRelease, "cuDevicePrimaryCtxRelease_v2")
    STITCH_CU_LOAD(cuCtxPushCurrent, "cuCtxPushCurrent_v2")
    STITCH_CU_LOAD(cuCtxPopCurrent, "cuCtxPopCurrent_v2")
    STITCH_CU_LOAD(cuModuleLoadData, "cuModuleLoadData")
    STITCH_CU_LOAD(cuModuleUnload, "cuModuleUnload")
    STITCH_CU_LOAD(cuModuleGetFunction, "cuModuleGetFunction")
    STITCH_CU_LOAD(cuFuncSetAttribute, "cuFuncSetAttribute")
    STITCH_CU_LOAD(cuFuncGetAttribute, "cuFuncGetAttribute")
    STITCH_CU_LOAD(cuOccupancyMaxActiveBlocksPerMultiprocessor, "cuOccupancyMaxActiveBlocksPerMultiprocessor")
    STITCH_CU_LOAD(cuLaunchKernelEx, "cuLaunchKernelEx")
    STITCH_CU_LOAD(cuMemAlloc, "cuMemAlloc_v2")
    STITCH_CU_LOAD(cuMemFree, "cuMemFree_v2")
    STITCH_CU_LOAD(cuMemsetD8Async, "cuMemsetD8Async")
    STITCH_CU_LOAD(cuMemcpyHtoDAsync, "cuMemcpyHtoDAsync_v2")
    STITCH_CU_LOAD(cuMemcpyDtoHAsync, "cuMemcpyDtoHAsync_v2")
    STITCH_CU_LOAD(cuMemcpyDtoDAsync, "cuMemcpyDtoDAsync_v2")
    STITCH_CU_LOAD(cuStreamSynchronize, "cuStreamSynchronize")
    STITCH_CU_LOAD(cuStreamCreate, "cuStreamCreate")
    STITCH_CU_LOAD(cuCtxGetStreamPriorityRange, "cuCtxGetStreamPriorityRange")
    STITCH_CU_LOAD(cuStreamDestroy, "cuStreamDestroy_v2")
    STITCH_CU_LOAD(cuStreamWaitEvent, "cuStreamWaitEvent")
    STITCH_CU_LOAD(cuEventCreate, "cuEventCreate")
    STITCH_CU_LOAD(cuEventDestroy, "cuEventDestroy_v2")
    STITCH_CU_LOAD(cuEventRecord, "cuEventRecord")
    STITCH_CU_LOAD(cuEventSynchronize, "cuEventSynchronize")
    STITCH_CU_LOAD(cuEventElapsedTime, "cuEventElapsedTime")
    STITCH_CU_LOAD(cuStreamBeginCapture, "cuStreamBeginCapture_v2")
    STITCH_CU_LOAD(cuStreamEndCapture, "cuStreamEndCapture")
    STITCH_CU_LOAD(cuGraphInstantiate, "cuGraphInstantiateWithFlags")
    STITCH_CU_LOAD(cuGraphLaunch, "cuGraphLaunch")
    STITCH_CU_LOAD(cuGraphExecDestroy, "cuGraphExecDestroy")
    STITCH_CU_LOAD(cuGraphDestroy, "cuGraphDestroy")
    STITCH_CU_LOAD(cuGetErrorString, "cuGetErrorString")
    STITCH_CU_LOAD(cuTensorMapEncodeTiled, "cuTensorMapEncodeTiled")
#undef STITCH_CU_LOAD
    return a;
  }
};

inline void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* msg = nullptr;
  CudaApi::get().cuGetErrorString(r, &msg);
  throw std::runtime_error(std::string("CUDA error in ") + what + ": " + (msg ? msg : "unknown"));
}

// Makes `ctx` current on the calling thread for a scope (the executor's
// device primary context, whatever context the caller has current).
class CtxScope {
 public:
  explicit CtxScope(void* ctx) : on_(ctx != nullptr) {
    if (on_) cu_check(CudaApi::get().cuCtxPushCurrent(static_cast<CUcontext>(ctx)), "cuCtxPushCurrent");
  }
  ~CtxScope() {
    if (on_) {
      CUcontext old;
      CudaApi::get().cuCtxPopCurrent(&old);
    }
  }
  CtxScope(const CtxScope&) = delete;
  CtxScope& operator=(const CtxScope&) = delete;

 private:
  bool on_;
};

}  // namespace exec
}  // namespace stitch
