// Shareable device memory and CUDA IPC mappings for the fused NVLink
// all-gather (fkv_decode_exchange / fkv_merge_wait).  cudaMalloc'd (not the
// torch caching allocator) so every buffer is its own IPC-exportable
// allocation; peers map each other's receive buffers and flag arrays once.
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"

extern "C" int fkv_dev_alloc(int64_t bytes, void** out_ptr) {
  using namespace fkv;
  if (!out_ptr || bytes <= 0) return set_error(FKV_ERR_INVALID, "fkv_dev_alloc: bad arguments");
  if (int rc = cuda_check(cudaMalloc(out_ptr, static_cast<size_t>(bytes)), "cudaMalloc")) return rc;
  return cuda_check(cudaMemset(*out_ptr, 0, static_cast<size_t>(bytes)), "cudaMemset");
}

extern "C" int fkv_dev_free(void* ptr) {
  return fkv::cuda_check(cudaFree(ptr), "cudaFree");
}

extern "C" int fkv_ipc_get(void* dev_ptr, void* handle) {
  using namespace fkv;
  if (!dev_ptr || !handle) return set_error(FKV_ERR_INVALID, "fkv_ipc_get: null pointer");
  cudaIpcMemHandle_t h;
  if (int rc = cuda_check(cudaIpcGetMemHandle(&h, dev_ptr), "cudaIpcGetMemHandle")) return rc;
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  return FKV_OK;
}

extern "C" int fkv_ipc_open(const void* handle, void** out_ptr) {
  using namespace fkv;
  if (!handle || !out_ptr) return set_error(FKV_ERR_INVALID, "fkv_ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_check(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
}

extern "C" int fkv_ipc_close(void* ptr) {
  return fkv::cuda_check(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

// Device address of pinned host memory (cudaHostAlloc / cudaHostRegister),
// for kernels that write their small results straight to the host
// (fkv_snapkv_select's budgets in ops.compress_stack).
extern "C" int fkv_host_device_ptr(void* host_ptr, void** out_ptr) {
  using namespace fkv;
  if (!host_ptr || !out_ptr) return set_error(FKV_ERR_INVALID, "fkv_host_device_ptr: null pointer");
  return cuda_check(cudaHostGetDevicePointer(out_ptr, host_ptr, 0), "cudaHostGetDevicePointer");
}
