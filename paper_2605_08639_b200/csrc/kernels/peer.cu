// NVLink peer memory for the 8-GPU box: CUDA IPC allocations shared between the one-process-
// per-GPU ranks, copy-engine copies (K5 replica weight push) and a device-side flag barrier.
//
// The reference has no communication code: HardwareProfile.bw_nvlink / bw_rdma
// (topology.py:29-47) are flat modelled bandwidths.  On B200 every GPU pair is one NVSwitch
// hop, so receive buffers are plain cudaMalloc allocations exported with cudaIpcGetMemHandle
// and opened by every peer; kernels then load/store peer rows directly.
#include <cstring>
#include "capi_common.cuh"
#include "../../../include/mb_kernels.h"

namespace mb {

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// flags[p] points at rank p's flag array (world uint32 entries).  Barrier epoch = ++epoch[0].
// Each rank writes its epoch into slot `rank` of every peer's array (system-scope release),
// then waits until every slot of its own array reaches the epoch (system-scope acquire).
__global__ void peer_barrier_kernel(uint32_t* const* flags, int rank, int world, uint32_t* epoch, int64_t timeout_ns,
                                    int* error_flag) {
  if (threadIdx.x != 0) return;
  const uint32_t e = epoch[0] + 1;
  epoch[0] = e;
  __threadfence_system();
  for (int p = 0; p < world; ++p) {
    uint32_t* dst = flags[p] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(e) : "memory");
  }
  uint32_t* mine = flags[rank];
  const uint64_t t0 = globaltimer_ns();
  for (int q = 0; q < world; ++q) {
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + q) : "memory");
      if (static_cast<int32_t>(v - e) >= 0) break;
      if (globaltimer_ns() - t0 > static_cast<uint64_t>(timeout_ns)) {
        if (error_flag) atomicExch(error_flag, 1);
        __trap();
      }
      __nanosleep(64);
    }
  }
  __threadfence_system();
}

}  // namespace mb

using namespace mb;

extern "C" int mb_ipc_malloc(int64_t bytes, void** ptr, void* handle_out) {
  MB_CHECK_ARG(bytes > 0 && ptr && handle_out, "bad ipc_malloc args");
  void* p = nullptr;
  MB_CUDA_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
  MB_CUDA_TRY(cudaMemset(p, 0, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_error(MB_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  memcpy(handle_out, &h, sizeof(h));
  *ptr = p;
  return MB_OK;
}

extern "C" int mb_ipc_handle_size(void) { return static_cast<int>(sizeof(cudaIpcMemHandle_t)); }

extern "C" int mb_ipc_open(const void* handle, void** ptr) {
  MB_CHECK_ARG(handle && ptr, "bad ipc_open args");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  MB_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MB_OK;
}

extern "C" int mb_ipc_close(void* ptr) {
  MB_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return MB_OK;
}

extern "C" int mb_device_free(void* ptr) {
  MB_CUDA_TRY(cudaFree(ptr));
  return MB_OK;
}

extern "C" int mb_host_alloc_mapped(int64_t bytes, void** host, void** dev) {
  MB_CHECK_ARG(bytes > 0 && host && dev, "bad mapped host allocation args");
  MB_CUDA_TRY(cudaHostAlloc(host, static_cast<size_t>(bytes), cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(*host, 0, static_cast<size_t>(bytes));
  MB_CUDA_TRY(cudaHostGetDevicePointer(dev, *host, 0));
  return MB_OK;
}

extern "C" int mb_host_free(void* host) {
  if (host) MB_CUDA_TRY(cudaFreeHost(host));
  return MB_OK;
}

extern "C" int mb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  MB_CHECK_ARG(bytes >= 0, "negative copy size");
  if (bytes == 0) return MB_OK;
  MB_CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                              reinterpret_cast<cudaStream_t>(stream)));
  return MB_OK;
}

extern "C" int mb_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t world, uint32_t* epoch,
                               int64_t timeout_ns, int32_t* error_flag, void* stream) {
  MB_CHECK_ARG(flags && epoch && world >= 1 && rank >= 0 && rank < world, "bad barrier args");
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flags, rank, world, epoch, timeout_ns,
                                                                             error_flag);
  MB_CUDA_TRY(cudaGetLastError());
  return MB_OK;
}
