// Peer-memory plumbing for the AutoPipe stage hand-off over NVLink.
//
// One process per GPU: a stage exports its receive buffers (the cut
// activation rows, the activation-gradient rows and a small flag array) as
// CUDA IPC handles; the neighbour stage maps them and its executor writes the
// cut activation straight into the peer's buffer from the producing kernel
// (GEMM / LayerNorm epilogue stores over NVLink), then bumps the peer's flag
// with a system-scope release store.  The consumer's stream waits on its
// local flag with cuStreamWaitValue32 (no SM spins), so the transfer is part
// of the producing kernel instead of a separate NCCL send / recv.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "eps_capi.h"
#include "../kernels/ptx.cuh"

namespace {

using GetAddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
using StreamWaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

GetAddressRangeFn address_range() {
  static GetAddressRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { fn = driver_fn<GetAddressRangeFn>("cuMemGetAddressRange"); });
  return fn;
}

StreamWaitValue32Fn stream_wait() {
  static StreamWaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] { fn = driver_fn<StreamWaitValue32Fn>("cuStreamWaitValue32"); });
  return fn;
}

__global__ void signal_kernel(uint32_t* flag, uint32_t value) {
  // every store the stream issued before this kernel (the producer's epilogue
  // writes into the peer buffer) is ordered before the flag at system scope
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

}  // namespace

extern "C" {

int eps_ipc_export(const void* dev_ptr, void* handle, int64_t* offset) {
  GetAddressRangeFn range = address_range();
  if (dev_ptr == nullptr || handle == nullptr || offset == nullptr || range == nullptr)
    return EPS_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return EPS_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return EPS_ECUDA;
  std::memcpy(handle, &h, sizeof(h));
  *offset = int64_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return EPS_OK;
}

int eps_ipc_open(const void* handle, int64_t offset, void** base, void** dev_ptr) {
  if (handle == nullptr || base == nullptr || dev_ptr == nullptr) return EPS_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* b = nullptr;
  if (cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return EPS_ECUDA;
  *base = b;
  *dev_ptr = static_cast<char*>(b) + offset;
  return EPS_OK;
}

int eps_ipc_close(void* base) {
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

int eps_peer_signal(void* flag, uint32_t value, void* stream) {
  if (flag == nullptr) return EPS_EINVAL;
  eps_k::count_launch();
  signal_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint32_t*>(flag),
                                                                  value);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

int eps_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (dst == nullptr || src == nullptr || bytes < 0) return EPS_EINVAL;
  return cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDeviceToDevice,
                         static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? EPS_OK
             : EPS_ECUDA;
}

// Stream-ordered 2D copy between any two UVA addresses (host <-> device):
// `height` rows of `width` bytes, row pitches dpitch / spitch.  The AutoCache
// disk tier moves a batch from its padded host window rows into HBM staging
// with one call.
int eps_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                     int64_t height, void* stream) {
  if (dst == nullptr || src == nullptr || width < 0 || height < 0 || dpitch < width ||
      spitch < width)
    return EPS_EINVAL;
  if (width == 0 || height == 0) return EPS_OK;
  return cudaMemcpy2DAsync(dst, size_t(dpitch), src, size_t(spitch), size_t(width),
                           size_t(height), cudaMemcpyDefault,
                           static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? EPS_OK
             : EPS_ECUDA;
}

// Page-lock an existing host range (e.g. a node-wide shared-memory AutoCache
// host tier that every rank of the node maps) so the gather / scatter
// kernels can address it over the host link (UVA).
int eps_host_register(void* ptr, int64_t bytes) {
  if (ptr == nullptr || bytes <= 0) return EPS_EINVAL;
  return cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterPortable | cudaHostRegisterMapped) ==
                 cudaSuccess
             ? EPS_OK
             : EPS_ECUDA;
}

int eps_host_unregister(void* ptr) {
  if (ptr == nullptr) return EPS_EINVAL;
  return cudaHostUnregister(ptr) == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

int eps_peer_wait(const void* flag, uint32_t value, void* stream) {
  StreamWaitValue32Fn wait = stream_wait();
  if (flag == nullptr || wait == nullptr) return EPS_EINVAL;
  return wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
              CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
             ? EPS_OK
             : EPS_ECUDA;
}

}  // extern "C"
