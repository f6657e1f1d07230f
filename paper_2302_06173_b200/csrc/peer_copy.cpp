// Copy-engine transfers between GPUs of one node, ordered by stream memory
// operations instead of kernels: the parallel-recovery merge moves
// its gradient shards with cudaMemcpyAsync into CUDA-IPC-mapped peer buffers
// (the DMA engines carry them over NVLink, no SM is taken from the replay
// GEMMs) and signals completion by writing an epoch counter into the peer's
// memory from the same stream (cuStreamWriteValue64: ordered after the copies
// by its default memory barrier); the peer's stream blocks on that counter
// with cuStreamWaitValue64 (a front-end wait, again no kernel).
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "internal.h"

namespace {
int pfail(int code, const std::string& msg) {
  rwb::set_error(msg.c_str());
  return code;
}

using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
}  // namespace

extern "C" {

int rw_copy_async(void* const* dsts, const void* const* srcs, const uint64_t* bytes, uint32_t n, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of((n && srcs) ? srcs[0] : nullptr));
  if (n && (!dsts || !srcs || !bytes)) return pfail(RW_INVALID_ARGUMENT, "null argument");
  auto cs = static_cast<cudaStream_t>(stream);
  for (uint32_t i = 0; i < n; ++i) {
    if (!bytes[i]) continue;
    cudaError_t e = cudaMemcpyAsync(dsts[i], srcs[i], bytes[i], cudaMemcpyDeviceToDevice, cs);
    if (e != cudaSuccess) return pfail(RW_CUDA_ERROR, std::string("peer copy: ") + cudaGetErrorString(e));
  }
  return RW_OK;
}

int rw_stream_write_u64(void* stream, void* addr, uint64_t value) {
  static WriteFn fn = entry<WriteFn>("cuStreamWriteValue64");
  if (!fn) return pfail(RW_CUDA_ERROR, "cuStreamWriteValue64 unavailable");
  if (!addr) return pfail(RW_INVALID_ARGUMENT, "null address");
  // flags 0 = CU_STREAM_WRITE_VALUE_DEFAULT: memory barrier before the write
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value, 0);
  return r == CUDA_SUCCESS ? RW_OK : pfail(RW_CUDA_ERROR, "cuStreamWriteValue64 failed");
}

int rw_stream_wait_u64(void* stream, const void* addr, uint64_t value) {
  static WaitFn fn = entry<WaitFn>("cuStreamWaitValue64");
  if (!fn) return pfail(RW_CUDA_ERROR, "cuStreamWaitValue64 unavailable");
  if (!addr) return pfail(RW_INVALID_ARGUMENT, "null address");
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(const_cast<void*>(addr)), value,
                  CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? RW_OK : pfail(RW_CUDA_ERROR, "cuStreamWaitValue64 failed");
}

}  // extern "C"
