// CUDA stream memory write (cuStreamWriteValue32), bound through the
// runtime's driver entry-point query so libwavepipe.so keeps linking only the
// static CUDA runtime.
//
// The IPC transport's device-side signals: a 32-bit flag written by one
// GPU's stream (after a copy-engine transfer, no host round trip).  The
// waiting side is a bounded wait kernel (wpk::wait_flag), not
// cuStreamWaitValue32: a memory-op wait on a peer that never signals cannot
// be released, a wait kernel can (see the stall watchdog).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>

namespace wprt {

struct StreamOps {
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;

  static const StreamOps& get() {
    static StreamOps ops;
    static std::once_flag once;
    static std::string error;
    std::call_once(once, [] {
      auto bind = [&](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q{};
        const cudaError_t e = cudaGetDriverEntryPointByVersion(name, fn, 12000, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn) {
          error = std::string("driver entry point ") + name + " unavailable";
        }
      };
      bind("cuStreamWriteValue32", reinterpret_cast<void**>(&ops.write32));
    });
    if (!error.empty()) throw std::runtime_error(error);
    return ops;
  }

  // Stream writes *flag = value once all earlier work of the stream is done;
  // the default flags include a memory barrier, so the earlier transfer's
  // bytes are visible to whoever observes the flag.
  static void write(cudaStream_t s, uint32_t* flag, uint32_t value) {
    const CUresult r =
        get().write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value, 0);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuStreamWriteValue32 failed: " + std::to_string(r));
  }
};

}  // namespace wprt
