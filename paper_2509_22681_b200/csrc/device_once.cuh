// Host helper: one-time, per-device setup of kernel attributes.
//
// cudaFuncSetAttribute (e.g. MaxDynamicSharedMemorySize above 48 KB) applies to
// the current device's context only, so a process that drives several GPUs
// (one FlameCtx per device) must set it once per device, and two host threads
// launching for the first time must not race on the flag.
#pragma once
#include <cuda_runtime.h>
#include <mutex>

namespace flame {

constexpr int kMaxDevices = 64;

struct DeviceOnce {
  std::mutex m;
  unsigned long long done = 0;  // bit i: device i is set up

  // Runs f() once per current device; a failed f() is retried on the next call.
  template <class F>
  cudaError_t run(F&& f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(m);
    if ((done >> dev) & 1ull) return cudaSuccess;
    e = f(dev);
    if (e == cudaSuccess) done |= 1ull << dev;
    return e;
  }
};

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

}  // namespace flame
