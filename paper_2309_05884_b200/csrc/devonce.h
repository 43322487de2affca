// Per-device one-time setup (e.g. cudaFuncSetAttribute): function attributes belong to a
// device context, so a process driving several GPUs must set them once on EACH device.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

namespace sqoc {

// Runs fn() (returning cudaError_t) the first time it is reached on the current device for
// this call site's (mutex, mask) pair; thread-safe.  Failed setups are retried next time.
template <class Fn>
cudaError_t once_per_device(std::mutex& mu, uint64_t& done_mask, Fn&& fn) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done_mask >> dev & 1ull) return cudaSuccess;
  e = fn();
  if (e == cudaSuccess) done_mask |= 1ull << dev;
  return e;
}

}  // namespace sqoc
