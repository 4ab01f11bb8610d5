// Small device helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "plan.hpp"

namespace merit_dev {

inline merit_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_check(e, what);
  count_launch();
  return MERIT_OK;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel,
// size): keeps the per-launch host path short for microsecond-scale kernels.
cudaError_t set_smem_attr_impl(const void* fn, cudaFuncAttribute attr, int bytes);
template <typename K>
inline cudaError_t set_smem_attr(K kernel, cudaFuncAttribute attr, int bytes) {
  return set_smem_attr_impl(reinterpret_cast<const void*>(kernel), attr, bytes);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace merit_dev
