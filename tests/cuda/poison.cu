// Test helper (not part of the product library): fill the shared memory of
// every SM with a bit pattern, so that a kernel launched next that reads
// shared memory it has not written (or whose asynchronous copy has not landed
// yet) computes with that pattern instead of with its own bytes from an
// earlier launch.  tests/test_gpu_determinism.py runs it before every launch
// with 0xFFFFFFFF (a NaN as fp32 / bf16 pair, 255 as pixels).
#include <cuda_runtime.h>

#include <cstdint>

__global__ void poison_kernel(uint32_t pattern, uint32_t words, uint32_t* sink) {
  extern __shared__ uint32_t sm[];
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sm[i] = pattern;
  __syncthreads();
  // keep the stores: read one word back (never true for the patterns used)
  if (sm[(threadIdx.x * 97u) % words] == 0x12345678u && sink) *sink = 1u;
}

extern "C" int poison_shared_memory(uint32_t pattern, void* stream) {
  int dev = 0, sms = 0, max_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaError_t e = cudaFuncSetAttribute(poison_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
  if (e != cudaSuccess) return static_cast<int>(e);
  // one CTA of the maximum size fits per SM: 2 x SMs CTAs cover every SM
  poison_kernel<<<2 * sms, 1024, max_smem, static_cast<cudaStream_t>(stream)>>>(
      pattern, static_cast<uint32_t>(max_smem / 4), nullptr);
  return static_cast<int>(cudaGetLastError());
}
