#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
// which pipe do FMNMX / IMNMX / HMNMX2 use: run each in a dependent-free loop and read ncu pipe counters
template <int MODE>
__global__ void k(const float* in, float* out, int iters) {
  float a[8]; uint32_t u[8];
  for (int i = 0; i < 8; i++) { a[i] = in[threadIdx.x + i]; u[i] = __float_as_uint(a[i]); }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) a[i] = fminf(a[i], a[(i + 3) & 7]);
      if (MODE == 1) u[i] = min(u[i], u[(i + 3) & 7] + 1u);
      if (MODE == 2) { __half2 x = *reinterpret_cast<__half2*>(&u[i]); __half2 y = *reinterpret_cast<__half2*>(&u[(i+3)&7]); x = __hmin2(x, y); u[i] = *reinterpret_cast<uint32_t*>(&x); }
      if (MODE == 3) asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(u[i]) : "r"(u[(i+1)&7]), "r"(u[(i + 3) & 7]));
    }
  }
  float s = 0; for (int i = 0; i < 8; i++) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
#include <cuda_fp16.h>
int main() {
  float *din, *dout; cudaMalloc(&din, 4096*4); cudaMemset(din, 0, 4096*4); cudaMalloc(&dout, 148*8*256*4);
  k<0><<<148*8, 256>>>(din, dout, 1000); k<1><<<148*8, 256>>>(din, dout, 1000);
  k<2><<<148*8, 256>>>(din, dout, 1000); k<3><<<148*8, 256>>>(din, dout, 1000);
  cudaDeviceSynchronize(); printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
