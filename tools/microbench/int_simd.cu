// Microbenchmark: byte-SIMD abs-diff-accumulate issue rate on sm_100a.
// Measures VABSDIFF4.U8.ACC (PTX vabsdiff4.u32.u32.u32.add), PRMT and IMAD
// throughput with CUDA events so the SAD kernel's INT roofline is measured,
// not assumed.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 int_simd.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) kbench(const uint32_t* __restrict__ in, uint32_t* out, int iters) {
  uint32_t a[8], b[8], acc[8];
  for (int i = 0; i < 8; i++) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 8 + i]; acc[i] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
#pragma unroll
      for (int i = 0; i < 8; i++) {
        if (MODE == 0) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[(i + r) & 7]));
        } else if (MODE == 1) {
          asm volatile("prmt.b32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[(i + r) & 7]));
        } else if (MODE == 2) {
          asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[(i + r) & 7]));
        } else {
          // half VABSDIFF4.ACC, half IMAD: do two pipes co-issue?
          if (i & 1) asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[(i + r) & 7]));
          else asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i]) : "r"(a[i]), "r"(b[(i + r) & 7]));
        }
      }
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(uint32_t* din, uint32_t* dout, int blocks, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kbench<MODE><<<blocks, 256>>>(din, dout, iters);
  cudaEventRecord(e0);
  kbench<MODE><<<blocks, 256>>>(din, dout, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double instr = double(blocks) * 256 * iters * 16 * 8;
  return instr / (ms * 1e-3);  // thread-instructions per second
}

template <int MODE>
double run_occ(uint32_t* din, uint32_t* dout, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kbench<MODE><<<blocks, threads>>>(din, dout, iters);
  cudaEventRecord(e0);
  kbench<MODE><<<blocks, threads>>>(din, dout, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return double(blocks) * threads * iters * 16 * 8 / (ms * 1e-3);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // occupancy sweep: warps per SM -> VABSDIFF4 instr/s
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    uint32_t *din, *dout; cudaMalloc(&din, 4096 * 4); cudaMemset(din, 0x5a, 4096 * 4);
    cudaMalloc(&dout, 148 * 64 * 32 * 4 * 8);
    for (int wps : {4, 8, 12, 16, 24, 32, 64}) {
      const int threads = wps >= 8 ? 256 : wps * 32;
      const int bps = wps * 32 / threads;
      double v = run_occ<0>(din, dout, p.multiProcessorCount * bps, threads, 1000);
      printf("{\"warps_per_sm\": %d, \"vabsdiff4_instr_per_s\": %.4e, \"frac_of_64_lanes\": %.3f}\n", wps, v,
             v / (p.multiProcessorCount * 1.965e9 * 64));
    }
    return 0;
  }
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t *din, *dout; cudaMalloc(&din, 4096 * 4); cudaMemset(din, 0x5a, 4096 * 4);
  int blocks = p.multiProcessorCount * 8; cudaMalloc(&dout, blocks * 256 * 4);
  int iters = 2000;
  double v = run<0>(din, dout, blocks, iters);
  double pr = run<1>(din, dout, blocks, iters);
  double im = run<2>(din, dout, blocks, iters);
  double mx = run<3>(din, dout, blocks, iters);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"vabsdiff4_acc_instr_per_s\": %.4e, \"vabsdiff4_absdiff_ops_per_s\": %.4e, "
         "\"prmt_instr_per_s\": %.4e, \"imad_instr_per_s\": %.4e, \"mixed_vabs_imad_instr_per_s\": %.4e, "
         "\"vabsdiff4_lanes_per_clk_per_sm_at_max_clock\": %.2f}\n",
         p.multiProcessorCount, clk, v, 4 * v, pr, im, mx, v / (p.multiProcessorCount * (clk * 1e3)));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
