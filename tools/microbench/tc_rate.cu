// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion rate on sm_100a.
// One CTA per SM, one thread issues back-to-back M=128 x N x K=16 MMAs (bf16
// in, fp32 accumulate) from shared memory (SS) or with A in TMEM (TS), in the
// pattern of the stride-1 conv kernel (K3d): groups of 4 k-steps x `prod`
// products, a commit per group, the accumulator toggled every `grp` groups.
// Reports cycles per MMA (clock64 on the issuing thread, completion included)
// and TFLOP/s over the grid (CUDA events).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_rate.cu -o tc_rate
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
__host__ __device__ constexpr uint32_t make_idesc(int n, int m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

struct Cfg {
  int n, ts, prod, grp, total_groups, accs, warp_issue;
};

// Issue from a whole converged warp: warp-uniform operands stay in uniform
// registers and one lane is elected inside the instruction sequence.
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) kbench(const uint4* __restrict__ init, Cfg c, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  uint8_t* sbase = smem + (base - smem_u32(smem));
  // 96 KB of operand data (A planes 32 KB, B planes up to 64 KB), random bits
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sbase)[i] = init[i];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (c.warp_issue && threadIdx.x < 32) {
    // whole warp, descriptors advanced by adds (+2 per 32 bytes), 3 products
    // per k-step unrolled as in the conv kernel
    const uint32_t idesc = make_idesc(c.n, 128);
    const uint64_t ad = sw128_desc(base), bd = sw128_desc(base + 32 * 1024);
    const uint32_t acc_cols = c.accs == 2 ? 192u : 0u;
    const uint32_t ta = tmem + 384;
    const long long t0 = clock64();
    int acc = 0;
    for (int g = 0; g < c.total_groups; ++g) {
      const uint32_t d = tmem + acc * acc_cols;
      const uint32_t first = (g % c.grp) > 0 ? 1u : 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (c.ts) {
          mma_ts_elect(d, ta + 8 * k, bd + 2 * k, idesc, (first | k) ? 1u : 0u);
          mma_ts_elect(d, ta + 8 * k, bd + 1536 + 2 * k, idesc, 1u);
          mma_ts_elect(d, ta + 32 + 8 * k, bd + 2 * k, idesc, 1u);
        } else {
          mma_ss_elect(d, ad + 2 * k, bd + 2 * k, idesc, (first | k) ? 1u : 0u);
          mma_ss_elect(d, ad + 2 * k, bd + 1536 + 2 * k, idesc, 1u);
          mma_ss_elect(d, ad + 1024 + 2 * k, bd + 2 * k, idesc, 1u);
        }
      }
      if ((g + 1) % c.grp == 0 && c.accs == 2) acc ^= 1;
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
      asm volatile(
          "{\n\t.reg .pred P1;\n\tW2:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
          "@!P1 bra W2;\n\t}" ::"r"(smem_u32(&bar))
          : "memory");
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (!c.warp_issue && threadIdx.x == 0) {
    const uint32_t idesc = make_idesc(c.n, 128);
    const uint32_t a0 = base, b0 = base + 32 * 1024;
    const uint32_t acc_cols = c.accs == 2 ? 192u : 0u;
    const uint32_t ta = tmem + 384;  // A in TMEM (garbage values: rate only)
    const long long t0 = clock64();
    int acc = 0;
    for (int g = 0; g < c.total_groups; ++g) {
      const uint32_t d = tmem + acc * acc_cols;
      for (int k = 0; k < 4; ++k) {
        for (int pr = 0; pr < c.prod; ++pr) {
          const uint32_t accum = (g % c.grp) > 0 || k > 0 || pr > 0;
          const uint64_t bdesc = sw128_desc(b0 + (pr & 1) * 24 * 1024 + 32 * k);
          if (c.ts) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                "r"(ta + 32 * (pr >> 1) + 8 * k), "l"(bdesc), "r"(idesc), "r"(accum)
                : "memory");
          } else {
            const uint64_t adesc = sw128_desc(a0 + (pr >> 1) * 16 * 1024 + 32 * k);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
                : "memory");
          }
        }
      }
      if ((g + 1) % c.grp == 0 && c.accs == 2) acc ^= 1;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 97 * 1024 + 1024;
  cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<uint32_t> h(96 * 1024 / 4);
  uint64_t x = 12345;
  for (auto& v : h) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    const uint32_t r = static_cast<uint32_t>(x >> 32);
    v = (r & 0x3fff3fffu) | 0x3c003c00u;  // bf16 pairs in ~[1, 2): non-trivial switching
  }
  uint4* dinit;
  long long* dcyc;
  cudaMalloc(&dinit, h.size() * 4);
  cudaMemcpy(dinit, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dcyc, sms * sizeof(long long));
  const int ns[] = {64, 128, 192, 256};
  printf("{\"rows\": [\n");
  bool first = true;
  for (int wi = 0; wi < 2; ++wi)
  for (int ts = 0; ts < 2; ++ts)
    for (int prod : {1, 3})
      for (int n : ns) {
        if (wi && prod != 3) continue;
        Cfg c{n, ts, prod, 3, 3 * 400, 2, wi};
        if (n > 192) c.accs = 1;  // two 256-column accumulators would leave no room for A
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        kbench<<<sms, 128, smem>>>(dinit, c, dcyc);
        cudaEventRecord(e0);
        kbench<<<sms, 128, smem>>>(dinit, c, dcyc);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(err));
          return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> cyc(sms);
        cudaMemcpy(cyc.data(), dcyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (long long v : cyc) avg += v;
        avg /= sms;
        const double mmas = double(c.total_groups) * 4 * prod;
        const double flop = 2.0 * 128 * n * 16 * mmas * sms;
        printf("%s  {\"issue\": \"%s\", \"a\": \"%s\", \"n\": %d, \"products\": %d, \"cyc_per_mma\": %.1f, \"floor_cyc\": %.1f, "
               "\"tflops\": %.1f, \"clk_mhz\": %.0f}",
               first ? "" : ",\n", wi ? "warp+elect" : "lane0", ts ? "tmem" : "smem", n, prod, avg / mmas, 128.0 * n / 256, flop / (ms * 1e-3) / 1e12,
               avg / (ms * 1e-3) / 1e6);
        first = false;
      }
  printf("\n]}\n");
  return 0;
}
