// K1 — window max (the max-pool StrategyProgram, workloads.hpp:376-385:
// Pre_1 MOVC r <- init, Body MAX r <- max(r, A), Post_1 ADD emit <- r + 0)
// over a strided, offset, clamped 2-D window view (view.hpp:68-84).
//
// Semantics are the reference engine's bit for bit: r starts at the MOVC
// constant, every window element v is folded as r = (r < v) ? v : r
// (std::max, rip.hpp:175-176) in row-major (ky, kx) order, and the result is
// emitted as r + 0.0f (rip.hpp:167-168).  CLAMP clamps each coordinate
// (equivalent to -inf padding for max); ZERO_PAD reads 0 outside.
//
// Roofline: HBM.  Algorithmic bytes = input plane bytes + output bytes.
#include "common.cuh"

namespace merit_dev {
namespace {

__device__ __forceinline__ float fold_max(float r, float v) { return (r < v) ? v : r; }

__device__ __forceinline__ float post_op(float r, int post) {
  if (post == POST_RELU) return (r < 0.f) ? 0.f : r;
  return __fadd_rn(r, 0.f);
}

// General path: one thread per output element.
__global__ void maxpool_generic_kernel(const float* __restrict__ in, float* __restrict__ out,
                                       MaxpoolParams p) {
  const long long total = p.planes * (long long)p.Ho * p.Wo;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const int x = static_cast<int>(o % p.Wo);
    const long long t = o / p.Wo;
    const int y = static_cast<int>(t % p.Ho);
    const long long plane = t / p.Ho;
    const float* src = in + plane * (long long)p.H * p.W;
    float r = p.init;
    for (int ky = 0; ky < p.KH; ++ky) {
      int iy = y * p.sy + ky * p.dy + p.oy;
      bool rin = iy >= 0 && iy < p.H;
      if (!rin && p.boundary == MERIT_CLAMP) { iy = iy < 0 ? 0 : p.H - 1; rin = true; }
      for (int kx = 0; kx < p.KW; ++kx) {
        int ix = x * p.sx + kx * p.dx + p.ox;
        bool cin = ix >= 0 && ix < p.W;
        if (!cin && p.boundary == MERIT_CLAMP) { ix = ix < 0 ? 0 : p.W - 1; cin = true; }
        const float v = (rin && cin) ? __ldg(src + (long long)iy * p.W + ix) : 0.f;
        r = fold_max(r, v);
      }
    }
    out[o] = post_op(r, p.post);
  }
}

// Fast path for 3x3 / stride 2 / offset -1 / CLAMP with Ho = H/2, Wo = W/2,
// W % 4 == 0.  A warp owns one plane, RB output rows and a 128-column input
// segment: lane l holds input columns 4l..4l+3 of every input row it needs as
// one 128-bit load (all 2*RB+1 rows issued before any use), takes column 4l-1
// from lane l-1 with a shuffle, and writes output columns 2l, 2l+1 as one
// 64-bit store.  Every input row is read once per band (one shared row per
// band boundary).
template <int RB>
__global__ void __launch_bounds__(256, 3) maxpool3s2_kernel(const float* __restrict__ in,
                                                         float* __restrict__ out, MaxpoolParams p,
                                                         int nseg, int nband) {
  const long long wg = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int seg = static_cast<int>(wg % nseg);
  const long long t = wg / nseg;
  const int band = static_cast<int>(t % nband);
  const long long plane = t / nband;
  if (plane >= p.planes) return;
  const int H = p.H, W = p.W, Ho = p.Ho, Wo = p.Wo;
  const float* src = in + plane * (long long)H * W;
  const int col0 = seg * 128 + lane * 4;
  const bool active = col0 < W;
  const int y0 = band * RB;
  float4 v[2 * RB + 1];
  float left[2 * RB + 1];
#pragma unroll
  for (int r = 0; r < 2 * RB + 1; ++r) {
    int iy = 2 * y0 - 1 + r;
    iy = iy < 0 ? 0 : (iy > H - 1 ? H - 1 : iy);
    v[r] = active ? __ldg(reinterpret_cast<const float4*>(src + (long long)iy * W + col0))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // Column col0-1: lane 0 of a segment > 0 loads it; column -1 clamps to 0.
#pragma unroll
  for (int r = 0; r < 2 * RB + 1; ++r) {
    float w = __shfl_up_sync(0xffffffffu, v[r].w, 1);
    if (lane == 0) {
      if (col0 == 0) {
        w = v[r].x;
      } else if (active) {
        int iy = 2 * y0 - 1 + r;
        iy = iy < 0 ? 0 : (iy > H - 1 ? H - 1 : iy);
        w = __ldg(src + (long long)iy * W + col0 - 1);
      }
    }
    left[r] = w;
  }
  if (!active) return;
  float* dst = out + plane * (long long)Ho * Wo + col0 / 2;
#pragma unroll
  for (int yy = 0; yy < RB; ++yy) {
    const int y = y0 + yy;
    if (y >= Ho) break;
    float r0 = p.init, r1 = p.init;
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      const float4 q = v[2 * yy + ky];
      const float l = left[2 * yy + ky];
      r0 = fold_max(r0, l);
      r0 = fold_max(r0, q.x);
      r0 = fold_max(r0, q.y);
      r1 = fold_max(r1, q.y);
      r1 = fold_max(r1, q.z);
      r1 = fold_max(r1, q.w);
    }
    float2 o = make_float2(post_op(r0, p.post), post_op(r1, p.post));
    *reinterpret_cast<float2*>(dst + (long long)y * Wo) = o;
  }
}

}  // namespace

merit_status launch_maxpool(const merit_plan& plan, const void* a, void* out, void* stream) {
  const MaxpoolParams& p = plan.mp;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float* in = static_cast<const float*>(a);
  float* o = static_cast<float*>(out);
  const long long total = p.planes * (long long)p.Ho * p.Wo;
  if (total == 0) return MERIT_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(out) % 8 == 0);
  if (p.fast && aligned) {
    constexpr int RB = 4;
    const int nseg = (p.W + 127) / 128;
    const int nband = (p.Ho + RB - 1) / RB;
    const long long warps = p.planes * nband * nseg;
    const long long threads = warps * 32;
    const long long blocks = (threads + 255) / 256;
    maxpool3s2_kernel<RB><<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, o, p, nseg, nband);
    return launch_status("maxpool3s2_kernel");
  }
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  const long long cap = (long long)num_sms() * 32;
  if (blocks > cap) blocks = cap;
  maxpool_generic_kernel<<<static_cast<unsigned>(blocks), threads, 0, s>>>(in, o, p);
  return launch_status("maxpool_generic_kernel");
}

}  // namespace merit_dev
