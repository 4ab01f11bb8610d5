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
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "tmap.cuh"

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

template <int RB>
__device__ __forceinline__ void maxpool3s2_item(const float* __restrict__ in, float* __restrict__ out,
                                                const MaxpoolParams& p, int nseg, int nband,
                                                long long wg);

// Fast path for 3x3 / stride 2 / offset -1 / CLAMP with Ho = H/2, Wo = W/2,
// W % 4 == 0.  A warp owns one plane, RB output rows and a 128-column input
// segment: lane l holds input columns 4l..4l+3 of every input row it needs as
// one 128-bit load (all 2*RB+1 rows issued before any use), takes column 4l-1
// from lane l-1 with a shuffle, and writes output columns 2l, 2l+1 as one
// 64-bit store.  Every input row is read once per band (one shared row per
// band boundary).
template <int RB>
__global__ void __launch_bounds__(128, 6) maxpool3s2_kernel(const float* __restrict__ in,
                                                         float* __restrict__ out, MaxpoolParams p,
                                                         int nseg, int nband, long long n_items,
                                                         int per_warp) {
  // Each warp owns `per_warp` consecutive (plane, band, segment) items; the
  // grid is sized so that every warp is resident at once and all warps carry
  // the same number of items (no partial second wave).
  const long long w0 = ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5) * per_warp;
  for (long long wg = w0; wg < w0 + per_warp && wg < n_items; ++wg)
    maxpool3s2_item<RB>(in, out, p, nseg, nband, wg);
}

template <int RB>
__device__ __forceinline__ void maxpool3s2_item(const float* __restrict__ in, float* __restrict__ out,
                                                const MaxpoolParams& p, int nseg, int nband,
                                                long long wg) {
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


// Streaming path for the same shape: a band's input rows are contiguous in
// memory, so one cp.async.bulk (TMA engine) per band moves them into a
// shared-memory ring NS bands deep; warps compute from shared memory.  Bytes
// in flight no longer cost registers, so HBM stays busy.
constexpr int kMpMaxStages = 16;

__device__ __forceinline__ void mp_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mp_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int NT, int RB, bool TM>
__global__ void __launch_bounds__(NT) maxpool3s2_bulk_kernel(const float* __restrict__ in,
                                                             float* __restrict__ out, MaxpoolParams p,
                                                             int nband, int n_items, int ns,
                                                             const __grid_constant__ CUtensorMap rows_map) {
  extern __shared__ __align__(128) float sbuf[];
  const int H = p.H, W = p.W, Ho = p.Ho, Wo = p.Wo;
  const int rows_max = 2 * RB + 1;
  const int stage_floats = ((rows_max * W * 4 + 127) / 128) * 32;  // 128-B aligned stages (TMA)
  __shared__ __align__(8) unsigned long long bars[kMpMaxStages];
  const uint32_t bar0 = smem_u32(&bars[0]);
  const uint32_t buf0 = smem_u32(sbuf);
  // item -> (plane, band) with one 32-bit divide (64-bit div/mod is a long
  // emulated sequence: it dominated the per-item cost)
  auto rows_of = [&](int item, int& plane, int& r0, int& nr) {
    plane = item / nband;
    const int band = item - plane * nband;
    const int y0 = band * RB;
    const int lo = max(0, 2 * y0 - 1);
    const int hi = min(H - 1, 2 * (y0 + RB) - 1);
    r0 = lo;
    nr = hi - lo + 1;
  };
  auto issue = [&](int item, int st) {
    int plane, r0, nr;
    rows_of(item, plane, r0, nr);
    const uint32_t bar = bar0 + 8u * st;
    if (p.dbg & 2) {  // timing experiment: no loads
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
      return;
    }
    if (TM) {
      // one tensor-map box of 2 RB + 1 rows of the [planes * H][W] matrix
      // (rows past the last plane are zero-filled and never read)
      const uint32_t bytes = static_cast<uint32_t>(2 * RB + 1) * W * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(buf0 + 4u * st * stage_floats),
          "l"(reinterpret_cast<uint64_t>(&rows_map)), "r"(0), "r"(plane * H + r0), "r"(bar)
          : "memory");
    } else {
      const float* src = in + ((long long)plane * H + r0) * W;
      const uint32_t bytes = static_cast<uint32_t>(nr) * W * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(buf0 + 4u * st * stage_floats), "l"(src), "r"(bytes), "r"(bar) : "memory");
    }
  };
  const int first = blockIdx.x;
  const int step = gridDim.x;
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) mp_mbar_init(bar0 + 8u * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // warm L2 with this CTA's first p.pf bands while the previous launch drains
  // (when the CTAs of consecutive launches fit on an SM together, the whole
  // input of launch i+1 streams into L2 under launch i's tail)
  if (threadIdx.x < 32 && !(p.dbg & 4)) {
    for (int i = threadIdx.x; i < p.pf; i += 32) {
      const int item = first + i * step;
      if (item >= n_items) break;
      int plane, r0, nr;
      rows_of(item, plane, r0, nr);
      prefetch_l2(in + ((long long)plane * H + r0) * W, static_cast<uint32_t>(nr) * W * 4u);
    }
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0)
    for (int i = 0; i < ns; ++i)
      if (first + i * step < n_items) issue(first + i * step, i);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int it = 0;
  int st = 0;
  uint32_t parity = 0;
  for (int item = first; item < n_items; item += step, ++it) {
    mp_mbar_wait(bar0 + 8u * st, parity);
    int plane, r0, nr;
    rows_of(item, plane, r0, nr);
    const int y0 = (item - plane * nband) * RB;
    float* orow = out + (long long)plane * Ho * Wo;
    const float* sb = sbuf + st * stage_floats;
    if (p.vec_out) {
      // The band's output rows are contiguous (RB * Wo floats): thread t
      // writes outputs 4t .. 4t+3 of the band with one 16-byte store, so a
      // warp store covers whole 128-byte lines (a partial-line store per
      // row measured ~2x slower for the output stream).
      const int q = Wo / 4;  // 16-byte groups per output row
      const int rows = min(RB, Ho - y0);
      for (int t = threadIdx.x; t < rows * q; t += NT) {
        const int yy = t / q;
        const int x0 = (t - yy * q) * 4;  // first output column
        const int y = y0 + yy;
        const int c0 = 2 * x0;            // input columns c0 - 1 .. c0 + 7
        float r[4] = {p.init, p.init, p.init, p.init};
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
          int iy = 2 * y - 1 + ky;
          iy = iy < 0 ? 0 : (iy > H - 1 ? H - 1 : iy);
          const float* row = sb + (iy - r0) * W;
          const float4 a4 = *reinterpret_cast<const float4*>(row + c0);
          const float4 b4 = *reinterpret_cast<const float4*>(row + c0 + 4);
          const float l = c0 == 0 ? a4.x : row[c0 - 1];
          r[0] = fold_max(fold_max(fold_max(r[0], l), a4.x), a4.y);
          r[1] = fold_max(fold_max(fold_max(r[1], a4.y), a4.z), a4.w);
          r[2] = fold_max(fold_max(fold_max(r[2], a4.w), b4.x), b4.y);
          r[3] = fold_max(fold_max(fold_max(r[3], b4.y), b4.z), b4.w);
        }
        if (!(p.dbg & 1))
          *reinterpret_cast<float4*>(orow + y * Wo + x0) =
              make_float4(post_op(r[0], p.post), post_op(r[1], p.post), post_op(r[2], p.post), post_op(r[3], p.post));
      }
    } else {
      // warp w computes output rows y0 + w, y0 + w + NT/32, ...
      for (int yy = warp; yy < RB; yy += NT / 32) {
        const int y = y0 + yy;
        if (y >= Ho) break;
        for (int c4 = lane; c4 * 4 < W; c4 += 32) {
          const int col0 = c4 * 4;
          float r0v = p.init, r1v = p.init;
#pragma unroll
          for (int ky = 0; ky < 3; ++ky) {
            int iy = 2 * y - 1 + ky;
            iy = iy < 0 ? 0 : (iy > H - 1 ? H - 1 : iy);
            const float* row = sb + (iy - r0) * W;
            const float4 qv = *reinterpret_cast<const float4*>(row + col0);
            const float l = col0 == 0 ? qv.x : row[col0 - 1];
            r0v = fold_max(r0v, l);
            r0v = fold_max(r0v, qv.x);
            r0v = fold_max(r0v, qv.y);
            r1v = fold_max(r1v, qv.y);
            r1v = fold_max(r1v, qv.z);
            r1v = fold_max(r1v, qv.w);
          }
          if (!(p.dbg & 1))
            *reinterpret_cast<float2*>(orow + y * Wo + col0 / 2) =
                make_float2(post_op(r0v, p.post), post_op(r1v, p.post));
        }
      }
    }
    __syncthreads();  // everyone is done with stage st: refill it
    if (threadIdx.x == 0 && item + ns * step < n_items) issue(item + ns * step, st);
    if (++st == ns) { st = 0; parity ^= 1; }
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
  if (p.fast && aligned && p.W % 4 == 0) {
    // bands of RB output rows (2 RB + 1 input rows, one bulk copy each);
    // 7 four-warp CTAs per SM with a 4..8-band ring keep ~200 KB of copies in
    // flight per SM, which is what the HBM stream needs at this size
    int RBv = 8;
    {
      // Single-band CTAs when the launch is small: bands of 28 output rows
      // (57 input rows, one TMA box each), one load in flight per CTA, used
      // when the bands would fit 7 resident CTAs per SM (C1: 1,024 bands;
      // measured 6.67 us with the 8-warp, 6-per-SM launch below vs 7.41 us
      // for 8-row bands through a 4-deep ring)
      const size_t st28 = ((size_t)57 * p.W * 4 + 127) / 128 * 128;
      const long long fit = st28 <= 200 * 1024 ? std::min<long long>(7, (227 * 1024) / (st28 + 1024)) : 0;
      const long long items28 = p.planes * ((p.Ho + 27) / 28);
      if (p.Ho >= 28 && fit > 0 && items28 <= num_sms() * fit) RBv = 28;
      // smaller launches still: 14-row bands (29 input rows, 13 KB), one per
      // 4-warp CTA, 12 resident per SM (C1: 2,048 bands, 6.47-6.65 us vs
      // 6.72 us for the 28-row shape on the same box)
      const size_t st14 = ((size_t)29 * p.W * 4 + 127) / 128 * 128;
      const long long items14 = p.planes * ((p.Ho + 13) / 14);
      if (p.Ho >= 14 && st14 <= 16 * 1024 && items14 <= num_sms() * 14LL) RBv = 14;
    }
    if (const char* re = getenv("MERIT_MP_RB")) {
      const int v = atoi(re);
      RBv = (v == 4 || v == 14 || v == 16 || v == 28 || v == 56) ? v : 8;
    }
    const int nband = (p.Ho + RBv - 1) / RBv;
    const long long items = p.planes * nband;
    if (items >= (1LL << 31)) return fail(MERIT_E_UNSUPPORTED_VIEW, "too many max-pool bands for one launch");
    int ctas = RBv == 14 ? 14 : 7;  // 14-row bands: one band per CTA
    if (const char* ce = getenv("MERIT_MP_CTAS")) ctas = atoi(ce);
    const size_t stage = ((size_t)(2 * RBv + 1) * p.W * 4 + 127) / 128 * 128;
    int ns = RBv == 4 ? 8 : (RBv == 8 ? 4 : (RBv == 16 ? 2 : 1));
    if (const char* se = getenv("MERIT_MP_STAGES")) ns = atoi(se);
    if (ns > kMpMaxStages) ns = kMpMaxStages;
    while (ns > 1 && ns * stage > 100 * 1024) --ns;
    size_t smem = ns * stage;
    if (const char* pe = getenv("MERIT_MP_SMEM_PAD")) smem += static_cast<size_t>(atoi(pe));  // residency experiments
    if (smem <= 200 * 1024) {
      long long grid = (long long)num_sms() * ctas;
      if (grid > items) grid = items;
      grid = grid_cap(static_cast<int>(grid));
      // band loads: a 2-D tensor map over the [planes * H][W] rows (UTMALDG),
      // or plain bulk copies (MERIT_MP_TMAP=0)
      CUtensorMap rmap;
      std::memset(&rmap, 0, sizeof(rmap));
      const char* te = getenv("MERIT_MP_TMAP");
      bool tm = !(te && te[0] == '0') && tensor_map_encoder() != nullptr && p.W <= 256 &&
                p.planes * p.H < (1LL << 31);
      if (tm) {
        const cuuint64_t dims[2] = {(cuuint64_t)p.W, (cuuint64_t)(p.planes * p.H)};
        const cuuint64_t strides[1] = {(cuuint64_t)p.W * 4};
        const cuuint32_t box[2] = {(cuuint32_t)p.W, (cuuint32_t)(2 * RBv + 1)};
        const cuuint32_t estr[2] = {1, 1};
        tm = tensor_map_encoder()(&rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(in), dims, strides,
                                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
      auto k = tm ? maxpool3s2_bulk_kernel<128, 8, true> : maxpool3s2_bulk_kernel<128, 8, false>;
      if (RBv == 4) k = tm ? maxpool3s2_bulk_kernel<128, 4, true> : maxpool3s2_bulk_kernel<128, 4, false>;
      if (RBv == 16) k = tm ? maxpool3s2_bulk_kernel<128, 16, true> : maxpool3s2_bulk_kernel<128, 16, false>;
      if (RBv == 28) k = tm ? maxpool3s2_bulk_kernel<128, 28, true> : maxpool3s2_bulk_kernel<128, 28, false>;
      if (RBv == 56) k = tm ? maxpool3s2_bulk_kernel<128, 56, true> : maxpool3s2_bulk_kernel<128, 56, false>;
      if (RBv == 14) {  // 4 warps (MERIT_MP_NT=256: 8)
        const char* ne = getenv("MERIT_MP_NT");
        k = (ne && atoi(ne) == 256) ? (tm ? maxpool3s2_bulk_kernel<256, 14, true> : maxpool3s2_bulk_kernel<256, 14, false>)
                                    : (tm ? maxpool3s2_bulk_kernel<128, 14, true> : maxpool3s2_bulk_kernel<128, 14, false>);
      }
      // 28-row bands: 8 warps per CTA (a band's 392 16-byte output groups in
      // two passes instead of four shortens every CTA's compute-and-store
      // tail) and exactly 6 CTAs per SM (dynamic shared memory padded to 32
      // KB): C1 runs 888 bands as the first wave and 136 as a second one,
      // 6.67 us vs 7.33 us with all 1,024 resident at once (7 per SM)
      int nt = 128;
      if (RBv == 28) {
        const char* ne = getenv("MERIT_MP_NT");
        if (!(ne && atoi(ne) == 128)) {
          nt = 256;
          k = tm ? maxpool3s2_bulk_kernel<256, 28, true> : maxpool3s2_bulk_kernel<256, 28, false>;
          if (!getenv("MERIT_MP_SMEM_PAD") && smem < 32768) smem = 32768;
        }
      }
      cudaError_t e = set_smem_attr(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(maxpool)");
      MaxpoolParams pp = p;
      if (const char* de = debug_env("MERIT_MP_DEBUG")) pp.dbg = atoi(de);
      pp.vec_out = (p.Wo % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
      pp.pf = ns;
      if (const char* pe = getenv("MERIT_MP_PF")) pp.pf = atoi(pe) < 0 ? (1 << 30) : atoi(pe);
      if (RBv == 14) {
        const char* ne = getenv("MERIT_MP_NT");
        nt = (ne && atoi(ne) == 256) ? 256 : 128;
      }
      e = launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(nt), smem, s, 1, in, o, pp, nband,
                     static_cast<int>(items), ns,
                     rmap);
      if (e != cudaSuccess) return cuda_check(e, "launch(maxpool3s2_bulk_kernel)");
      return launch_status("maxpool3s2_bulk_kernel");
    }
    constexpr int RB = 4;
    const int nseg = (p.W + 127) / 128;
    const int nband4 = (p.Ho + RB - 1) / RB;
    const long long items4 = p.planes * nband4 * nseg;
    const long long resident = (long long)num_sms() * 6 * 4;  // 6 CTAs x 4 warps per SM
    const int per_warp = static_cast<int>((items4 + resident - 1) / resident);
    const long long warps = (items4 + per_warp - 1) / per_warp;
    const long long blocks = (warps + 3) / 4;
    maxpool3s2_kernel<RB><<<static_cast<unsigned>(blocks), 128, 0, s>>>(in, o, p, nseg, nband4, items4,
                                                                      per_warp);
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
