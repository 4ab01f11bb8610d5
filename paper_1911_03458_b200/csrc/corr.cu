// K4 — displacement correlation (the FlowNet `correlation` template,
// workloads.hpp:230-251, with mac_program(1, 0)):
//
//   out[y][x][dy][dx] = post( sum_c A[c][y + ay][x + ax] * B[c][y + dy + by][x + dx + bx] )
//
// with ZERO_PAD reads outside either source.  The engine's REAL32 MAC is
// r = float(r + float(double(b) * c)) (rip.hpp:161-178 with shift 0), i.e.
// __fadd_rn(r, __fmul_rn(a, b)) in channel order — so the kernel folds the
// channels in that order with exactly those two roundings (no FMA
// contraction) and is bit-identical to merit::run_full, like the exact
// interpreter it replaces for this view family, at CUDA-core throughput.
//
// Two kernels.  corr_tma_kernel (both sources W % 4 == 0, the usual case):
// 2-D output tiles whose 8-channel stages arrive as TMA boxes (out-of-bounds
// fill = the zero padding) through a 6-deep mbarrier ring; thread tile XB
// columns x DK displacements, chosen for dx-lane use and occupancy.
// corr_kernel (any width): one output row per CTA, predicated loads.  In both
// a thread owns XB columns x DK displacements dx of one (row, dy) and per
// channel folds XB * DK products from XB + DK - 1 staged B values.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_common.cuh"
#include "tmap.cuh"

namespace merit_dev {
namespace {

constexpr int kXB = 4;  // output columns per thread
constexpr int kDK = 8;  // displacements dx per thread
constexpr int kCC = 8;  // channels per shared-memory stage

struct CorrLaunch {
  CorrParams p;
  int TX;    // output columns per CTA (multiple of kXB)
  int DXC;   // dx chunks of kDK
  int WB;    // B strip width = TX + kDK * DXC - 1 (padded to 4)
  int nxt;   // column tiles per row
};

__global__ void __launch_bounds__(1024) corr_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                     float* __restrict__ out, CorrLaunch L) {
  extern __shared__ __align__(16) float sm[];
  const CorrParams& p = L.p;
  float* As = sm;                       // [kCC][TX]
  float* Bs = sm + kCC * L.TX;          // [kCC][DY][WB]
  const int y = blockIdx.x / L.nxt;
  const int x0 = (blockIdx.x - y * L.nxt) * L.TX;
  const int t = threadIdx.x;
  const int nxq = L.TX / kXB;
  const int dxc = t % L.DXC;
  const int r1 = t / L.DXC;
  const int xq = r1 % nxq;
  const int dy = r1 / nxq;
  const bool active = dy < p.DY;
  const int warp = t >> 5, lane = t & 31, nwarps = blockDim.x >> 5;
  const long long a_plane = (long long)p.Ha * p.Wa, b_plane = (long long)p.Hb * p.Wb;
  const int ya = y + p.ay;
  const bool ya_in = ya >= 0 && ya < p.Ha;

  float acc[kXB][kDK];
#pragma unroll
  for (int i = 0; i < kXB; ++i)
#pragma unroll
    for (int k = 0; k < kDK; ++k) acc[i][k] = 0.f;

  pdl_launch_dependents();
  pdl_wait();
  for (int c0 = 0; c0 < p.C; c0 += kCC) {
    const int cn = min(kCC, p.C - c0);
    __syncthreads();  // the previous stage's reads are done
    // stage A: cn rows of TX (one row per warp step, lanes along x)
    for (int c = warp; c < cn; c += nwarps) {
      const float* src = A + (c0 + c) * a_plane + (long long)(ya_in ? ya : 0) * p.Wa;
      for (int xx = lane; xx < L.TX; xx += 32) {
        const int xa = x0 + xx + p.ax;
        As[c * L.TX + xx] = (ya_in && xa >= 0 && xa < p.Wa) ? __ldg(src + xa) : 0.f;
      }
    }
    // stage B: cn x DY rows of WB
    for (int row = warp; row < cn * p.DY; row += nwarps) {
      const int c = row / p.DY;
      const int r = row - c * p.DY;
      const int yb = y + r + p.by;
      const bool yin = yb >= 0 && yb < p.Hb;
      const float* src = B + (c0 + c) * b_plane + (long long)(yin ? yb : 0) * p.Wb;
      float* dst = Bs + row * L.WB;
      for (int xx = lane; xx < L.WB; xx += 32) {
        const int xb = x0 + xx + p.bx;
        dst[xx] = (yin && xb >= 0 && xb < p.Wb) ? __ldg(src + xb) : 0.f;
      }
    }
    __syncthreads();
    if (active) {
      for (int c = 0; c < cn; ++c) {
        const float4 a4 = *reinterpret_cast<const float4*>(As + c * L.TX + xq * kXB);
        const float a[kXB] = {a4.x, a4.y, a4.z, a4.w};
        const float* br = Bs + (c * p.DY + dy) * L.WB + xq * kXB + dxc * kDK;
        float b[kXB + kDK - 1];
#pragma unroll
        for (int j = 0; j < kXB + kDK - 1; ++j) b[j] = br[j];
#pragma unroll
        for (int i = 0; i < kXB; ++i)
#pragma unroll
          for (int k = 0; k < kDK; ++k) acc[i][k] = __fadd_rn(acc[i][k], __fmul_rn(a[i], b[i + k]));
      }
    }
  }
  if (!active) return;
  // Post_1: emit r + 0 (a -0 sum becomes +0) or max(r, 0) (std::max(r, 0): r unless r < 0)
#pragma unroll
  for (int i = 0; i < kXB; ++i) {
    const int x = x0 + xq * kXB + i;
    if (x >= p.Wo) continue;
    float* o = out + (((long long)y * p.Wo + x) * p.DY + dy) * p.DX;
#pragma unroll
    for (int k = 0; k < kDK; ++k) {
      const int dx = dxc * kDK + k;
      if (dx < p.DX) {
        const float r = acc[i][k];
        __stcs(o + dx, p.post == POST_RELU ? (r < 0.f ? 0.f : r) : __fadd_rn(r, 0.f));
      }
    }
  }
}

// ---- TMA path (W % 4 == 0 on both sources) --------------------------------
// A CTA owns TY output rows x TX columns for every displacement; one stage =
// kCC channels: an A box {WA, TY, kCC} at (floor4(x0 + ax), y0 + ay, c0) and a
// B box {WB, TY + DY - 1, kCC} at (floor4(x0 + bx), y0 + by, c0), whose
// out-of-bounds fill is the view's zero padding (no per-element predicates).
// The B rows of a stage are shared by every (row, dy) pair of the tile.
// NS-stage mbarrier ring; thread 0 refills a slot after the CTA barrier that
// ends its use.  Thread = (dxc, xq, ty, dy): 4 columns x 8 dx of one (row, dy).
struct CorrTma {
  CorrParams p;
  int TX, TY, DXC;
  int WA, WB, RB;       // box widths (floats, multiples of 4) and B box rows
  int nxt;              // column tiles per tile row
  int n_stages;         // ceil(C / kCC)
  int NS;               // ring depth
  uint32_t stage_bytes, a_bytes;
};

__device__ __forceinline__ int floor4(int x) { return x >= 0 ? (x & ~3) : -((-x + 3) & ~3); }

__device__ __forceinline__ void corr_tma_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(c), "r"(bar)
      : "memory");
}

template <int XB, int DK>
__global__ void __launch_bounds__(1024) corr_tma_kernel(const __grid_constant__ CUtensorMap amap,
                                                         const __grid_constant__ CUtensorMap bmap,
                                                         float* __restrict__ out, CorrTma L) {
  extern __shared__ __align__(128) uint8_t smem_c[];
  const CorrParams& p = L.p;
  const uint32_t base = (smem_u32(smem_c) + 127u) & ~127u;
  float* fbase = reinterpret_cast<float*>(smem_c + (base - smem_u32(smem_c)));
  const uint32_t bars = base + L.NS * L.stage_bytes;
  const int y0 = (blockIdx.x / L.nxt) * L.TY;
  const int x0 = (blockIdx.x - (blockIdx.x / L.nxt) * L.nxt) * L.TX;
  const int xa0 = floor4(x0 + p.ax), xb0 = floor4(x0 + p.bx);
  const int da = x0 + p.ax - xa0, db = x0 + p.bx - xb0;
  const int t = threadIdx.x;
  const int nxq = L.TX / XB;
  const int dxc = t % L.DXC;
  int r1 = t / L.DXC;
  const int xq = r1 % nxq;
  r1 /= nxq;
  const int ty = r1 % L.TY;
  const int dy = r1 / L.TY;
  const bool active = dy < p.DY;

  if (t == 0) {
    for (int s = 0; s < L.NS; ++s) tc::mbar_init(bars + 8u * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();
  auto issue = [&](int st) {
    const int s = st % L.NS;
    const uint32_t dst = base + s * L.stage_bytes;
    tc::mbar_expect_tx(bars + 8u * s, L.stage_bytes);
    corr_tma_3d(dst, &amap, xa0, y0 + p.ay, st * kCC, bars + 8u * s);
    corr_tma_3d(dst + L.a_bytes, &bmap, xb0, y0 + p.by, st * kCC, bars + 8u * s);
  };
  if (t == 0)
    for (int st = 0; st < L.NS && st < L.n_stages; ++st) issue(st);

  float acc[XB][DK];
#pragma unroll
  for (int i = 0; i < XB; ++i)
#pragma unroll
    for (int k = 0; k < DK; ++k) acc[i][k] = 0.f;
  const int a_plane = L.TY * L.WA, b_plane = L.RB * L.WB;  // floats per channel
  const int a_off = ty * L.WA + da + xq * XB;
  const int b_off = (ty + dy) * L.WB + db + xq * XB + dxc * DK;
  for (int st = 0; st < L.n_stages; ++st) {
    const int s = st % L.NS;
    tc::mbar_wait(bars + 8u * s, (st / L.NS) & 1);
    const float* As = fbase + s * (L.stage_bytes / 4);
    const float* Bs = As + L.a_bytes / 4;
    const int cn = min(kCC, p.C - st * kCC);
    if (active) {
      for (int c = 0; c < cn; ++c) {
        const float* ar = As + c * a_plane + a_off;
        const float* br = Bs + c * b_plane + b_off;
        float a[XB], b[XB + DK - 1];
#pragma unroll
        for (int i = 0; i < XB; ++i) a[i] = ar[i];
#pragma unroll
        for (int j = 0; j < XB + DK - 1; ++j) b[j] = br[j];
#pragma unroll
        for (int i = 0; i < XB; ++i)
#pragma unroll
          for (int k = 0; k < DK; ++k) acc[i][k] = __fadd_rn(acc[i][k], __fmul_rn(a[i], b[i + k]));
      }
    }
    __syncthreads();  // slot s consumed by every thread
    if (t == 0 && st + L.NS < L.n_stages) issue(st + L.NS);
  }
  if (!active) return;
  const int y = y0 + ty;
  if (y >= p.Ho) return;
#pragma unroll
  for (int i = 0; i < XB; ++i) {
    const int x = x0 + xq * XB + i;
    if (x >= p.Wo) continue;
    float* o = out + (((long long)y * p.Wo + x) * p.DY + dy) * p.DX;
#pragma unroll
    for (int k = 0; k < DK; ++k) {
      const int dx = dxc * DK + k;
      if (dx < p.DX) {
        const float r = acc[i][k];
        __stcs(o + dx, p.post == POST_RELU ? (r < 0.f ? 0.f : r) : __fadd_rn(r, 0.f));
      }
    }
  }
}

merit_status launch_corr_tma(const CorrParams& p, const float* a, const float* b, float* out, cudaStream_t s,
                             bool& used) {
  used = false;
  if (p.Wa % 4 || p.Wb % 4 || (reinterpret_cast<uintptr_t>(a) % 16) || (reinterpret_cast<uintptr_t>(b) % 16) ||
      tensor_map_encoder() == nullptr)
    return MERIT_OK;
  if (const char* e = getenv("MERIT_CORR_TMA"); e && e[0] == '0') return MERIT_OK;
  // per-thread tile XB columns x DK displacements: the sequential channel
  // chain of every output is the engine's order, so parallelism comes from
  // outputs only — smaller thread tiles when there are too few outputs to
  // keep ~16 warps per SM busy
  // (measured, tools/corr_time.py: FlowNetC 48x48 d=21 -> 2x8, 96x128 d=9 -> 2x4 / 4x8)
  int XB = 4, DK = 8;
  {
    const long long outs = (long long)p.Ho * p.Wo * p.DY * p.DX;
    const long long want = 16LL * 32 * num_sms();
    const int dxc8 = (p.DX + 7) / 8;
    const bool dx8_full = 5 * p.DX >= 4 * 8 * dxc8;  // 8-wide dx chunks >= 80% used
    if (!dx8_full) { XB = 2; DK = 4; }
    else if (outs / 32 < want) { XB = 2; DK = 8; }
    if (const char* te = getenv("MERIT_CORR_TILE")) {
      if (!strcmp(te, "4x8")) { XB = 4; DK = 8; }
      if (!strcmp(te, "2x8")) { XB = 2; DK = 8; }
      if (!strcmp(te, "2x4")) { XB = 2; DK = 4; }
      if (!strcmp(te, "1x8")) { XB = 1; DK = 8; }
    }
  }
  CorrTma L;
  L.p = p;
  L.DXC = (p.DX + DK - 1) / DK;
  const int per_quad = p.DY * L.DXC;  // threads per XB output columns
  // column tile: 8 unless the image is narrower; rows: the most that keep
  // the CTA within 1024 threads and the grid at >= 90% of the SMs
  L.TX = std::min(8, (p.Wo + XB - 1) / XB * XB);
  L.TY = std::max(1, std::min(p.Ho, 1024 / (per_quad * (L.TX / XB))));
  auto grid_of = [&](int ty) { return (long long)((p.Ho + ty - 1) / ty) * ((p.Wo + L.TX - 1) / L.TX); };
  while (L.TY > 1 && grid_of(L.TY) * 10 < 9LL * num_sms()) --L.TY;
  if (const char* e = getenv("MERIT_CORR_TY")) L.TY = std::max(1, atoi(e));
  const int threads = (per_quad * L.TY * (L.TX / XB) + 31) / 32 * 32;
  if (threads > 1024) return MERIT_OK;
  L.WA = L.TX + 4;
  L.WB = (L.TX + DK * L.DXC - 1 + 3 + 3) / 4 * 4;
  L.RB = L.TY + p.DY - 1;
  if (L.WA > 256 || L.WB > 256 || L.RB > 256) return MERIT_OK;
  L.nxt = (p.Wo + L.TX - 1) / L.TX;
  L.n_stages = (p.C + kCC - 1) / kCC;
  L.a_bytes = static_cast<uint32_t>(kCC * L.TY * L.WA * 4);
  L.stage_bytes = (L.a_bytes + static_cast<uint32_t>(kCC * L.RB * L.WB * 4) + 127u) & ~127u;
  // ring depth: enough stages in flight to cover the TMA latency (one stage
  // of a FlowNet tile computes in ~0.5 us), within the shared memory of one CTA
  L.NS = 6;
  if (const char* ne = getenv("MERIT_CORR_NS")) L.NS = std::max(1, std::min(16, atoi(ne)));
  while (L.NS > 1 && 128 + L.NS * (size_t)L.stage_bytes + 8 * 16 > 200 * 1024) --L.NS;
  if (L.NS > L.n_stages) L.NS = std::max(1, L.n_stages);
  const size_t smem = 128 + L.NS * (size_t)L.stage_bytes + 8 * 16;
  if (smem > 200 * 1024) return MERIT_OK;
  CUtensorMap amap, bmap;
  std::memset(&amap, 0, sizeof(amap));
  std::memset(&bmap, 0, sizeof(bmap));
  const cuuint32_t es[3] = {1, 1, 1};
  {
    const cuuint64_t dims[3] = {(cuuint64_t)p.Wa, (cuuint64_t)p.Ha, (cuuint64_t)p.C};
    const cuuint64_t str[2] = {(cuuint64_t)p.Wa * 4, (cuuint64_t)p.Wa * p.Ha * 4};
    const cuuint32_t box[3] = {(cuuint32_t)L.WA, (cuuint32_t)L.TY, (cuuint32_t)kCC};
    if (tensor_map_encoder()(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a), dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return MERIT_OK;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)p.Wb, (cuuint64_t)p.Hb, (cuuint64_t)p.C};
    const cuuint64_t str[2] = {(cuuint64_t)p.Wb * 4, (cuuint64_t)p.Wb * p.Hb * 4};
    const cuuint32_t box[3] = {(cuuint32_t)L.WB, (cuuint32_t)L.RB, (cuuint32_t)kCC};
    if (tensor_map_encoder()(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(b), dims, str, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return MERIT_OK;
  }
  const long long grid = grid_of(L.TY);
  if (grid >= (1LL << 31)) return MERIT_OK;
  auto kern = corr_tma_kernel<4, 8>;
  if (XB == 2 && DK == 8) kern = corr_tma_kernel<2, 8>;
  if (XB == 2 && DK == 4) kern = corr_tma_kernel<2, 4>;
  if (XB == 1 && DK == 8) kern = corr_tma_kernel<1, 8>;
  cudaError_t e = set_smem_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(corr_tma)");
  e = launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(threads), smem, s, 1, amap, bmap, out, L);
  if (e != cudaSuccess) return cuda_check(e, "launch(corr_tma)");
  used = true;
  return launch_status("corr_tma_kernel");
}

}  // namespace

// Threads per CTA for a displacement window, 0 if it does not fit one CTA
// (the lowering then keeps the exact interpreter).
int corr_threads_per_column_quad(int DY, int DX) {
  const int dxc = (DX + kDK - 1) / kDK;
  return DY * dxc <= 1024 ? DY * dxc : 0;
}

merit_status launch_corr(const merit_plan& plan, const void* a, const void* b, void* out, void* stream) {
  const CorrParams& p = plan.corr;
  if (p.C > 0 && p.Ho > 0 && p.Wo > 0) {
    bool used = false;
    const merit_status st = launch_corr_tma(p, static_cast<const float*>(a), static_cast<const float*>(b),
                                            static_cast<float*>(out), static_cast<cudaStream_t>(stream), used);
    if (st != MERIT_OK || used) return st;
  }
  CorrLaunch L;
  L.p = p;
  L.DXC = (p.DX + kDK - 1) / kDK;
  const int per_quad = p.DY * L.DXC;  // threads per kXB output columns
  if (per_quad > 1024) return fail(MERIT_E_UNSUPPORTED_VIEW, "correlation window too large for one CTA");
  // the widest column tile within 512 threads that still gives every SM a CTA
  const int wo4 = (p.Wo + kXB - 1) / kXB * kXB;
  int tx = std::max(kXB, std::min(128, (512 / per_quad) * kXB));
  tx = std::min(tx, wo4);
  while (tx > kXB && (long long)p.Ho * ((p.Wo + tx - 1) / tx) < num_sms()) tx -= kXB;
  if (const char* e = getenv("MERIT_CORR_TX")) tx = std::max(kXB, atoi(e) / kXB * kXB);
  L.TX = tx;
  L.WB = (tx + kDK * L.DXC - 1 + 3) / 4 * 4;
  L.nxt = (p.Wo + tx - 1) / tx;
  const int threads = (per_quad * (tx / kXB) + 31) / 32 * 32;
  const size_t smem = sizeof(float) * ((size_t)kCC * tx + (size_t)kCC * p.DY * L.WB);
  if (threads > 1024 || smem > 200 * 1024) return fail(MERIT_E_UNSUPPORTED_VIEW, "correlation tile too large");
  const long long grid = (long long)p.Ho * L.nxt;
  if (grid == 0) return MERIT_OK;
  if (grid >= (1LL << 31)) return fail(MERIT_E_UNSUPPORTED_VIEW, "correlation grid too large");
  cudaError_t e = set_smem_attr(corr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(corr)");
  e = launch_pdl(corr_kernel, dim3(static_cast<unsigned>(grid)), dim3(threads), smem,
                 static_cast<cudaStream_t>(stream), 1, static_cast<const float*>(a), static_cast<const float*>(b),
                 static_cast<float*>(out), L);
  if (e != cudaSuccess) return cuda_check(e, "launch(corr)");
  return launch_status("corr_kernel");
}

}  // namespace merit_dev
