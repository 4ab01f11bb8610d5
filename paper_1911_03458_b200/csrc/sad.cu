// K2 — L1 block matching (the motion-estimation workload, workloads.hpp:
// 255-279, with sad_program(2), workloads.hpp:64-68) plus the caller-side
// argmin stage the reference leaves to users.
//
// out[.., by, bx, dy, dx] = sum_{i<BH, j<BW} |cur[by*BH+i, bx*BW+j]
//                                           - ref[by*BH+dy+i+oy, bx*BW+dx+j+ox]|
// with the reference view's boundary rule (ZERO_PAD: 0 outside the frame,
// the semantics of oracle_motion_estimation, workloads.hpp:569-576).  On
// 8-bit frames every partial sum is an exact integer < 2^24, so the int32
// result equals the reference's REAL32 accumulation bit for bit.
//
// Design (sm_100a):
//  * A CTA owns one block row band: TBX horizontally adjacent blocks of one
//    frame pair.  It stages the Eq. 6 footprint of the reference window
//    (footprint_box, view.hpp:143-149) into shared memory once, as FOUR
//    byte-shifted word copies, so that any dx reads 32-bit aligned words
//    without a per-thread PRMT.
//  * A thread owns one (block, dx, dy-group of D rows) item: the current
//    block lives in registers (BH x BW/4 words), and every reference row it
//    streams is folded into all D displacement accumulators it overlaps with
//    VABSDIFF4.U8.ACC — 4 abs-diff-accumulates per instruction, the native
//    byte-SIMD op (measured 64 lanes/clk/SM, tools/microbench/int_simd.cu).
//  * Argmin: per-thread min over its D rows, then a shared-memory atomicMin
//    on the packed key (sad << 16 | dy*WX + dx) — lowest SAD, then lowest
//    raster index, exactly the tie-break BASELINE.json asks for.
#include "common.cuh"

namespace merit_dev {
namespace {

constexpr int kSadMaxThreads = 384;

__device__ __forceinline__ uint32_t vabsdiff4_acc(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

struct SadLaunch {
  SadParams p;
  int TBX;       // blocks per CTA
  int G;         // dy groups
  int n_tiles_x; // ceil(BX / TBX)
  int R;         // staged reference rows = G*D + BH - 1
  int span;      // staged reference columns = TBX*BW + WX - 1
  int Ww;        // words per staged row per copy
  int CS;        // words per shifted copy (padded to 8 mod 32 against bank conflicts)
  int raw_pitch; // bytes per raw staged row (multiple of 4, >= 4*(Ww+1))
  int items;     // TBX * WX * G
  int word_path; // 4-byte aligned staging
};

template <int BLK, int D>
__global__ void __launch_bounds__(kSadMaxThreads, 2)
sad_kernel(const uint8_t* __restrict__ cur, const uint8_t* __restrict__ ref, void* __restrict__ out,
           int32_t* __restrict__ aux, SadLaunch L) {
  extern __shared__ __align__(16) uint32_t smem[];
  const SadParams& p = L.p;
  constexpr int BWW = BLK / 4;  // words per block row
  // --- tile coordinates
  const int tx = blockIdx.x % L.n_tiles_x;
  const long long t2 = blockIdx.x / L.n_tiles_x;
  const int by = static_cast<int>(t2 % p.BY);
  const long long pair = t2 / p.BY;
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);
  // --- shared memory carve-up
  uint32_t* copies = smem;                                   // 4 * CS words
  uint8_t* raw = reinterpret_cast<uint8_t*>(smem + 4 * L.CS);  // R * raw_pitch bytes
  uint8_t* curs = raw + L.R * L.raw_pitch;                   // TBX * BLK * BLK bytes
  uint32_t* keys = reinterpret_cast<uint32_t*>(curs + L.TBX * BLK * BLK);  // TBX keys
  const uint8_t* refp = ref + pair * (long long)p.Hr * p.Wr;
  const uint8_t* curp = cur + pair * (long long)p.Hc * p.Wc;
  // Reference footprint origin (Eq. 6): row by*BH + oy, column bx0*BW + ox.
  const int ry0 = by * BLK + p.oy;
  const int rx0 = bx0 * BLK + p.ox;
  const int nthreads = blockDim.x;
  // 1) raw bytes of the reference window, boundary applied.  When the window
  //    origin and the frame pitch are 4-byte aligned (every BASELINE config)
  //    whole words are fetched, four per thread in flight.
  const int rawcols = L.raw_pitch;
  if (L.word_path) {
    const int rw = rawcols / 4;
    const int total = L.R * rw;
    uint32_t* raww = reinterpret_cast<uint32_t*>(raw);
    for (int e0 = threadIdx.x; e0 < total; e0 += 4 * nthreads) {
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * nthreads;
        v[u] = 0u;
        if (e < total) {
          const int r = e / rw, c = (e % rw) * 4;
          int y = ry0 + r, x = rx0 + c;
          if (c < L.span) {
            bool in = y >= 0 && y < p.Hr && x >= 0 && x < p.Wr;
            if (!in && p.boundary == MERIT_CLAMP) {
              if (x >= 0 && x < p.Wr) {  // only the row is outside: clamp it
                y = y < 0 ? 0 : p.Hr - 1;
                in = true;
              }
            }
            if (in) {
              v[u] = __ldg(reinterpret_cast<const uint32_t*>(refp + (long long)y * p.Wr + x));
            } else if (p.boundary == MERIT_CLAMP) {  // column outside: byte-wise clamp
              y = y < 0 ? 0 : (y >= p.Hr ? p.Hr - 1 : y);
              uint32_t w = 0;
              for (int q = 0; q < 4; ++q) {
                int xx = x + q;
                xx = xx < 0 ? 0 : (xx >= p.Wr ? p.Wr - 1 : xx);
                w |= static_cast<uint32_t>(__ldg(refp + (long long)y * p.Wr + xx)) << (8 * q);
              }
              v[u] = w;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * nthreads;
        if (e < total) raww[e] = v[u];
      }
    }
  } else {
    for (int e = threadIdx.x; e < L.R * rawcols; e += nthreads) {
      const int r = e / rawcols, c = e % rawcols;
      int y = ry0 + r, x = rx0 + c;
      uint8_t v = 0;
      if (c < L.span) {
        bool in = y >= 0 && y < p.Hr && x >= 0 && x < p.Wr;
        if (!in && p.boundary == MERIT_CLAMP) {
          y = y < 0 ? 0 : (y >= p.Hr ? p.Hr - 1 : y);
          x = x < 0 ? 0 : (x >= p.Wr ? p.Wr - 1 : x);
          in = true;
        }
        if (in) v = __ldg(refp + (long long)y * p.Wr + x);
      }
      raw[e] = v;
    }
  }
  // 2) current blocks.
  if (L.word_path) {
    constexpr int WPB = BLK * BLK / 4;
    uint32_t* cursw = reinterpret_cast<uint32_t*>(curs);
    for (int e = threadIdx.x; e < L.TBX * WPB; e += nthreads) {
      const int b = e / WPB, r = (e % WPB) / (BLK / 4), c = (e % (BLK / 4)) * 4;
      uint32_t v = 0;
      if (b < nb) {
        const int y = by * BLK + r + p.cy, x = (bx0 + b) * BLK + c + p.cx;
        v = __ldg(reinterpret_cast<const uint32_t*>(curp + (long long)y * p.Wc + x));
      }
      cursw[e] = v;
    }
  } else {
    for (int e = threadIdx.x; e < L.TBX * BLK * BLK; e += nthreads) {
      const int b = e / (BLK * BLK), r = (e / BLK) % BLK, c = e % BLK;
      uint8_t v = 0;
      if (b < nb) {
        const int y = by * BLK + r + p.cy, x = (bx0 + b) * BLK + c + p.cx;
        v = __ldg(curp + (long long)y * p.Wc + x);
      }
      curs[e] = v;
    }
  }
  if (threadIdx.x < L.TBX) keys[threadIdx.x] = 0xffffffffu;
  __syncthreads();
  // 3) four byte-shifted word copies: copy_s[r][w] = bytes (4w+s .. 4w+s+3).
  {
    const int rw = L.raw_pitch / 4;
    const uint32_t* raww = reinterpret_cast<const uint32_t*>(raw);
    for (int e = threadIdx.x; e < L.R * L.Ww; e += nthreads) {
      const int r = e / L.Ww, w = e % L.Ww;
      const uint32_t lo = raww[r * rw + w];
      const uint32_t hi = (w + 1 < rw) ? raww[r * rw + w + 1] : 0u;
      const int o = r * L.Ww + w;
      copies[o] = lo;
      copies[L.CS + o] = __byte_perm(lo, hi, 0x4321);
      copies[2 * L.CS + o] = __byte_perm(lo, hi, 0x5432);
      copies[3 * L.CS + o] = __byte_perm(lo, hi, 0x6543);
    }
  }
  __syncthreads();
  // 4) per-thread item: (block, dy-group, dx)
  const int item = threadIdx.x;
  if (item < L.items) {
    const int per_block = p.WX * L.G;
    const int b = item / per_block;
    const int rem = item % per_block;
    const int g = rem / p.WX;
    const int dx = rem % p.WX;
    if (b < nb) {
      uint32_t cw[BLK][BWW];
      const uint32_t* cb = reinterpret_cast<const uint32_t*>(curs + b * BLK * BLK);
#pragma unroll
      for (int i = 0; i < BLK; ++i)
#pragma unroll
        for (int j = 0; j < BWW; ++j) cw[i][j] = cb[i * BWW + j];
      const int col = b * BLK + dx;  // byte column in the staged window
      const uint32_t* cp = copies + (col & 3) * L.CS + (col >> 2);
      uint32_t acc[D];
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = 0;
      const int row0 = g * D;
#pragma unroll
      for (int r = 0; r < D + BLK - 1; ++r) {
        uint32_t rw[BWW];
        const uint32_t* rp = cp + (row0 + r) * L.Ww;
#pragma unroll
        for (int j = 0; j < BWW; ++j) rw[j] = rp[j];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int i = r - d;
          if (i >= 0 && i < BLK) {
#pragma unroll
            for (int j = 0; j < BWW; ++j) acc[d] = vabsdiff4_acc(cw[i][j], rw[j], acc[d]);
          }
        }
      }
      const int bx = bx0 + b;
      const long long blk_index = (pair * p.BY + by) * (long long)p.BX + bx;
      uint32_t best = 0xffffffffu;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int dy = row0 + d;
        if (dy < p.WY) {
          const uint32_t key = (acc[d] << 16) | static_cast<uint32_t>(dy * p.WX + dx);
          best = key < best ? key : best;
          if (p.write_map) {
            const long long o = (blk_index * p.WY + dy) * p.WX + dx;
            if (p.out_f32)
              static_cast<float*>(out)[o] = static_cast<float>(acc[d]);
            else
              static_cast<int32_t*>(out)[o] = static_cast<int32_t>(acc[d]);
          }
        }
      }
      if (p.argmin) atomicMin(&keys[b], best);
    }
  }
  if (p.argmin) {
    __syncthreads();
    if (threadIdx.x < nb) {
      const uint32_t key = keys[threadIdx.x];
      const int idx = static_cast<int>(key & 0xffffu);
      const int dy = idx / p.WX, dx = idx % p.WX;
      const long long blk_index = (pair * p.BY + by) * (long long)p.BX + bx0 + threadIdx.x;
      int32_t* a = aux + blk_index * 3;
      a[0] = dy + p.oy - p.cy;
      a[1] = dx + p.ox - p.cx;
      a[2] = static_cast<int32_t>(key >> 16);
    }
  }
}

template <int BLK, int D>
merit_status launch_sad_t(const SadParams& p, const uint8_t* cur, const uint8_t* ref, void* out,
                          int32_t* aux, cudaStream_t s) {
  SadLaunch L;
  L.p = p;
  L.G = (p.WY + D - 1) / D;
  const int per_block = p.WX * L.G;
  if (per_block > kSadMaxThreads)
    return fail(MERIT_E_UNSUPPORTED_VIEW, "search window too wide for the SAD kernel");
  // Blocks per CTA: least idle-lane fraction within the thread budget.
  L.TBX = 1;
  double best_waste = 2.0;
  for (int t = 1; t <= 8 && t <= p.BX; ++t) {
    const int items = t * per_block;
    const int threads = (items + 31) / 32 * 32;
    if (threads > kSadMaxThreads) break;
    const double waste = double(threads - items) / threads;
    if (waste < best_waste - 1e-9 || (waste < best_waste + 0.02 && t > L.TBX && items < 256)) {
      best_waste = waste;
      L.TBX = t;
    }
  }
  L.items = L.TBX * per_block;
  L.n_tiles_x = (p.BX + L.TBX - 1) / L.TBX;
  L.R = L.G * D + BLK - 1;
  L.span = L.TBX * BLK + p.WX - 1;
  L.Ww = (L.span + 3) / 4;
  L.raw_pitch = (L.Ww + 1) * 4;
  L.CS = L.R * L.Ww;
  L.CS += ((8 - (L.CS % 32)) + 32) % 32;
  L.word_path = ((p.ox % 4) == 0 && (p.cx % 4) == 0 && (p.Wr % 4) == 0 && (p.Wc % 4) == 0 &&
                 (reinterpret_cast<uintptr_t>(cur) % 4) == 0 && (reinterpret_cast<uintptr_t>(ref) % 4) == 0)
                    ? 1 : 0;
  const size_t smem = 4ull * L.CS * 4 + (size_t)L.R * L.raw_pitch + (size_t)L.TBX * BLK * BLK +
                      (size_t)L.TBX * 4 + 16;
  const long long ctas = p.pairs * (long long)p.BY * L.n_tiles_x;
  if (ctas == 0) return MERIT_OK;
  if (smem > 227 * 1024) return fail(MERIT_E_UNSUPPORTED_VIEW, "SAD footprint exceeds shared memory");
  auto kern = sad_kernel<BLK, D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(sad)");
  const int threads = (L.items + 31) / 32 * 32;
  kern<<<static_cast<unsigned>(ctas), threads, smem, s>>>(cur, ref, out, aux, L);
  return launch_status("sad_kernel");
}

}  // namespace

merit_status launch_sad(const merit_plan& plan, const void* a, const void* b, void* out, void* aux,
                        void* stream) {
  const SadParams& p = plan.sad;
  const uint8_t* cur = static_cast<const uint8_t*>(p.ref_is_b ? a : b);
  const uint8_t* ref = static_cast<const uint8_t*>(p.ref_is_b ? b : a);
  int32_t* ax = static_cast<int32_t*>(aux);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool wide = p.WY > 33;
  if (p.BH == 16) {
    return wide ? launch_sad_t<16, 13>(p, cur, ref, out, ax, s)
                : launch_sad_t<16, 11>(p, cur, ref, out, ax, s);
  }
  return wide ? launch_sad_t<8, 13>(p, cur, ref, out, ax, s)
              : launch_sad_t<8, 11>(p, cur, ref, out, ax, s);
}

}  // namespace merit_dev
