// K2 — L1 block matching (the motion-estimation workload, workloads.hpp:
// 255-279, with sad_program(2), workloads.hpp:64-68) plus the caller-side
// argmin stage the reference leaves to users.
//
// out[.., by, bx, dy, dx] = sum_{i<BH, j<BW} |cur[by*BH+i+cy, bx*BW+j+cx]
//                                           - ref[by*BH+dy+i+oy, bx*BW+dx+j+ox]|
// with the reference view's boundary rule (ZERO_PAD: 0 outside the frame,
// the semantics of oracle_motion_estimation, workloads.hpp:569-576; CLAMP:
// clamped coordinates).  On 8-bit frames every partial sum is an exact
// integer < 2^24, so the int32 result equals the reference's REAL32
// accumulation bit for bit.
//
// Design (sm_100a):
//  * Persistent CTAs (2 per SM).  A tile is TBX horizontally adjacent blocks
//    of one block row of one frame pair.  The Eq. 6 footprint of the tile's
//    reference window (footprint_box, view.hpp:143-149) is fetched with
//    cp.async into a raw smem buffer one tile AHEAD (double buffered), so
//    the global-memory latency hides behind the current tile's arithmetic.
//  * From the raw window the CTA builds FOUR byte-shifted word copies, so a
//    thread at any dx reads 32-bit aligned words with no per-thread PRMT.
//  * A thread owns one (block, dy-group of D rows, dx) item: the current
//    block lives in registers (BH x BW/4 words) and every reference row it
//    streams from smem is folded into all D displacement accumulators it
//    overlaps with VABSDIFF4.U8.ACC — 4 abs-diff-accumulates per
//    instruction (measured 64 lanes/clk/SM, tools/microbench/int_simd.cu).
//  * Argmin: per-thread min over its D rows, then a shared-memory atomicMin
//    on the packed key (sad << 16 | dy*WX + dx): lowest SAD, then lowest
//    raster index — the tie-break BASELINE.json asks for.
#include <cstdlib>

#include "common.cuh"

namespace merit_dev {
namespace {

constexpr int kSadThreads = 256;     // 8 warps: 2 per SM sub-partition, 2 CTAs/SM at <= 128 regs
constexpr int kSadMaxThreads = kSadThreads;

__device__ __forceinline__ uint32_t vabsdiff4_acc(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 4 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct SadLaunch {
  SadParams p;
  int TBX;        // blocks per tile
  int G;          // dy groups
  int n_tiles_x;  // ceil(BX / TBX)
  long long n_tiles;
  int R;          // staged reference rows = G*D + BH - 1
  int span;       // staged reference columns = TBX*BW + WX - 1
  int Ww;         // words per staged row per copy
  int CS;         // words per shifted copy (padded to 8 mod 32 against bank conflicts)
  int rw;         // words per raw row (= Ww + 1)
  int items;      // TBX * WX * G
  int word_path;  // 4-byte aligned reference rows / current blocks
  int vec_path;   // 16-byte aligned reference rows
};

template <int BLK>
__device__ __forceinline__ void stage_tile(const SadLaunch& L, const uint8_t* __restrict__ cur,
                                           const uint8_t* __restrict__ ref, long long tile,
                                           uint32_t raw_s, uint8_t* raw, uint32_t cur_s,
                                           uint8_t* curs) {
  const SadParams& p = L.p;
  const int tx = static_cast<int>(tile % L.n_tiles_x);
  const long long t2 = tile / L.n_tiles_x;
  const int by = static_cast<int>(t2 % p.BY);
  const long long pair = t2 / p.BY;
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);
  const uint8_t* refp = ref + pair * (long long)p.Hr * p.Wr;
  const uint8_t* curp = cur + pair * (long long)p.Hc * p.Wc;
  const int ry0 = by * BLK + p.oy, rx0 = bx0 * BLK + p.ox;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  constexpr int BWW = BLK / 4;
  if (L.word_path && p.boundary == MERIT_ZERO_PAD) {
    if (L.vec_path) {
      const int rq = L.rw / 4;  // 16-byte chunks per raw row (rw % 4 == 0)
      for (int e = threadIdx.x; e < L.R * rq; e += blockDim.x) {
        const int r = e / rq, q = e - r * rq;
        const int y = ry0 + r, x = rx0 + 16 * q;
        const bool in = y >= 0 && y < p.Hr && 16 * q < L.span && x >= 0 && x + 16 <= p.Wr;
        cp_async16(raw_s + 16u * e, in ? refp + (long long)y * p.Wr + x : refp, in);
      }
    } else {
      for (int r = warp; r < L.R; r += nwarps) {
        const int y = ry0 + r;
        const bool yin = y >= 0 && y < p.Hr;
        const uint8_t* rowp = refp + (long long)(yin ? y : 0) * p.Wr;
        for (int w = lane; w < L.rw; w += 32) {
          const int x = rx0 + 4 * w;
          const bool in = yin && 4 * w < L.span && x >= 0 && x < p.Wr;
          cp_async4(raw_s + 4u * (r * L.rw + w), in ? rowp + x : refp, in);
        }
      }
    }
    for (int rr = warp; rr < L.TBX * BLK; rr += nwarps) {
      const int b = rr / BLK, r = rr - b * BLK;
      if (lane < BWW) {
        const bool in = b < nb;
        const int y = by * BLK + r + p.cy, x = (bx0 + b) * BLK + lane * 4 + p.cx;
        cp_async4(cur_s + 4u * (rr * BWW + lane), in ? curp + (long long)y * p.Wc + x : curp, in);
      }
    }
  } else {
    // Byte path (unaligned rows or CLAMP): synchronous, boundary per pixel.
    const int rawcols = 4 * L.rw;
    for (int r = warp; r < L.R; r += nwarps) {
      for (int c = lane; c < rawcols; c += 32) {
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
        raw[r * rawcols + c] = v;
      }
    }
    for (int rr = warp; rr < L.TBX * BLK; rr += nwarps) {
      const int b = rr / BLK, r = rr - b * BLK;
      for (int c = lane; c < BLK; c += 32) {
        uint8_t v = 0;
        if (b < nb) {
          const int y = by * BLK + r + p.cy, x = (bx0 + b) * BLK + c + p.cx;
          v = __ldg(curp + (long long)y * p.Wc + x);
        }
        curs[rr * BLK + c] = v;
      }
    }
  }
}

template <int BLK, int D>
__global__ void __launch_bounds__(kSadThreads, 2)
sad_kernel(const uint8_t* __restrict__ cur, const uint8_t* __restrict__ ref, void* __restrict__ out,
           int32_t* __restrict__ aux, SadLaunch L) {
  extern __shared__ __align__(16) uint32_t smem[];
  const SadParams& p = L.p;
  constexpr int BWW = BLK / 4;  // words per block row
  const int raw_words = L.R * L.rw;
  const int cur_words = L.TBX * BLK * BWW;
  // --- shared memory carve-up: raw[2] | cur[2] | keys | counters
  uint32_t* copies = smem;
  uint32_t* raw0 = copies + 4 * L.CS;
  uint32_t* cur0 = raw0 + 2 * raw_words;
  uint32_t* keys = cur0 + 2 * cur_words;   // per block: running argmin key
  uint32_t* cnt = keys + L.TBX;             // per block: contributions so far
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;

  // per-thread item: (block, dx); the thread walks all dy groups
  const int item = threadIdx.x;
  const int ib = item / p.WX;
  const int idx = item - ib * p.WX;
  const bool has_item = item < L.items;

  if (threadIdx.x < L.TBX) {
    keys[threadIdx.x] = 0xffffffffu;
    cnt[threadIdx.x] = 0u;
  }
  long long tile = blockIdx.x;
  int buf = 0;
  pdl_launch_dependents();
  pdl_wait();  // first global access follows
  if (tile < L.n_tiles) {
    stage_tile<BLK>(L, cur, ref, tile, smem_u32(raw0), reinterpret_cast<uint8_t*>(raw0),
                    smem_u32(cur0), reinterpret_cast<uint8_t*>(cur0));
    cp_async_commit();
  }
  for (; tile < L.n_tiles; tile += gridDim.x, buf ^= 1) {
    uint32_t* raw = raw0 + buf * raw_words;
    uint32_t* curw = cur0 + buf * cur_words;
    cp_async_wait_all();
    __syncthreads();  // raw[buf] landed; previous tile's compute finished
    // four byte-shifted word copies: copy_s[r][w] = bytes (4w+s .. 4w+s+3)
    for (int r = warp; r < L.R; r += nwarps) {
      for (int w = lane; w < L.Ww; w += 32) {
        const uint32_t lo = raw[r * L.rw + w];
        const uint32_t hi = raw[r * L.rw + w + 1];
        const int o = r * L.Ww + w;
        copies[o] = lo;
        copies[L.CS + o] = __byte_perm(lo, hi, 0x4321);
        copies[2 * L.CS + o] = __byte_perm(lo, hi, 0x5432);
        copies[3 * L.CS + o] = __byte_perm(lo, hi, 0x6543);
      }
    }
    __syncthreads();
    // prefetch the next tile into the other buffer while this one computes
    const long long next = tile + gridDim.x;
    if (next < L.n_tiles) {
      stage_tile<BLK>(L, cur, ref, next, smem_u32(raw0 + (buf ^ 1) * raw_words),
                      reinterpret_cast<uint8_t*>(raw0 + (buf ^ 1) * raw_words),
                      smem_u32(cur0 + (buf ^ 1) * cur_words),
                      reinterpret_cast<uint8_t*>(cur0 + (buf ^ 1) * cur_words));
      cp_async_commit();
    }
    // tile coordinates
    const int tx = static_cast<int>(tile % L.n_tiles_x);
    const long long t2 = tile / L.n_tiles_x;
    const int by = static_cast<int>(t2 % p.BY);
    const long long pair = t2 / p.BY;
    const int bx0 = tx * L.TBX;
    const int nb = min(L.TBX, p.BX - bx0);
    if (has_item && ib < nb) {
      uint32_t cw[BLK][BWW];
      const uint32_t* cb = curw + ib * BLK * BWW;
#pragma unroll
      for (int i = 0; i < BLK; ++i)
#pragma unroll
        for (int j = 0; j < BWW; ++j) cw[i][j] = cb[i * BWW + j];
      const int col = ib * BLK + idx;  // byte column in the staged window
      const uint32_t* cp0 = copies + (col & 3) * L.CS + (col >> 2);
      const long long blk_index = (pair * p.BY + by) * (long long)p.BX + bx0 + ib;
      uint32_t best = 0xffffffffu;
      for (int ig = 0; ig < L.G; ++ig) {
        const uint32_t* cp = cp0 + ig * D * L.Ww;
        uint32_t acc[D];
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] = 0;
#pragma unroll
        for (int r = 0; r < D + BLK - 1; ++r) {
          uint32_t rwv[BWW];
#pragma unroll
          for (int j = 0; j < BWW; ++j) rwv[j] = cp[j];
          cp += L.Ww;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const int i = r - d;
            if (i >= 0 && i < BLK) {
#pragma unroll
              for (int j = 0; j < BWW; ++j) acc[d] = vabsdiff4_acc(cw[i][j], rwv[j], acc[d]);
            }
          }
        }
        const int dy0 = ig * D;
        const int nd = min(D, p.WY - dy0);
        uint32_t key = (static_cast<uint32_t>(dy0) * p.WX + idx);
        const uint32_t kstep = static_cast<uint32_t>(p.WX);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const uint32_t k = (acc[d] << 16) | (key + d * kstep);
          if (d < nd) best = k < best ? k : best;
        }
        if (p.write_map) {
          const long long obase = (blk_index * p.WY + dy0) * p.WX + idx;
          if (p.out_f32) {
            float* o = static_cast<float*>(out) + obase;
#pragma unroll
            for (int d = 0; d < D; ++d)
              if (d < nd) __stcs(o + d * p.WX, static_cast<float>(acc[d]));
          } else {
            int32_t* o = static_cast<int32_t*>(out) + obase;
#pragma unroll
            for (int d = 0; d < D; ++d)
              if (d < nd) __stcs(o + d * p.WX, static_cast<int32_t>(acc[d]));
          }
        }
      }
      if (p.argmin) {
        // Barrier-free per-block argmin: every (block, dx) thread folds its key
        // in; the thread that arrives last writes the record and re-arms the
        // slot for the next tile (the next tile's atomics follow the barrier at
        // the top of the loop).
        atomicMin(&keys[ib], best);
        __threadfence_block();
        if (atomicAdd(&cnt[ib], 1u) == static_cast<uint32_t>(p.WX - 1)) {
          __threadfence_block();
          const uint32_t key = atomicExch(&keys[ib], 0xffffffffu);
          cnt[ib] = 0u;
          const int k = static_cast<int>(key & 0xffffu);
          const int dy = k / p.WX, dx = k - (k / p.WX) * p.WX;
          int32_t* a = aux + blk_index * 3;
          a[0] = dy + p.oy - p.cy;
          a[1] = dx + p.ox - p.cx;
          a[2] = static_cast<int32_t>(key >> 16);
        }
      }
    }
  }
  cp_async_wait_all();
}

template <int BLK, int D>
merit_status launch_sad_t(const SadParams& p, const uint8_t* cur, const uint8_t* ref, void* out,
                          int32_t* aux, cudaStream_t s) {
  SadLaunch L;
  L.p = p;
  L.G = (p.WY + D - 1) / D;
  const int per_block = p.WX;
  if (per_block > kSadMaxThreads)
    return fail(MERIT_E_UNSUPPORTED_VIEW, "search window too wide for the SAD kernel");
  // Blocks per tile: least idle-lane fraction within the thread budget.
  L.TBX = 1;
  double best_waste = 2.0;
  for (int t = 1; t <= 16 && t <= p.BX; ++t) {
    const int items = t * per_block;
    const int threads = (items + 31) / 32 * 32;
    if (threads > kSadMaxThreads) break;
    const double waste = double(threads - items) / threads;
    if (waste < best_waste - 0.02) {
      best_waste = waste;
      L.TBX = t;
    }
  }
  L.items = L.TBX * per_block;
  L.n_tiles_x = (p.BX + L.TBX - 1) / L.TBX;
  L.n_tiles = p.pairs * (long long)p.BY * L.n_tiles_x;
  L.R = L.G * D + BLK - 1;
  L.span = L.TBX * BLK + p.WX - 1;
  L.Ww = (L.span + 3) / 4;
  L.rw = (L.Ww + 1 + 3) / 4 * 4;  // raw rows (+1 word for the shift) padded to 16-byte chunks
  L.CS = L.R * L.Ww;
  L.CS += ((8 - (L.CS % 32)) + 32) % 32;
  L.word_path = ((p.ox % 4) == 0 && (p.cx % 4) == 0 && (p.Wr % 4) == 0 && (p.Wc % 4) == 0 &&
                 (reinterpret_cast<uintptr_t>(cur) % 4) == 0 && (reinterpret_cast<uintptr_t>(ref) % 4) == 0)
                    ? 1 : 0;
  L.vec_path = (L.word_path && (p.ox % 16) == 0 && (p.Wr % 16) == 0 && (BLK % 16) == 0 &&
                (reinterpret_cast<uintptr_t>(ref) % 16) == 0) ? 1 : 0;
  const size_t smem = 4ull * (4ull * L.CS + 2ull * L.R * L.rw + 2ull * L.TBX * BLK * (BLK / 4) + 2ull * L.TBX);
  if (L.n_tiles == 0) return MERIT_OK;
  if (smem > 110 * 1024) return fail(MERIT_E_UNSUPPORTED_VIEW, "SAD footprint exceeds shared memory");
  auto kern = sad_kernel<BLK, D>;
  cudaError_t e = set_smem_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(sad)");
  const int threads = (L.items + 31) / 32 * 32;
  long long grid = 2LL * num_sms();
  if (grid > L.n_tiles) grid = L.n_tiles;
  e = launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(threads), smem, s, 1, cur, ref, out, aux, L);
  if (e != cudaSuccess) return cuda_check(e, "launch(sad)");
  return launch_status("sad_kernel");
}

}  // namespace

// Kernel variant for a window: D rows per thread such that WX * ceil(WY/D)
// fits the thread budget.  Used by the lowering to decide eligibility.
int sad_rows_per_thread(int BH, int WY, int WX) {
  if (WX > kSadMaxThreads || WY > 256) return 0;
  if (BH == 16) {
    const char* e = getenv("MERIT_SAD_D");  // tuning override: 11 or 33
    if (WY <= 33) return (e && atoi(e) == 11) ? 11 : 33;
    return 17;
  }
  return WY <= 33 ? 11 : 22;
}

merit_status launch_sad(const merit_plan& plan, const void* a, const void* b, void* out, void* aux,
                        void* stream) {
  const SadParams& p = plan.sad;
  const uint8_t* cur = static_cast<const uint8_t*>(p.ref_is_b ? a : b);
  const uint8_t* ref = static_cast<const uint8_t*>(p.ref_is_b ? b : a);
  int32_t* ax = static_cast<int32_t*>(aux);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int D = sad_rows_per_thread(p.BH, p.WY, p.WX);
  if (p.BH == 16) {
    if (D == 33) return launch_sad_t<16, 33>(p, cur, ref, out, ax, s);
    if (D == 11) return launch_sad_t<16, 11>(p, cur, ref, out, ax, s);
    if (D == 17) return launch_sad_t<16, 17>(p, cur, ref, out, ax, s);
  } else {
    if (D == 11) return launch_sad_t<8, 11>(p, cur, ref, out, ax, s);
    if (D == 22) return launch_sad_t<8, 22>(p, cur, ref, out, ax, s);
  }
  return fail(MERIT_E_UNSUPPORTED_VIEW, "no SAD kernel variant for this window");
}

}  // namespace merit_dev
