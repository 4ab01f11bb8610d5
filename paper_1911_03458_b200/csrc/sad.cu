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
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "tmap.cuh"

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
  int n_tiles;
  int R;          // staged reference rows = G*D + BH - 1
  int span;       // staged reference columns = TBX*BW + WX - 1
  int Ww;         // words per staged row per copy
  int CS;         // words per shifted copy (padded to 8 mod 32 against bank conflicts)
  int rw;         // words per raw row (= Ww + 1)
  int items;      // TBX * WX * G
  int word_path;  // 4-byte aligned reference rows / current blocks
  int vec_path;   // 16-byte aligned reference rows
  int tma;        // reference window + current blocks staged by TMA (ZERO_PAD)
  int R_box;      // TMA box rows (= R)
  int nby;        // block rows per tile / per thread (1, or 2 for 8x8 blocks on the TMA path)
  int BYT;        // tile rows = ceil(BY / nby)
  int cur_pitch;  // bytes per staged current-frame row: TBX*BW rounded up to 16
  uint32_t raw_buf, cur_buf;  // bytes per raw / current buffer (128-byte multiples)
  uint32_t ntx_m, ntx_s;      // n / n_full_x as a multiply-high (fast_div)
  int n_full_x;               // full (TBX-block) tiles per block row
  int n_full_tiles;           // tiles [0, n_full_tiles) are full; the partial last
                              // tiles of every row follow (cheap ones in the final wave)
  uint32_t byt_m, byt_s;      // n / BYT
  int cp_sr, cp_sw;           // copy builder: blockDim.x = cp_sr * Ww + cp_sw
  int by0, by1;               // block-row band [by0, by1) of this launch
  int dbl;                    // double-buffered shifted copies: one barrier per tile (TMA staging)
  int dbg;                    // timing experiments (MERIT_SAD_DBG): 1 skip the copy builder, 2 skip the epilogue
  uint32_t key_mul;           // 65536 as a launch parameter: argmin keys acc * key_mul + d * WX
                              // stay IMADs (FMA pipe) instead of folding into ALU shift-adds
  uint32_t one;               // 1 as a launch parameter: sums written as IMADs (FMA pipe)
  int fast_build;             // fused kernel: the staged geometry is the compile-time one
                              // (sad_build_copies_fused) and the window starts word-aligned
  int dref_w;                 // fused kernel: words of the staged rows before the window
};

// n / d for n < 2^31 by multiply-high (Granlund-Montgomery): s = ceil(log2 d),
// m = floor(2^32 (2^s - d) / d) + 1.  Replaces the ~25-instruction signed
// division the compiler emits per tile.
inline void fast_div_init(uint32_t d, uint32_t& m, uint32_t& s) {
  s = 0;
  while ((1ull << s) < d) ++s;
  m = static_cast<uint32_t>(((1ull << 32) * ((1ull << s) - d)) / d + 1);
}
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t m, uint32_t s) {
  return (__umulhi(n, m) + n) >> s;
}

// Tile order: every full tile first (row-major over (pair, block row), TBX
// blocks each), then the partial last tile of every row.  The partial tiles
// carry BX % TBX blocks (C2: 1 of 7), so the ragged final wave is made of
// cheap tiles instead of full ones.  t2 = pair * BYT + tile row, tx = tile column.
__device__ __forceinline__ void sad_tile_coords(int tile, int n_full_tiles, int n_full_x, uint32_t m, uint32_t s,
                                                int& t2, int& tx) {
  if (tile < n_full_tiles) {
    t2 = static_cast<int>(fast_div(static_cast<uint32_t>(tile), m, s));
    tx = tile - t2 * n_full_x;
  } else {
    t2 = tile - n_full_tiles;
    tx = n_full_x;
  }
}

template <int BLK>
__device__ __forceinline__ void stage_tile(const SadLaunch& L, const uint8_t* __restrict__ cur,
                                           const uint8_t* __restrict__ ref, int tile,
                                           uint32_t raw_s, uint8_t* raw, uint32_t cur_s,
                                           uint8_t* curs) {
  const SadParams& p = L.p;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const long long pair = fast_div(t2, L.byt_m, L.byt_s);
  const int by = L.by0 + t2 - static_cast<int>(pair) * L.BYT;  // nby == 1 on this path
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
        cp_async4(cur_s + static_cast<uint32_t>(r * L.cur_pitch + b * BLK + 4 * lane),
                  in ? curp + (long long)y * p.Wc + x : curp, in);
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
        curs[r * L.cur_pitch + b * BLK + c] = v;
      }
    }
  }
}

// TMA boxes of 8-bit tensors must start at a 16-byte multiple in the
// innermost dimension (measured on sm_100a, tools/microbench/tma_u8.cu: any
// other start faults with an illegal instruction), so boxes start at
// floor16(x) and the kernel skips the 0..15 leading bytes.
__host__ __device__ __forceinline__ int floor16(int x) { return x >= 0 ? (x & ~15) : -((-x + 15) & ~15); }

__device__ __forceinline__ void sad_tma_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z,
                                           uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void sad_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
#ifdef MERIT_SAD_SUSPEND
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, " MERIT_SAD_SUSPEND ";\n\t"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
#endif
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// The TMA part of a tile's staging, issued by the calling thread.
template <int BLK>
__device__ __forceinline__ void issue_tile_tma(const SadLaunch& L, const CUtensorMap* ref_map,
                                               const CUtensorMap* cur_map, int tile, uint32_t raw_s,
                                               uint32_t cur_s, uint32_t bar) {
  const SadParams& p = L.p;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int pair = static_cast<int>(fast_div(t2, L.byt_m, L.byt_s));
  const int by = L.by0 + (t2 - pair * L.BYT) * L.nby;
  const int bx0 = tx * L.TBX;
  const uint32_t bytes = L.R_box * L.rw * 4 + L.nby * BLK * L.cur_pitch;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  sad_tma_3d(raw_s, ref_map, floor16(bx0 * BLK + p.ox), by * BLK + p.oy, pair, bar);
  sad_tma_3d(cur_s, cur_map, floor16(bx0 * BLK + p.cx), by * BLK + p.cy, pair, bar);
}

// One tile's staging: TMA (one 3-D box for the reference window, one for the
// current blocks, completion on the buffer's mbarrier; zero fill outside the
// frame = ZERO_PAD) or the cp.async / byte paths.
template <int BLK>
__device__ __forceinline__ void issue_tile(const SadLaunch& L, const uint8_t* __restrict__ cur,
                                           const uint8_t* __restrict__ ref, const CUtensorMap* ref_map,
                                           const CUtensorMap* cur_map, int tile, uint32_t raw_s, uint8_t* raw,
                                           uint32_t cur_s, uint8_t* curs, uint32_t bar) {
  if (L.tma) {
    if (threadIdx.x == 0) issue_tile_tma<BLK>(L, ref_map, cur_map, tile, raw_s, cur_s, bar);
  } else {
    stage_tile<BLK>(L, cur, ref, tile, raw_s, raw, cur_s, curs);
    cp_async_commit();
  }
}

// One SAD-map entry: int32, float (a REAL32 map) or uint16 (exact: every
// 8-bit 8x8 / 16x16 SAD is <= 65,280), streaming store.
__device__ __forceinline__ void sad_store1(void* out, const SadParams& p, long long i, uint32_t v) {
  if (p.out_f32) __stcs(static_cast<float*>(out) + i, static_cast<float>(v));
  else if (p.out_u16) __stcs(static_cast<unsigned short*>(out) + i, static_cast<unsigned short>(v));
  else __stcs(static_cast<int32_t*>(out) + i, static_cast<int32_t>(v));
}

// SAD-map rows d < nd of one (block, dx) thread: out[obase + d * WX]
// (int32, float for a REAL32 map, or uint16), streaming stores.
template <int D>
__device__ __forceinline__ void sad_store_map(void* out, int out_f32, long long obase, int WX, const uint32_t* acc,
                                              int nd, int out_u16 = 0) {
  if (out_f32) {
    float* o = static_cast<float*>(out) + obase;
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < nd) __stcs(o + d * WX, static_cast<float>(acc[d]));
  } else if (out_u16) {
    unsigned short* o = static_cast<unsigned short*>(out) + obase;
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < nd) __stcs(o + d * WX, static_cast<unsigned short>(acc[d]));
  } else {
    int32_t* o = static_cast<int32_t*>(out) + obase;
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < nd) __stcs(o + d * WX, static_cast<int32_t>(acc[d]));
  }
}

// WXC: the displacement-window width as a compile-time constant (0 = runtime
// p.WX).  A constant width turns the per-displacement key and SAD-map store
// offsets into immediates (the epilogue was ~8% of the issued instructions).
// The four byte-shifted word copies of a tile's staged reference window:
// copy_s[r][w] = window bytes (4w+s .. 4w+s+3), one (row, word) per thread per
// step over the flattened R x Ww range, starting at (cp_r0, cp_w0).
template <int BLK>
__device__ __forceinline__ void sad_build_copies(const SadLaunch& L, int tile, const uint32_t* raw,
                                                 uint32_t* copies, int cp_r0, int cp_w0) {
  const SadParams& p = L.p;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int bx0 = tx * L.TBX;
  // leading bytes of the staged rows before the window (TMA boxes start at
  // a 16-byte multiple)
  const int dref = L.tma ? (bx0 * BLK + p.ox) - floor16(bx0 * BLK + p.ox) : 0;
  const uint32_t cs4 = static_cast<uint32_t>(L.CS) * 4u;
  const uint32_t raw_s = smem_u32(raw) + static_cast<uint32_t>(dref >> 2) * 4u;
  const uint32_t cop_s = smem_u32(copies);
  const int dr = dref & 3;
  int r = (L.dbg & 1) ? L.R : cp_r0, w = cp_w0;
  while (r < L.R) {
    const uint32_t ra = raw_s + static_cast<uint32_t>(r * L.rw + w) * 4u;
    const uint32_t ca = cop_s + static_cast<uint32_t>(r * L.Ww + w) * 4u;
    uint32_t a0, a1, a2;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a0) : "r"(ra));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a1) : "r"(ra + 4));
    uint32_t c0, c1, c2, c3;
    if (dr == 0) {
      c0 = a0;
      c1 = __byte_perm(a0, a1, 0x4321);
      c2 = __byte_perm(a0, a1, 0x5432);
      c3 = __byte_perm(a0, a1, 0x6543);
    } else {
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a2) : "r"(ra + 8));
      c0 = __funnelshift_r(a0, a1, 8 * dr);
      c1 = dr + 1 < 4 ? __funnelshift_r(a0, a1, 8 * (dr + 1)) : a1;
      c2 = dr + 2 < 4 ? __funnelshift_r(a0, a1, 8 * (dr + 2)) : __funnelshift_r(a1, a2, 8 * (dr - 2));
      c3 = __funnelshift_r(a1, a2, 8 * (dr - 1));
    }
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca), "r"(c0) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + cs4), "r"(c1) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + 2 * cs4), "r"(c2) : "memory");
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + 3 * cs4), "r"(c3) : "memory");
    w += L.cp_sw;
    r += L.cp_sr;
    if (w >= L.Ww) {
      w -= L.Ww;
      ++r;
    }
  }
}

// Compile-time staging geometry of the warp-per-block kernels (8-block tiles,
// TMA staging), the values the launcher derives at run time:
// span = 8 BLK + WX - 1 bytes, Ww = ceil(span / 4) made odd, R = G D + NBY BLK
// - 1 rows, raw rows of rw = 4 ceil((Ww + 5) / 4) words, CS = R Ww padded to 8
// mod 32.  C2 (16x16, +/-16): Ww 41, R 48, rw 48,
// CS 1992; C5 8x8 / fused (+/-32, two block rows): Ww 33, R 81, rw 40, CS 2696.
template <int BLK, int WX, int NBY>
struct WarpGeo {
  static constexpr int D = 33, G = (WX + D - 1) / D;
  static constexpr int span = 8 * BLK + WX - 1;
  static constexpr int WW = ((span + 3) / 4) | 1;
  static constexpr int R = G * D + NBY * BLK - 1;
  static constexpr int RW = (WW + 5 + 3) / 4 * 4;
  static constexpr int CS = R * WW + ((8 - (R * WW) % 32) + 32) % 32;
};
using FusedGeo = WarpGeo<8, 65, 2>;
constexpr int kFusedCPW = (8 * 8 + 12 + 15) / 16 * 16 / 4;  // fused kernel: words per staged current row
static_assert(FusedGeo::WW == 33 && FusedGeo::R == 81 && FusedGeo::RW == 40 && FusedGeo::CS == 2696, "fused geometry");
static_assert(WarpGeo<16, 33, 1>::WW == 41 && WarpGeo<16, 33, 1>::CS == 1992, "C2 geometry");

// The warp kernels' copy builder on that fixed geometry, for windows that
// start on a word: item it = (r, w) of the flattened R x Ww walk reads raw
// word it + (rw - Ww) r and writes copy word it of each of the four byte
// shifts: no per-item row/column bookkeeping (the generic builder spends ~45
// instructions per item on it).
template <class GEO, int NT>
__device__ __forceinline__ void sad_build_copies_geo(const uint32_t* raw, uint32_t* copies) {
  constexpr int N = GEO::R * GEO::WW;
  const uint32_t raw_s = smem_u32(raw), cop_s = smem_u32(copies);
#pragma unroll
  for (int k = 0; k < (N + NT - 1) / NT; ++k) {
    const int it = static_cast<int>(threadIdx.x) + k * NT;
    if ((k + 1) * NT <= N || it < N) {
      const int r = it / GEO::WW;
      const uint32_t ra = raw_s + static_cast<uint32_t>(it + (GEO::RW - GEO::WW) * r) * 4u;
      const uint32_t ca = cop_s + static_cast<uint32_t>(it) * 4u;
      uint32_t a0, a1;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a0) : "r"(ra));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a1) : "r"(ra + 4));
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca), "r"(a0) : "memory");
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + 4 * GEO::CS), "r"(__byte_perm(a0, a1, 0x4321)) : "memory");
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + 8 * GEO::CS), "r"(__byte_perm(a0, a1, 0x5432)) : "memory");
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(ca + 12 * GEO::CS), "r"(__byte_perm(a0, a1, 0x6543)) : "memory");
    }
  }
}

// One tile's matching for this thread's (block, dx) item: the current
// block(s) into registers from the staged rows, `after_cw()` (called by every
// thread of the CTA once the staged current rows are no longer needed), the
// SAD accumulation over the shifted copies, then the SAD-map stores and the
// argmin fold into keys / cnt.
template <int BLK, int D, int NBY, int WXC, typename AfterCw>
__device__ __forceinline__ void sad_tile_work(const SadLaunch& L, void* __restrict__ out, int32_t* __restrict__ aux,
                                              int tile, const uint32_t* curw, const uint32_t* copies,
                                              uint32_t* keys, uint32_t* cnt, AfterCw after_cw) {
  const SadParams& p = L.p;
  const int WX = WXC ? WXC : p.WX;
  constexpr int BWW = BLK / 4;  // words per block row
  const int cpw = L.cur_pitch / 4;  // words per staged current row
  const int item = threadIdx.x;
  const int ib = item / WX;
  const int idx = item - ib * WX;
  const bool has_item = item < L.items;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int pair_i = static_cast<int>(fast_div(t2, L.byt_m, L.byt_s));
  const int by = L.by0 + (t2 - pair_i * L.BYT) * NBY;  // first block row of the tile
  const long long pair = pair_i;
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);
  const int dcur = L.tma ? (bx0 * BLK + p.cx) - floor16(bx0 * BLK + p.cx) : 0;
  // lanes with an item in this tile (warp-converged here; the argmin
  // folds each block's lanes with a warp reduction before the shared atomics)
  const unsigned act = __ballot_sync(0xffffffffu, has_item && ib < nb);
  // current blocks (NBY block rows) in registers: rows of cur_pitch bytes,
  // block ib at byte dcur + ib*BLK (dcur % 4 == 0), block row n at row n*BLK
  uint32_t cw[NBY][BLK][BWW];
  if (has_item && ib < nb) {
    const uint32_t* cb = curw + (dcur >> 2) + ib * BWW;
    if (BWW == 4 && ((dcur & 15) == 0)) {
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int i = 0; i < BLK; ++i) {
          const uint4 q4 = *reinterpret_cast<const uint4*>(cb + (n * BLK + i) * cpw);
          cw[n][i][0] = q4.x; cw[n][i][1 % BWW] = q4.y; cw[n][i][2 % BWW] = q4.z; cw[n][i][3 % BWW] = q4.w;
        }
    } else {
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int i = 0; i < BLK; ++i)
#pragma unroll
          for (int j = 0; j < BWW; ++j) cw[n][i][j] = cb[(n * BLK + i) * cpw + j];
    }
  }
  after_cw();
  if (!(has_item && ib < nb)) return;
  const int col = ib * BLK + idx;  // byte column in the staged window
  const uint32_t* cp0 = copies + (col & 3) * L.CS + (col >> 2);
  const long long blk_index = (pair * p.BY + by) * (long long)p.BX + bx0 + ib;
  uint32_t best[NBY];
#pragma unroll
  for (int n = 0; n < NBY; ++n) best[n] = 0xffffffffu;
  for (int ig = 0; ig < L.G; ++ig) {
    const uint32_t* cp = cp0 + ig * D * L.Ww;
    uint32_t acc[NBY][D];
#pragma unroll
    for (int n = 0; n < NBY; ++n)
#pragma unroll
      for (int d = 0; d < D; ++d) acc[n][d] = 0;
    // block row n at displacement d reads staged row r = n*BLK + d + i:
    // every loaded reference word feeds all NBY block rows
#pragma unroll
    for (int r = 0; r < D + NBY * BLK - 1; ++r) {
      uint32_t rwv[BWW];
#pragma unroll
      for (int j = 0; j < BWW; ++j) rwv[j] = cp[j];
      cp += L.Ww;
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int i = r - d - n * BLK;
          if (i >= 0 && i < BLK) {
#pragma unroll
            for (int j = 0; j < BWW; ++j) acc[n][d] = vabsdiff4_acc(cw[n][i][j], rwv[j], acc[n][d]);
          }
        }
    }
    if (L.dbg & 2) {
      uint32_t x = 0;
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int d = 0; d < D; ++d) x ^= acc[n][d];
      best[0] ^= x;
      continue;
    }
    const int dy0 = ig * D;
    const int nd = min(D, p.WY - dy0);
    // argmin key = sad << 16 | (dy * WX + dx): the per-thread part
    // dy0 * WX + idx is added after the min (it does not change the order)
    const uint32_t key0 = static_cast<uint32_t>(dy0 * WX + idx);
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      uint32_t bn = 0xffffffffu;
      const bool store = p.write_map && by + n < L.by1;
      const long long obase = ((blk_index + n * (long long)p.BX) * p.WY + dy0) * WX + idx;
      // keys on the FMA pipe (IMAD), mins on the ALU: the ALU is the
      // VABSDIFF4 pipe.  Full groups and the one-short last group of an
      // odd window (C5: 65 = 33 + 32) need no per-displacement predicates.
      const uint32_t kmul = L.key_mul;
      if (nd == D) {
#pragma unroll
        for (int d = 0; d < D; ++d) bn = min(bn, acc[n][d] * kmul + static_cast<uint32_t>(d * WX));
        if (store) sad_store_map<D>(out, p.out_f32, obase, WX, acc[n], D, p.out_u16);
      } else if (WXC != 0 && nd == D - 1) {
#pragma unroll
        for (int d = 0; d < D - 1; ++d) bn = min(bn, acc[n][d] * kmul + static_cast<uint32_t>(d * WX));
        if (store) sad_store_map<D>(out, p.out_f32, obase, WX, acc[n], D - 1, p.out_u16);
      } else {
#pragma unroll
        for (int d = 0; d < D; ++d)
          if (d < nd) bn = min(bn, acc[n][d] * kmul + static_cast<uint32_t>(d * WX));
        if (store) sad_store_map<D>(out, p.out_f32, obase, WX, acc[n], nd, p.out_u16);
      }
      best[n] = min(best[n], bn + key0);
    }
  }
  if ((L.dbg & 2) && best[0] == 0x12345u) aux[0] = 1;  // keep the work live
  if (p.argmin && !(L.dbg & 2)) {
    // Barrier-free per-block argmin: every (block, dx) thread folds its key
    // in; the thread that arrives last writes the record and re-arms the
    // slot for a later tile.
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      if (by + n >= L.by1) break;
      const int slot = n * L.TBX + ib;
      // the lanes of this warp on the same block fold their keys first
      // (REDUX): one shared atomic per (warp, block) instead of one per lane
      const unsigned grp = __match_any_sync(act, slot);
      const uint32_t wmin = __reduce_min_sync(grp, best[n]);
      const int lane = threadIdx.x & 31;
      if (lane != __ffs(grp) - 1) continue;
      atomicMin(&keys[slot], wmin);
      __threadfence_block();
      const uint32_t np = static_cast<uint32_t>(__popc(grp));
      if (atomicAdd(&cnt[slot], np) == static_cast<uint32_t>(WX) - np) {
        __threadfence_block();
        const uint32_t key = atomicExch(&keys[slot], 0xffffffffu);
        cnt[slot] = 0u;
        const int k = static_cast<int>(key & 0xffffu);
        const int dy = k / WX, dx = k - (k / WX) * WX;
        int32_t* a = aux + (blk_index + n * (long long)p.BX) * 3;
        a[0] = dy + p.oy - p.cy;
        a[1] = dx + p.ox - p.cx;
        a[2] = static_cast<int32_t>(key >> 16);
      }
    }
  }
}

// Warp-per-block matching for a square window of 32k + 1 displacements per
// axis (WXC = 33: the +/-16 search of C2; 65: +/-32, C5): the k warps of a
// block column own its columns dx = 32 w + lane for every dy (dy groups of
// D = 33 accumulators per block row, the loop of sad_tile_work; NBY = 2
// vertically adjacent 8x8 blocks share every loaded reference word), and the
// last column dx = 32k is split over the lanes: lane l of warp w also
// matches (dy = 32 w + l, dx = 32k) in a side loop, and the corner
// (dy = 32k, dx = 32k) is shared by the last warp (two products per lane,
// REDUX sum).  Every lane does useful work (C2: 231 of 256 lanes in the
// (block, dx) mapping), tiles are 8 block columns wide (C2: 120 = 15 x 8, no
// partial tiles) and the argmin is a warp REDUX per block (plus one shared
// atomic per warp when k = 2).
template <int BLK, int NBY, int WXC, typename AfterCw>
__device__ __forceinline__ void sad_tile_work_warp(const SadLaunch& L, void* __restrict__ out,
                                                   int32_t* __restrict__ aux, int tile, const uint32_t* curw,
                                                   const uint32_t* copies, uint32_t* keys, uint32_t* cnt,
                                                   AfterCw after_cw) {
  constexpr int D = 33, WX = WXC, WY = WXC, BWW = BLK / 4;
  constexpr int WPB = (WX - 1) / 32;  // warps per block column
  constexpr int WW = WarpGeo<BLK, WX, NBY>::WW;  // staged row pitch in words (the launcher checks L.Ww)
  constexpr int G = (WY + D - 1) / D;
  const SadParams& p = L.p;
  const int cpw = L.cur_pitch / 4;
  const int warp = static_cast<int>(threadIdx.x) >> 5;
  const int ib = warp / WPB, wsub = warp - (warp / WPB) * WPB;
  const int lane = static_cast<int>(threadIdx.x) & 31;
  const int dxl = 32 * wsub + lane;  // this lane's column
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int pair_i = static_cast<int>(fast_div(t2, L.byt_m, L.byt_s));
  const int by = L.by0 + (t2 - pair_i * L.BYT) * NBY;  // first block row of the tile
  const long long pair = pair_i;
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);
  if (ib >= nb) {  // warp-uniform
    after_cw();
    return;
  }
  const int dcur = L.tma ? (bx0 * BLK + p.cx) - floor16(bx0 * BLK + p.cx) : 0;
  // current blocks in registers: block row n at staged rows n*BLK .., bytes dcur + ib*BLK
  const uint32_t* cb = curw + (dcur >> 2) + ib * BWW;
  uint32_t cw[NBY][BLK][BWW];
  if (BWW == 4 && (dcur & 15) == 0) {
#pragma unroll
    for (int n = 0; n < NBY; ++n)
#pragma unroll
      for (int i = 0; i < BLK; ++i) {
        const uint4 q4 = *reinterpret_cast<const uint4*>(cb + (n * BLK + i) * cpw);
        cw[n][i][0] = q4.x; cw[n][i][1 % BWW] = q4.y; cw[n][i][2 % BWW] = q4.z; cw[n][i][3 % BWW] = q4.w;
      }
  } else {
#pragma unroll
    for (int n = 0; n < NBY; ++n)
#pragma unroll
      for (int i = 0; i < BLK; ++i)
#pragma unroll
        for (int j = 0; j < BWW; ++j) cw[n][i][j] = cb[(n * BLK + i) * cpw + j];
  }
  // the corner's current-block words (lane-dependent rows: not from cw), read
  // before the staged rows are released
  constexpr int PER = BLK * BWW / 32;  // words per lane: 2 (16x16) or 0 (8x8: 16 lanes, one word)
  uint32_t ccw[NBY][PER >= 1 ? PER : 1];
  if (wsub == WPB - 1) {
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      if constexpr (PER >= 1) {
        const int i = lane / (BWW / PER), j0 = PER * (lane % (BWW / PER));
#pragma unroll
        for (int q = 0; q < PER; ++q) ccw[n][q] = cb[(n * BLK + i) * cpw + j0 + q];
      } else {
        ccw[n][0] = lane < BLK * BWW ? cb[(n * BLK + lane / BWW) * cpw + lane % BWW] : 0u;
      }
    }
  }
  after_cw();
  const long long blk_index = (pair * p.BY + by) * (long long)p.BX + bx0 + ib;
  const uint32_t kmul = L.key_mul;
  uint32_t best[NBY];
#pragma unroll
  for (int n = 0; n < NBY; ++n) best[n] = 0xffffffffu;
  const int col = ib * BLK + dxl;  // byte column of this lane's dx in the staged window
#pragma unroll 1
  for (int ig = 0; ig < G; ++ig) {
    const uint32_t* cp = copies + (col & 3) * L.CS + (col >> 2) + ig * D * WW;
    uint32_t acc[NBY][D];
#pragma unroll
    for (int n = 0; n < NBY; ++n)
#pragma unroll
      for (int d = 0; d < D; ++d) acc[n][d] = 0;
#pragma unroll
    for (int r = 0; r < D + NBY * BLK - 1; ++r) {
      uint32_t rwv[BWW];
#pragma unroll
      for (int j = 0; j < BWW; ++j) rwv[j] = cp[j];
      cp += WW;
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int i = r - d - n * BLK;
          if (i >= 0 && i < BLK) {
#pragma unroll
            for (int j = 0; j < BWW; ++j) acc[n][d] = vabsdiff4_acc(cw[n][i][j], rwv[j], acc[n][d]);
          }
        }
    }
    // the last group of a 65-row window has 32 rows (65 = 33 + 32)
    const int nd = (ig + 1) * D <= WY ? D : WY - ig * D;
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      const bool store = p.write_map && by + n < L.by1;
      const long long obase = ((blk_index + n * (long long)p.BX) * WY + ig * D) * WX + dxl;
      uint32_t bn = 0xffffffffu;
      if (nd == D) {
#pragma unroll
        for (int d = 0; d < D; ++d) bn = min(bn, acc[n][d] * kmul + static_cast<uint32_t>(d * WX));
        if (store) sad_store_map<D>(out, p.out_f32, obase, WX, acc[n], D, p.out_u16);
      } else {
#pragma unroll
        for (int d = 0; d < D - 1; ++d) bn = min(bn, acc[n][d] * kmul + static_cast<uint32_t>(d * WX));
        if (store) sad_store_map<D>(out, p.out_f32, obase, WX, acc[n], D - 1, p.out_u16);
      }
      best[n] = min(best[n], bn + static_cast<uint32_t>(ig * D * WX + dxl));
    }
  }
  // the last column dx = 32k (byte column ib*BLK + 32k: a multiple of 4,
  // shifted copy 0): this lane takes dy = dxl; block row n reads staged rows
  // dxl + n*BLK ..
  const int colx = ib * BLK + (WX - 1);
  const uint32_t* cx0 = copies + (colx & 3) * L.CS + (colx >> 2);
#pragma unroll
  for (int n = 0; n < NBY; ++n) {
    uint32_t ax = 0;
    const uint32_t* cx = cx0 + (dxl + n * BLK) * WW;
#pragma unroll
    for (int i = 0; i < BLK; ++i) {
#pragma unroll
      for (int j = 0; j < BWW; ++j) ax = vabsdiff4_acc(cw[n][i][j], cx[j], ax);
      cx += WW;
    }
    best[n] = min(best[n], ax * kmul + static_cast<uint32_t>(dxl * WX + (WX - 1)));
    const long long bb = (blk_index + n * (long long)p.BX) * (long long)(WY * WX);
    if (p.write_map && by + n < L.by1) {
      sad_store1(out, p, bb + dxl * WX + (WX - 1), ax);
    }
    if (wsub == WPB - 1) {
      // corner (dy = 32k, dx = 32k): BLK x BWW words over the 32 lanes
      uint32_t v = 0;
      if constexpr (PER >= 1) {
        const int i = lane / (BWW / PER), j0 = PER * (lane % (BWW / PER));
#pragma unroll
        for (int q = 0; q < PER; ++q) v = vabsdiff4_acc(ccw[n][q], cx0[(WY - 1 + n * BLK + i) * WW + j0 + q], v);
      } else if (lane < BLK * BWW) {
        const int i = lane / BWW, j = lane % BWW;
        v = vabsdiff4_acc(ccw[n][0], cx0[(WY - 1 + n * BLK + i) * WW + j], 0u);
      }
      const uint32_t axx = __reduce_add_sync(0xffffffffu, v);
      if (lane == 0) best[n] = min(best[n], axx * kmul + static_cast<uint32_t>((WY - 1) * WX + (WX - 1)));
      if (p.write_map && by + n < L.by1 && lane == 0) {
        sad_store1(out, p, bb + (WY - 1) * WX + (WX - 1), axx);
      }
    }
  }
  if (p.argmin) {
    // key = sad << 16 | (dy * WX + dx): lowest SAD, then lowest raster index
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      if (by + n >= L.by1) break;
      const uint32_t key = __reduce_min_sync(0xffffffffu, best[n]);
      if (lane != 0) continue;
      uint32_t fin = key;
      bool last = true;
      if (WPB > 1) {  // the block's warps meet in a shared slot; the last one writes
        const int slot = n * L.TBX + ib;
        atomicMin(&keys[slot], key);
        __threadfence_block();
        last = atomicAdd(&cnt[slot], 1u) == static_cast<uint32_t>(WPB - 1);
        if (last) {
          __threadfence_block();
          fin = atomicExch(&keys[slot], 0xffffffffu);
          cnt[slot] = 0u;
        }
      }
      if (last) {
        const int k = static_cast<int>(fin & 0xffffu);
        const int dy = k / WX, dx = k - (k / WX) * WX;
        int32_t* a = aux + (blk_index + n * (long long)p.BX) * 3;
        a[0] = dy + p.oy - p.cy;
        a[1] = dx + p.ox - p.cx;
        a[2] = static_cast<int32_t>(fin >> 16);
      }
    }
  }
}


// Fused 8x8 + 16x16 matching (multi-workload plans, merit_dev_plan_create_multi):
// the +/-32 search of 8x8 blocks (WX = WY = 65, two block rows per tile, as
// sad_tile_work_warp<8, 2, 65>) also yields the SAD of every 16x16 block made
// of 2 x 2 of them at every displacement — the four 8x8 SADs at the same
// (dy, dx) sum to it exactly (integers) — so the 16x16 workload costs a few
// adds and a shuffle per displacement instead of a second pass over the
// frames.  Lane mapping: the 16 warps of the CTA are (block-column pair q,
// dx quarter h) = (w / 4, w % 4); lanes 0-15 own 8x8 block column 2q,
// lanes 16-31 block column 2q + 1, both at dx = 16 h + (lane & 15), so lanes
// l and l ^ 16 hold the left and right halves of one 16x16 block at the same
// displacement: u = (top + bottom)(l) + (top + bottom)(l ^ 16).  The 65th
// column dx = 64 is split over the lanes by dy = 16 h + (lane & 15), the
// corner (64, 64) is shared by warp h = 3.  Argmin: REDUX over each
// half-warp (8x8) and the whole warp (16x16), then one shared atomic per
// warp and slot; the fourth warp to arrive writes the record.
template <typename AfterCw>
__device__ __forceinline__ void sad_tile_work_fused(const SadLaunch& L, int32_t* __restrict__ aux, int tile,
                                                    const uint32_t* curw, const uint32_t* copies, uint32_t* keys,
                                                    uint32_t* cnt, AfterCw after_cw) {
  constexpr int BLK = 8, NBY = 2, D = 33, WX = 65, WY = 65, BWW = 2;
  constexpr int WW = FusedGeo::WW;  // staged row pitch in words (fixed geometry: the launcher checks L.Ww)
  const SadParams& p = L.p;
  constexpr int cpw = kFusedCPW;  // words per staged current row (fixed geometry)
  const int warp = static_cast<int>(threadIdx.x) >> 5;
  const int q = warp >> 2, h = warp & 3;
  const int lane = static_cast<int>(threadIdx.x) & 31;
  const int half = lane >> 4, l16 = lane & 15;
  const int ib = 2 * q + half;     // this lane's 8x8 block column in the tile
  const int dxl = 16 * h + l16;    // this lane's column
  const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int pair_i = static_cast<int>(fast_div(t2, L.byt_m, L.byt_s));
  const int by = L.by0 + (t2 - pair_i * L.BYT) * NBY;  // first 8x8 block row of the tile (even)
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);  // even (BX = 2 BX2)
  if (2 * q >= nb) {  // warp-uniform
    after_cw();
    return;
  }
  const int dcur = (bx0 * BLK + p.cx) - floor16(bx0 * BLK + p.cx);
  const uint32_t* cb = curw + (dcur >> 2) + ib * BWW;
  uint32_t cw[NBY][BLK][BWW];
#pragma unroll
  for (int n = 0; n < NBY; ++n)
#pragma unroll
    for (int i = 0; i < BLK; ++i)
#pragma unroll
      for (int j = 0; j < BWW; ++j) cw[n][i][j] = cb[(n * BLK + i) * cpw + j];
  // corner words: 8 rows x 2 words of this half's block, one per lane
  uint32_t ccw[NBY];
  if (h == 3) {
#pragma unroll
    for (int n = 0; n < NBY; ++n) ccw[n] = cb[(n * BLK + (l16 >> 1)) * cpw + (l16 & 1)];
  }
  after_cw();
  const uint32_t kmul = L.key_mul;
  uint32_t best[NBY], best2 = 0xffffffffu;
#pragma unroll
  for (int n = 0; n < NBY; ++n) best[n] = 0xffffffffu;
  const int col = ib * BLK + dxl;
  const uint32_t one = L.one;
  // dy groups [0, 33) and [33, 65) as two specialised bodies (C5 37.2 ->
  // 36.3 ms against one 33-row body run for [0, 33) and [32, 65) with the
  // duplicated dy = 32, which MERIT_FUSED_ONEBODY keeps for A/B timing)
#ifndef MERIT_FUSED_HOTX  // timing experiment: run the dy groups MERIT_FUSED_HOTX times (same result)
#define MERIT_FUSED_HOTX 1
#endif
  auto group = [&](auto dg_tag, const int dy0) {
    constexpr int DG = decltype(dg_tag)::value;
    const uint32_t* cp = copies + (col & 3) * L.CS + (col >> 2) + dy0 * WW;
    uint32_t acc[NBY][DG];
#pragma unroll
    for (int n = 0; n < NBY; ++n)
#pragma unroll
      for (int d = 0; d < DG; ++d) acc[n][d] = 0;
    uint32_t bn0 = 0xffffffffu, bn1 = 0xffffffffu, bn2 = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < DG + NBY * BLK - 1; ++r) {
      uint32_t rwv[BWW];
#pragma unroll
      for (int j = 0; j < BWW; ++j) rwv[j] = cp[j];
      cp += WW;
#pragma unroll
      for (int n = 0; n < NBY; ++n)
#pragma unroll
        for (int d = 0; d < DG; ++d) {
          const int i = r - d - n * BLK;
          if (i >= 0 && i < BLK) {
#pragma unroll
            for (int j = 0; j < BWW; ++j) acc[n][d] = vabsdiff4_acc(cw[n][i][j], rwv[j], acc[n][d]);
          }
        }
      // displacement d is complete once its bottom block's last row
      // (r = d + 2 BLK - 1) is in: fold its keys here, so the key IMADs,
      // the shuffle and the mins interleave with the VABSDIFF4 stream and the
      // two accumulators die early (two displacements per fold: 3-way mins).
      // Keys: 8x8 acc * 2^16 + dy * WX; 16x16 (sum of the four 8x8 SADs)
      // * 2^16 + 4 dy * WX, built from the two 8x8 keys (t = k0 + k1 = (top +
      // bottom) * 2^16 + 2c, plus the other half's t from lane ^ 16): three
      // IMADs and a shuffle per displacement; the 4x index scaling keeps the
      // raster order (4 * 65 * 65 < 2^16) and is undone when the record is written
      const int d = r - (NBY * BLK - 1);
      auto keys = [&](int dd, uint32_t& k0v, uint32_t& k1v, uint32_t& k2v) {
        const uint32_t c = static_cast<uint32_t>(dd * WX);
        k0v = acc[0][dd] * kmul + c;
        k1v = acc[1][dd] * kmul + c;
        const uint32_t t = k0v * one + k1v;
        const uint32_t to = __shfl_xor_sync(0xffffffffu, t, 16);
        k2v = t * one + to;
      };
      if (d >= 1 && (d & 1)) {
        uint32_t a0, a1, a2, b0, b1, b2;
        keys(d - 1, a0, a1, a2);
        keys(d, b0, b1, b2);
        bn0 = __vimin3_u32(bn0, a0, b0);
        bn1 = __vimin3_u32(bn1, a1, b1);
        bn2 = __vimin3_u32(bn2, a2, b2);
      } else if (d == DG - 1 && (d & 1) == 0) {  // odd DG: the last one alone
        uint32_t a0, a1, a2;
        keys(d, a0, a1, a2);
        bn0 = min(bn0, a0);
        bn1 = min(bn1, a1);
        bn2 = min(bn2, a2);
      }
    }
    const uint32_t k0 = static_cast<uint32_t>(dy0 * WX + dxl);
    best[0] = min(best[0], bn0 + k0);
    best[1] = min(best[1], bn1 + k0);
    best2 = min(best2, bn2 + 4 * k0);
  };
#ifndef MERIT_FUSED_ONEBODY
#pragma unroll 1
  for (int rep = 0; rep < MERIT_FUSED_HOTX; ++rep) {
    group(std::integral_constant<int, D>{}, 0);
    group(std::integral_constant<int, WY - D>{}, D);
  }
#else
  constexpr int DY1 = WY - D;
#pragma unroll 1
  for (int igx = 0; igx < 2 * MERIT_FUSED_HOTX; ++igx) group(std::integral_constant<int, D>{}, (igx & 1) * DY1);
#endif
  // the last column dx = 64 (byte column ib*8 + 64: shifted copy 0): this
  // lane takes dy = 16 h + (lane & 15); block row n reads staged rows dy + 8 n ..
  const int colx = ib * BLK + (WX - 1);
  const uint32_t* cx0 = copies + (colx & 3) * L.CS + (colx >> 2);
  {
    uint32_t ax[NBY];
#pragma unroll
    for (int n = 0; n < NBY; ++n) {
      ax[n] = 0;
      const uint32_t* cx = cx0 + (dxl + n * BLK) * WW;
#pragma unroll
      for (int i = 0; i < BLK; ++i) {
#pragma unroll
        for (int j = 0; j < BWW; ++j) ax[n] = vabsdiff4_acc(cw[n][i][j], cx[j], ax[n]);
        cx += WW;
      }
    }
    const uint32_t c = static_cast<uint32_t>(dxl * WX + (WX - 1));
    best[0] = min(best[0], ax[0] * kmul + c);
    best[1] = min(best[1], ax[1] * kmul + c);
    const uint32_t sv = ax[0] + ax[1];
    const uint32_t so = __shfl_xor_sync(0xffffffffu, sv, 16);
    best2 = min(best2, (sv + so) * kmul + 4 * c);
  }
  if (h == 3) {
    // corner (64, 64): each half's 8x8 block from its 16 lanes, the 16x16 block from all 32
    uint32_t v[NBY];
#pragma unroll
    for (int n = 0; n < NBY; ++n)
      v[n] = vabsdiff4_acc(ccw[n], cx0[(WY - 1 + n * BLK + (l16 >> 1)) * WW + (l16 & 1)], 0u);
    const uint32_t c = static_cast<uint32_t>((WY - 1) * WX + (WX - 1));
    const uint32_t s0 = __reduce_add_sync(hmask, v[0]);
    const uint32_t s1 = __reduce_add_sync(hmask, v[1]);
    const uint32_t s2 = __reduce_add_sync(0xffffffffu, v[0] + v[1]);
    if (l16 == 0) {
      best[0] = min(best[0], s0 * kmul + c);
      best[1] = min(best[1], s1 * kmul + c);
    }
    if (lane == 0) best2 = min(best2, s2 * kmul + 4 * c);
  }
  if (by >= L.by1) return;
  // this warp's partial argmin keys (its dx quarter h) for the tile's 8x8
  // blocks (half-warp REDUX) and 16x16 block (warp REDUX): plain shared
  // stores into part[slot][h]; one warp of the CTA combines the four
  // quarters and writes the records once every warp has finished the tile
  // (sad_fused_finalize: no shared atomics or fences on this path)
#pragma unroll
  for (int n = 0; n < NBY; ++n) {
    const uint32_t key = __reduce_min_sync(hmask, best[n]);
    if (l16 == 0) keys[(n * L.TBX + ib) * 4 + h] = key;
  }
  const uint32_t key2 = __reduce_min_sync(0xffffffffu, best2);
  if (lane == 0) keys[(NBY * L.TBX + q) * 4 + h] = key2;
  (void)aux;
  (void)cnt;
}

// The argmin records of fused tile `tile` from its four dx-quarter partial
// keys (part[slot][h]), by one warp: lane s takes slot s (8x8 blocks n * TBX
// + ib, then the 16x16 blocks).  Keys: sad << 16 | index, the 16x16 index
// scaled by 4 (sad_tile_work_fused).
__device__ __forceinline__ void sad_fused_finalize(const SadLaunch& L, int32_t* __restrict__ aux, int tile,
                                                   const uint32_t* part) {
  constexpr int NBY = 2, WX = 65;
  const SadParams& p = L.p;
  const int lane = static_cast<int>(threadIdx.x) & 31;
  int t2, tx;
  sad_tile_coords(tile, L.n_full_tiles, L.n_full_x, L.ntx_m, L.ntx_s, t2, tx);
  const int pair_i = static_cast<int>(fast_div(t2, L.byt_m, L.byt_s));
  const int by = L.by0 + (t2 - pair_i * L.BYT) * NBY;
  if (by >= L.by1) return;
  const long long pair = pair_i;
  const int bx0 = tx * L.TBX;
  const int nb = min(L.TBX, p.BX - bx0);
  const int n8 = NBY * L.TBX;
  if (lane >= n8 + L.TBX / 2) return;
  const bool is16 = lane >= n8;
  const int n = is16 ? 0 : lane / L.TBX;
  const int ib = is16 ? 2 * (lane - n8) : lane - n * L.TBX;  // 16x16: its left 8x8 column
  if (ib >= nb) return;
  const uint32_t* pk = part + lane * 4;
  const uint32_t fin = min(__vimin3_u32(pk[0], pk[1], pk[2]), pk[3]);
  const int k = static_cast<int>(fin & 0xffffu) >> (is16 ? 2 : 0);
  const int dy = k / WX, dx = k - (k / WX) * WX;
  int32_t* a;
  if (is16) {
    const long long b2 = (pair * p.BY2 + by / 2) * (long long)p.BX2 + (bx0 >> 1) + (lane - n8);
    a = aux + p.aux2_delta + b2 * 3;
  } else {
    a = aux + ((pair * p.BY + by + n) * (long long)p.BX + bx0 + ib) * 3;
  }
  a[0] = dy + p.oy - p.cy;
  a[1] = dx + p.ox - p.cx;
  a[2] = static_cast<int32_t>(fin >> 16);
}

template <int BLK, int D, int NBY, int NT, int WXC, int MODE = 0>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1)
sad_kernel(const uint8_t* __restrict__ cur, const uint8_t* __restrict__ ref, void* __restrict__ out,
           int32_t* __restrict__ aux, SadLaunch L, const __grid_constant__ CUtensorMap ref_map,
           const __grid_constant__ CUtensorMap cur_map) {
  extern __shared__ __align__(128) uint8_t smem_b[];
  const int raw_words = static_cast<int>(L.raw_buf / 4);
  const int cur_words = static_cast<int>(L.cur_buf / 4);
  // --- shared memory carve-up: raw[2] | cur[2] | copies[4 or 2 x 4] | keys | counters | mbarriers
  uint32_t* raw0 = reinterpret_cast<uint32_t*>(smem_b + ((128u - (smem_u32(smem_b) & 127u)) & 127u));
  uint32_t* cur0 = raw0 + 2 * raw_words;
  uint32_t* copies0 = cur0 + 2 * cur_words;
  uint32_t* keys = copies0 + (L.dbl ? 8 : 4) * L.CS;  // per block: running argmin key
  uint32_t* cnt = keys + NBY * L.TBX;       // per block: contributions so far
  const uint32_t bar0 = (smem_u32(cnt + NBY * L.TBX) + 7u) & ~7u;
  // copy-builder start (row, word) of this thread in the flattened R x Ww walk
  const int cp_r0 = static_cast<int>(threadIdx.x) / L.Ww;
  const int cp_w0 = static_cast<int>(threadIdx.x) - cp_r0 * L.Ww;

  if (threadIdx.x < NBY * L.TBX) {
    keys[threadIdx.x] = 0xffffffffu;
    cnt[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int tile = blockIdx.x;
  int buf = 0;
  uint32_t phase_bits = 0;  // bit b: parity of buffer b's next completion
  pdl_launch_dependents();
  pdl_wait();  // first global access follows
  if (tile < L.n_tiles)
    issue_tile<BLK>(L, cur, ref, &ref_map, &cur_map, tile, smem_u32(raw0), reinterpret_cast<uint8_t*>(raw0),
                    smem_u32(cur0), reinterpret_cast<uint8_t*>(cur0), bar0);
  for (; tile < L.n_tiles; tile += gridDim.x, buf ^= 1) {
    uint32_t* raw = raw0 + buf * raw_words;
    uint32_t* curw = cur0 + buf * cur_words;
    uint32_t* copies = copies0 + (L.dbl ? buf * 4 * L.CS : 0);
    if (L.tma) {
      sad_mbar_wait(bar0 + 8u * buf, (phase_bits >> buf) & 1u);
      phase_bits ^= 1u << buf;
    } else {
      cp_async_wait_all();
    }
    // Single copy buffer: the previous tile's compute must finish before it is
    // rebuilt (and cp.async / byte staging must become visible).  Double
    // buffer (TMA staging only): copies[buf] was last read by tile - 2, which
    // every thread finished before the previous iteration's barrier.
    if (!L.dbl) __syncthreads();
    sad_build_copies<BLK>(L, tile, raw, copies, cp_r0, cp_w0);
    __syncthreads();
    // prefetch the next tile into the other buffer while this one computes
    const int next = tile + gridDim.x;
    if (next < L.n_tiles)
      issue_tile<BLK>(L, cur, ref, &ref_map, &cur_map, next, smem_u32(raw0 + (buf ^ 1) * raw_words),
                      reinterpret_cast<uint8_t*>(raw0 + (buf ^ 1) * raw_words),
                      smem_u32(cur0 + (buf ^ 1) * cur_words),
                      reinterpret_cast<uint8_t*>(cur0 + (buf ^ 1) * cur_words), bar0 + 8u * (buf ^ 1));
    if constexpr (MODE == 1)
      sad_tile_work_warp<BLK, NBY, WXC>(L, out, aux, tile, curw, copies, keys, cnt, [] {});
    else
      sad_tile_work<BLK, D, NBY, WXC>(L, out, aux, tile, curw, copies, keys, cnt, [] {});
  }
  cp_async_wait_all();
}

// Barrier-free variant for TMA staging: the warps of a CTA run their tiles
// without ever meeting at a CTA barrier in steady state.  The raw window is
// single-buffered, the current rows double-buffered and the shifted copies
// triple-buffered; after finishing tile k a warp builds its share of tile
// k + 2's copies, then starts tile k + 1, whose copies every warp finished
// one tile earlier.  So the copy building, the epilogue and the staging
// waits of one warp overlap the VABSDIFF4 streams of the others instead of
// being aligned across the SM by tile barriers.
//   tma[b]  (b = k % 2): TMA of tile k landed in raw / cur[b]
//   full[c] (c = k % 3): all threads built their share of copies[c] for tile k
//   done[c]:             all threads finished tile k's matching (copies[c] free)
// The last warp to load its current blocks of tile k issues tile k + 2's TMA
// into raw / cur[b]: every thread built its share of tile k + 1 (the last
// reader of raw) before it started tile k.
template <int BLK, int D, int NBY, int NT, int WXC, int MODE = 0>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1)
sad_async_kernel(const uint8_t* __restrict__ cur, const uint8_t* __restrict__ ref, void* __restrict__ out,
                 int32_t* __restrict__ aux, SadLaunch L, const __grid_constant__ CUtensorMap ref_map,
                 const __grid_constant__ CUtensorMap cur_map) {
  extern __shared__ __align__(128) uint8_t smem_b[];
  const int raw_words = static_cast<int>(L.raw_buf / 4);
  const int cur_words = static_cast<int>(L.cur_buf / 4);
  // --- carve-up: raw | cur[2] | copies[3 x 4] | keys[2] | cnt[2] | ctr[2] | mbarriers tma[2] full[3] done[3]
  uint32_t* raw0 = reinterpret_cast<uint32_t*>(smem_b + ((128u - (smem_u32(smem_b) & 127u)) & 127u));
  uint32_t* cur0 = raw0 + raw_words;
  uint32_t* copies0 = cur0 + 2 * cur_words;
  const int nslot = NBY * L.TBX + (MODE == 2 ? L.TBX / 2 : 0);  // fused: + the 16x16 slots
  // MODE 2: three tiles' partial keys [slot][dx quarter] (tile k at k % 3);
  // else two tiles' running keys + arrival counters
  uint32_t* keys0 = copies0 + 12 * L.CS;
  uint32_t* cnt0 = keys0 + (MODE == 2 ? 12 : 2) * nslot;
  uint32_t* ctr = cnt0 + 2 * nslot;
  const uint32_t bar_tma = (smem_u32(ctr + 2) + 7u) & ~7u;
  const uint32_t bar_full = bar_tma + 16u;
  const uint32_t bar_done = bar_full + 24u;
  const int cp_r0 = static_cast<int>(threadIdx.x) / L.Ww;
  const int cp_w0 = static_cast<int>(threadIdx.x) - cp_r0 * L.Ww;
  const int nwarps = static_cast<int>(blockDim.x) >> 5;

  if (threadIdx.x < 2 * nslot) {
    keys0[threadIdx.x] = 0xffffffffu;
    cnt0[threadIdx.x] = 0u;
  }
  if (threadIdx.x < 2) ctr[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_tma + 8u * i) : "memory");
    for (int i = 0; i < 3; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_full + 8u * i), "r"(blockDim.x) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_done + 8u * i), "r"(blockDim.x) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // first global access follows
  const int first = blockIdx.x, step = gridDim.x;
  const int nk = first < L.n_tiles ? (L.n_tiles - 1 - first) / step + 1 : 0;  // tiles of this CTA
  auto tile_of = [&](int k) { return first + k * step; };
  auto issue = [&](int k) {  // one thread: TMA of tile k into raw / cur[k % 2]
    const int b = k & 1;
    issue_tile_tma<BLK>(L, &ref_map, &cur_map, tile_of(k), smem_u32(raw0), smem_u32(cur0 + b * cur_words),
                        bar_tma + 8u * b);
  };
  auto arrive = [](uint32_t bar) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory"); };
  auto build = [&](int k) {  // this thread's share of tile k's copies
    const int b = k & 1, c = k % 3;
    if (k >= 3) sad_mbar_wait(bar_done + 8u * c, static_cast<uint32_t>((k - 3) / 3) & 1u);  // copies[c] free
    if constexpr (MODE == 2) {
      // every warp finished tile k - 3: one warp writes its argmin records
      // (before building tile k, whose partial keys reuse that buffer)
      if (k >= 3 && ((k - 3) % nwarps) == (static_cast<int>(threadIdx.x) >> 5))
        sad_fused_finalize(L, aux, tile_of(k - 3), keys0 + c * 4 * nslot);
    }
    sad_mbar_wait(bar_tma + 8u * b, static_cast<uint32_t>(k >> 1) & 1u);
    bool built = false;
    if constexpr (MODE == 2) {
      if (L.fast_build) {
        sad_build_copies_geo<FusedGeo, NT>(raw0 + L.dref_w, copies0 + c * 4 * L.CS);
        built = true;
      }
    } else if constexpr (MODE == 1 && WXC > 0) {
      if (L.fast_build) {
        sad_build_copies_geo<WarpGeo<BLK, WXC, NBY>, NT>(raw0 + L.dref_w, copies0 + c * 4 * L.CS);
        built = true;
      }
    }
    if (!built) sad_build_copies<BLK>(L, tile_of(k), raw0, copies0 + c * 4 * L.CS, cp_r0, cp_w0);
    arrive(bar_full + 8u * c);
  };
  if (threadIdx.x == 0 && nk > 0) issue(0);
  if (nk > 0) build(0);
  if (nk > 1) {
    if (threadIdx.x == 0) {  // raw is free once every thread built tile 0
      sad_mbar_wait(bar_full, 0u);
      issue(1);
    }
    build(1);
  }
  for (int k = 0; k < nk; ++k) {
    const int b = k & 1, c = k % 3;
    sad_mbar_wait(bar_full + 8u * c, static_cast<uint32_t>(k / 3) & 1u);
    auto refill = [&] {
          // the last warp done with cur[b] for tile k refills buffer b with tile k + 2
          // (every lane's loads of its current rows must have returned first:
          // they were only requested so far, conv_tma_s1.cu raw_release)
          __threadfence_block();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) {
            __threadfence_block();
            if (atomicAdd(&ctr[b], 1u) == static_cast<uint32_t>(nwarps - 1)) {
              ctr[b] = 0u;
              __threadfence_block();
              if (k + 2 < nk) issue(k + 2);
            }
          }
        };
    if constexpr (MODE == 2)
      sad_tile_work_fused(L, aux, tile_of(k), cur0 + b * cur_words, copies0 + c * 4 * L.CS, keys0 + c * 4 * nslot,
                          cnt0, refill);
    else if constexpr (MODE == 1)
      sad_tile_work_warp<BLK, NBY, WXC>(L, out, aux, tile_of(k), cur0 + b * cur_words, copies0 + c * 4 * L.CS,
                                        keys0 + b * nslot, cnt0 + b * nslot, refill);
    else
      sad_tile_work<BLK, D, NBY, WXC>(L, out, aux, tile_of(k), cur0 + b * cur_words, copies0 + c * 4 * L.CS,
                                      keys0 + b * nslot, cnt0 + b * nslot, refill);
    arrive(bar_done + 8u * c);
    if (k + 2 < nk) build(k + 2);
  }
  if constexpr (MODE == 2) {  // the records of the last (up to three) tiles
    __syncthreads();
    const int w = static_cast<int>(threadIdx.x) >> 5;
    for (int t = nk > 3 ? nk - 3 : 0; t < nk; ++t)
      if ((t % nwarps) == w) sad_fused_finalize(L, aux, tile_of(t), keys0 + (t % 3) * 4 * nslot);
  }
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
  // Blocks per tile: the most busy lanes per SM sub-partition.  Warps of a
  // CTA are spread warp % 4 over the four sub-partitions, so a CTA of w
  // warps costs ceil(w / 4) * 4 warp slots of VABSDIFF4 time (7 warps load
  // three sub-partitions with two warps and one with one: profiled as 12% of
  // all stall samples at the tile barrier).
  auto best_tbx = [&](int budget, double& eff_out) {
    int tbx = 1;
    double best_eff = -1.0;
    for (int t = 1; t <= 16 && t <= p.BX; ++t) {
      const int items = t * per_block;
      const int warps = (items + 31) / 32;
      if (warps * 32 > budget) break;
      const int tiles = (p.BX + t - 1) / t;  // the last tile of a row may be partial
      const double eff = double(items) / (((warps + 3) / 4) * 4 * 32) * double(p.BX) / (tiles * t);
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        tbx = t;
      }
    }
    eff_out = best_eff;
    return tbx;
  };
  // 256-thread CTAs, two per SM; or one 512-thread CTA per SM when a wide
  // window leaves many lanes idle in 256 threads (C5 +/-32: 3 blocks = 76%
  // of lanes busy, 7 blocks in 512 threads = 89%)
  double eff256 = 0, eff512 = 0;
  const int tbx256 = best_tbx(256, eff256);
  const int tbx512 = best_tbx(512, eff512);
  // measured: C5 (eff 0.76 -> 0.87) 120 -> 99 ms; C2 (0.86 -> 0.97) 64 -> 67 us,
  // the single CTA per SM exposes the tile barriers
  int nt = (eff256 < 0.80 && eff512 > 1.08 * eff256) ? 512 : 256;
  if (const char* te = getenv("MERIT_SAD_THREADS")) nt = atoi(te) == 512 ? 512 : 256;
  L.TBX = nt == 512 ? tbx512 : tbx256;
  L.items = L.TBX * per_block;
  // warp-per-block mapping for the +/-16 search of 16x16 blocks (C2): 8-block
  // tiles, every lane busy (sad_tile_work_warp)
  const char* wme = getenv("MERIT_SAD_WARP");
  const bool warp_mode = D == 33 && (BLK == 16 ? (p.WX == 33 || p.WX == 65) : p.WX == 65) && p.WY == p.WX &&
                         p.BX >= 8 && (!(wme && wme[0] == '0') || p.fuse2);
  if (p.fuse2 && !(BLK == 8 && warp_mode && p.write_map == 0 && p.argmin && p.BX == 2 * p.BX2 &&
                   p.BY == 2 * p.BY2))
    return fail(MERIT_E_UNSUPPORTED_VIEW, "fused 8x8 + 16x16 SAD needs the +/-32 warp kernel");
  if (warp_mode) {
    nt = 8 * (p.WX - 1);  // 8 blocks x (WX - 1) / 32 warps
    L.TBX = 8;
    L.items = nt;
  }
  L.n_tiles_x = (p.BX + L.TBX - 1) / L.TBX;
  L.span = L.TBX * BLK + p.WX - 1;
  L.Ww = (L.span + 3) / 4;
  // warp mode: the 33rd column's side loop has lane l read staged row l + i,
  // so an odd row pitch keeps the 32 lanes on 32 banks (40 words: 8-way conflicts)
  if (warp_mode && (L.Ww & 1) == 0) L.Ww += 1;
  // TMA staging lands rows from floor16(x): up to 15 leading bytes, and the
  // copy builder reads 2 words past the window
  const char* te = getenv("MERIT_SAD_TMA");
  const bool tma_ok = !(te && te[0] == '0') && p.boundary == MERIT_ZERO_PAD && tensor_map_encoder() != nullptr &&
                      p.Wr % 16 == 0 && p.Wc % 16 == 0 && p.cx % 4 == 0 &&
                      (reinterpret_cast<uintptr_t>(ref) % 16) == 0 && (reinterpret_cast<uintptr_t>(cur) % 16) == 0 &&
                      p.pairs < (1LL << 31);
  L.word_path = ((p.ox % 4) == 0 && (p.cx % 4) == 0 && (p.Wr % 4) == 0 && (p.Wc % 4) == 0 &&
                 (reinterpret_cast<uintptr_t>(cur) % 4) == 0 && (reinterpret_cast<uintptr_t>(ref) % 4) == 0)
                    ? 1 : 0;
  L.vec_path = (L.word_path && (p.ox % 16) == 0 && (p.Wr % 16) == 0 && (BLK % 16) == 0 &&
                (reinterpret_cast<uintptr_t>(ref) % 16) == 0) ? 1 : 0;
  // geometry for nby block rows per tile; TMA staging only where the boxes fit
  L.by0 = p.by_begin;
  L.by1 = p.by_count > 0 ? p.by_begin + p.by_count : p.BY;
  if (L.by0 < 0 || L.by1 > p.BY || L.by0 >= L.by1) return fail(MERIT_E_INVALID_ARGUMENT, "bad SAD block-row band");
  auto geometry = [&](int nby, bool tma) {
    L.nby = nby;
    L.BYT = (L.by1 - L.by0 + nby - 1) / nby;
    L.R = L.G * D + nby * BLK - 1;
    L.rw = tma ? (L.Ww + 5 + 3) / 4 * 4 : (L.Ww + 1 + 3) / 4 * 4;  // raw words per row, 16-byte chunks
    L.CS = L.R * L.Ww;
    L.CS += ((8 - (L.CS % 32)) + 32) % 32;
    L.cur_pitch = (L.TBX * BLK + (tma ? 12 : 0) + 15) / 16 * 16;
    L.R_box = L.R;
    L.raw_buf = (static_cast<uint32_t>(L.R_box * L.rw * 4) + 127u) & ~127u;
    L.cur_buf = (static_cast<uint32_t>(nby * BLK * L.cur_pitch) + 127u) & ~127u;
    return tma && L.rw * 4 <= 256 && L.R_box <= 256 && L.cur_pitch <= 256 && nby * BLK <= 256;
  };
  // 8x8 blocks: two block rows per thread (every loaded reference word feeds
  // both), on the TMA staging path
  const char* ne = getenv("MERIT_SAD_NBY");
  const int nby_want = (BLK == 8 && !(ne && ne[0] == '1')) ? 2 : 1;
  L.tma = geometry(nby_want, tma_ok);
  if (!L.tma && nby_want != 1) L.tma = geometry(1, tma_ok);
  if (!L.tma) geometry(1, false);
  const long long n_tiles = p.pairs * (long long)L.BYT * L.n_tiles_x;
  if (n_tiles >= (1LL << 31)) return fail(MERIT_E_UNSUPPORTED_VIEW, "too many SAD tiles for one launch");
  L.n_tiles = static_cast<int>(n_tiles);
  CUtensorMap ref_map, cur_map;
  std::memset(&ref_map, 0, sizeof(ref_map));
  std::memset(&cur_map, 0, sizeof(cur_map));
  if (L.tma) {
    const cuuint64_t rd[3] = {(cuuint64_t)p.Wr, (cuuint64_t)p.Hr, (cuuint64_t)p.pairs};
    const cuuint64_t rs[2] = {(cuuint64_t)p.Wr, (cuuint64_t)p.Wr * p.Hr};
    const cuuint32_t rb[3] = {(cuuint32_t)(L.rw * 4), (cuuint32_t)L.R_box, 1};
    const cuuint64_t cd[3] = {(cuuint64_t)p.Wc, (cuuint64_t)p.Hc, (cuuint64_t)p.pairs};
    const cuuint64_t cs[2] = {(cuuint64_t)p.Wc, (cuuint64_t)p.Wc * p.Hc};
    const cuuint32_t cbx[3] = {(cuuint32_t)L.cur_pitch, (cuuint32_t)(L.nby * BLK), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    L.tma = tensor_map_encoder()(&ref_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(ref), rd, rs, rb,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
            tensor_map_encoder()(&cur_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(cur), cd, cs, cbx,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    if (!L.tma) return fail(MERIT_E_CUDA, "cuTensorMapEncodeTiled failed for the SAD frames");
  }
  const size_t smem_cap = (nt == 512 ? 220 : 110) * 1024;
  auto smem_for = [&](int ncopy) {
    return 128 + 2ull * L.raw_buf + 2ull * L.cur_buf + 4ull * (4ull * ncopy * L.CS + 2ull * L.nby * L.TBX) + 8 + 16;
  };
  L.dbg = 0;
  if (const char* ge = debug_env("MERIT_SAD_DBG")) L.dbg = atoi(ge);
  const char* de = getenv("MERIT_SAD_DBL");
  L.dbl = (L.tma && !(de && de[0] == '0') && smem_for(2) <= smem_cap) ? 1 : 0;
  const size_t smem = smem_for(L.dbl ? 2 : 1);
  if (L.n_tiles == 0) return MERIT_OK;
  if (smem > smem_cap) return fail(MERIT_E_UNSUPPORTED_VIEW, "SAD footprint exceeds shared memory");
  // barrier-free variant (TMA staging): two staging buffers, three copy buffers
  const size_t nslot_h = static_cast<size_t>(L.nby * L.TBX + (p.fuse2 ? L.TBX / 2 : 0));
  const size_t smem_async = 128 + 1ull * L.raw_buf + 2ull * L.cur_buf +
                            4ull * (12ull * L.CS + (p.fuse2 ? 14ull : 4ull) * nslot_h + 2) + 8 + 64;
  const char* ae = getenv("MERIT_SAD_ASYNC");
  const bool use_async = L.tma && (!(ae && ae[0] == '0') || p.fuse2) && smem_async <= smem_cap;
  if (p.fuse2 && !(use_async && L.nby == 2 && L.by0 % 2 == 0 && L.by1 % 2 == 0))
    return fail(MERIT_E_UNSUPPORTED_VIEW, "fused 8x8 + 16x16 SAD needs TMA staging of two-row tiles");
  auto kern = nt == 512 ? sad_kernel<BLK, D, 1, 512, 0> : sad_kernel<BLK, D, 1, 256, 0>;
  if constexpr (BLK == 8) {
    if (L.nby == 2) kern = nt == 512 ? sad_kernel<BLK, D, 2, 512, 0> : sad_kernel<BLK, D, 2, 256, 0>;
  }
  // compile-time window widths for the +/-16 and +/-32 searches (C2, C5)
  if constexpr (D == 33) {
    if constexpr (BLK == 16) {
      if (p.WX == 33) kern = nt == 512 ? sad_kernel<16, 33, 1, 512, 33> : sad_kernel<16, 33, 1, 256, 33>;
      if (p.WX == 65) kern = nt == 512 ? sad_kernel<16, 33, 1, 512, 65> : sad_kernel<16, 33, 1, 256, 65>;
      if (warp_mode) kern = p.WX == 33 ? sad_kernel<16, 33, 1, 256, 33, true> : sad_kernel<16, 33, 1, 512, 65, true>;
    } else {
      if (p.WX == 65 && L.nby == 2) kern = nt == 512 ? sad_kernel<8, 33, 2, 512, 65> : sad_kernel<8, 33, 2, 256, 65>;
      if (warp_mode) kern = L.nby == 2 ? sad_kernel<8, 33, 2, 512, 65, true> : sad_kernel<8, 33, 1, 512, 65, true>;
    }
  }
  if (warp_mode) {
    const int ww = BLK == 16 ? (p.WX == 33 ? WarpGeo<16, 33, 1>::WW : WarpGeo<16, 65, 1>::WW)
                             : WarpGeo<8, 65, 1>::WW;
    if (L.Ww != ww) return fail(MERIT_E_UNSUPPORTED_VIEW, "warp-per-block SAD row pitch");
  }
  if (const char* we = getenv("MERIT_SAD_WXC"); we && we[0] == '0' && !warp_mode) {  // A/B: runtime width
    kern = nt == 512 ? sad_kernel<BLK, D, 1, 512, 0> : sad_kernel<BLK, D, 1, 256, 0>;
    if constexpr (BLK == 8) {
      if (L.nby == 2) kern = nt == 512 ? sad_kernel<BLK, D, 2, 512, 0> : sad_kernel<BLK, D, 2, 256, 0>;
    }
  }
  if (use_async) {
    // same template arguments, barrier-free kernel
#define MERIT_SAD_ASYNC_OF(B, DD, NB, T, W) \
  if (kern == sad_kernel<B, DD, NB, T, W>) kern = sad_async_kernel<B, DD, NB, T, W>;
    MERIT_SAD_ASYNC_OF(BLK, D, 1, 512, 0)
    MERIT_SAD_ASYNC_OF(BLK, D, 1, 256, 0)
    if constexpr (BLK == 8) {
      MERIT_SAD_ASYNC_OF(BLK, D, 2, 512, 0)
      MERIT_SAD_ASYNC_OF(BLK, D, 2, 256, 0)
    }
    if constexpr (D == 33) {
      if constexpr (BLK == 16) {
        MERIT_SAD_ASYNC_OF(16, 33, 1, 512, 33)
        MERIT_SAD_ASYNC_OF(16, 33, 1, 256, 33)
        MERIT_SAD_ASYNC_OF(16, 33, 1, 512, 65)
        MERIT_SAD_ASYNC_OF(16, 33, 1, 256, 65)
      } else {
        MERIT_SAD_ASYNC_OF(8, 33, 2, 512, 65)
        MERIT_SAD_ASYNC_OF(8, 33, 2, 256, 65)
      }
    }
#undef MERIT_SAD_ASYNC_OF
    if constexpr (D == 33) {
      if constexpr (BLK == 16) {
        if (kern == sad_kernel<16, 33, 1, 256, 33, true>) kern = sad_async_kernel<16, 33, 1, 256, 33, true>;
        if (kern == sad_kernel<16, 33, 1, 512, 65, true>) kern = sad_async_kernel<16, 33, 1, 512, 65, true>;
      } else {
        if (kern == sad_kernel<8, 33, 2, 512, 65, true>) kern = sad_async_kernel<8, 33, 2, 512, 65, true>;
        if (kern == sad_kernel<8, 33, 1, 512, 65, true>) kern = sad_async_kernel<8, 33, 1, 512, 65, true>;
        if (p.fuse2) kern = sad_async_kernel<8, 33, 2, 512, 65, 2>;
        if (p.fuse2 && (L.Ww != FusedGeo::WW || L.R != FusedGeo::R || L.rw != FusedGeo::RW ||
                        L.CS != FusedGeo::CS || L.cur_pitch != 4 * kFusedCPW))
          return fail(MERIT_E_UNSUPPORTED_VIEW, "fused SAD staging geometry");
      }
    }
  }
  const size_t smem_launch = use_async ? smem_async : smem;
  cudaError_t e = set_smem_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_launch));
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(sad)");
  const int threads = (L.items + 31) / 32 * 32;
  L.key_mul = 65536u;
  L.one = 1u;
  // warp-per-block / fused kernels: the copy builder on the compile-time
  // staging geometry when it matches (TMA staging, 8-block tiles) and the
  // window starts on a word (ox % 4 == 0)
  L.dref_w = ((p.ox % 16) + 16) % 16 / 4;
  auto geo_is = [&](auto geo) {
    using GEO = decltype(geo);
    return L.Ww == GEO::WW && L.R == GEO::R && L.rw == GEO::RW && L.CS == GEO::CS;
  };
  bool geo_ok = false;
  if constexpr (D == 33) {
    if (p.fuse2)
      geo_ok = geo_is(FusedGeo{}) && threads == 512;
    else if (warp_mode && BLK == 16)
      geo_ok = p.WX == 33 ? geo_is(WarpGeo<16, 33, 1>{}) && threads == 256 : geo_is(WarpGeo<16, 65, 1>{}) && threads == 512;
    else if (warp_mode && BLK == 8)
      geo_ok = L.nby == 2 ? geo_is(WarpGeo<8, 65, 2>{}) : geo_is(WarpGeo<8, 65, 1>{});
  }
  L.fast_build = (use_async && L.tma && geo_ok && p.ox % 4 == 0) ? 1 : 0;
#ifdef MERIT_NO_FAST_BUILD
  L.fast_build = 0;
#endif
  L.cp_sr = threads / L.Ww;
  L.cp_sw = threads - L.cp_sr * L.Ww;
  L.n_full_x = p.BX / L.TBX;
  L.n_full_tiles = static_cast<int>(p.pairs * (long long)L.BYT * L.n_full_x);
  if (const char* oe = getenv("MERIT_SAD_ORDER"); oe && oe[0] == '0') {  // A/B: row-major order
    L.n_full_x = L.n_tiles_x;
    L.n_full_tiles = L.n_tiles;
  }
  L.ntx_m = L.ntx_s = 0;
  if (L.n_full_x > 0) fast_div_init(static_cast<uint32_t>(L.n_full_x), L.ntx_m, L.ntx_s);
  fast_div_init(static_cast<uint32_t>(L.BYT), L.byt_m, L.byt_s);
  long long grid = (nt == 512 ? 1LL : 2LL) * num_sms();
  if (grid > L.n_tiles) grid = L.n_tiles;
  grid = grid_cap(static_cast<int>(grid));
  e = launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(threads), smem_launch, s, 1, cur, ref, out, aux, L,
                 ref_map, cur_map);
  if (e != cudaSuccess) return cuda_check(e, "launch(sad)");
  if (p.fuse2) return launch_status("sad_async_kernel<fused 8x8 + 16x16>");
  return launch_status(warp_mode ? (use_async ? "sad_async_kernel<warp per block>" : "sad_kernel<warp per block>")
                                 : (use_async ? "sad_async_kernel" : "sad_kernel"));
}

}  // namespace

// Kernel variant for a window: D rows per thread such that WX * ceil(WY/D)
// fits the thread budget.  Used by the lowering to decide eligibility.
int sad_rows_per_thread(int BH, int WY, int WX) {
  if (WX > kSadMaxThreads || WY > 256) return 0;
  const char* e = getenv("MERIT_SAD_D");  // tuning override
  const int want = e ? atoi(e) : 0;
  if (BH == 16) {
    if (want == 11 || want == 17 || want == 33) return want;
    return WY <= 66 ? 33 : 17;
  }
  if (want == 11 || want == 22 || want == 33) return want;
  return WY <= 33 ? 11 : (WY <= 66 ? 33 : 22);  // measured on C5 (+/-32): 33 beats 22 by 3%
}

namespace {
// f32 -> u8 for both frames of a narrowed plan; *bad |= 1 if any value is
// not an integer in [0, 255] (NaN fails the comparisons).
__global__ void narrow_u8_kernel(const float* __restrict__ a, uint8_t* __restrict__ ua, long long na,
                                 const float* __restrict__ b, uint8_t* __restrict__ ub, long long nb,
                                 int32_t* __restrict__ bad) {
  pdl_launch_dependents();
  pdl_wait();
  bool ok = true;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < na + nb; i += stride) {
    const float v = i < na ? a[i] : b[i - na];
    const bool good = v >= 0.f && v <= 255.f && v == rintf(v);
    ok = ok && good;
    const uint8_t u = good ? static_cast<uint8_t>(v) : 0;
    if (i < na) ua[i] = u; else ub[i - na] = u;
  }
  if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}
}  // namespace

merit_status launch_sad_narrowed(const merit_plan& plan, const void* a, const void* b, void* out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long na = plan.info.src_a_bytes / 4, nb = plan.info.src_b_bytes / 4;
  uint8_t* ua = static_cast<uint8_t*>(plan.d_narrow);
  uint8_t* ub = ua + ((na + 127) / 128) * 128;
  int32_t* bad = reinterpret_cast<int32_t*>(ub + ((nb + 127) / 128) * 128);
  merit_status st = cuda_check(cudaMemsetAsync(bad, 0, 4, s), "cudaMemsetAsync(narrow flag)");
  if (st != MERIT_OK) return st;
  long long blocks = (na + nb + 255) / 256;
  if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
  cudaError_t e = launch_pdl(narrow_u8_kernel, dim3(static_cast<unsigned>(std::max(1LL, blocks))), dim3(256), 0, s,
                             1, static_cast<const float*>(a), ua, na, static_cast<const float*>(b), ub, nb, bad);
  if (e != cudaSuccess) return cuda_check(e, "launch(narrow)");
  if ((st = launch_status("narrow_u8_kernel")) != MERIT_OK) return st;
  SadParams p = plan.sad;
  merit_plan sub;  // the same plan on the u8 copies
  sub.kernel = MERIT_KERNEL_SAD;
  sub.sad = p;
  sub.info = plan.info;
  if ((st = launch_sad(sub, ua, ub, out, nullptr, stream)) != MERIT_OK) return st;
  // exact interpreter on the f32 frames, only if a pixel did not narrow
  return launch_generic(plan, a, b, out, stream, bad);
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
    if (D == 33) return launch_sad_t<8, 33>(p, cur, ref, out, ax, s);
  }
  return fail(MERIT_E_UNSUPPORTED_VIEW, "no SAD kernel variant for this window");
}

}  // namespace merit_dev
