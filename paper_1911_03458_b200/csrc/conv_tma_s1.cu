// K3d — stride-1, 3-wide convolution with the three horizontal taps stacked
// along the MMA's N dimension (the C3 shape: NCHW fp32, 3x3, stride 1, pad 1,
// Cout <= 80).
//
// For a fixed kernel row ky and channel block, the tap-kx partial sums
//   P_kx[x][co] = sum_ci in[ci][y + ky - 1][x] * w[co][ci][ky][kx]
// are ONE product A x B with A = input columns (M = 128 slots) and
// B = the three tap matrices stacked (N = 3 * Cout).  The convolution is
//   out[x] = P_0[x - 1] + P_1[x] + P_2[x + 1],
// so the epilogue applies the column shifts with warp shuffles.  Compared
// with three N = Cout MMAs per k-step, each A tile is read by the tensor core
// once instead of three times, which is what bounds the narrow-Cout case
// (shared-memory bandwidth, not MMA issue).
//
// Gather: one TMA tensor load per (tile, ky, 32-channel half) lands the raw
// rows [c][rows][W] (zero fill = the view's zero padding in y and c); eight
// repack warps split fp32 into bf16 hi/lo (3-product split: hi*hi + hi*lo +
// lo*hi) and write the K-major SW128 A planes.  Slots: `slots` per output
// row (power of two >= W + 2), input column x at slot x + 1, so every row
// carries the zero columns x = -1 and x = W the shifts read.
//
// Warps: 0-7 repack, 8 B loader + TMEM alloc, 9 MMA, 10-13 and 15-18
// epilogue (two sets, alternating 8-channel chunks), 14 TMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"
#include "tmap.cuh"

namespace merit_dev {
namespace {

using namespace tc;

constexpr int kRepackWarps = 8;
constexpr int kRepackers = kRepackWarps * 32;
constexpr int kWarpB = 8, kWarpMma = 9, kWarpEpi0 = 10, kWarpTma = 14, kWarpEpi1 = 15;
// Shared-memory-A variant: every repack thread arrives on a_full itself after
// its own fence.proxy.async (the CUTLASS transform -> MMA form); 0 = one
// elected lane per warp after a __syncwarp (A/B).
#ifndef MERIT_S1_ALLARRIVE
#define MERIT_S1_ALLARRIVE 1
#endif
constexpr int kThreads = 19 * 32;
constexpr int kEpiWarps = 8;  // two sets of four (one warp per TMEM lane quadrant each)
constexpr int kEC = 8;        // output channels per epilogue chunk
constexpr int kMaxRing = 8;
constexpr uint32_t kAccCols = 256;  // TMEM columns per accumulator (N <= 240)

struct S1Args {
  ConvParams p;
  const uint8_t* wpk;
  float* out;
  int slots_log2;      // slots per output row = 1 << slots_log2
  int segs_log2;       // 32-lane segments per output row (slots / 32)
  int seg_w;           // output columns per segment (<= 30: the segment's lanes 1 .. seg_w)
  int rows;            // output rows per tile = 128 / slots
  int tiles_per_img;   // ceil(Ho / rows)
  int n_tiles;
  int n_full;          // units below n_full are whole tiles; the last (n_tiles - n_full)
  int n_units;         // tiles from n_full on run as `parts` N-part units each (the final, partial wave)
  int parts;           // 2 or 4: output-channel parts of a tail tile (N = 3 BN / parts)
  int parts_log2;      // log2(parts)
  int n_groups;        // KH * CB
  uint32_t raw_bytes;  // 128 slots * 32 ch * 4 = 16 KB (half a 64-channel k-block)
  uint32_t a_slot;     // nsplit planes x 16 KB
  uint32_t b_plane;    // BN * 128: one tap, one split plane
  uint32_t b_slot;     // 3 taps x nsplit planes
  int nr, na, nb;
  int resident;        // nb == n_groups: every group's weights stay in their B slot (loaded once per CTA)
  unsigned long long* prof;  // MERIT_CONV_DEBUG & 64: per-warp [total, wait1, wait2, wait3]
  int debug;
};

__device__ __forceinline__ void tma_load_4d_s1(uint32_t dst, const CUtensorMap* map, int x, int y, int c, int n,
                                               uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(c), "r"(n), "r"(bar)
      : "memory");
}

// Hand a raw slot back to the TMA warp.  The slot's values were only REQUESTED
// by the ld.shared instructions before this point: the arrive does not wait
// for them (no register dependence; the SASS shows no scoreboard wait before
// SYNCS.ARRIVE), and with the shared-memory pipe saturated by the tensor
// core's operand reads the last loads were still queued when the next box
// landed in the slot (the N = 240 fault: rows loaded last
// came from the next group).  A CTA-scope fence first: it completes only when
// this thread's prior loads have returned.  MERIT_RAW_RELEASE_FENCE=0: the
// bare arrive (diagnosis).
#ifndef MERIT_RAW_RELEASE_FENCE
#define MERIT_RAW_RELEASE_FENCE 1
#endif
__device__ __forceinline__ void raw_release(uint32_t bar) {
#if MERIT_RAW_RELEASE_FENCE
  __threadfence_block();
#endif
  mbar_arrive(bar);
}

__device__ __forceinline__ void twait_s1(uint32_t bar, uint32_t par, unsigned long long& acc, bool on) {
  if (on) {
    const unsigned long long t0 = clock64();
    mbar_wait(bar, par);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, par);
  }
}

// TMEMA: the A planes live in TMEM (columns 384..511: two slots of hi | lo,
// 32 columns each) and the MMA reads A from there (tcgen05.mma [a_tmem]):
// the repack writes them with tcgen05.st and the tensor core's shared-memory
// traffic drops to B alone.  Needs 3 BN <= 192 (two 192-column accumulators).
constexpr uint32_t kTmemA = 384;
template <bool SPLIT3, bool TMEMA>
__global__ void __maxnreg__(96)  // 19 warps: <= 5 per SM sub-partition x 96 regs
conv_s1_kernel(const __grid_constant__ CUtensorMap in_map, S1Args A) {
  constexpr uint32_t acc_cols = TMEMA ? 192u : kAccCols;
  extern __shared__ uint8_t smem_raw[];
  const ConvParams& p = A.p;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t aring = base;                          // na x a_slot
  const uint32_t bring = aring + A.na * A.a_slot;       // nb x b_slot
  const uint32_t rring = bring + A.nb * A.b_slot + 128;  // nr x raw_bytes after a 128-B zero pad
  const uint32_t bars = rring + A.nr * A.raw_bytes;
  auto r_full = [&](int s) { return bars + 8u * s; };
  auto r_empty = [&](int s) { return bars + 8u * (kMaxRing + s); };
  auto a_full = [&](int s) { return bars + 8u * (2 * kMaxRing + s); };
  auto a_empty = [&](int s) { return bars + 8u * (3 * kMaxRing + s); };
  auto b_full = [&](int s) { return bars + 8u * (4 * kMaxRing + s); };
  auto b_empty = [&](int s) { return bars + 8u * (5 * kMaxRing + s); };
  auto tfull = [&](int a) { return bars + 8u * (6 * kMaxRing + a); };
  auto tempty = [&](int a) { return bars + 8u * (6 * kMaxRing + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (6 * kMaxRing + 4);
  volatile uint32_t* tmem_slot_ptr =
      reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  if (threadIdx.x < 32) {  // zero pad read as the x = -1 column of slot 0's first row
    const uint32_t z = rring - 128 + 4u * threadIdx.x;
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(z), "r"(0u) : "memory");
    // ... and of slot s > 0: the last word of slot s - 1 (channel 31, last
    // row, column slots - 1 >= W: every box writes a zero there).  On the
    // first lap that box may still be in flight when slot s is read, and the
    // word would be whatever the previous kernel left in shared memory.
    if (static_cast<int>(threadIdx.x) < A.nr) {
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(rring + (threadIdx.x + 1u) * A.raw_bytes - 4u), "r"(0u) : "memory");
      fence_proxy_async();
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nr; ++s) {
      mbar_init(r_full(s), 1);
      mbar_init(r_empty(s), kRepackers / 2);  // one half of the repack warps
    }
    for (int s = 0; s < A.na; ++s) {
#if MERIT_S1_ALLARRIVE
      // shared-memory A: every repack thread arrives after its own proxy fence;
      // TMEM A: one elected lane per warp after tcgen05.wait::st + __syncwarp
      mbar_init(a_full(s), TMEMA ? kRepackWarps : kRepackers);
#else
      mbar_init(a_full(s), kRepackWarps);  // one elected lane per repack warp
#endif
      mbar_init(a_empty(s), 1);
    }
    for (int s = 0; s < A.nb; ++s) {
      mbar_init(b_full(s), 1);
      mbar_init(b_empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), kEpiWarps);  // one elected lane per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpB) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(2 * kAccCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  pdl_launch_dependents();
  pdl_wait();  // prologue done: from here on global memory is touched
  const int BN = p.BN;
  const int W = p.W;
  // scheduling unit -> (tile, half): half = -1 for a whole tile, else the
  // part 0 .. parts - 1 of the output channels of a tail tile (BN / parts
  // channels each; the name `half` is kept for parts = 2)
  auto unit_of = [&](int u, int& tile, int& half) {
    if (u < A.n_full) {
      tile = u;
      half = -1;
    } else {
      tile = A.n_full + ((u - A.n_full) >> A.parts_log2);
      half = (u - A.n_full) & (A.parts - 1);
    }
  };
  // Segmented slot layout: TMEM lane quadrant q (A rows 32q .. 32q + 31) is
  // segment sg = q % S of output row r = q / S (S = slots / 32): lane l holds
  // input column x = sg * seg_w - 1 + l, so lanes 1 .. seg_w produce outputs
  // sg * seg_w .. + seg_w - 1 and both neighbours of every output column
  // (x - 1, x + 1) are in the same warp: the epilogue's tap shifts are plain
  // lane shuffles.  Raw row r holds column x at word r * slots + x (x = -1:
  // the previous row's zero-filled tail, or the pad before the ring; x >= W:
  // the box's zero fill).
  auto seg_word = [&](int q, int l) {
    const int r = q >> A.segs_log2, sg = q & ((1 << A.segs_log2) - 1);
    return (r << A.slots_log2) + sg * A.seg_w - 1 + l;
  };
  const bool pon = (A.debug & 64) && lane == 0 && warp < 16;
  unsigned long long w1 = 0, w2 = 0, w3 = 0;
  const unsigned long long t_start = clock64();

  if (warp == kWarpTma) {
    // ============ raw-row loader: the MERIT gather on the TMA engine ======
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&in_map)) : "memory");
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
#ifdef MERIT_DEV_DEBUG
        if (A.debug & 8192) break;  // no raw rows in the A-release experiment
#endif
        int tile, half;
        unit_of(u, tile, half);
        const int n = tile / A.tiles_per_img;
        const int y0 = (tile - n * A.tiles_per_img) * A.rows;
        for (int g = 0; g < A.n_groups; ++g) {
          const int ky = g / p.CB, cb = g - ky * p.CB;
          for (int h = 0; h < 2; ++h) {
            twait_s1(r_empty(st), ph ^ 1, w1, pon);
            mbar_expect_tx(r_full(st), A.raw_bytes);
            // input rows y0 + ky*dy + oy + {0 .. rows-1}, all W columns, 32
            // channels; rows / channels out of range read as zero
            tma_load_4d_s1(rring + st * A.raw_bytes, &in_map, 0, y0 + ky * p.dy + p.oy, cb * 64 + 32 * h, n,
                           r_full(st));
            if (++st == A.nr) { st = 0; ph ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (TMEMA && warp < kRepackWarps) {
    // ============ repack into TMEM: lane = A row (slot), 32 channels per warp
    // warp w: TMEM lane quadrant w & 3 (the warp's own), channel half w >> 2
    // (raw half slot); every lane loads its pixel's 32 channels (consecutive
    // lanes = consecutive x: conflict-free), splits them and stores 16 hi +
    // 16 lo columns.
    const int w = warp;
    const int q = w & 3, h = w >> 2;
    // raw [c][128 slots]: A row 32q + lane reads the raw word of its segment
    // column (seg_word); channel stride 512 B, an immediate
    const uint32_t lane_off = static_cast<uint32_t>(seg_word(q, lane)) * 4u;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + kTmemA + 16u * h;
    int rs = h, as = 0;
    uint32_t rph = 0, aph = 0;
    for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
      for (int g = 0; g < A.n_groups; ++g) {
#ifdef MERIT_DEV_DEBUG
        if (A.debug & 8192) {  // timing experiment: A slots released without raw rows or repack (wrong values)
          twait_s1(a_empty(as), aph ^ 1, w2, pon);
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full(as));
          if (++as == A.na) { as = 0; aph ^= 1; }
          continue;
        }
#endif
        twait_s1(r_full(rs), rph, w1, pon);
        float v[32];
        const uint32_t src = rring + rs * A.raw_bytes + lane_off;
        const float* sp = reinterpret_cast<const float*>(smem_raw + (src - smem_u32(smem_raw)));
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = sp[c * 128];
        raw_release(r_empty(rs));
        rs += 2;
        while (rs >= A.nr) { rs -= A.nr; rph ^= 1; }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) split_bf16x2(v[2 * i], v[2 * i + 1], hi[i], lo[i]);
        twait_s1(a_empty(as), aph ^ 1, w2, pon);
        tc_fence_after();
        const uint32_t ta = t_lane + static_cast<uint32_t>(as) * 64u;
        TMEM_ST16(ta, hi);
        if (SPLIT3) TMEM_ST16(ta + 32u, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(as));
        if (++as == A.na) { as = 0; aph ^= 1; }
      }
    }
  } else if (warp < kRepackWarps) {
    // ============ repack: raw fp32 [c][r][W] -> bf16 hi/lo K-major planes ===
    // warp w: channels 8w..8w+7 of the k-block (chunk column w of every A
    // row; warps 0-3 read the even raw entries = channels 0-31, warps 4-7
    // the odd ones); lane l: A rows 32j + l, j = 0..3, so an STS.128 phase
    // writes 8 consecutive rows and the 128-B swizzle spreads the banks.
    const int w = warp;
    const uint32_t cbase = static_cast<uint32_t>(8 * (w & 3)) * 512u;  // raw [c][128 slots]
    int rs = w >> 2, as = 0;
    uint32_t rph = 0, aph = 0;
    for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
        int tile, half;
        unit_of(u, tile, half);
      for (int g = 0; g < A.n_groups; ++g) {
        twait_s1(r_full(rs), rph, w1, pon);
        float v[4][8];
        const uint32_t src = rring + rs * A.raw_bytes + cbase;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t a0 = src + static_cast<uint32_t>(seg_word(j, lane)) * 4u;
          const float* sp = reinterpret_cast<const float*>(smem_raw + (a0 - smem_u32(smem_raw)));
#pragma unroll
          for (int c = 0; c < 8; ++c) v[j][c] = sp[c * 128];
        }
        raw_release(r_empty(rs));
        rs += 2;
        while (rs >= A.nr) { rs -= A.nr; rph ^= 1; }
        twait_s1(a_empty(as), aph ^ 1, w2, pon);
        const uint32_t phi = aring + as * A.a_slot;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int row = 32 * j + lane;
          const uint32_t off = (row >> 3) * 1024u + (row & 7) * 128u + (((uint32_t)w ^ (uint32_t)(row & 7)) << 4);
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) split_bf16x2(v[j][2 * c], v[j][2 * c + 1], hi[c], lo[c]);
          st_shared_v4(phi + off, hi[0], hi[1], hi[2], hi[3]);
          if (SPLIT3) st_shared_v4(phi + kAPlane + off, lo[0], lo[1], lo[2], lo[3]);
        }
        fence_proxy_async();
#if MERIT_S1_ALLARRIVE
        mbar_arrive(a_full(as));
#else
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(as));
#endif
        if (++as == A.na) { as = 0; aph ^= 1; }
      }
    }
  } else if (warp == kWarpB) {
    // ============ B loader: stack the three tap matrices along N ==========
    // packed (conv_pack_kernel) k-block (ky, cb, kx) = [hi][lo] planes of
    // BN rows; the slot holds [hi: kx 0 | 1 | 2][lo: kx 0 | 1 | 2], i.e. one
    // K-major SW128 image of N = 3 BN rows per split plane.
    if (lane == 0 && A.resident) {
      // weights resident: every group's full stacked-tap image into its own
      // slot once; half units address their rows inside it (MMA warp)
      constexpr int nsp = SPLIT3 ? 2 : 1;
      if (blockIdx.x < A.n_units) {
        for (int g = 0; g < A.n_groups; ++g) {
          mbar_expect_tx(b_full(g), 3u * nsp * A.b_plane);
          for (int kx = 0; kx < 3; ++kx)
            for (int sp = 0; sp < nsp; ++sp)
              bulk_g2s(bring + g * A.b_slot + (sp * 3 + kx) * A.b_plane,
                       A.wpk + ((long long)(g * 3 + kx) * nsp + sp) * A.b_plane, A.b_plane, b_full(g));
        }
      }
    } else if (lane == 0) {
      constexpr int nsp = SPLIT3 ? 2 : 1;
      int st = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
        int tile, half;
        unit_of(u, tile, half);
        for (int g = 0; g < A.n_groups; ++g) {
          twait_s1(b_empty(st), ph ^ 1, w1, pon);
          // a part unit stacks the taps' rows of its channel part: N = 3 BN / parts
          const uint32_t rows = half < 0 ? A.b_plane : A.b_plane >> A.parts_log2;
          const uint32_t src_off = half < 0 ? 0u : static_cast<uint32_t>(half) * rows;
          mbar_expect_tx(b_full(st), 3u * nsp * rows);
          for (int kx = 0; kx < 3; ++kx)
            for (int sp = 0; sp < nsp; ++sp)
              bulk_g2s(bring + st * A.b_slot + (sp * 3 + kx) * rows,
                       A.wpk + ((long long)(g * 3 + kx) * nsp + sp) * A.b_plane + src_off, rows, b_full(st));
          if (++st == A.nb) { st = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma) {
    // ============ MMA issuer: the whole warp runs the loop (warp-uniform
    // operands in uniform registers), one elected lane issues each MMA ======
    const bool pon_w = (A.debug & 64) != 0;
    const uint32_t idesc_full = make_idesc(3 * BN);
    const uint32_t idesc_half = make_idesc(3 * (BN >> A.parts_log2));
    int as = 0, bs = 0, acc = 0;
    uint32_t aph = 0, bph = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
      int tile, half;
      unit_of(u, tile, half);
      const uint32_t idesc = half < 0 ? idesc_full : idesc_half;
      const uint32_t b_lo16 = (3 * (half < 0 ? A.b_plane : A.b_plane >> A.parts_log2)) >> 4;  // lo planes, descriptor units
      twait_s1(tempty(acc), acc_phase ^ 1, w3, pon_w);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * acc_cols;
      for (int g = 0; g < A.n_groups; ++g) {
        if (A.resident) bs = g, bph = 0;  // loaded once: phase 0 stays complete
        if (!(A.debug & 2048)) {  // 2048: timing experiment, MMAs without operand waits
          twait_s1(a_full(as), aph, w1, pon_w);
          twait_s1(b_full(bs), bph, w2, pon_w);
        }
        tc_fence_after();
        const uint64_t bd = sw128_desc(bring + bs * A.b_slot);
        if (A.resident && half >= 0) {
          // part unit on the resident full image: one N = BN / parts MMA per tap
          // (rows kx * BN + part * BN / parts of each split plane) into columns kx * BN / parts
          const uint32_t hb = static_cast<uint32_t>(p.BN >> A.parts_log2);
          const uint32_t lo16 = (3u * A.b_plane) >> 4;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const uint64_t bk = bd + ((static_cast<uint32_t>(kx * p.BN + half * (p.BN >> A.parts_log2)) * 128u) >> 4);
            const uint32_t dk = d_tmem + static_cast<uint32_t>(kx) * hb;
            const uint32_t idk = make_idesc(p.BN >> A.parts_log2);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if constexpr (TMEMA) {
                const uint32_t ta = tmem_base + kTmemA + static_cast<uint32_t>(as) * 64u;
                tc_mma_ts_w(dk, ta + 8 * k, bk + 2 * k, idk, (g > 0 || k > 0) ? 1u : 0u);
                if (SPLIT3) {
                  tc_mma_ts_w(dk, ta + 8 * k, bk + lo16 + 2 * k, idk, 1u);
                  tc_mma_ts_w(dk, ta + 32 + 8 * k, bk + 2 * k, idk, 1u);
                }
              } else {
                const uint64_t ad = sw128_desc(aring + as * A.a_slot);
                tc_mma_w(dk, ad + 2 * k, bk + 2 * k, idk, (g > 0 || k > 0) ? 1u : 0u);
                if (SPLIT3) {
                  tc_mma_w(dk, ad + 2 * k, bk + lo16 + 2 * k, idk, 1u);
                  tc_mma_w(dk, ad + (kAPlane >> 4) + 2 * k, bk + 2 * k, idk, 1u);
                }
              }
            }
          }
        } else if constexpr (TMEMA) {
          const uint32_t ta = tmem_base + kTmemA + static_cast<uint32_t>(as) * 64u;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            tc_mma_ts_w(d_tmem, ta + 8 * k, bd + 2 * k, idesc, (g > 0 || k > 0) ? 1u : 0u);
            if (SPLIT3) {
              tc_mma_ts_w(d_tmem, ta + 8 * k, bd + b_lo16 + 2 * k, idesc, 1u);
              tc_mma_ts_w(d_tmem, ta + 32 + 8 * k, bd + 2 * k, idesc, 1u);
            }
          }
        } else {
          const uint64_t ad = sw128_desc(aring + as * A.a_slot);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            tc_mma_w(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (g > 0 || k > 0) ? 1u : 0u);
            if (SPLIT3) {
              tc_mma_w(d_tmem, ad + 2 * k, bd + b_lo16 + 2 * k, idesc, 1u);
              tc_mma_w(d_tmem, ad + (kAPlane >> 4) + 2 * k, bd + 2 * k, idesc, 1u);
            }
          }
        }
        if (!A.resident) {
          tc_commit_w(b_empty(bs));
          if (++bs == A.nb) { bs = 0; bph ^= 1; }
        }
        tc_commit_w(a_empty(as));
        if (++as == A.na) { as = 0; aph ^= 1; }
      }
      tc_commit_w(tfull(acc));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    __syncwarp();
  } else if ((warp >= kWarpEpi0 && warp < kWarpEpi0 + 4) || warp >= kWarpEpi1) {
    // ============ epilogue: out[x] = P0[x-1] + P1[x] + P2[x+1] =============
    // Warp quadrant q holds A rows 32q..32q+31 (one row segment with its two
    // halo columns); set k (0: warps 10-13, 1: warps 15-18) takes chunks of
    // kEC channels c0 = kEC * (2i + k).  The x - 1 / x + 1 neighbours are lane
    // shuffles inside the segment: no cross-warp exchange, no barrier.
    const int q = warp & 3;
    const int set = warp >= kWarpEpi1 ? 1 : 0;
    const int r = q >> A.segs_log2;
    const int x = (q & ((1 << A.segs_log2) - 1)) * A.seg_w + lane - 1;
    const bool in_seg = lane >= 1 && lane <= A.seg_w;
    const bool relu = p.post == POST_RELU;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < A.n_units; u += gridDim.x) {
        int tile, half;
        unit_of(u, tile, half);
      const int n = tile / A.tiles_per_img;
      const int y = (tile - n * A.tiles_per_img) * A.rows + r;
      const bool store = in_seg && x < W && y < p.Ho && !(A.debug & 128);
      // a part unit holds BN / parts channels: P_kx at columns kx * bn
      const int bn = half < 0 ? BN : BN >> A.parts_log2;
      const int co_off = half < 0 ? 0 : half * bn;
      const int n_chunks = bn / kEC;
      const int my_last = ((n_chunks - 1 - set) / 2) * 2 + set;  // this set's last chunk
      float* dst = A.out + ((long long)n * p.Cout * p.Ho + y) * W + x + (long long)co_off * p.Ho * W;
      const long long co_stride = (long long)p.Ho * W;
      twait_s1(tfull(acc), acc_phase, w1, pon);
      tc_fence_after();
      if (A.debug & 1024) {  // timing experiment: release the accumulator unread
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const uint32_t t_row = tmem_base + acc * acc_cols + (static_cast<uint32_t>(q * 32) << 16);
      for (int ch = set; ch < n_chunks; ch += 2) {
        const int c0 = ch * kEC;
        uint32_t p0[kEC], p1[kEC], p2[kEC];
        TMEM_LD8(t_row + c0, p0);
        TMEM_LD8(t_row + bn + c0, p1);
        TMEM_LD8(t_row + 2 * bn + c0, p2);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ch == my_last) {  // accumulator drained by this warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(acc));
        }
        const int cmax = p.Cout - co_off - c0;  // channels of this chunk that exist
        float* ptr = dst + (long long)c0 * co_stride;
#pragma unroll
        for (int e = 0; e < kEC; ++e) {
          const float left = __shfl_up_sync(0xffffffffu, __uint_as_float(p0[e]), 1);
          const float right = __shfl_down_sync(0xffffffffu, __uint_as_float(p2[e]), 1);
          float v = __fadd_rn(__fadd_rn(left, __uint_as_float(p1[e])), right);
          v = relu ? fmaxf(v, 0.f) : __fadd_rn(v, 0.f);
          if (store && e < cmax) *ptr = v;
          ptr += co_stride;
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (pon) {
    unsigned long long* pr = A.prof + (blockIdx.x * 16 + warp) * 4;
    pr[0] = clock64() - t_start; pr[1] = w1; pr[2] = w2; pr[3] = w3;
  }
  __syncthreads();
  if (warp == kWarpB) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * kAccCols)
                 : "memory");
  }
}

// N = 3 BN <= 240: Cout <= 64 runs with A in TMEM (N <= 192), Cout 65..80 with
// A in shared memory.  MERIT_S1_N240=0 sends the latter to the general 3-wide
// kernels (where they ran while the raw-slot release fault was open).
int s1_max_n() {
  const char* e = getenv("MERIT_S1_N240");
  return (e && e[0] == '0') ? 192 : 240;
}

int slots_log2_for(int W) {
  for (int l = 5; l <= 7; ++l)
    if (W + 2 <= (1 << l)) return l;
  return -1;
}

}  // namespace

// Geometric eligibility (plan time: decides nothing about packing, which is
// shared with the other conv kernels).
bool conv_s1_eligible(const ConvParams& p, const void* a) {
  if (p.gemm) return false;
  const char* e = getenv("MERIT_CONV_S1");
  if (e && e[0] == '0') return false;
  return p.KW == 3 && p.dx == 1 && p.ox == -1 && p.sx == 1 && p.sy == 1 && p.Wo == p.W && !p.in_bf16 &&
         p.n_tiles_n == 1 && 3 * p.BN <= s1_max_n() && p.BN % 16 == 0 && slots_log2_for(p.W) > 0 && p.W % 4 == 0 &&
         // row segments of at most 30 output columns (32 lanes with both halo columns)
         (p.W + (1 << (slots_log2_for(p.W) - 5)) - 1) >> (slots_log2_for(p.W) - 5) <= 30 &&
         (reinterpret_cast<uintptr_t>(a) % 16) == 0 && tensor_map_encoder() != nullptr;
}

merit_status launch_conv_s1(const merit_plan& plan, const void* a, const void* packed_b, void* out,
                            void* stream) {
  const ConvParams& p = plan.conv;
  S1Args A;
  A.p = p;
  A.wpk = static_cast<const uint8_t*>(packed_b);
  A.out = static_cast<float*>(out);
  A.slots_log2 = slots_log2_for(p.W);
  A.segs_log2 = A.slots_log2 - 5;
  A.seg_w = (p.W + (1 << A.segs_log2) - 1) >> A.segs_log2;
  A.rows = 128 >> A.slots_log2;
  A.tiles_per_img = (p.Ho + A.rows - 1) / A.rows;
  A.n_tiles = p.N * A.tiles_per_img;
  A.n_groups = p.KH * p.CB;
  const bool split3 = p.split == 3;
  const uint32_t nsp = split3 ? 2u : 1u;
  const char* te = getenv("MERIT_S1_TMEMA");
  const bool tmema = !(te && te[0] == '0') && 3 * p.BN <= 192;
  A.raw_bytes = 128u * 32u * 4u;  // box {slots, rows, 32 ch}: slots * rows = 128
  A.a_slot = tmema ? 0u : nsp * kAPlane;  // TMEM-resident A: no shared-memory ring
  A.b_plane = static_cast<uint32_t>(p.BN) * 128u;
  A.b_slot = 3u * nsp * A.b_plane;
  const size_t fixed = 1024 + 128 + 8 * (6 * kMaxRing + 4) + 16;
  const size_t budget = 227 * 1024 - fixed;
  A.na = 2;
  A.nb = 2;
  A.nr = 2;
  auto used_bytes = [&]() {
    return A.na * (size_t)A.a_slot + A.nb * (size_t)A.b_slot + A.nr * (size_t)A.raw_bytes;
  };
  // Weights resident when every (ky, channel block) group fits a B slot next
  // to a 4-deep raw ring (C3: 3 x 48 KB): loaded once per CTA instead of
  // once per tile (C3: 144 KB x 896 tiles = 129 MB of L2 -> SM traffic);
  // measured at C3: 25.2-25.5 us resident vs 24.2 us streamed (the B slots
  // are not the bottleneck), so opt-in (MERIT_S1_RESIDENT=1)
  const char* rese = getenv("MERIT_S1_RESIDENT");
  A.resident = (rese && rese[0] == '1') && A.n_groups <= kMaxRing &&
               A.n_groups * (size_t)A.b_slot + 4 * (size_t)A.raw_bytes + 2 * (size_t)A.a_slot <= budget;
  if (A.resident) A.nb = A.n_groups;
  for (;;) {  // grow: raw (even), A, B
    const size_t used = used_bytes();
    if (A.nr < 4 && used + 2 * A.raw_bytes <= budget) { A.nr += 2; continue; }
    if (!tmema && A.na < 3 && used + A.a_slot <= budget) { ++A.na; continue; }
    if (!A.resident && A.nb < 3 && used + A.b_slot <= budget) { ++A.nb; continue; }
    if (A.resident && A.nr < kMaxRing && used + 2 * A.raw_bytes <= budget) { A.nr += 2; continue; }
    break;
  }
  if (const char* re = getenv("MERIT_S1_RINGS")) {  // "na,nb,nr" (tuning)
    int na, nb, nr;
    if (sscanf(re, "%d,%d,%d", &na, &nb, &nr) == 3 && na >= 1 && nb >= 1 && nr >= 2 && nr % 2 == 0 &&
        na <= kMaxRing && nb <= kMaxRing && nr <= kMaxRing) {
      A.na = tmema ? 2 : na; A.nb = A.resident ? A.n_groups : nb; A.nr = nr;
    }
  }
  if (used_bytes() > budget) return fail(MERIT_E_UNSUPPORTED_VIEW, "stride-1 conv rings exceed shared memory");
  const size_t smem = fixed + used_bytes();
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.Cin, (cuuint64_t)p.N};
  const cuuint64_t strides[3] = {(cuuint64_t)p.W * 4, (cuuint64_t)p.H * p.W * 4,
                                 (cuuint64_t)p.Cin * p.H * p.W * 4};
  // box width = slots (> W): columns x >= W land as zeros, so the raw rows
  // already have the A-row layout (x at slot x + 1, read at word m - 1)
  const cuuint32_t box[4] = {(cuuint32_t)(1u << A.slots_log2), (cuuint32_t)A.rows, 32, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult cr = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(a), dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(MERIT_E_CUDA, "cuTensorMapEncodeTiled failed for the conv input");
  if (A.n_tiles == 0) return MERIT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto kfn = split3 ? (tmema ? conv_s1_kernel<true, true> : conv_s1_kernel<true, false>)
                    : (tmema ? conv_s1_kernel<false, true> : conv_s1_kernel<false, false>);
  cudaError_t e = set_smem_attr(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(conv_s1)");
  int grid = num_sms();
  if (grid > A.n_tiles) grid = A.n_tiles;
  grid = grid_cap(grid);
  // Tail split: the final partial wave of r = n_tiles % grid tiles runs as
  // `parts` r units of BN / parts output channels each, so it costs 1 / parts
  // of a tile instead of a whole one (C3: 896 tiles on 148 SMs, r = 8: four
  // parts of 16 channels, the busiest SM runs 6.25 tiles against 6.05 on
  // average; halves: 6.5).  A part keeps BN / parts a multiple of 16 (N =
  // 3 BN / parts a multiple of 16, whole 8-row B atoms, two epilogue chunks).
  // MERIT_S1_SPLIT=0 / 2 / 4: no split / halves / quarters (A/B).
  {
    const int r = A.n_tiles % grid;
    const char* se = getenv("MERIT_S1_SPLIT");
    const int want = se ? atoi(se) : 4;
    A.parts = 1;
    for (int parts : {4, 2})
      if (A.parts == 1 && parts <= want && r > 0 && parts * r <= grid && p.BN % (16 * parts) == 0) A.parts = parts;
    A.n_full = A.parts > 1 ? A.n_tiles - r : A.n_tiles;
    A.n_units = A.n_full + A.parts * (A.n_tiles - A.n_full);
    if (A.parts == 1) A.parts = 2;  // unused (no part units)
    A.parts_log2 = A.parts == 4 ? 2 : 1;
  }
  {
    const char* dbg = debug_env("MERIT_CONV_DEBUG");
    A.debug = dbg ? atoi(dbg) : 0;
  }
  A.prof = nullptr;
  if (A.debug & 64) {
    cudaMalloc(&A.prof, 8ull * 4 * 16 * grid);
    cudaMemset(A.prof, 0, 8ull * 4 * 16 * grid);
  }
  e = launch_pdl(kfn, dim3(grid), dim3(kThreads), smem, s, 1, map, A);
  if (e != cudaSuccess) return cuda_check(e, "launch(conv_s1)");
  if (A.debug & 64) {
    cudaStreamSynchronize(s);
    std::vector<unsigned long long> h(4 * 16 * grid);
    cudaMemcpy(h.data(), A.prof, h.size() * 8, cudaMemcpyDeviceToHost);
    auto frac = [&](int w0, int w1_, int idx) {
      double t = 0, v = 0;
      for (int b = 0; b < grid; ++b)
        for (int ww = w0; ww < w1_; ++ww) { t += h[(b * 16 + ww) * 4]; v += h[(b * 16 + ww) * 4 + idx]; }
      return t > 0 ? 100.0 * v / t : 0.0;
    };
    fprintf(stderr,
            "[s1 prof] rings nr=%d na=%d nb=%d | tma: r_empty-wait %.1f%% | repack: r_full-wait %.1f%% a_empty-wait "
            "%.1f%% | B: b_empty-wait %.1f%% | mma: a_full %.1f%% b_full %.1f%% tempty %.1f%% | epi: tfull-wait "
            "%.1f%%\n",
            A.nr, A.na, A.nb, frac(kWarpTma, kWarpTma + 1, 1), frac(0, 8, 1), frac(0, 8, 2), frac(kWarpB, kWarpB + 1, 1),
            frac(kWarpMma, kWarpMma + 1, 1), frac(kWarpMma, kWarpMma + 1, 2), frac(kWarpMma, kWarpMma + 1, 3),
            frac(kWarpEpi0, kWarpEpi0 + 4, 1));
    cudaFree(A.prof);
  }
  return launch_status(split3 ? (tmema ? "conv_s1_kernel<split3, taps stacked on N, A in TMEM>"
                                       : "conv_s1_kernel<split3, taps stacked on N>")
                              : (tmema ? "conv_s1_kernel<bf16, taps stacked on N, A in TMEM>"
                                       : "conv_s1_kernel<bf16, taps stacked on N>"));
}

}  // namespace merit_dev
