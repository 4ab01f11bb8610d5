// K3c — stride-2, 3-wide bf16 convolution with the MERIT gather done by the
// TMA engine (the C4 shape: NCHW, KW = 3, ox = -1, sx = 2).
//
// The view's strided row term (y*2 + ky - 1) is a TMA tensor-map traversal
// stride on the H dimension, its zero padding is the TMA out-of-bounds fill,
// and one cp.async.bulk.tensor per (tile, ky, 64-channel block) lands the raw
// rows [c][4 rows][W] in a shared-memory ring several groups deep — no
// registers are spent on bytes in flight and no load instructions are issued
// by the SM.  Eight repack warps turn the raw rows into the two UMMA A planes
// (tap 1 = even columns, tap 2 = odd columns; tap 0 is tap 2 read one slot row
// earlier, the shifted-view trick of conv_tap3.cu), and the MMA / epilogue
// roles are those of conv_tap3.cu.
//
// Slots: 32 per output row (4 leading pads + Wo = 28), a tile = 128 slots =
// 4 output rows of one image, so every tile starts on a pad slot and tap 0
// never needs a guard row.
//
// Warps: 0-7 repack, 8 B loader + TMEM alloc, 9 MMA, 10-13 epilogue, 14 TMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "tc_common.cuh"
#include "tmap.cuh"

namespace merit_dev {
namespace {

using namespace tc;

constexpr int kRepackWarps = 8;
constexpr int kRepackers = kRepackWarps * 32;
constexpr int kWarpB = 8, kWarpMma = 9, kWarpEpi0 = 10, kWarpTma = 14;
// A-ready signal: every repack thread arrives on a_full itself, right after
// its own fence.proxy.async (the release pattern of the CUTLASS transform ->
// MMA pipelines), instead of one elected lane per warp after a __syncwarp
// (time-neutral at C4); 0 = that form, for A/B timing.
#ifndef MERIT_TMA_ALLARRIVE
#define MERIT_TMA_ALLARRIVE 1
#endif
#ifndef MERIT_RAW_RELEASE_FENCE
#define MERIT_RAW_RELEASE_FENCE 1
#endif
constexpr int kThreads = 15 * 32;
constexpr int kMaxRing = 8;
constexpr uint32_t kPlane = kAPlane;           // 16 KB
constexpr uint32_t kASlot = 2 * kPlane;        // [tap2][tap1]
constexpr int kEpiCo = 16;                     // output channels per TMA store

struct TmaArgs {
  ConvParams p;
  const uint8_t* wpk;
  float* out;
  int tiles_per_img;   // Ho / 4
  int n_tiles;
  int n_units;         // scheduling units: tiles, or (pair of M tiles, N tile) in pair mode
  int n_groups;        // KH * CB
  uint32_t raw_bytes;  // W * 4 rows * 32 ch * 2 (half a 64-channel k-block)
  uint32_t b_bytes;    // one (k-block, tap) of B: BN rows x 64 ch
  uint32_t b_slot;     // this CTA's share of it: b_bytes, or b_bytes / 2 in pair mode
  int nr, na, nb;
  uint32_t tmem_cols;
  uint32_t stage_bytes;  // epilogue staging: kEpiCo co x 4 rows x Wo fp32
  unsigned long long* prof;  // MERIT_CONV_DEBUG & 64: per-warp [total, wait1, wait2, wait3]
  int debug;
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int x, int y, int c,
                                            int n, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(c), "r"(n), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void twait(uint32_t bar, uint32_t par, unsigned long long& acc, bool on) {
  if (on) {
    const unsigned long long t0 = clock64();
    mbar_wait(bar, par);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, par);
  }
}

// B tile of one CTA of a pair: completion is signalled on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
// The same, multicast to the CTAs of `mask` (same shared offset in each); each
// destination's bytes complete on its own pair leader's barrier at the same
// offset (CUTLASS's 2-SM multicast load)
__device__ __forceinline__ void tma_load_2d_pair_mc(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                    uint32_t leader_bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int x, int y, int c, int n) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "r"(c), "r"(n)
               : "memory");
}

// PAIR: the kernel runs as clusters of two CTAs that issue cta_group::2 MMAs
// (M = 256): each CTA gathers and repacks its own 128-slot tile (A) and loads
// HALF of every weight tile (B rows = output channels), so each weight byte
// fetched from L2 feeds 256 output slots.  The leader (rank 0) issues the
// MMAs; operand-ready signals of the peer arrive on the leader's barriers,
// and the MMA commits multicast back to both CTAs.
//
// QUAD (needs PAIR): clusters of two such pairs that share every weight tile:
// the CTAs holding the same half of it (ranks 0 / 2 and 1 / 3) each load a
// quarter and multicast it to both, so a weight byte read from L2 feeds 512
// output slots.  A weight slot is refilled once both pairs' MMAs released it.
template <bool PAIR, bool QUAD = false>
__global__ void __maxnreg__(128)  // 15 warps: <= 4 per SM sub-partition x 128 regs
conv_tma_kernel(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
                const __grid_constant__ CUtensorMap b_map, TmaArgs A) {
  extern __shared__ uint8_t smem_raw[];
  const ConvParams& p = A.p;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  // B first: tap 0's view of A row 0 starts 128 B before the tap-2 plane,
  // which must be a valid shared address (its value only feeds the pad slot
  // of output row 0, which is never stored).
  const uint32_t bring = base;                          // nb x b_bytes
  const uint32_t aring = bring + A.nb * A.b_slot;       // na x kASlot
  const uint32_t rring = aring + A.na * kASlot;         // nr x raw_bytes
  const uint32_t ering = rring + A.nr * A.raw_bytes;    // 2 x stage_bytes (epilogue)
  const uint32_t bars = (ering + 2 * A.stage_bytes + 7u) & ~7u;
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
  auto tap2_plane = [&](int s) { return aring + s * kASlot; };
  auto tap1_plane = [&](int s) { return aring + s * kASlot + kPlane; };

  constexpr uint32_t kSplit = PAIR ? 2u : 1u;  // CTAs feeding one MMA
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;  // rank in the cluster
  const uint32_t rank = crank & 1u;                          // rank in the pair
  const uint32_t lead = crank & ~1u;                         // the pair's leader
  const uint16_t pair_mask = static_cast<uint16_t>(3u << lead);
  // operand-ready / accumulator-free signals go to the MMA-issuing CTA
  auto to_leader = [&](uint32_t bar) {
    if (PAIR) mbar_arrive_cluster(mapa_shared(bar, lead)); else mbar_arrive(bar);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < A.nr; ++s) {
      mbar_init(r_full(s), 1);
      mbar_init(r_empty(s), kRepackers / 2);  // one half of the repack warps
    }
    for (int s = 0; s < A.na; ++s) {
#if MERIT_TMA_ALLARRIVE
      mbar_init(a_full(s), kRepackers * kSplit);  // every repack thread, after its own proxy fence
#else
      mbar_init(a_full(s), kRepackWarps * kSplit);  // one elected lane per repack warp
#endif
      mbar_init(a_empty(s), 1);
    }
    for (int s = 0; s < A.nb; ++s) {
      mbar_init(b_full(s), 1);
      mbar_init(b_empty(s), QUAD ? 2 : 1);  // quad: both pairs' MMAs release it
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), 4 * kSplit);  // one elected lane per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpB) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "r"(A.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "r"(A.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  pdl_launch_dependents();
  pdl_wait();  // prologue done: from here on global memory is touched
  const int BN = p.BN;
  const int W = p.W;
  const bool pon = (A.debug & 64) && lane == 0;
  unsigned long long w1 = 0, w2 = 0, w3 = 0;
  const unsigned long long t_start = clock64();
  // scheduling unit -> (M tile, N tile); in pair mode the two CTAs of a
  // cluster take adjacent M tiles (an odd last one reads / writes out of
  // bounds image N, which TMA zero-fills / clips)
  constexpr int kCl = QUAD ? 4 : (PAIR ? 2 : 1);  // CTAs per cluster = M tiles per unit
  const int unit0 = static_cast<int>(blockIdx.x) / kCl;
  const int ustep = static_cast<int>(gridDim.x) / kCl;
  auto m_tile = [&](int u) { return kCl * (u / p.n_tiles_n) + static_cast<int>(crank); };

  if (warp == kWarpTma) {
    // ============ raw-row loader: the MERIT gather on the TMA engine ======
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&in_map)) : "memory");
      int st = 0;
      uint32_t ph = 0;
      for (int tile = unit0; tile < A.n_units; tile += ustep) {
        const int mt = m_tile(tile);
        const int n = mt / A.tiles_per_img;
        const int y0 = (mt - n * A.tiles_per_img) * 4;
        for (int g = 0; g < A.n_groups; ++g) {
          const int ky = g / p.CB, cb = g - (g / p.CB) * p.CB;
          for (int h = 0; h < 2; ++h) {
            twait(r_empty(st), ph ^ 1, w1, pon);
            mbar_expect_tx(r_full(st), A.raw_bytes);
            // rows 2*y0 + ky - 1 + {0, 2, 4, 6} (traversal stride 2), all W
            // columns, 32 channels; out-of-range rows / channels read as zero.
            tma_load_4d(rring + st * A.raw_bytes, &in_map, 0, y0 * p.sy + ky * p.dy + p.oy, cb * 64 + 32 * h,
                        n, r_full(st));
            if (++st == A.nr) { st = 0; ph ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < kRepackWarps) {
    // ============ repack: raw [c][r][W] -> UMMA K-major planes =============
    // warp w: channels 8w..8w+7 (chunk column w of every A row); lane l:
    // output column x = l - 4 (lanes 0-3 are the row's pad slots) of all four
    // output rows, i.e. A rows 32k + l, k = 0..3.  One 32-bit shared load per
    // (channel, row) brings input columns 2x, 2x+1 = taps 1 and 2; in step k
    // the 8 lanes of an STS.128 phase write 8 consecutive rows, so the 128-B
    // swizzle spreads them over all banks.
    const int w = warp, l = lane;
    const int x = l - 4;
    const bool pad = x < 0;
    const uint32_t rowbytes = static_cast<uint32_t>(W) * 2u;
    // raw entries alternate channel halves: warps 0-3 consume the even
    // entries (channels 0-31 of the k-block), warps 4-7 the odd ones.  nr is
    // even, so every slot belongs to one half and its mbarrier phases follow
    // that half's program order (an odd ring would let the halves' phases
    // alias).
    const uint32_t roff = static_cast<uint32_t>(8 * (w & 3)) * 4u * rowbytes + (pad ? 0u : 4u * x);
    int rs = w >> 2, as = 0;
    uint32_t rph = 0, aph = 0;
    for (int tile = unit0; tile < A.n_units; tile += ustep) {
      for (int g = 0; g < A.n_groups; ++g) {
        twait(r_full(rs), rph, w1, pon);
        uint32_t v[4][8];  // [row k][channel c]: (tap1 | tap2 << 16)
        const uint32_t src = rring + rs * A.raw_bytes + roff;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint32_t t = 0u;
            if (!pad)
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(src + (c * 4u + k) * rowbytes));
            v[k][c] = t;
          }
        // the loads above must have RETURNED before the slot is handed back
        // (the arrive alone does not wait for them: conv_tma_s1.cu raw_release)
#if MERIT_RAW_RELEASE_FENCE
        __threadfence_block();
#endif
        mbar_arrive(r_empty(rs));
        rs += 2;
        while (rs >= A.nr) { rs -= A.nr; rph ^= 1; }
        twait(a_empty(as), aph ^ 1, w2, pon);
        const uint32_t p2 = tap2_plane(as), p1 = tap1_plane(as);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int row = 32 * k + l;
          const uint32_t off = (row >> 3) * 1024u + (row & 7) * 128u + (((uint32_t)w ^ (uint32_t)(row & 7)) << 4);
          const uint32_t* wv = v[k];
          st_shared_v4(p1 + off, __byte_perm(wv[0], wv[1], 0x5410), __byte_perm(wv[2], wv[3], 0x5410),
                       __byte_perm(wv[4], wv[5], 0x5410), __byte_perm(wv[6], wv[7], 0x5410));
          st_shared_v4(p2 + off, __byte_perm(wv[0], wv[1], 0x7632), __byte_perm(wv[2], wv[3], 0x7632),
                       __byte_perm(wv[4], wv[5], 0x7632), __byte_perm(wv[6], wv[7], 0x7632));
        }
        fence_proxy_async();
#if MERIT_TMA_ALLARRIVE
        to_leader(a_full(as));
#else
        __syncwarp();
        if (l == 0) to_leader(a_full(as));
#endif
        if (++as == A.na) { as = 0; aph ^= 1; }
      }
    }
  } else if (warp == kWarpB) {
    // ============ B loader =====================================================
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int tile = unit0; tile < A.n_units; tile += ustep) {
        const int nt = tile % p.n_tiles_n;
        for (int kb = 0; kb < p.n_kb; ++kb) {
          twait(b_empty(st), ph ^ 1, w1, pon);
          if (QUAD) {
            // this CTA's quarter: sub-half (crank >> 1) of weight half `rank`,
            // multicast to the two CTAs holding that half; every pair leader
            // still receives its whole tile
            if (rank == 0) mbar_expect_tx(b_full(st), A.b_bytes);
            const uint32_t q = A.b_slot / 2;
            const uint32_t sub = crank >> 1;
            const long long off = ((long long)nt * p.n_kb + kb) * A.b_bytes + rank * A.b_slot + sub * q;
            tma_load_2d_pair_mc(bring + st * A.b_slot + sub * q, &b_map, 0, static_cast<int>(off >> 8),
                                mapa_shared(b_full(st), lead), static_cast<uint16_t>(rank ? 0xAu : 0x5u));
          } else if (PAIR) {
            // both halves complete on the leader's barrier, which expects the
            // whole tile
            if (rank == 0) mbar_expect_tx(b_full(st), A.b_bytes);
            const long long off = ((long long)nt * p.n_kb + kb) * A.b_bytes + rank * A.b_slot;
            tma_load_2d_pair(bring + st * A.b_slot, &b_map, 0, static_cast<int>(off >> 8),
                             mapa_shared(b_full(st), lead));
          } else {
            mbar_expect_tx(b_full(st), A.b_bytes);
            bulk_g2s(bring + st * A.b_bytes, A.wpk + ((long long)nt * p.n_kb + kb) * A.b_bytes, A.b_bytes,
                     b_full(st));
          }
          if (++st == A.nb) { st = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma) {
    // ============ MMA issuer: the leader CTA's whole warp runs the loop
    // (warp-uniform operands), one elected lane issues (tc_common.cuh) ======
    if (rank == 0) {
      const bool pon_w = (A.debug & 64) != 0;
      const uint32_t idesc = PAIR ? make_idesc_pair(BN) : make_idesc(BN);
      int as = 0, bs = 0, acc = 0;
      uint32_t aph = 0, bph = 0, acc_phase = 0;
      for (int tile = unit0; tile < A.n_units; tile += ustep) {
        twait(tempty(acc), acc_phase ^ 1, w3, pon_w);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int g = 0; g < A.n_groups; ++g) {
          twait(a_full(as), aph, w1, pon_w);
          tc_fence_after();
          for (int kx = 0; kx < 3; ++kx) {
            twait(b_full(bs), bph, w2, pon_w);
            tc_fence_after();
            // tap 0 = tap-2 plane one slot row earlier; tap 1; tap 2
            const uint32_t a0 = kx == 1 ? tap1_plane(as) : tap2_plane(as) - (kx == 0 ? 128u : 0u);
            const uint64_t ad = sw128_desc(a0), bd = sw128_desc(bring + bs * A.b_slot);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t accum = (g > 0 || kx > 0 || k > 0) ? 1u : 0u;
              if (PAIR)
                tc_mma_pair_w(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
              else
                tc_mma_w(d_tmem, ad + 2 * k, bd + 2 * k, idesc, accum);
            }
            if (PAIR) tc_commit_pair_w(b_empty(bs), QUAD ? 0xF : pair_mask); else tc_commit_w(b_empty(bs));
            if (++bs == A.nb) { bs = 0; bph ^= 1; }
          }
          if (PAIR) tc_commit_pair_w(a_empty(as), pair_mask); else tc_commit_w(a_empty(as));
          if (++as == A.na) { as = 0; aph ^= 1; }
        }
        if (PAIR) tc_commit_pair_w(tfull(acc), pair_mask); else tc_commit_w(tfull(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kWarpEpi0 && warp < kWarpEpi0 + 4) {
    // ============ epilogue: TMEM -> smem [co][4][Wo] -> TMA store =========
    // Warp quadrant qd holds slot rows 32qd..32qd+31 = output row y0 + qd,
    // lane = x + 4.  Each kEpiCo-channel chunk is staged in shared memory and
    // written to NCHW by ONE tensor store (box Wo x 4 x kEpiCo) issued by one
    // thread; TMEM is released right after the last tcgen05.ld of the tile.
    const int qd = warp & 3;
    const int x = lane - 4;
    const bool valid = x >= 0 && x < p.Wo;
    const bool leader = warp == kWarpEpi0 && lane == 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int sb = 0;  // staging buffer
    for (int tile = unit0; tile < A.n_units; tile += ustep) {
      const int mt = m_tile(tile), nt = tile % p.n_tiles_n;
      const int n = mt / A.tiles_per_img;
      const int y0 = (mt - n * A.tiles_per_img) * 4;
      twait(tfull(acc), acc_phase, w1, pon);
      tc_fence_after();
#ifdef MERIT_DEV_DEBUG
      if (A.debug & 1024) {  // timing experiment: release the accumulator unread (no output)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) to_leader(tempty(acc));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
#endif
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(qd * 32) << 16);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t rr[32];
        TMEM_LD32(t_row + c0, rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 + 32 >= BN) {  // accumulator drained: let the MMA reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) to_leader(tempty(acc));
        }
#pragma unroll
        for (int hh = 0; hh < 32 / kEpiCo; ++hh) {
          // staging buffer sb must no longer be read by an in-flight store
          if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const uint32_t sbase = ering + sb * A.stage_bytes;
          if (valid) {
#pragma unroll
            for (int j = 0; j < kEpiCo; ++j) {
              float v = __uint_as_float(rr[kEpiCo * hh + j]);
              v = p.post == POST_RELU ? ((v < 0.f) ? 0.f : v) : __fadd_rn(v, 0.f);
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(sbase + 4u * ((j * 4 + qd) * p.Wo + x)), "f"(v)
                           : "memory");
            }
          }
          fence_proxy_async();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (leader && nt * BN + c0 + kEpiCo * hh < p.Cout) {
            tma_store_4d(&out_map, sbase, 0, y0, nt * BN + c0 + kEpiCo * hh, n);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          sb ^= 1;
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (pon) {
    unsigned long long* pr = A.prof + (blockIdx.x * 16 + warp) * 4;
    pr[0] = clock64() - t_start; pr[1] = w1; pr[2] = w2; pr[3] = w3;
  }
  // pair: neither CTA may exit while the other can still signal it or the
  // leader's MMAs can still read its shared memory
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == kWarpB) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(A.tmem_cols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(A.tmem_cols)
                   : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() { return tensor_map_encoder(); }

}  // namespace

bool conv_tma_eligible(const ConvParams& p, const void* a) {
  if (p.gemm) return false;
  const char* e = getenv("MERIT_CONV_TMA");
  if (e && e[0] == '0') return false;
  return p.KW == 3 && p.dx == 1 && p.ox == -1 && p.sx == 2 && p.in_bf16 && p.split == 1 &&
         p.W % 8 == 0 && 2 * p.Wo == p.W && p.Wo + 4 == 32 && p.Ho % 4 == 0 && p.W <= 256 &&
         (p.Wo * 4) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(a) % 16) == 0 && get_encode() != nullptr;
}

merit_status launch_conv_tma(const merit_plan& plan, const void* a, const void* packed_b, void* out,
                             void* stream) {
  const ConvParams& p = plan.conv;
  TmaArgs A;
  A.p = p;
  A.wpk = static_cast<const uint8_t*>(packed_b);
  A.out = static_cast<float*>(out);
  A.tiles_per_img = p.Ho / 4;
  const int m_tiles = p.N * A.tiles_per_img;
  A.n_tiles = m_tiles * p.n_tiles_n;
  // CTA pairs (cta_group::2) unless disabled; BN % 16 == 0 keeps each half of
  // a weight tile a whole number of 8-row swizzle atoms
  const char* pe = getenv("MERIT_CONV_PAIR");
  const bool pair = !(pe && pe[0] == '0') && p.BN % 16 == 0 && num_sms() >= 2;
  // two pairs per cluster sharing weight tiles by multicast: each quarter of
  // a tile must be whole 1 KB swizzle atoms (BN % 32 == 0)
  const char* qe = getenv("MERIT_CONV_QUAD");
  const bool quad = pair && (qe && qe[0] == '1') && p.BN % 32 == 0 && num_sms() >= 4;
  const int mpu = quad ? 4 : (pair ? 2 : 1);  // M tiles per scheduling unit
  A.n_units = ((m_tiles + mpu - 1) / mpu) * p.n_tiles_n;
  A.n_groups = p.KH * p.CB;
  A.raw_bytes = static_cast<uint32_t>(p.W) * 4u * 32u * 2u;
  A.b_bytes = static_cast<uint32_t>(p.BN) * 128u;
  A.b_slot = pair ? A.b_bytes / 2 : A.b_bytes;
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * p.BN)) cols <<= 1;
  A.tmem_cols = cols;
  const size_t fixed = 1024 + 8 * (6 * kMaxRing + 4) + 16 + 8;
  const size_t budget = 227 * 1024 - fixed;
  A.stage_bytes = kEpiCo * 4u * static_cast<uint32_t>(p.Wo) * 4u;
  A.na = 2;
  A.nr = 2;
  A.nb = 2;
  int nb_first = 4;  // weight slots granted before the raw ring grows
  if (const char* r = getenv("MERIT_TMA_NB_FIRST")) nb_first = atoi(r);
  auto used_bytes = [&]() {
    return A.na * (size_t)kASlot + A.nb * (size_t)A.b_slot + A.nr * (size_t)A.raw_bytes + 2 * (size_t)A.stage_bytes;
  };
  // grow the rings in the order that hides the most latency: B, raw, B, A
  for (;;) {
    const size_t used = used_bytes();
    if (A.nb < nb_first && used + A.b_slot <= budget) { ++A.nb; continue; }
    if (A.nr < 4 && used + 2 * A.raw_bytes <= budget) { A.nr += 2; continue; }  // even
    if (A.nb < kMaxRing && used + A.b_slot <= budget) { ++A.nb; continue; }
    if (A.na < 3 && used + kASlot <= budget) { ++A.na; continue; }
    break;
  }
  const size_t used = used_bytes();
  if (used > budget) return fail(MERIT_E_UNSUPPORTED_VIEW, "TMA conv rings exceed shared memory");
  const size_t smem = fixed + used;
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.Cin, (cuuint64_t)p.N};
  const cuuint64_t strides[3] = {(cuuint64_t)p.W * 2, (cuuint64_t)p.H * p.W * 2,
                                 (cuuint64_t)p.Cin * p.H * p.W * 2};
  const cuuint32_t box[4] = {(cuuint32_t)p.W, 8, 32, 1};
  const cuuint32_t estr[4] = {1, (cuuint32_t)p.sy, 1, 1};
  CUresult cr = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a), dims, strides,
                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(MERIT_E_CUDA, "cuTensorMapEncodeTiled failed for the conv input");
  CUtensorMap omap;
  const cuuint64_t odims[4] = {(cuuint64_t)p.Wo, (cuuint64_t)p.Ho, (cuuint64_t)p.Cout, (cuuint64_t)p.N};
  const cuuint64_t ostr[3] = {(cuuint64_t)p.Wo * 4, (cuuint64_t)p.Ho * p.Wo * 4, (cuuint64_t)p.Cout * p.Ho * p.Wo * 4};
  const cuuint32_t obox[4] = {(cuuint32_t)p.Wo, 4, kEpiCo, 1};
  const cuuint32_t oestr[4] = {1, 1, 1, 1};
  cr = get_encode()(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, odims, ostr, obox, oestr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(MERIT_E_CUDA, "cuTensorMapEncodeTiled failed for the conv output");
  // packed weights as rows of 256 bytes: one box = this CTA's half tile
  CUtensorMap bmap;
  std::memset(&bmap, 0, sizeof(bmap));
  if (pair) {
    const cuuint64_t bdims[2] = {256, (cuuint64_t)(p.packed_b_bytes / 256)};
    const cuuint64_t bstr[1] = {256};
    const cuuint32_t bbox[2] = {256, (quad ? A.b_slot / 2 : A.b_slot) / 256};
    const cuuint32_t bestr[2] = {1, 1};
    cr = get_encode()(&bmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(packed_b), bdims, bstr, bbox,
                      bestr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(MERIT_E_CUDA, "cuTensorMapEncodeTiled failed for the conv weights");
  }
  if (A.n_tiles == 0) return MERIT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto kfn = quad ? conv_tma_kernel<true, true> : (pair ? conv_tma_kernel<true> : conv_tma_kernel<false>);
  cudaError_t e = set_smem_attr(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(conv_tma)");
  int grid;
  if (quad) {
    int quads = num_sms() / 4;
    static std::mutex qmu;
    static std::vector<std::pair<size_t, int>> qcache;  // smem bytes -> 4-CTA clusters
    int mc = -1;
    {
      std::lock_guard<std::mutex> lk(qmu);
      for (auto& c : qcache)
        if (c.first == smem) mc = c.second;
      if (mc < 0) {
        mc = max_active_clusters(kfn, dim3(kThreads), smem, 4u);
        qcache.push_back({smem, mc});
      }
    }
    if (mc > 0 && quads > mc) quads = mc;
    if (A.debug & 4096) fprintf(stderr, "[conv_tma] max active 4-CTA clusters %d, quads %d\n", mc, quads);
    if (quads > A.n_units) quads = A.n_units;
    grid = 4 * grid_cap(quads);
  } else if (pair) {
    int pairs = num_sms() / 2;
    // only as many pairs as can be co-resident (TPC / GPC placement): a
    // surplus pair would run its units as a second wave after everyone else
    static std::mutex mu;
    static std::vector<std::pair<size_t, int>> cache;  // smem bytes -> clusters
    int max_clusters = -1;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& c : cache)
        if (c.first == smem) max_clusters = c.second;
      if (max_clusters < 0) {
        max_clusters = max_active_clusters(kfn, dim3(kThreads), smem, 2u);
        cache.push_back({smem, max_clusters});
      }
    }
    if (max_clusters > 0 && pairs > max_clusters) pairs = max_clusters;
    if (A.debug & 4096) fprintf(stderr, "[conv_tma] max active 2-CTA clusters %d, pairs %d\n", max_clusters, pairs);
    if (pairs > A.n_units) pairs = A.n_units;
    grid = 2 * grid_cap(pairs);
  } else {
    grid = num_sms();
    if (grid > A.n_tiles) grid = A.n_tiles;
    grid = grid_cap(grid);
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
  e = launch_pdl(kfn, dim3(grid), dim3(kThreads), smem, s, static_cast<unsigned>(mpu), map, omap, bmap, A);
  if (e != cudaSuccess) return cuda_check(e, "launch(conv_tma)");
  if (A.debug & 64) {
    cudaStreamSynchronize(s);
    std::vector<unsigned long long> h(4 * 16 * grid);
    cudaMemcpy(h.data(), A.prof, h.size() * 8, cudaMemcpyDeviceToHost);
    auto frac = [&](int w0, int w1_, int idx, int bstep) {
      double t = 0, v = 0;
      for (int b = 0; b < grid; b += bstep)
        for (int ww = w0; ww < w1_; ++ww) { t += h[(b * 16 + ww) * 4]; v += h[(b * 16 + ww) * 4 + idx]; }
      return t > 0 ? 100.0 * v / t : 0.0;
    };
    const int ms = pair ? 2 : 1;  // MMA issuers: leaders only
    fprintf(stderr, "[tma prof] %s rings nr=%d na=%d nb=%d | tma: r_empty-wait %.1f%% | repack: r_full-wait %.1f%% a_empty-wait %.1f%% | B: b_empty-wait %.1f%% | mma: a_full %.1f%% b_full %.1f%% tempty %.1f%% | epi: tfull-wait %.1f%%\n",
            pair ? "pair" : "single", A.nr, A.na, A.nb, frac(kWarpTma, kWarpTma + 1, 1, 1), frac(0, 8, 1, 1),
            frac(0, 8, 2, 1), frac(kWarpB, kWarpB + 1, 1, 1), frac(kWarpMma, kWarpMma + 1, 1, ms),
            frac(kWarpMma, kWarpMma + 1, 2, ms), frac(kWarpMma, kWarpMma + 1, 3, ms), frac(kWarpEpi0, kWarpEpi0 + 4, 1, 1));
    cudaFree(A.prof);
  }
  return launch_status(quad ? "conv_tma_kernel<quad, cta_group::2, weight multicast>"
                              : (pair ? "conv_tma_kernel<pair, cta_group::2>" : "conv_tma_kernel<single>"));
}

}  // namespace merit_dev
