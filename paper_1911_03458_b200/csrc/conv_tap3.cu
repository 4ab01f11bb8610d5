// K3b — 3-wide convolution windows (KW = 3, dx = 1, ox = -1, stride 1 or 2)
// on tcgen05 with TAP-SHARING SHIFTED VIEWS.
//
// The MERIT view of a convolution (workloads.hpp:180-195) maps output pixel x
// and tap kx to input column sx*x + kx - 1.  Along a row of pixels the three
// taps overlap: for stride 2, tap 0 of pixel x is tap 2 of pixel x-1 (column
// 2x-1); for stride 1, taps 0 and 2 of pixel x are tap 1 of pixels x-1 and
// x+1.  If the GEMM rows are laid out as "slots" with one padding slot before
// every output row (and one after it for stride 1), these identities hold at
// row boundaries too (the padding slot reads only padding).  So the A-operand
// tile of the shifted tap is the SAME shared-memory tile, read one row earlier
// or later: the UMMA descriptor's start address moves by +-128 B (the
// hardware applies the 128-B swizzle from physical address bits, so the
// descriptor's base_offset field stays 0 — measured).  The producers write two
// tiles per (ky, channel-block) group for stride 2 and ONE for stride 1,
// instead of three, with no shuffles: the view's kx term is executed by the
// tensor core's operand addressing.
//
// Pipeline (persistent, one CTA per SM, warp-specialised, 448 threads):
//   warps 0-7  producers: thread = (slot row r, channel half h); one coalesced
//              load per (channel, input row) per thread, software-pipelined one
//              group ahead; guard rows (-1 / 128) come from one channel per lane
//              of the edge warps and are stored as 16-bit elements.
//   warp 8     TMEM allocation + B loader (cp.async.bulk of packed weights)
//   warp 9     MMA issuer: per group, 3 taps x 4 K-steps (x3 for the f32 split)
//   warps 10-13 epilogue: tcgen05.ld -> NCHW fp32 stores, skipping pad slots
// Separate rings for A (per group) and B (per k-block) so B can run ahead.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

namespace merit_dev {
namespace {

using namespace tc;

constexpr int kProducerWarps = 8;
constexpr int kProducers = kProducerWarps * 32;
constexpr int kWarpLoad = kProducerWarps;
constexpr int kWarpMma = kProducerWarps + 1;
constexpr int kThreads = (kProducerWarps + 2 + 4) * 32;
constexpr uint32_t kGuard = 1024;                     // guard atom before / after each plane
constexpr uint32_t kPlaneG = kGuard + kAPlane + kGuard;
constexpr int kMaxRing = 8;

struct Tap3Args {
  ConvParams p;
  const void* in;
  const uint8_t* wpk;
  float* out;
  int S;            // slots per output row
  int padL;         // 1
  long long slots;  // N * Ho * S
  int n_tiles;      // ceil(slots / 128) * n_tiles_n
  int n_groups;     // KH * CB
  int nplanes;      // tap planes x (split3 ? 2 : 1)
  uint32_t a_slot;  // nplanes * kPlaneG
  uint32_t b_bytes; // per k-block
  int na, nb;
  uint32_t tmem_cols;
  unsigned long long* prof;  // MERIT_CONV_DEBUG & 64: per-role cycle counters
  int debug;
};

__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(static_cast<unsigned short>(v)) : "memory");
}

template <bool IN_BF16, bool SPLIT3, int SX>
__global__ void __launch_bounds__(kThreads, 1) conv_tap3_kernel(Tap3Args A) {
  extern __shared__ uint8_t smem_raw[];
  const ConvParams& p = A.p;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int NTP = SX == 2 ? 2 : 1;      // tap planes: [tap2, tap1] or [tap1]
  constexpr int NSPL = SPLIT3 ? 2 : 1;      // hi / lo
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t aring = base;
  const uint32_t bring = aring + A.na * A.a_slot;
  const uint32_t bars = bring + A.nb * A.b_bytes;
  auto a_full = [&](int s) { return bars + 8u * s; };
  auto a_empty = [&](int s) { return bars + 8u * (kMaxRing + s); };
  auto b_full = [&](int s) { return bars + 8u * (2 * kMaxRing + s); };
  auto b_empty = [&](int s) { return bars + 8u * (3 * kMaxRing + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (4 * kMaxRing + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (4 * kMaxRing + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (4 * kMaxRing + 4);
  volatile uint32_t* tmem_slot_ptr =
      reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));
  // plane data address: slot s, tap plane tp, hi/lo hl
  auto plane = [&](int s, int tp, int hl) {
    return aring + s * A.a_slot + (tp * NSPL + hl) * kPlaneG + kGuard;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < A.na; ++s) {
      mbar_init(a_full(s), kProducers);
      mbar_init(a_empty(s), 1);
    }
    for (int s = 0; s < A.nb; ++s) {
      mbar_init(b_full(s), 1);
      mbar_init(b_empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kWarpLoad) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(A.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  pdl_launch_dependents();
  pdl_wait();  // prologue done: from here on global memory is touched

  const long long HW = (long long)p.H * p.W;
  const int BN = p.BN;
  const long long HoS = (long long)p.Ho * A.S;

  if (warp < kProducerWarps) {
    // ============ A producers =================================================
    const int r = threadIdx.x & 127;  // slot row in the tile
    const int h = threadIdx.x >> 7;   // channel half
    const uint32_t row_off = (r >> 3) * 1024u + (r & 7) * 128u;
    const uint32_t swz = r & 7;
    // edge warps: row 0 (warps 0, 4) own the guard row -1; row 127 (warps 3, 7)
    // own guard row 128 (stride 1 only)
    const bool edge_lo = (warp & 3) == 0;
    const bool edge_hi = SX == 1 && (warp & 3) == 3;
    const bool prof_on = (A.debug & 64) && lane == 0;
    unsigned long long c_ldwait = 0, c_empty = 0, c_emit = 0, c_issue = 0;
    const unsigned long long c_start = clock64();
    int stage = 0;
    uint32_t phase = 0;
    struct Grp {
      uint32_t w[32];
      uint32_t g;  // guard value for channel `lane` (edge warps)
    };
    // Pixel of this thread's slot row for a tile (32-bit math, once per tile).
    struct Pix {
      int n, y, x;
      bool in;
    };
    const int S = A.S, Ho = p.Ho;
    auto pix_of = [&](int tile) {
      Pix q;
      const int slot = (tile / p.n_tiles_n) * kBM + r;  // slots < 2^31 (checked at launch)
      q.in = slot < static_cast<int>(A.slots);
      const int rowi = slot / S;          // n * Ho + y
      q.x = slot - rowi * S - A.padL;
      q.n = rowi / Ho;
      q.y = rowi - q.n * Ho;
      if (!q.in) { q.n = 0; q.y = 0; q.x = -1; }
      return q;
    };
    auto load_grp = [&](Grp& G, const Pix& P, int ky, int cb) {
      const int n = P.n, y = P.y, x = P.x;
      const bool in_slot = P.in;
      const int iy = y * p.sy + ky * p.dy + p.oy;
      const bool rowok = in_slot && iy >= 0 && iy < p.H;
      const int c0 = cb * 64 + h * 32;
      const int nc = rowok ? min(32, p.Cin - c0) : 0;
      const long long pl = ((long long)n * p.Cin + c0) * HW + (long long)iy * p.W;
      // column of the stored tap: stride 2 -> 2x (word 2x,2x+1); stride 1 -> x
      const int col = SX == 2 ? 2 * x : x;
      const bool colok = col >= 0 && (SX == 2 ? col + 1 < p.W : col < p.W);
      if (IN_BF16) {
        const uint16_t* src = static_cast<const uint16_t*>(A.in) + pl + col;
        if (SX == 2) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            G.w[c] = (c < nc && colok) ? __ldg(reinterpret_cast<const uint32_t*>(src + c * HW)) : 0u;
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) G.w[c] = (c < nc && colok) ? __ldg(src + c * HW) : 0u;
        }
      } else {
        const float* src = static_cast<const float*>(A.in) + pl + col;
#pragma unroll
        for (int c = 0; c < 32; ++c) G.w[c] = (c < nc && colok) ? __float_as_uint(__ldg(src + c * HW)) : 0u;
      }
      // guard: edge lane's pixel, neighbouring column; channel = lane
      G.g = 0u;
      if (edge_lo || edge_hi) {
        const int src_lane = edge_lo ? 0 : 31;
        const int xe = __shfl_sync(0xffffffffu, x, src_lane);
        const long long ple = __shfl_sync(0xffffffffu, pl, src_lane);
        const int nce = __shfl_sync(0xffffffffu, nc, src_lane);
        const int gcol = edge_lo ? (SX == 2 ? 2 * xe - 1 : xe - 1) : xe + 1;
        if (lane < nce && gcol >= 0 && gcol < p.W) {
          if (IN_BF16) G.g = __ldg(static_cast<const uint16_t*>(A.in) + ple + (long long)lane * HW + gcol);
          else G.g = __float_as_uint(__ldg(static_cast<const float*>(A.in) + ple + (long long)lane * HW + gcol));
        }
      }
    };
    auto emit_grp = [&](const Grp& G) {
      unsigned long long t0 = prof_on ? clock64() : 0;
      if (prof_on) {
        uint32_t dep = G.g;
#pragma unroll
        for (int c = 0; c < 32; ++c) dep ^= G.w[c];
        asm volatile("" ::"r"(dep));
        const unsigned long long t1 = clock64();
        c_ldwait += t1 - t0;
        t0 = t1;
      }
      mbar_wait(a_empty(stage), phase ^ 1);
      if (prof_on) { const unsigned long long t1 = clock64(); c_empty += t1 - t0; t0 = t1; }
#pragma unroll
      for (int tp = 0; tp < NTP; ++tp) {
        const uint32_t ph = plane(stage, tp, 0);
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          const uint32_t dst = ph + row_off + (((h * 4 + q8) ^ swz) << 4);
          if (IN_BF16) {
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t w0 = G.w[q8 * 8 + 2 * e], w1 = G.w[q8 * 8 + 2 * e + 1];
              // stride 2: plane 0 = tap 2 (high halves), plane 1 = tap 1 (low halves)
              pk[e] = (SX == 2 && tp == 0) ? __byte_perm(w0, w1, 0x7632) : __byte_perm(w0, w1, 0x5410);
            }
            st_shared_v4(dst, pk[0], pk[1], pk[2], pk[3]);
          } else {
            float q[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) q[e] = __uint_as_float(G.w[q8 * 8 + e]);
            st_shared_v4(dst, pack_bf16(q[0], q[1]), pack_bf16(q[2], q[3]), pack_bf16(q[4], q[5]),
                         pack_bf16(q[6], q[7]));
            if (SPLIT3) {
              float l[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) l[e] = q[e] - bf16_round(q[e]);
              st_shared_v4(dst - ph + plane(stage, tp, 1), pack_bf16(l[0], l[1]), pack_bf16(l[2], l[3]),
                           pack_bf16(l[4], l[5]), pack_bf16(l[6], l[7]));
            }
          }
        }
      }
      // guard rows: element (channel h*32 + lane) of row -1 (plane of the
      // shifted tap: tap2 for stride 2, tap1 for stride 1) or row 128.
      if (edge_lo || edge_hi) {
        const int ch = h * 32 + lane;
        const uint32_t gj = ch >> 3, ge = ch & 7;
        const uint32_t goff = edge_lo ? (static_cast<uint32_t>(-128) + ((gj ^ 7u) << 4) + 2 * ge)
                                      : (kAPlane + ((gj ^ 0u) << 4) + 2 * ge);
        const uint32_t gbase = plane(stage, 0, 0);
        if (IN_BF16) {
          st_shared_u16(gbase + goff, G.g);
        } else {
          const float v = __uint_as_float(G.g);
          const uint32_t hb = __float_as_uint(bf16_round(v)) >> 16;
          st_shared_u16(gbase + goff, hb);
          if (SPLIT3) {
            const float lo = v - bf16_round(v);
            st_shared_u16(plane(stage, 0, 1) + goff, __float_as_uint(bf16_round(lo)) >> 16);
          }
        }
      }
      fence_proxy_async();
      mbar_arrive(a_full(stage));
      if (prof_on) c_emit += clock64() - t0;
      if (++stage == A.na) {
        stage = 0;
        phase ^= 1;
      }
    };
    // (tile, group) sequence with a one-group-deep load pipeline
    Grp ga, gb;
    const int ngrp = A.n_groups;
    int tile = blockIdx.x;                 // tile of the group being emitted
    int gi = 0;                            // its group index
    Pix pc = pix_of(tile);                 // pixel for `tile`
    Pix pn = pc;                           // pixel for the tile of the next load
    int lt = tile, lg = 0;                 // (tile, group) of the next load
    auto next_load = [&](Grp& G) {         // issue the loads of (lt, lg) and advance
      const int ky = lg / p.CB, cb = lg - (lg / p.CB) * p.CB;
      load_grp(G, pn, ky, cb);
      if (++lg == ngrp) {
        lg = 0;
        lt += gridDim.x;
        if (lt < A.n_tiles) pn = pix_of(lt);
      }
    };
    auto have_load = [&]() { return lt < A.n_tiles; };
    if (tile < A.n_tiles) next_load(ga);
    while (tile < A.n_tiles) {
      const bool more = have_load();
      if (more) {
        const unsigned long long ti = prof_on ? clock64() : 0;
        next_load(gb);
        if (prof_on) c_issue += clock64() - ti;
      }
      emit_grp(ga);
      if (++gi == ngrp) { gi = 0; tile += gridDim.x; }
      if (!more) break;
      const bool more2 = have_load();
      if (more2) {
        const unsigned long long ti = prof_on ? clock64() : 0;
        next_load(ga);
        if (prof_on) c_issue += clock64() - ti;
      }
      emit_grp(gb);
      if (++gi == ngrp) { gi = 0; tile += gridDim.x; }
      if (!more2) break;
    }
    (void)pc;
    if (prof_on) {
      unsigned long long* pr = A.prof + (blockIdx.x * 16 + warp) * 8;
      pr[0] = clock64() - c_start; pr[1] = c_ldwait; pr[2] = c_empty; pr[3] = c_emit; pr[4] = c_issue;
    }
  } else if (warp == kWarpLoad) {
    // ============ B loader =====================================================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < A.n_tiles; tile += gridDim.x) {
        const int nt = tile % p.n_tiles_n;
        for (int kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait(b_empty(stage), phase ^ 1);
          mbar_expect_tx(b_full(stage), A.b_bytes);
          bulk_g2s(bring + stage * A.b_bytes, A.wpk + ((long long)nt * p.n_kb + kb) * A.b_bytes, A.b_bytes,
                   b_full(stage));
          if (++stage == A.nb) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma) {
    // ============ MMA issuer (whole warp, elected lane) ===================================================
    {
      const uint32_t idesc = make_idesc(BN);
      const bool mprof = (A.debug & 64) != 0;
      unsigned long long m_a = 0, m_b = 0, m_t = 0;
      const unsigned long long m_start = clock64();
      int as = 0, bs = 0, acc = 0;
      uint32_t aph = 0, bph = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < A.n_tiles; tile += gridDim.x) {
        { const unsigned long long t0 = clock64(); mbar_wait(tempty_bar(acc), acc_phase ^ 1); if (mprof) m_t += clock64() - t0; }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int g = 0; g < A.n_groups; ++g) {
          { const unsigned long long t0 = clock64(); mbar_wait(a_full(as), aph); if (mprof) m_a += clock64() - t0; }
          tc_fence_after();
          for (int kx = 0; kx < 3; ++kx) {
            { const unsigned long long t0 = clock64(); mbar_wait(b_full(bs), bph); if (mprof) m_b += clock64() - t0; }
            tc_fence_after();
            // A operand of tap kx: which plane, and the row shift
            const int tp = SX == 2 ? (kx == 1 ? 1 : 0) : 0;
            const int shift = SX == 2 ? (kx == 0 ? -1 : 0) : (kx - 1);
            const uint32_t a_hi = plane(as, tp, 0) + static_cast<uint32_t>(shift * 128);
            const uint32_t a_lo = plane(as, tp, NSPL - 1) + static_cast<uint32_t>(shift * 128);
            const uint32_t b_hi = bring + bs * A.b_bytes;
            const uint32_t b_lo = b_hi + BN * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t accum = (g > 0 || kx > 0 || k > 0) ? 1u : 0u;
              tc_mma_w(d_tmem, (sw128_desc(a_hi) + 2 * k), (sw128_desc(b_hi) + 2 * k), idesc, accum);
              if (SPLIT3) {
                tc_mma_w(d_tmem, (sw128_desc(a_hi) + 2 * k), (sw128_desc(b_lo) + 2 * k), idesc, 1u);
                tc_mma_w(d_tmem, (sw128_desc(a_lo) + 2 * k), (sw128_desc(b_hi) + 2 * k), idesc, 1u);
              }
            }
            tc_commit_w(b_empty(bs));
            if (++bs == A.nb) {
              bs = 0;
              bph ^= 1;
            }
          }
          tc_commit_w(a_empty(as));
          if (++as == A.na) {
            as = 0;
            aph ^= 1;
          }
        }
        tc_commit_w(tfull_bar(acc));
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (mprof && lane == 0) {
        unsigned long long* pr = A.prof + (blockIdx.x * 16 + warp) * 8;
        pr[0] = clock64() - m_start; pr[1] = m_a; pr[2] = m_b; pr[3] = m_t;
      }
    }
    __syncwarp();
  } else {
    // ============ epilogue: TMEM -> NCHW fp32, pad slots skipped =============
    const int q = warp & 3;
    const int HoWo = p.Ho * p.Wo;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < A.n_tiles; tile += gridDim.x) {
      const int mt = tile / p.n_tiles_n, nt = tile % p.n_tiles_n;
      const long long slot = (long long)mt * kBM + q * 32 + lane;
      bool valid = slot < A.slots;
      long long obase = 0;
      if (valid) {
        const long long n = slot / HoS;
        const long long rem = slot - n * HoS;
        const int y = static_cast<int>(rem / A.S);
        const int x = static_cast<int>(rem - (long long)y * A.S) - A.padL;
        valid = x >= 0 && x < p.Wo;
        obase = n * (long long)p.Cout * HoWo + (long long)y * p.Wo + x;
      }
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t rr[32];
        TMEM_LD32(t_row + c0, rr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int co0 = nt * BN + c0;
        if (valid) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int co = co0 + j;
            if (co < p.Cout) {
              float v = __uint_as_float(rr[j]);
              v = p.post == POST_RELU ? ((v < 0.f) ? 0.f : v) : __fadd_rn(v, 0.f);
              __stcs(A.out + obase + (long long)co * HoWo, v);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar(acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  __syncthreads();
  if (warp == kWarpLoad) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(A.tmem_cols)
                 : "memory");
  }
}

}  // namespace

bool conv_tap3_eligible(const ConvParams& p) {
  if (p.gemm) return false;
  return p.KW == 3 && p.dx == 1 && p.ox == -1 &&
         ((p.sx == 2 && p.in_bf16 && p.split == 1 && p.W % 2 == 0) ||
          (p.sx == 1 && p.Wo == p.W && (p.split == 1 ? p.in_bf16 : !p.in_bf16)));
}

merit_status launch_conv_tap3(const merit_plan& plan, const void* a, const void* packed_b, void* out,
                              void* stream) {
  const ConvParams& p = plan.conv;
  Tap3Args A;
  A.p = p;
  A.in = a;
  A.wpk = static_cast<const uint8_t*>(packed_b);
  A.out = static_cast<float*>(out);
  A.padL = 1;
  A.S = p.Wo + 1 + (p.sx == 1 ? 1 : 0);
  A.slots = (long long)p.N * p.Ho * A.S;
  const long long tiles_m = (A.slots + kBM - 1) / kBM;
  A.n_tiles = static_cast<int>(tiles_m * p.n_tiles_n);
  A.n_groups = p.KH * p.CB;
  const bool split3 = p.split == 3;
  A.nplanes = (p.sx == 2 ? 2 : 1) * (split3 ? 2 : 1);
  A.a_slot = A.nplanes * kPlaneG;
  A.b_bytes = static_cast<uint32_t>(p.BN) * 128u * (split3 ? 2u : 1u);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * p.BN)) cols <<= 1;
  A.tmem_cols = cols;
  // ring depths: 3 A slots (one group each) if possible, B fills the rest
  const size_t fixed = 1024 + 8 * (4 * kMaxRing + 4) + 16;
  const size_t budget = 227 * 1024 - fixed;
  A.na = 3;
  while (A.na > 2 && A.na * (size_t)A.a_slot + 3 * (size_t)A.b_bytes > budget) --A.na;
  A.nb = static_cast<int>((budget - A.na * (size_t)A.a_slot) / A.b_bytes);
  if (A.nb > kMaxRing) A.nb = kMaxRing;
  if (A.nb < 2 || A.na * (size_t)A.a_slot + 2 * (size_t)A.b_bytes > budget)
    return fail(MERIT_E_UNSUPPORTED_VIEW, "tap3 conv tiles exceed shared memory");
  const size_t smem = fixed + A.na * (size_t)A.a_slot + A.nb * (size_t)A.b_bytes;
  if (A.n_tiles == 0) return MERIT_OK;
  if (A.slots + kBM >= (1LL << 31)) return fail(MERIT_E_UNSUPPORTED_VIEW, "too many output slots for one launch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int grid = num_sms();
  if (grid > A.n_tiles) grid = A.n_tiles;
  grid = grid_cap(grid);
  const char* dbg = debug_env("MERIT_CONV_DEBUG");
  A.debug = dbg ? atoi(dbg) : 0;
  A.prof = nullptr;
  if (A.debug & 64) {
    cudaMalloc(&A.prof, 8ull * 8 * 16 * grid);
    cudaMemset(A.prof, 0, 8ull * 8 * 16 * grid);
  }
  cudaError_t e;
#define MERIT_LAUNCH_TAP3(INB, S3, SXV)                                                     \
  do {                                                                                        \
    auto k = conv_tap3_kernel<INB, S3, SXV>;                                                  \
    e = set_smem_attr(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    if (e != cudaSuccess) return cuda_check(e, "set_smem_attr(conv_tap3)");            \
    e = launch_pdl(k, dim3(grid), dim3(kThreads), smem, s, 1, A);                              \
    if (e != cudaSuccess) return cuda_check(e, "launch(conv_tap3)");                         \
  } while (0)
  if (p.sx == 2) MERIT_LAUNCH_TAP3(true, false, 2);
  else if (p.in_bf16) MERIT_LAUNCH_TAP3(true, false, 1);
  else if (split3) MERIT_LAUNCH_TAP3(false, true, 1);
  else MERIT_LAUNCH_TAP3(false, false, 1);
#undef MERIT_LAUNCH_TAP3
  if (A.debug & 64) {
    cudaStreamSynchronize(s);
    std::vector<unsigned long long> h(8 * 16 * grid);
    cudaMemcpy(h.data(), A.prof, h.size() * 8, cudaMemcpyDeviceToHost);
    double pt = 0, pl = 0, pe = 0, pm = 0, pi = 0, mt = 0, ma = 0, mb = 0, mtt = 0;
    for (int b = 0; b < grid; ++b) {
      for (int w = 0; w < kProducerWarps; ++w) {
        const unsigned long long* q = &h[(b * 16 + w) * 8];
        pt += q[0]; pl += q[1]; pe += q[2]; pm += q[3]; pi += q[4];
      }
      const unsigned long long* q = &h[(b * 16 + kWarpMma) * 8];
      mt += q[0]; ma += q[1]; mb += q[2]; mtt += q[3];
    }
    fprintf(stderr, "[tap3 prof] producer: load-issue %.1f%% load-wait %.1f%% empty-wait %.1f%% emit %.1f%% | mma: A-wait %.1f%% B-wait %.1f%% tmem-wait %.1f%% | cycles/CTA %.0f\n",
            100 * pi / pt, 100 * pl / pt, 100 * pe / pt, 100 * pm / pt, 100 * ma / mt, 100 * mb / mt, 100 * mtt / mt, mt / grid);
    cudaFree(A.prof);
  }
  return launch_status("conv_tap3_kernel");
}

}  // namespace merit_dev
