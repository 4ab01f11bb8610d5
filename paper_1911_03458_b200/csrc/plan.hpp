// Internal plan representation shared by the lowering (lower.cpp), the C ABI
// (capi.cpp) and the kernel launchers (*.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "merit_dev.h"

namespace merit_dev {

constexpr int kMaxRank = MERIT_MAX_RANK;
constexpr int kMaxK = 2 * MERIT_MAX_RANK;  // concatenated (p, a) rank

// Affine form of one ViewSpec (view.hpp:37-42, Eq. 5): for source axis i,
// x_i = sum_j coef[i][j] * k_j + off[i].
struct ViewAffine {
  int src_rank = 0;
  int k_rank = 0;
  int boundary = MERIT_ZERO_PAD;
  int64_t src_shape[kMaxRank] = {};
  int64_t coef[kMaxRank][kMaxK] = {};
  int64_t off[kMaxRank] = {};
};

// Flattened StrategyProgram for the generic device interpreter.
struct ProgramImage {
  int32_t depth = 0;
  int32_t outputs = 1;
  int32_t n_segments = 0;
  int32_t n_instrs = 0;
  int32_t seg_start[2 * kMaxRank + 2] = {};
  int32_t seg_len[2 * kMaxRank + 2] = {};
  merit_alu_instr instrs[MERIT_MAX_INSTRS] = {};
  double constants[MERIT_MAX_CONSTANTS] = {};
  int32_t n_constants = 0;
  int32_t n_tables = 0;
  double tab_lo[MERIT_MAX_TABLES] = {};
  double tab_hi[MERIT_MAX_TABLES] = {};
  int32_t tab_n[MERIT_MAX_TABLES] = {};
  int32_t tab_clamp[MERIT_MAX_TABLES] = {};
  int32_t tab_off[MERIT_MAX_TABLES] = {};
  int32_t n_table_samples = 0;
  double table_samples[MERIT_MAX_TABLES * MERIT_MAX_TABLE_SAMPLES] = {};
};

// K0: exact interpreter (engine.hpp:120-143 with rip.hpp:210-267 semantics).
struct GenericParams {
  int32_t fix16 = 0;   // Fix16Mode (rip.hpp:144-158) instead of Real32Mode
  int32_t p_rank = 0, a_rank = 0;
  int64_t p_shape[kMaxRank] = {};
  int64_t a_shape[kMaxRank] = {};
  int64_t rows = 0;    // prod(p_shape)
  int64_t a_vol = 0;
  int32_t dtype_a = MERIT_F32, dtype_b = MERIT_F32, dtype_out = MERIT_F32;
  int32_t uses_a = 1, uses_b = 1;
  ViewAffine va, vb;
};

// Epilogue of the MAC / MAX skeletons (Post_1 of the program).
enum PostOp : int32_t { POST_ADD_ZERO = 0, POST_RELU = 1 };

// K1: window max (maxpool program, workloads.hpp:376-385).
struct MaxpoolParams {
  int64_t planes = 0;  // product of the leading (batch, channel) extents
  int32_t H = 0, W = 0, Ho = 0, Wo = 0, KH = 0, KW = 0;
  int32_t sy = 1, sx = 1, dy = 1, dx = 1, oy = 0, ox = 0;
  int32_t boundary = MERIT_CLAMP;  // CLAMP (coordinate clamp) or ZERO_PAD (value 0)
  int32_t post = POST_ADD_ZERO;
  float init = -3.0e38f;           // MOVC constant of Pre_1
  int32_t fast = 0;                // 3x3 / stride 2 / offset -1 warp-row path
  int32_t vec_out = 0;             // launch-time: Wo % 4 == 0 and 16-byte aligned output
  int32_t dbg = 0;                 // launch-time timing experiments (MERIT_MP_DEBUG)
  int32_t pf = 0;                  // launch-time: bands per CTA prefetched into L2 before the PDL wait
};

// K2: L1 block matching (motion estimation, workloads.hpp:255-279).
struct SadParams {
  int64_t pairs = 1;
  int32_t Hc = 0, Wc = 0;   // current-frame extents
  int32_t Hr = 0, Wr = 0;   // reference-frame extents
  int32_t BY = 0, BX = 0;   // block grid
  int32_t BH = 16, BW = 16; // block extents (a_shape)
  int32_t WY = 0, WX = 0;   // displacement window (p extents)
  int32_t oy = 0, ox = 0;   // reference offset at displacement 0
  int32_t cy = 0, cx = 0;   // current-frame offset of block (0,0)
  int32_t boundary = MERIT_ZERO_PAD;  // reference-frame boundary
  int32_t ref_is_b = 1;     // port B carries the displaced reference view
  int32_t write_map = 1;
  int32_t argmin = 0;
  int32_t out_f32 = 0;      // SAD map as float (REAL32) instead of int32
  int32_t out_u16 = 0;      // SAD map as uint16 (exact for 8-bit 8x8 / 16x16 blocks)
  // Block-row band of one launch (pipelined host-buffer runs): block rows
  // [by_begin, by_begin + by_count) of every pair; by_count 0 = all BY rows.
  int32_t by_begin = 0, by_count = 0;
  // Fused coarse level (multi-workload plans): also the argmin of the
  // 2BH x 2BW blocks made of 2 x 2 of these blocks, same window and frames,
  // written at d_aux + aux2_delta int32 elements (merged grid BY2 x BX2).
  int32_t fuse2 = 0;
  int32_t BY2 = 0, BX2 = 0;
  int64_t aux2_delta = 0;
  // REAL32 frames (the reference Tensor's only float type): narrowed to u8 on
  // the device before matching, exact-interpreter fallback (launch_sad_narrowed)
  int32_t narrow = 0;
};

// K3: implicit-GEMM convolution on tcgen05 (mac_program over conv views).
struct ConvParams {
  int32_t N = 1, Cin = 0, H = 0, W = 0;
  int32_t Cout = 0, Ho = 0, Wo = 0, KH = 0, KW = 0;
  int32_t sy = 1, sx = 1, dy = 1, dx = 1, oy = 0, ox = 0;
  int32_t in_bf16 = 0;      // activations stored as bf16 (else f32)
  int32_t w_bf16 = 0;       // weights stored as bf16 (else f32)
  int32_t split = 3;        // bf16 terms per product: 1 (bf16) or 3 (f32 via hi/lo)
  int32_t post = POST_ADD_ZERO;
  int32_t BN = 0;           // N tile (multiple of 16, <= 256)
  int32_t n_tiles_n = 0;
  int32_t CB = 0;           // 64-channel blocks
  int32_t n_kb = 0;         // k-blocks per tile = KH*KW*CB
  int64_t npix = 0;         // N*Ho*Wo
  int64_t packed_b_bytes = 0;
  // Element strides of the operands (NCHW / OIHW / NCHW by default; a GEMM
  // view maps onto the same kernel with A rows as pixels and K as channels,
  // workloads.hpp:122-136).  Only the general kernel K3a reads them.
  int64_t a_sn = 0, a_sc = 0, a_sy = 0, a_sx = 0;  // input: image, channel, row, column
  int64_t o_sn = 0, o_sc = 0, o_sp = 0;            // output: image, channel, pixel (y*Wo + x)
  int64_t w_so = 0, w_si = 0;                      // weights: output channel, input channel
  int32_t gemm = 0;                                // not NCHW: general kernel only
};

// K4: displacement correlation (correlation template, workloads.hpp:230-251):
// out[y][x][dy][dx] = post(sum_c A[c][y + ay][x + ax] * B[c][y + dy + by][x + dx + bx])
// with the engine's REAL32 MAC (fl(fl(a * b) + r), channel order), ZERO_PAD
// reads outside either source.  A is the undisplaced view.
struct CorrParams {
  int32_t C = 0;
  int32_t Ha = 0, Wa = 0, Hb = 0, Wb = 0;  // source extents
  int32_t Ho = 0, Wo = 0, DY = 0, DX = 0;  // p extents
  int32_t ay = 0, ax = 0, by = 0, bx = 0;  // view offsets
  int32_t post = POST_ADD_ZERO;
};

}  // namespace merit_dev

struct merit_plan;

namespace merit_dev {
// One piece of a pipelined host-buffer run (merit_dev_run_host): a sub-plan
// over a slice of the outermost independent axis (max-pool planes, conv
// images, SAD frame pairs or block-row bands), the source prefixes it reads
// and the output byte ranges it writes.
struct HostSlice {
  merit_plan* sub = nullptr;            // owned by the parent plan
  int64_t a_off = 0, b_off = 0;         // launch pointer offsets (bytes)
  int64_t out_off = 0, aux_off = 0;
  int64_t a_need = 0, b_need = 0;       // source prefix (bytes) that must have landed
  int64_t out_lo = 0, out_hi = 0;       // bytes written (D2H ranges)
  int64_t aux_lo = 0, aux_hi = 0;
  int64_t aux2_lo = 0, aux2_hi = 0;     // fused plans: the coarse level's records
};
}  // namespace merit_dev

struct merit_plan {
  int32_t kernel = MERIT_KERNEL_GENERIC;
  merit_workload_desc desc{};
  merit_plan_info info{};
  merit_dev::ProgramImage prog{};
  merit_dev::GenericParams gen{};
  merit_dev::MaxpoolParams mp{};
  merit_dev::SadParams sad{};
  merit_dev::ConvParams conv{};
  merit_dev::CorrParams corr{};
  bool conv_swapped = false;  // input tensor is src_b, weights are src_a
  bool corr_swapped = false;  // the displaced view is src_a
  // Lazily created device state (plan creation itself needs no GPU).
  mutable std::mutex mu;
  mutable void* d_prog = nullptr;      // ProgramImage copy for K0
  mutable void* d_err = nullptr;       // int32 device error flag
  mutable void* d_packed_b = nullptr;  // K3 packed weights
  mutable void* d_narrow = nullptr;    // narrowed SAD plans: u8 copies of both frames
  mutable bool packed_valid = false;  // set by merit_dev_plan_pack_b only
  mutable int device = -1;
  // Concurrent runs of one plan (several threads / streams): a run that packs
  // the weights on the fly writes the shared d_packed_b, so such runs hold
  // pack_mu while they enqueue, wait on pack_event (the previous packing
  // run's last launch) and record it after their own; exact-interpreter runs
  // share d_err and hold run_mu from launch to error check.
  mutable std::mutex pack_mu;
  mutable void* pack_event = nullptr;
  mutable std::mutex run_mu;
  // Device staging of merit_dev_run_host (a, b, out, aux), kept across calls
  // on the device they were made on; host_mu serialises host-buffer calls.
  mutable std::mutex host_mu;
  mutable void* stage[4] = {nullptr, nullptr, nullptr, nullptr};
  mutable size_t stage_bytes[4] = {0, 0, 0, 0};
  mutable int stage_dev = -1;
  // Pipelined host-buffer runs: slices (built on first use, host only) and
  // the H2D / D2H copy streams + events (on stage_dev).
  mutable bool slices_built = false;
  mutable std::vector<merit_dev::HostSlice> slices;
  mutable void* copy_stream[2] = {nullptr, nullptr};
  mutable std::vector<void*> copy_events;
  // Multi-workload plans (merit_dev_plan_create_multi): the owned member
  // plans, their output (bytes) / argmin (int32 elements) offsets, and for a
  // fused plan (kernel SAD, sad.fuse2) the fine level's record offset.
  std::vector<merit_plan*> members;
  std::vector<int64_t> member_out_off, member_aux_off;
  int64_t fused_aux_off = 0;
  ~merit_plan();
};

namespace merit_dev {

// Set the thread-local error message and return the status.
merit_status fail(merit_status st, const std::string& msg);

merit_status lower(const merit_workload_desc& d, merit_plan& plan);

// Pipelined host-buffer run (host_pipeline.cpp): H2D of slice k+1, the kernel
// of slice k and the D2H of slice k-1 overlap on three streams.  Returns
// MERIT_E_UNSUPPORTED_VIEW (and does nothing) when the plan does not slice.
merit_status run_host_pipelined(const merit_plan& plan, void* da, void* db, void* dout, void* daux,
                                const void* h_a, const void* h_b, void* h_out, void* h_aux, bool need_b,
                                void* stream);
// Lazily allocate a plan's device state on the current device (capi.cpp).
merit_status ensure_device_state(const merit_plan& plan);
// Order a write of plan.d_packed_b after the runs that read it / record this
// stream's position as the new last reader (caller holds plan.pack_mu).
merit_status pack_wait(const merit_plan& plan, void* stream);
merit_status pack_done(const merit_plan& plan, void* stream);
// Release the pipeline's streams/events (plan destruction, device switch).
void release_host_pipeline(const merit_plan& plan);

// Kernel launchers (defined in the .cu files).  All asynchronous on `stream`.
merit_status launch_generic(const merit_plan& plan, const void* a, const void* b, void* out,
                            void* stream, const int32_t* run_if = nullptr);
// REAL32 block matching on the SAD kernel (SadParams::narrow): narrow both
// frames to 8 bits on the device, match, and re-run the exact interpreter
// (stream-ordered, device-side condition) if any pixel is not an integer in
// [0, 255].  Results are the engine's bit for bit either way.
merit_status launch_sad_narrowed(const merit_plan& plan, const void* a, const void* b, void* out,
                                 void* stream);
merit_status launch_maxpool(const merit_plan& plan, const void* a, void* out, void* stream);
// Rows per thread of the SAD kernel variant for a window, 0 if none fits.
int sad_rows_per_thread(int BH, int WY, int WX);
merit_status launch_sad(const merit_plan& plan, const void* a, const void* b, void* out,
                        void* aux, void* stream);
merit_status launch_conv_pack(const merit_plan& plan, const void* b, void* packed, void* stream);
merit_status launch_conv(const merit_plan& plan, const void* a, const void* packed_b, void* out,
                         void* stream);
merit_status launch_corr(const merit_plan& plan, const void* a, const void* b, void* out, void* stream);
// K4 threads per 4 output columns for a DY x DX window (0: does not fit a CTA).
int corr_threads_per_column_quad(int DY, int DX);

// Check a CUDA status from C++ host code; returns MERIT_E_CUDA with context.
merit_status cuda_check(int err, const char* what);
void count_launch(int n = 1);
void note_kernel(const char* name);  // static string: last kernel launched

int64_t elem_size(int dtype);

}  // namespace merit_dev
