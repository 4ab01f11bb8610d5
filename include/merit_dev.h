/*
 * merit_dev.h — C ABI of the B200 (sm_100a) MERIT device operator.
 *
 * This is the drop-in boundary for the reference's single execution entry
 * point `merit::Tensor merit::run_full(const merit::Workload&)`
 * (/root/reference/proj/include/merit/engine.hpp:282-287).  A reference
 * caller describes the same Workload — two gather views (ViewSpec,
 * view.hpp:24-49), two source tensors and a ranged-inner-product
 * StrategyProgram (rip.hpp:85-107) — as plain C structs, asks the library to
 * lower it to a device plan, and runs the plan on device or host buffers.
 * No torch types, no C++ types cross this boundary.
 *
 * Lowering (merit_dev_plan_create) recognises the reduction skeletons the
 * reference's templates emit (workloads.hpp:47-68, :376-385) and the affine
 * view structure that goes with them, and picks one of four sm_100a kernels:
 *   MERIT_KERNEL_MAXPOOL  window max on CUDA cores (K1)
 *   MERIT_KERNEL_SAD      byte-SIMD block matching + fused argmin (K2)
 *   MERIT_KERNEL_CONV_TC  implicit-GEMM convolution on tcgen05/TMEM (K3)
 *   MERIT_KERNEL_CORR     displacement correlation on CUDA cores (K4), bit-exact
 *   MERIT_KERNEL_GENERIC  exact device interpreter of any REAL32/FIX16 program
 * There is no CPU execution path: a plan that cannot run on the device fails
 * with a status code (mirroring merit::ErrorCode, tensor.hpp:15-29).
 *
 * Every entry point returns merit_status; on failure the thread-local message
 * is available from merit_dev_last_error().
 *
 * Threading (engine.hpp's run_full is a pure function; SPEC.md:294-295 lets
 * p-tiles run concurrently).  All functions are thread-safe.  A plan is
 * immutable after creation apart from lazily created device state and the
 * packed-weight copy of merit_dev_plan_pack_b; it may be run from several
 * host threads on several streams at once:
 *   - kernels that only read their sources (max-pool, SAD, correlation, a
 *     conv plan after merit_dev_plan_pack_b) run fully concurrently;
 *   - a conv run that packs its weights on the fly (no pack_b) writes the
 *     plan's packed buffer, so such runs of ONE plan are stream-ordered one
 *     after another (an event chain), and pack_b itself waits for them;
 *   - exact-interpreter runs of one plan (they synchronise their stream to
 *     read the device error flag) are serialised by the plan;
 *   - merit_dev_run_host calls of one plan are serialised (they share the
 *     plan's staging buffers).
 * A plan's device state lives on the device of its first run; running it on
 * another device fails with MERIT_E_INVALID_ARGUMENT: for multi-GPU create one
 * plan per device (tests/test_concurrency.py).
 */
#ifndef MERIT_DEV_H_
#define MERIT_DEV_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MERIT_DEV_ABI_VERSION 1
#define MERIT_MAX_RANK 8
#define MERIT_MAX_TERMS 24
#define MERIT_MAX_CONSTANTS 16
#define MERIT_MAX_TABLES 4
#define MERIT_MAX_TABLE_SAMPLES 1024
#define MERIT_MAX_INSTRS 64

/* Status codes.  1..13 mirror merit::ErrorCode in declaration order
 * (tensor.hpp:15-29) offset by one so that 0 is success. */
typedef enum merit_status {
  MERIT_OK = 0,
  MERIT_E_OUT_OF_RANGE = 1,        /* ErrorCode::OutOfRange (REJECT gather)     */
  MERIT_E_BAD_MAGIC = 2,           /* ErrorCode::BadMagic                        */
  MERIT_E_TRUNCATED_PAYLOAD = 3,   /* ErrorCode::TruncatedPayload                */
  MERIT_E_UNKNOWN_DTYPE = 4,       /* ErrorCode::UnknownDtype                    */
  MERIT_E_NEGATIVE_STRIDE = 5,     /* ErrorCode::NegativeStride                  */
  MERIT_E_LUT_RANGE = 6,           /* ErrorCode::LutRange                        */
  MERIT_E_DIV_BY_ZERO = 7,         /* ErrorCode::DivByZero                       */
  MERIT_E_SCRATCHPAD_OVERFLOW = 8, /* ErrorCode::ScratchpadOverflow             */
  MERIT_E_OUT_OF_FOOTPRINT = 9,    /* ErrorCode::OutOfFootprint                  */
  MERIT_E_INDIVISIBLE = 10,        /* ErrorCode::Indivisible                     */
  MERIT_E_UNKNOWN_TEMPLATE = 11,   /* ErrorCode::UnknownTemplate                 */
  MERIT_E_BAD_PARAMS = 12,         /* ErrorCode::BadParams (Workload::validate)  */
  MERIT_E_USAGE = 13,              /* ErrorCode::Usage                           */
  MERIT_E_UNSUPPORTED_PROGRAM = 100, /* no device kernel for this program       */
  MERIT_E_UNSUPPORTED_VIEW = 101,    /* no device kernel for this view shape    */
  MERIT_E_CUDA = 102,                /* CUDA runtime / launch failure           */
  MERIT_E_INVALID_ARGUMENT = 103     /* null pointer, bad enum, size mismatch   */
} merit_status;

/* view.hpp:11 */
typedef enum merit_boundary {
  MERIT_ZERO_PAD = 0,
  MERIT_CLAMP = 1,
  MERIT_REJECT = 2
} merit_boundary;

/* view.hpp:15-20: component j of the concatenated (p, a) index contributes
 * k_j * stride + offset to source axis `axis`. */
typedef struct merit_view_term {
  int32_t component;
  int32_t axis;
  int64_t stride;
  int64_t offset;
} merit_view_term;

/* view.hpp:24-49 */
typedef struct merit_view_spec {
  int32_t src_rank;
  int32_t p_rank;
  int32_t a_rank;
  int32_t n_terms;
  int64_t src_shape[MERIT_MAX_RANK];
  int64_t p_shape[MERIT_MAX_RANK];
  int64_t a_shape[MERIT_MAX_RANK];
  merit_view_term terms[MERIT_MAX_TERMS];
  int32_t boundary; /* merit_boundary */
  int32_t _pad;
} merit_view_spec;

/* rip.hpp:15-31, same order. */
typedef enum merit_op {
  MERIT_OP_ADD = 0, MERIT_OP_SUB, MERIT_OP_L1, MERIT_OP_MAC, MERIT_OP_MAX,
  MERIT_OP_MIN, MERIT_OP_SEL, MERIT_OP_BAND, MERIT_OP_BOR, MERIT_OP_BXOR,
  MERIT_OP_BNOT, MERIT_OP_IDX, MERIT_OP_LUT, MERIT_OP_MOVC, MERIT_OP_DIV
} merit_op;

/* rip.hpp:33-41 Operand::Kind */
typedef enum merit_operand_kind {
  MERIT_OPND_REG = 0, MERIT_OPND_PORT_A = 1, MERIT_OPND_PORT_B = 2, MERIT_OPND_ZERO = 3
} merit_operand_kind;

/* rip.hpp:51-57 AluInstr (+ Operand, Dst) */
typedef struct merit_alu_instr {
  int32_t op;        /* merit_op */
  int32_t dst_out;   /* Dst::out: 1 = emit to the output stream */
  int32_t dst_reg;   /* Dst::reg */
  int32_t a_kind, a_reg;
  int32_t b_kind, b_reg;
  int32_t c_kind, c_reg;
  int32_t shift;
  int32_t aux;
} merit_alu_instr;

/* rip.hpp:61-78 LookupTable */
typedef struct merit_lookup_table {
  double lo, hi;
  int32_t n_samples;
  int32_t clamp;
  const double* samples;
} merit_lookup_table;

/* rip.hpp:85-107 StrategyProgram.  Segment s holds seg_len[s] instructions,
 * stored back to back in `instrs` in segment order Pre_1..Pre_D, Body,
 * Post_D..Post_1 (2*depth+1 segments). */
typedef struct merit_program {
  int32_t depth;
  int32_t outputs;
  int32_t n_segments;
  int32_t n_constants;
  int32_t n_tables;
  int32_t _pad;
  const int32_t* seg_len;
  const merit_alu_instr* instrs;
  const double* constants;
  const merit_lookup_table* tables;
} merit_program;

/* Element types of the buffers crossing the ABI.  F32 and I16 are the
 * reference's REAL32 / FIX16 (tensor.hpp:67); BF16 and U8 are device
 * storage types for the same values (bf16-rounded activations, 8-bit frames);
 * I32 / U16 are exact integer SAD outputs. */
typedef enum merit_dtype {
  MERIT_F32 = 0, MERIT_I16 = 1, MERIT_BF16 = 2, MERIT_U8 = 3, MERIT_I32 = 4,
  MERIT_U16 = 5  /* exact SAD map of 8-bit 8x8 / 16x16 blocks (every SAD <= 65,280): half the bytes of I32 */
} merit_dtype;

/* Request flags. */
enum {
  MERIT_FLAG_EXACT = 1u << 0,   /* force the bit-exact generic interpreter     */
  MERIT_FLAG_ARGMIN = 1u << 1,  /* L1 block matching: also write (mv_y, mv_x,
                                   min SAD) per block, lowest-raster tie-break */
  MERIT_FLAG_NO_MAP = 1u << 2,  /* with ARGMIN: skip the full SAD map output   */
  MERIT_FLAG_FAST_BF16 = 1u << 3 /* f32 MAC conv: one bf16 product instead of
                                    the 3-term bf16 split (looser tolerance)  */
};

/* engine.hpp:16-39 Workload, as a descriptor.  Data pointers are supplied
 * at run time. */
typedef struct merit_workload_desc {
  merit_view_spec view_a;
  merit_view_spec view_b;
  int32_t dtype_a;    /* merit_dtype of src_a buffers */
  int32_t dtype_b;    /* merit_dtype of src_b buffers */
  int32_t dtype_out;  /* merit_dtype of the output buffer */
  int32_t frac_bits;  /* Tensor::frac_bits of FIX16 sources (tensor.hpp:78) */
  uint32_t flags;
  int32_t _pad;
  merit_program program;
} merit_workload_desc;

typedef enum merit_kernel_kind {
  MERIT_KERNEL_GENERIC = 0,
  MERIT_KERNEL_MAXPOOL = 1,
  MERIT_KERNEL_SAD = 2,
  MERIT_KERNEL_CONV_TC = 3,
  MERIT_KERNEL_CORR = 4,
  MERIT_KERNEL_MULTI = 5   /* multi-workload plan run member by member */
} merit_kernel_kind;

/* What a plan needs and produces. */
typedef struct merit_plan_info {
  int32_t kernel;          /* merit_kernel_kind */
  int32_t out_rank;        /* Workload::output_shape() rank */
  int64_t out_shape[MERIT_MAX_RANK + 1];
  int64_t out_elems;       /* 0 when MERIT_FLAG_NO_MAP */
  int64_t out_bytes;
  int64_t aux_elems;       /* int32 elements of the argmin record (3 per block) */
  int64_t src_a_bytes;
  int64_t src_b_bytes;
  int64_t n_outputs;       /* ranged inner products computed = prod(p_shape) */
  double algorithmic_ops;  /* MACs / abs-diffs / compares per run, counted as
                              the reference's run_full executes them */
  double algorithmic_bytes;/* compulsory HBM bytes per run */
  double executed_ops;     /* the ops the device executes per run: equal to
                              algorithmic_ops unless a fused multi-workload
                              plan shares work between members */
  int32_t launches_per_run;/* kernel launches issued by merit_dev_run */
  int32_t _pad;
  char description[256];
} merit_plan_info;

typedef struct merit_plan merit_plan;

/* Library identification. */
int32_t merit_dev_abi_version(void);
const char* merit_dev_build_info(void);

/* Thread-local message of the last failing call ("" if none). */
const char* merit_dev_last_error(void);

/* Validate (engine.hpp:30-38 Workload::validate, rip.hpp:96-106) and lower a
 * workload to a device plan.  Host-only; needs no GPU. */
merit_status merit_dev_plan_create(const merit_workload_desc* desc, merit_plan** out_plan);
merit_status merit_dev_plan_destroy(merit_plan* plan);
merit_status merit_dev_plan_query(const merit_plan* plan, merit_plan_info* info);

/* Pack the B operand (e.g. convolution weights) into the kernel's operand
 * layout on the device, once.  d_src_b is a device pointer.  After it, runs
 * use the packed copy and ignore their d_src_b.  Optional: without it every
 * run packs its own d_src_b on the fly. */
merit_status merit_dev_plan_pack_b(merit_plan* plan, const void* d_src_b, void* cuda_stream);

/* Several workloads over the SAME two source tensors as one plan: what a
 * caller of the reference does with one run_full per workload
 * (engine.hpp:282-287), e.g. the 16x16 and 8x8 block searches of C5.
 * Every member is validated and lowered like merit_dev_plan_create; all
 * members must have the same source shapes and dtypes (BAD_PARAMS
 * otherwise).  merit_dev_run / _run_host take the shared sources once and
 * write the members' outputs back to back in member order: d_out holds
 * every member's output, d_aux every member's argmin records (offsets from
 * merit_dev_plan_member).  Members that the device can compute in one pass
 * are fused into one launch:
 *   L1 block matching with BxB and 2Bx2B blocks (B = 8) over the same frames,
 *   window (+/-32) and boundary, argmin without SAD maps: one byte-SIMD pass
 *   computes the BxB SADs and sums 2 x 2 of them into the 2Bx2B SAD at every
 *   displacement (exact integers, results identical to separate runs).
 * Otherwise the members run one after another on the stream
 * (info.kernel = MERIT_KERNEL_MULTI).  Host-only, like plan creation. */
merit_status merit_dev_plan_create_multi(const merit_workload_desc* descs, int32_t n, merit_plan** out_plan);
/* Member i of a multi-workload plan (or member 0 = the plan itself for a
 * single-workload plan): its own plan info and the byte / int32-element
 * offsets of its output and argmin records in the plan's d_out / d_aux. */
merit_status merit_dev_plan_member(const merit_plan* plan, int32_t i, merit_plan_info* info,
                                   int64_t* out_offset_bytes, int64_t* aux_offset_elems);

/* Run on device buffers, asynchronously on `cuda_stream` (0 = default).
 * d_out receives Workload::output_shape() elements of dtype_out (may be null
 * with MERIT_FLAG_NO_MAP); d_aux receives the argmin records (may be null
 * without MERIT_FLAG_ARGMIN). */
merit_status merit_dev_run(const merit_plan* plan, const void* d_src_a, const void* d_src_b,
                           void* d_out, void* d_aux, void* cuda_stream);

/* Run on host buffers: H2D copies, run, D2H copies, synchronise — the
 * reference's run_full calling convention (host tensors in, host tensor out). */
merit_status merit_dev_run_host(const merit_plan* plan, const void* h_src_a, const void* h_src_b,
                                void* h_out, void* h_aux, void* cuda_stream);

/* How merit_dev_run_host pipelines this plan (host-only, no device needed):
 * the run is cut along the outermost independent axis (max-pool planes, conv
 * images, SAD frame pairs or block-row bands) and slice k's H2D, kernel and
 * D2H overlap slice k+1's.  Writes up to `cap` slices and sets *n_slices to
 * the count (0: the plan runs unsliced).  a_need / b_need: source bytes that
 * must have landed before the slice's kernel; out / aux: the byte ranges it
 * writes.  MERIT_HOST_CHUNKS=n in the environment forces n slices. */
typedef struct merit_host_slice {
  int64_t a_need, b_need;
  int64_t out_lo, out_hi;
  int64_t aux_lo, aux_hi;
  int64_t aux2_lo, aux2_hi;  /* a second aux range (fused multi-workload plans) */
} merit_host_slice;
merit_status merit_dev_plan_slices(const merit_plan* plan, merit_host_slice* slices, int64_t cap,
                                   int64_t* n_slices);

/* merit::run_tiled's traffic report (engine.hpp:72-80, :189-278) for a
 * TilingPlan {t_p, t_a} over this plan's workload: the plan is validated like
 * TilingPlan::validate (engine.hpp:50-63; MERIT_E_BAD_PARAMS) and every pass
 * is charged its Eq. 6 footprint box (view.hpp:121-149; negative strides ->
 * MERIT_E_NEGATIVE_STRIDE), exactly as the reference counts words.  The
 * device executes its own tiling, so the scratchpad
 * capacities of EngineConfig are not enforced.  Host-only: no
 * device needed.  t_p / t_a hold p_rank / a_rank extents. */
typedef struct merit_traffic_report {
  uint64_t dram_read_words_a;
  uint64_t dram_read_words_b;
  uint64_t dram_write_words;
  uint64_t scratchpad_peak_words_a;
  uint64_t scratchpad_peak_words_b;
  uint64_t passes;
  uint64_t macs;
} merit_traffic_report;
merit_status merit_dev_tiled_traffic(const merit_plan* plan, const int64_t* t_p, const int64_t* t_a,
                                     merit_traffic_report* report);

/* The measured counterpart of the TrafficReport: run the plan on device
 * buffers with the GPU's performance counters armed (CUPTI range profiler,
 * one user range around the run, user replay: the run repeats once per
 * counter pass) after a read-only L2 flush, and report the DRAM bytes the
 * run actually moved (all of its launches).  Where the reference counts the
 * words its scratchpad loads pass by pass (engine.hpp:233-241), this is what
 * HBM served.  Output lines still dirty in L2 when the run ends are not
 * written yet, and evictions of unrelated lines may add a few MB of writes.
 * range_time_ns is the GPU time spanned by the range (launch gaps included,
 * not a kernel time).  Synchronous; fails with MERIT_E_UNSUPPORTED_PROGRAM
 * when CUPTI (libcupti.so, the copy already in the process if any, else
 * loaded at the first call) or profiling permission is missing, or the
 * profiler refuses the session (e.g. the counters are held by another client
 * of the GPU); merit_dev_last_error() then starts with
 * "measure_traffic unavailable on this system: " and names the CUPTI step. */
typedef struct merit_measured_traffic {
  double dram_read_bytes;
  double dram_write_bytes;
  double range_time_ns;
  int64_t ranges;     /* profiled ranges (1) */
  int64_t launches;   /* kernel launches the library issued per run */
  int32_t passes;     /* replay passes (runs) the metrics needed */
  int32_t _pad;
} merit_measured_traffic;
merit_status merit_dev_measure_traffic(const merit_plan* plan, const void* d_src_a, const void* d_src_b,
                                       void* d_out, void* d_aux, void* cuda_stream,
                                       merit_measured_traffic* report);
/* The same from host sources (copied to device buffers the call allocates
 * and frees; outputs are discarded). */
merit_status merit_dev_measure_traffic_host(const merit_plan* plan, const void* h_src_a, const void* h_src_b,
                                            merit_measured_traffic* report);

/* Deterministic input synthesis shared by tests and the benchmark
 * (workloads.hpp:74-105 SplitMix64 / fill_random, and the seeded frame
 * generator of SURVEY §8(d)).  Host-only. */
void merit_gen_uniform_f32(float* out, int64_t n, uint64_t seed, double lo, double hi);
void merit_gen_normal_f32(float* out, int64_t n, uint64_t seed, double sigma);
void merit_gen_range_i16(int16_t* out, int64_t n, uint64_t seed, int64_t lo, int64_t hi);
void merit_gen_me_pair(uint8_t* cur, uint8_t* ref, int64_t h, int64_t w, int64_t blk,
                       int64_t max_shift, int64_t noise, uint64_t seed);
void merit_f32_to_bf16(const float* in, uint16_t* out, int64_t n);

/* Counters of kernels launched through this library by the calling process
 * (evidence for the benchmark's gpu_launches claim). */
int64_t merit_dev_launch_count(void);
/* Name of the last kernel this library launched (a static string; "" before
 * the first launch). */
const char* merit_dev_last_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* MERIT_DEV_H_ */
