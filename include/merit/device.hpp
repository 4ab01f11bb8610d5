// merit/device.hpp — header swap for reference callers.
//
// The reference executes a workload with
//     merit::Tensor merit::run_full(const merit::Workload&)   (engine.hpp:282-287)
// on the host.  Including this header after the reference's merit/engine.hpp
// gives the same call on the B200:
//     merit::Tensor merit::device::run_full(const merit::Workload&, uint32_t flags = 0)
// with identical argument meaning, output shape (Workload::output_shape(),
// engine.hpp:24-28), dtype (REAL32 -> fdata, FIX16 -> qdata) and error
// behaviour (merit::Error carrying the reference ErrorCode).  Failures that
// have no reference counterpart (no device, a program the device cannot run)
// are reported as merit::Error(ErrorCode::BadParams, "device: ...").
//
// The workload is lowered through the C ABI (merit_dev.h); link against
// paper_1911_03458_b200/libmerit_dev.so.  There is no host fallback.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "merit/engine.hpp"
#include "merit_dev.h"

namespace merit {
namespace device {

namespace detail {

inline void fill_view(merit_view_spec& c, const ViewSpec& v) {
  if (v.source_shape.size() > MERIT_MAX_RANK || v.p_shape.size() > MERIT_MAX_RANK ||
      v.a_shape.size() > MERIT_MAX_RANK || v.terms.size() > MERIT_MAX_TERMS)
    throw Error(ErrorCode::BadParams, "device: view exceeds the ABI limits");
  c = merit_view_spec{};
  c.src_rank = static_cast<int32_t>(v.source_shape.size());
  c.p_rank = static_cast<int32_t>(v.p_shape.size());
  c.a_rank = static_cast<int32_t>(v.a_shape.size());
  c.n_terms = static_cast<int32_t>(v.terms.size());
  for (size_t i = 0; i < v.source_shape.size(); ++i) c.src_shape[i] = v.source_shape[i];
  for (size_t i = 0; i < v.p_shape.size(); ++i) c.p_shape[i] = v.p_shape[i];
  for (size_t i = 0; i < v.a_shape.size(); ++i) c.a_shape[i] = v.a_shape[i];
  for (size_t t = 0; t < v.terms.size(); ++t)
    c.terms[t] = merit_view_term{v.terms[t].component, v.terms[t].axis, v.terms[t].stride,
                                 v.terms[t].offset};
  c.boundary = static_cast<int32_t>(v.boundary);
}

// Owns the flattened program arrays the descriptor points into.
struct Desc {
  merit_workload_desc d{};
  std::vector<int32_t> seg_len;
  std::vector<merit_alu_instr> instrs;
  std::vector<merit_lookup_table> tables;
};

inline void fill(Desc& D, const Workload& w, uint32_t flags) {
  fill_view(D.d.view_a, w.view_a);
  fill_view(D.d.view_b, w.view_b);
  const bool fix = w.src_a.dtype == Dtype::Fix16;
  D.d.dtype_a = fix ? MERIT_I16 : MERIT_F32;
  D.d.dtype_b = w.src_b.dtype == Dtype::Fix16 ? MERIT_I16 : MERIT_F32;
  D.d.dtype_out = fix ? MERIT_I16 : MERIT_F32;
  D.d.frac_bits = w.src_a.frac_bits;
  D.d.flags = flags;
  const StrategyProgram& p = w.program;
  for (const auto& seg : p.segments) {
    D.seg_len.push_back(static_cast<int32_t>(seg.size()));
    for (const AluInstr& in : seg) {
      merit_alu_instr c{};
      c.op = static_cast<int32_t>(in.op);
      c.dst_out = in.dst.out ? 1 : 0;
      c.dst_reg = in.dst.reg;
      c.a_kind = static_cast<int32_t>(in.a.kind);
      c.a_reg = in.a.reg;
      c.b_kind = static_cast<int32_t>(in.b.kind);
      c.b_reg = in.b.reg;
      c.c_kind = static_cast<int32_t>(in.c.kind);
      c.c_reg = in.c.reg;
      c.shift = in.shift;
      c.aux = in.aux;
      D.instrs.push_back(c);
    }
  }
  for (const LookupTable& t : p.tables)
    D.tables.push_back(merit_lookup_table{t.lo, t.hi, static_cast<int32_t>(t.samples.size()),
                                          t.clamp ? 1 : 0, t.samples.data()});
  merit_program& pc = D.d.program;
  pc.depth = p.depth;
  pc.outputs = p.outputs;
  pc.n_segments = static_cast<int32_t>(p.segments.size());
  pc.n_constants = static_cast<int32_t>(p.constants.size());
  pc.n_tables = static_cast<int32_t>(p.tables.size());
  pc.seg_len = D.seg_len.data();
  pc.instrs = D.instrs.data();
  pc.constants = p.constants.data();
  pc.tables = D.tables.data();
}

[[noreturn]] inline void raise(merit_status st) {
  const std::string msg = merit_dev_last_error();
  if (st >= 1 && st <= 13) throw Error(static_cast<ErrorCode>(st - 1), msg);
  throw Error(ErrorCode::BadParams, "device: " + msg);
}

struct PlanGuard {
  merit_plan* p = nullptr;
  ~PlanGuard() { merit_dev_plan_destroy(p); }
};

}  // namespace detail

/// engine.hpp:282-287 on the device: validate, lower, run, copy back.
///
/// Numerics: max-pool, L1 / SAD, correlation, FIX16 and every program on the
/// exact interpreter are bit-identical to merit::run_full.  REAL32 MAC
/// convolutions run on the tensor cores with a 3-term bf16 split and fp32
/// accumulation: |got - ref| <= 1e-4 (1 + |ref|) against the double oracle —
/// looser than the 1e-5 of the reference's own REAL32 acceptance tests
/// (SPEC.md:61,570).  Pass flags = MERIT_FLAG_EXACT for the engine's own
/// summation order and rounding (bit-identical, on the interpreter).
inline Tensor run_full(const Workload& w, uint32_t flags = 0) {
  w.validate();  // the reference's own checks first (engine.hpp:30-38)
  detail::Desc D;
  detail::fill(D, w, flags);
  detail::PlanGuard g;
  merit_status st = merit_dev_plan_create(&D.d, &g.p);
  if (st != MERIT_OK) detail::raise(st);
  Tensor out = w.src_a.dtype == Dtype::Real32 ? Tensor::real(w.output_shape())
                                              : Tensor::fix(w.output_shape(), w.src_a.frac_bits);
  const bool fix = w.src_a.dtype == Dtype::Fix16;
  const void* a = fix ? static_cast<const void*>(w.src_a.qdata.data())
                      : static_cast<const void*>(w.src_a.fdata.data());
  const void* b = w.src_b.dtype == Dtype::Fix16 ? static_cast<const void*>(w.src_b.qdata.data())
                                                : static_cast<const void*>(w.src_b.fdata.data());
  void* o = fix ? static_cast<void*>(out.qdata.data()) : static_cast<void*>(out.fdata.data());
  st = merit_dev_run_host(g.p, a, b, o, nullptr, nullptr);
  if (st != MERIT_OK) detail::raise(st);
  return out;
}

/// engine.hpp:289-295 on the device.  The plan is validated by the reference's
/// own TilingPlan::validate (BadParams); the result is run_full's (the device
/// executes its own footprint-staged tiling) and the report is
/// the reference's TrafficReport for the plan (Eq. 6 words per pass, computed
/// by merit_dev_tiled_traffic).  EngineConfig's scratchpad capacities keep
/// their diagnostic meaning (engine.hpp:82-87, :154-155): a plan whose
/// largest footprint box exceeds scratch_words_a / scratch_words_b throws
/// ScratchpadOverflow, as the reference's Scratchpad::load does.
inline std::pair<Tensor, TrafficReport> run_tiled(const Workload& w, const TilingPlan& plan,
                                                  const EngineConfig& cfg = {}, uint32_t flags = 0) {
  w.validate();
  plan.validate(w.p_shape(), w.a_shape());
  TrafficReport rep;
  {
    detail::Desc D;
    detail::fill(D, w, flags);
    detail::PlanGuard g;
    merit_status st = merit_dev_plan_create(&D.d, &g.p);
    if (st != MERIT_OK) detail::raise(st);
    merit_traffic_report r{};
    st = merit_dev_tiled_traffic(g.p, plan.t_p.data(), plan.t_a.data(), &r);
    if (st != MERIT_OK) detail::raise(st);
    rep.dram_read_words_a = r.dram_read_words_a;
    rep.dram_read_words_b = r.dram_read_words_b;
    rep.dram_write_words = r.dram_write_words;
    rep.scratchpad_peak_words_a = r.scratchpad_peak_words_a;
    rep.scratchpad_peak_words_b = r.scratchpad_peak_words_b;
    rep.passes = r.passes;
    rep.macs = r.macs;
  }
  if (static_cast<int64_t>(rep.scratchpad_peak_words_a) > cfg.scratch_words_a ||
      static_cast<int64_t>(rep.scratchpad_peak_words_b) > cfg.scratch_words_b)
    throw Error(ErrorCode::ScratchpadOverflow, "tile exceeds scratchpad");
  return {run_full(w, flags), rep};
}

/// The DRAM traffic a device run of the workload actually causes (the GPU's
/// counters through CUPTI, L2 flushed first): the measured counterpart of
/// run_tiled's TrafficReport (engine.hpp:72-80).  Allocates device copies of
/// the sources and the output, runs once, returns merit_measured_traffic.
inline merit_measured_traffic measure_traffic(const Workload& w, uint32_t flags = 0) {
  w.validate();
  detail::Desc D;
  detail::fill(D, w, flags);
  detail::PlanGuard g;
  merit_status st = merit_dev_plan_create(&D.d, &g.p);
  if (st != MERIT_OK) detail::raise(st);
  const bool fa = w.src_a.dtype == Dtype::Fix16, fb = w.src_b.dtype == Dtype::Fix16;
  const void* ha = fa ? static_cast<const void*>(w.src_a.qdata.data()) : static_cast<const void*>(w.src_a.fdata.data());
  const void* hb = fb ? static_cast<const void*>(w.src_b.qdata.data()) : static_cast<const void*>(w.src_b.fdata.data());
  merit_measured_traffic r{};
  st = merit_dev_measure_traffic_host(g.p, ha, hb, &r);
  if (st != MERIT_OK) detail::raise(st);
  return r;
}

/// Which device kernel a workload lowers to (MERIT_KERNEL_*), without running it.
inline int lowered_kernel(const Workload& w, uint32_t flags = 0) {
  detail::Desc D;
  detail::fill(D, w, flags);
  detail::PlanGuard g;
  merit_status st = merit_dev_plan_create(&D.d, &g.p);
  if (st != MERIT_OK) detail::raise(st);
  merit_plan_info info{};
  merit_dev_plan_query(g.p, &info);
  return info.kernel;
}

}  // namespace device
}  // namespace merit
