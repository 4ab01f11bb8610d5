// Probe of merit_dev_measure_traffic_host without PyTorch in the process.
#include <cstdio>
#include <vector>
#include "merit_dev.h"

int main() {
  // 2-D max-pool, 3x3 / s2 / pad 1 (CLAMP) over (4, 64, 112, 112) fp32
  const int64_t n = 4, c = 64, h = 112, w = 112, ho = 56, wo = 56;
  merit_workload_desc d{};
  d.view_a.src_rank = 4; d.view_a.p_rank = 4; d.view_a.a_rank = 2; d.view_a.n_terms = 6;
  const int64_t src[4] = {n, c, h, w}, p[4] = {n, c, ho, wo};
  for (int i = 0; i < 4; ++i) { d.view_a.src_shape[i] = src[i]; d.view_a.p_shape[i] = p[i]; d.view_b.p_shape[i] = p[i]; }
  d.view_a.a_shape[0] = d.view_a.a_shape[1] = 3;
  const merit_view_term t[6] = {{0, 0, 1, 0}, {1, 1, 1, 0}, {2, 2, 2, -1}, {4, 2, 1, 0}, {3, 3, 2, -1}, {5, 3, 1, 0}};
  for (int i = 0; i < 6; ++i) d.view_a.terms[i] = t[i];
  d.view_a.boundary = MERIT_CLAMP;
  d.view_b.src_rank = 1; d.view_b.src_shape[0] = 1; d.view_b.p_rank = 4; d.view_b.a_rank = 2;
  d.view_b.a_shape[0] = d.view_b.a_shape[1] = 3;
  d.dtype_a = d.dtype_b = d.dtype_out = MERIT_F32;
  int32_t seg[5] = {1, 0, 1, 0, 1};
  merit_alu_instr ins[3] = {};
  ins[0].op = MERIT_OP_MOVC; ins[0].a_kind = ins[0].b_kind = ins[0].c_kind = MERIT_OPND_ZERO;
  ins[1].op = MERIT_OP_MAX; ins[1].a_kind = MERIT_OPND_REG; ins[1].b_kind = MERIT_OPND_PORT_A; ins[1].c_kind = MERIT_OPND_ZERO;
  ins[2].op = MERIT_OP_ADD; ins[2].dst_out = 1; ins[2].a_kind = MERIT_OPND_REG; ins[2].b_kind = ins[2].c_kind = MERIT_OPND_ZERO;
  double consts[1] = {-3.0e38};
  d.program.depth = 2; d.program.outputs = 1; d.program.n_segments = 5; d.program.n_constants = 1;
  d.program.seg_len = seg; d.program.instrs = ins; d.program.constants = consts;
  merit_plan* plan = nullptr;
  if (merit_dev_plan_create(&d, &plan)) { std::printf("plan: %s\n", merit_dev_last_error()); return 1; }
  merit_plan_info info{};
  merit_dev_plan_query(plan, &info);
  std::printf("kernel %d: %s\n", info.kernel, info.description);
  std::vector<float> a(n * c * h * w, 0.25f), b(1, 0.f);
  merit_measured_traffic r{};
  const int st = merit_dev_measure_traffic_host(plan, a.data(), b.data(), &r);
  std::printf("status %d %s\nread %.0f write %.0f time_ns %.0f ranges %lld launches %lld passes %d (sources %lld B)\n", st,
              merit_dev_last_error(), r.dram_read_bytes, r.dram_write_bytes, r.kernel_time_ns, (long long)r.ranges,
              (long long)r.launches, r.passes, (long long)info.src_a_bytes);
  merit_dev_plan_destroy(plan);
  return st;
}
