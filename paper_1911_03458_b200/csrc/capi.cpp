// C ABI entry points (include/merit_dev.h).  Host-side plumbing only: plan
// lifetime, lazy device state, host<->device copies for merit_dev_run_host,
// and deterministic input synthesis.  All compute is in the .cu kernels.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <utility>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <cstdio>

#include "plan.hpp"

namespace merit_dev {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
std::atomic<const char*> g_last_kernel{""};
}  // namespace

merit_status fail(merit_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

merit_status cuda_check(int err, const char* what) {
  if (err == cudaSuccess) return MERIT_OK;
  return fail(MERIT_E_CUDA, std::string(what) + ": " +
                                cudaGetErrorString(static_cast<cudaError_t>(err)));
}

void count_launch(int n) { g_launches += n; }
void note_kernel(const char* name) { g_last_kernel.store(name); }
bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("MERIT_PDL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return on != 0;
}

cudaError_t set_smem_attr_impl(const void* fn, cudaFuncAttribute attr, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first.first == dev && e.first.second == fn && e.second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, attr, bytes);
  if (e == cudaSuccess) done.push_back({{dev, fn}, bytes});
  return e;
}

}  // namespace merit_dev

using namespace merit_dev;

// Device-side state a plan needs lazily (program image, error flag).
merit_status merit_dev::ensure_device_state(const merit_plan& plan) {
  std::lock_guard<std::mutex> lk(plan.mu);
  int dev = 0;
  merit_status st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (st != MERIT_OK) return st;
  if (plan.device >= 0 && plan.device != dev)
    return fail(MERIT_E_INVALID_ARGUMENT, "plan was first used on another device");
  plan.device = dev;
  if (!plan.d_err) {
    if ((st = cuda_check(cudaMalloc(&plan.d_err, 16), "cudaMalloc(err)")) != MERIT_OK) return st;
    if ((st = cuda_check(cudaMemset(plan.d_err, 0, 16), "cudaMemset(err)")) != MERIT_OK) return st;
  }
  const bool narrow = plan.kernel == MERIT_KERNEL_SAD && plan.sad.narrow;
  if ((plan.kernel == MERIT_KERNEL_GENERIC || narrow) && !plan.d_prog) {
    if ((st = cuda_check(cudaMalloc(&plan.d_prog, sizeof(ProgramImage)), "cudaMalloc(prog)")) !=
        MERIT_OK)
      return st;
    if ((st = cuda_check(cudaMemcpy(plan.d_prog, &plan.prog, sizeof(ProgramImage),
                                    cudaMemcpyHostToDevice),
                         "cudaMemcpy(prog)")) != MERIT_OK)
      return st;
  }
  if (narrow && !plan.d_narrow) {
    // u8 copies of both frames + the validity flag
    const size_t bytes = (plan.info.src_a_bytes + plan.info.src_b_bytes) / 4 + 64;
    if ((st = cuda_check(cudaMalloc(&plan.d_narrow, bytes), "cudaMalloc(narrow)")) != MERIT_OK) return st;
  }
  if (plan.kernel == MERIT_KERNEL_CONV_TC && !plan.d_packed_b) {
    if ((st = cuda_check(cudaMalloc(&plan.d_packed_b, plan.conv.packed_b_bytes),
                         "cudaMalloc(packed_b)")) != MERIT_OK)
      return st;
  }
  return MERIT_OK;
}

// Stream-order a write of plan.d_packed_b after every earlier run that read
// it (caller holds plan.pack_mu).
merit_status merit_dev::pack_wait(const merit_plan& plan, void* stream) {
  if (!plan.pack_event) return MERIT_OK;
  return cuda_check(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(plan.pack_event), 0),
                    "cudaStreamWaitEvent(pack)");
}
merit_status merit_dev::pack_done(const merit_plan& plan, void* stream) {
  if (!plan.pack_event) {
    cudaEvent_t e;
    merit_status st = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate(pack)");
    if (st != MERIT_OK) return st;
    plan.pack_event = e;
  }
  return cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(plan.pack_event), static_cast<cudaStream_t>(stream)),
                    "cudaEventRecord(pack)");
}

extern "C" {

int32_t merit_dev_abi_version(void) { return MERIT_DEV_ABI_VERSION; }

const char* merit_dev_build_info(void) {
  return "merit_dev: sm_100a kernels {generic, maxpool, sad(vabsdiff4), conv_tc(tcgen05)}";
}

const char* merit_dev_last_error(void) { return g_last_error.c_str(); }

int64_t merit_dev_launch_count(void) { return g_launches.load(); }

const char* merit_dev_last_kernel(void) { return g_last_kernel.load(); }

merit_status merit_dev_plan_create(const merit_workload_desc* desc, merit_plan** out_plan) {
  if (!desc || !out_plan) return fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  *out_plan = nullptr;
  merit_plan* plan = new (std::nothrow) merit_plan();
  if (!plan) return fail(MERIT_E_INVALID_ARGUMENT, "out of host memory");
  plan->desc = *desc;
  // The program's arrays are copied into plan->prog by lower(); the copied
  // descriptor must not keep dangling caller pointers.
  merit_status st = lower(*desc, *plan);
  plan->desc.program.seg_len = nullptr;
  plan->desc.program.instrs = nullptr;
  plan->desc.program.constants = nullptr;
  plan->desc.program.tables = nullptr;
  if (st != MERIT_OK) {
    delete plan;
    return st;
  }
  g_last_error.clear();
  *out_plan = plan;
  return MERIT_OK;
}

// ----------------------------------------------------- multi-workload plans --
namespace {
// The 8x8 + 16x16 (fine, coarse) pair of L1 block-matching members the fused
// SAD kernel computes in one pass: same frames, window, offsets and
// boundary, argmin without maps, the coarse grid exactly 2 x 2 fine blocks.
bool fusable_sad(const merit_plan& fine, const merit_plan& coarse) {
  if (fine.kernel != MERIT_KERNEL_SAD || coarse.kernel != MERIT_KERNEL_SAD) return false;
  const SadParams &f = fine.sad, &c = coarse.sad;
  return f.BH == 8 && f.BW == 8 && c.BH == 16 && c.BW == 16 && f.pairs == c.pairs && f.Hc == c.Hc &&
         f.Wc == c.Wc && f.Hr == c.Hr && f.Wr == c.Wr && f.WY == 65 && f.WX == 65 && c.WY == 65 && c.WX == 65 &&
         f.oy == c.oy && f.ox == c.ox && f.cy == 0 && f.cx == 0 && c.cy == 0 && c.cx == 0 &&
         f.boundary == c.boundary && f.ref_is_b == c.ref_is_b && f.argmin && c.argmin && !f.write_map &&
         !c.write_map && f.BY == 2 * c.BY && f.BX == 2 * c.BX && f.by_count == 0 && c.by_count == 0 &&
         f.by_begin == 0 && c.by_begin == 0;
}
}  // namespace

merit_status merit_dev_plan_create_multi(const merit_workload_desc* descs, int32_t n, merit_plan** out_plan) {
  if (!descs || !out_plan || n < 1) return fail(MERIT_E_INVALID_ARGUMENT, "null argument or empty workload list");
  *out_plan = nullptr;
  merit_plan* g = new (std::nothrow) merit_plan();
  if (!g) return fail(MERIT_E_INVALID_ARGUMENT, "out of host memory");
  for (int32_t i = 0; i < n; ++i) {
    merit_plan* m = nullptr;
    merit_status st = merit_dev_plan_create(&descs[i], &m);
    if (st != MERIT_OK) {
      const std::string msg = "workload " + std::to_string(i) + ": " + g_last_error;
      delete g;
      return fail(st, msg);
    }
    g->members.push_back(m);
  }
  // shared sources (Workload::validate's shape check, engine.hpp:35-36, across members)
  const merit_workload_desc& d0 = descs[0];
  for (int32_t i = 1; i < n; ++i) {
    const merit_workload_desc& d = descs[i];
    bool same = d.dtype_a == d0.dtype_a && d.dtype_b == d0.dtype_b &&
                d.view_a.src_rank == d0.view_a.src_rank && d.view_b.src_rank == d0.view_b.src_rank;
    for (int k = 0; same && k < d.view_a.src_rank; ++k) same = d.view_a.src_shape[k] == d0.view_a.src_shape[k];
    for (int k = 0; same && k < d.view_b.src_rank; ++k) same = d.view_b.src_shape[k] == d0.view_b.src_shape[k];
    if (!same) {
      delete g;
      return fail(MERIT_E_BAD_PARAMS, "multi-workload plans share their two source tensors (shape / dtype mismatch)");
    }
  }
  merit_plan_info& info = g->info;
  std::memset(&info, 0, sizeof(info));
  info.src_a_bytes = g->members[0]->info.src_a_bytes;
  info.src_b_bytes = g->members[0]->info.src_b_bytes;
  int64_t out_off = 0, aux_off = 0;
  for (merit_plan* m : g->members) {
    g->member_out_off.push_back(out_off);
    g->member_aux_off.push_back(aux_off);
    out_off += m->info.out_bytes;
    aux_off += m->info.aux_elems;
    info.out_elems += m->info.out_elems;
    info.n_outputs += m->info.n_outputs;
    info.algorithmic_ops += m->info.algorithmic_ops;
    info.executed_ops += m->info.executed_ops;
    info.launches_per_run += m->info.launches_per_run;
  }
  info.out_bytes = out_off;
  info.aux_elems = aux_off;
  info.out_rank = 1;
  info.out_shape[0] = info.out_elems;
  info.algorithmic_bytes = (double)info.src_a_bytes + (double)info.src_b_bytes + (double)out_off + 4.0 * aux_off;
  info.kernel = MERIT_KERNEL_MULTI;
  // fusion: the fine / coarse block-matching pair
  int fi = -1, ci = -1;
  if (n == 2) {
    if (fusable_sad(*g->members[0], *g->members[1])) fi = 0, ci = 1;
    else if (fusable_sad(*g->members[1], *g->members[0])) fi = 1, ci = 0;
  }
  if (fi >= 0) {
    const merit_plan& f = *g->members[fi];
    g->kernel = MERIT_KERNEL_SAD;
    g->sad = f.sad;
    g->sad.fuse2 = 1;
    g->sad.BY2 = g->members[ci]->sad.BY;
    g->sad.BX2 = g->members[ci]->sad.BX;
    g->fused_aux_off = g->member_aux_off[fi];
    g->sad.aux2_delta = g->member_aux_off[ci] - g->member_aux_off[fi];
    info.kernel = MERIT_KERNEL_SAD;
    info.launches_per_run = 1;
    info.executed_ops = f.info.algorithmic_ops;  // the coarse SADs are sums of fine ones
    std::snprintf(info.description, sizeof(info.description),
                  "sad fused %dx%d + %dx%d pairs=%lld frame=%dx%d blocks=%dx%d+%dx%d window=%dx%d off=%d,%d %s "
                  "+argmin (no map)",
                  f.sad.BH, f.sad.BW, 2 * f.sad.BH, 2 * f.sad.BW, (long long)f.sad.pairs, f.sad.Hc, f.sad.Wc,
                  f.sad.BY, f.sad.BX, g->sad.BY2, g->sad.BX2, f.sad.WY, f.sad.WX, f.sad.oy, f.sad.ox,
                  f.sad.boundary == MERIT_CLAMP ? "clamp" : "zero");
  } else {
    g->kernel = MERIT_KERNEL_MULTI;
    std::snprintf(info.description, sizeof(info.description), "multi %d workloads (run one after another)", n);
  }
  g->desc = d0;
  g->desc.program = {};
  g_last_error.clear();
  *out_plan = g;
  return MERIT_OK;
}

merit_status merit_dev_plan_member(const merit_plan* plan, int32_t i, merit_plan_info* info, int64_t* out_off,
                                   int64_t* aux_off) {
  if (!plan) return fail(MERIT_E_INVALID_ARGUMENT, "null plan");
  const int32_t nm = plan->members.empty() ? 1 : static_cast<int32_t>(plan->members.size());
  if (i < 0 || i >= nm) return fail(MERIT_E_INVALID_ARGUMENT, "member index out of range");
  if (plan->members.empty()) {
    if (info) *info = plan->info;
    if (out_off) *out_off = 0;
    if (aux_off) *aux_off = 0;
    return MERIT_OK;
  }
  if (info) *info = plan->members[i]->info;
  if (out_off) *out_off = plan->member_out_off[i];
  if (aux_off) *aux_off = plan->member_aux_off[i];
  return MERIT_OK;
}

merit_status merit_dev_plan_destroy(merit_plan* plan) {
  if (!plan) return MERIT_OK;
  if (plan->device >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(plan->device);
    if (plan->d_prog) cudaFree(plan->d_prog);
    if (plan->d_err) cudaFree(plan->d_err);
    if (plan->d_packed_b) cudaFree(plan->d_packed_b);
    if (plan->d_narrow) cudaFree(plan->d_narrow);
    if (plan->pack_event) cudaEventDestroy(static_cast<cudaEvent_t>(plan->pack_event));
    cudaSetDevice(cur);
  }
  if (plan->stage_dev >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(plan->stage_dev);
    for (void* p : plan->stage)
      if (p) cudaFree(p);
    release_host_pipeline(*plan);
    cudaSetDevice(cur);
  }
  delete plan;
  return MERIT_OK;
}

merit_status merit_dev_plan_query(const merit_plan* plan, merit_plan_info* info) {
  if (!plan || !info) return fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  *info = plan->info;
  return MERIT_OK;
}

merit_status merit_dev_plan_pack_b(merit_plan* plan, const void* d_src_b, void* stream) {
  if (!plan) return fail(MERIT_E_INVALID_ARGUMENT, "null plan");
  if (plan->kernel != MERIT_KERNEL_CONV_TC) return MERIT_OK;  // nothing to pack
  if (!d_src_b) return fail(MERIT_E_INVALID_ARGUMENT, "null weights");
  merit_status st = ensure_device_state(*plan);
  if (st != MERIT_OK) return st;
  std::lock_guard<std::mutex> lk(plan->pack_mu);
  if ((st = pack_wait(*plan, stream)) != MERIT_OK) return st;
  st = launch_conv_pack(*plan, d_src_b, plan->d_packed_b, stream);
  if (st == MERIT_OK) st = pack_done(*plan, stream);
  if (st == MERIT_OK) plan->packed_valid = true;
  return st;
}

static merit_status check_error_flag(const merit_plan& plan, cudaStream_t s) {
  int32_t err[2] = {0, 0};
  merit_status st = cuda_check(
      cudaMemcpyAsync(err, plan.d_err, sizeof(err), cudaMemcpyDeviceToHost, s), "read error flag");
  if (st != MERIT_OK) return st;
  if ((st = cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize")) != MERIT_OK) return st;
  if (err[0] != 0) {
    cudaMemsetAsync(plan.d_err, 0, 16, s);
    cudaStreamSynchronize(s);
    const char* what = "device execution error";
    switch (err[0]) {
      case MERIT_E_OUT_OF_RANGE: what = "gather outside source tensor"; break;
      case MERIT_E_DIV_BY_ZERO: what = "DIV by zero"; break;
      case MERIT_E_LUT_RANGE: what = "lookup outside table range"; break;
      case MERIT_E_BAD_PARAMS: what = "program emitted wrong output count or bad aux index"; break;
      default: break;
    }
    return fail(static_cast<merit_status>(err[0]), what);
  }
  return MERIT_OK;
}

merit_status merit_dev_run(const merit_plan* plan, const void* d_a, const void* d_b, void* d_out,
                           void* d_aux, void* stream) {
  if (!plan) return fail(MERIT_E_INVALID_ARGUMENT, "null plan");
  const merit_plan_info& info = plan->info;
  if (info.out_elems > 0 && !d_out) return fail(MERIT_E_INVALID_ARGUMENT, "null output");
  if (info.aux_elems > 0 && !d_aux) return fail(MERIT_E_INVALID_ARGUMENT, "null aux output");
  merit_status st = MERIT_OK;
  if (!plan->members.empty()) {
    // multi-workload plan: one fused launch, or the members in order
    if (plan->kernel == MERIT_KERNEL_SAD) {
      if (!d_a || !d_b) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      if ((st = ensure_device_state(*plan)) != MERIT_OK) return st;
      st = launch_sad(*plan, d_a, d_b, nullptr, static_cast<int32_t*>(d_aux) + plan->fused_aux_off, stream);
      if (st != MERIT_E_UNSUPPORTED_VIEW) return st;  // else: not fusable for these buffers
    }
    for (size_t i = 0; i < plan->members.size(); ++i) {
      st = merit_dev_run(plan->members[i], d_a, d_b,
                         d_out ? static_cast<char*>(d_out) + plan->member_out_off[i] : nullptr,
                         d_aux ? static_cast<int32_t*>(d_aux) + plan->member_aux_off[i] : nullptr, stream);
      if (st != MERIT_OK) return st;
    }
    return MERIT_OK;
  }
  st = ensure_device_state(*plan);
  if (st != MERIT_OK) return st;
  switch (plan->kernel) {
    case MERIT_KERNEL_GENERIC: {
      if (!d_a || !d_b) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      std::lock_guard<std::mutex> lk(plan->run_mu);  // one error flag per plan
      st = launch_generic(*plan, d_a, d_b, d_out, stream);
      if (st == MERIT_OK) st = check_error_flag(*plan, static_cast<cudaStream_t>(stream));
      return st;
    }
    case MERIT_KERNEL_MAXPOOL:
      if (!d_a) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      return launch_maxpool(*plan, d_a, d_out, stream);
    case MERIT_KERNEL_SAD: {
      if (!d_a || !d_b) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      if (!plan->sad.narrow) return launch_sad(*plan, d_a, d_b, d_out, d_aux, stream);
      // the plan's u8 frame copies are shared: stream-ordered like on-the-fly packing
      std::lock_guard<std::mutex> lk(plan->pack_mu);
      if ((st = pack_wait(*plan, stream)) != MERIT_OK) return st;
      st = launch_sad_narrowed(*plan, d_a, d_b, d_out, stream);
      if (st == MERIT_OK) st = pack_done(*plan, stream);
      return st;
    }
    case MERIT_KERNEL_CONV_TC: {
      const void* in = plan->conv_swapped ? d_b : d_a;
      const void* w = plan->conv_swapped ? d_a : d_b;
      if (!in) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      if (plan->packed_valid) return launch_conv(*plan, in, plan->d_packed_b, d_out, stream);
      // weights packed on the fly into the plan's buffer, ordered after any
      // other stream's run that still reads it
      if (!w) return fail(MERIT_E_INVALID_ARGUMENT, "null weights and no packed copy");
      std::lock_guard<std::mutex> lk(plan->pack_mu);
      if ((st = pack_wait(*plan, stream)) != MERIT_OK) return st;
      st = launch_conv_pack(*plan, w, plan->d_packed_b, stream);
      if (st == MERIT_OK) st = launch_conv(*plan, in, plan->d_packed_b, d_out, stream);
      if (st == MERIT_OK) st = pack_done(*plan, stream);
      return st;
    }
    case MERIT_KERNEL_CORR:
      if (!d_a || !d_b) return fail(MERIT_E_INVALID_ARGUMENT, "null source");
      return plan->corr_swapped ? launch_corr(*plan, d_b, d_a, d_out, stream)
                                : launch_corr(*plan, d_a, d_b, d_out, stream);
    default:
      return fail(MERIT_E_INVALID_ARGUMENT, "corrupt plan");
  }
}

merit_status merit_dev_run_host(const merit_plan* plan, const void* h_a, const void* h_b,
                                void* h_out, void* h_aux, void* stream) {
  if (!plan) return fail(MERIT_E_INVALID_ARGUMENT, "null plan");
  const merit_plan_info& info = plan->info;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Port B is copied whenever the caller provides it (for a packed
  // convolution plan the run ignores it).
  const bool need_b = h_b != nullptr && info.src_b_bytes > 0;
  std::lock_guard<std::mutex> lock(plan->host_mu);
  // Device staging cached in the plan: a fresh stream-ordered allocation of
  // the buffers per call measured ~0.7 ms of C2's 1.5 ms call (40 MB
  // returned to and re-mapped from the driver every time).
  int dev = 0;
  merit_status st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (st != MERIT_OK) return st;
  if (plan->stage_dev != dev) {
    if (plan->stage_dev >= 0) {
      cudaSetDevice(plan->stage_dev);
      for (void*& p : plan->stage) {
        if (p) cudaFree(p);
        p = nullptr;
      }
      release_host_pipeline(*plan);
      cudaSetDevice(dev);
    }
    for (size_t& b : plan->stage_bytes) b = 0;
    plan->stage_dev = dev;
  }
  const size_t want[4] = {static_cast<size_t>(info.src_a_bytes), need_b ? static_cast<size_t>(info.src_b_bytes) : 0,
                          static_cast<size_t>(info.out_bytes), static_cast<size_t>(info.aux_elems) * 4};
  for (int i = 0; i < 4; ++i) {
    if (want[i] == 0 || want[i] <= plan->stage_bytes[i]) continue;
    if (plan->stage[i]) cudaFree(plan->stage[i]);
    plan->stage[i] = nullptr;
    plan->stage_bytes[i] = 0;
    st = cuda_check(cudaMalloc(&plan->stage[i], want[i]), "cudaMalloc(run_host staging)");
    if (st != MERIT_OK) return st;
    plan->stage_bytes[i] = want[i];
  }
  void* da = plan->stage[0];
  void* db = need_b ? plan->stage[1] : nullptr;
  void* dout = info.out_bytes > 0 ? plan->stage[2] : nullptr;
  void* daux = info.aux_elems > 0 ? plan->stage[3] : nullptr;
#define MERIT_TRY(expr, what)                                  \
  do {                                                         \
    st = cuda_check((expr), what);                             \
    if (st != MERIT_OK) { cudaStreamSynchronize(s); return st; } \
  } while (0)
  // Sliced plans overlap H2D, kernel and D2H slice by slice (host_pipeline.cpp)
  st = run_host_pipelined(*plan, da, db, dout, daux, h_a, h_b, h_out, h_aux, need_b, stream);
  if (st != MERIT_E_UNSUPPORTED_VIEW) return st;
  MERIT_TRY(cudaMemcpyAsync(da, h_a, info.src_a_bytes, cudaMemcpyHostToDevice, s), "H2D a");
  if (need_b) MERIT_TRY(cudaMemcpyAsync(db, h_b, info.src_b_bytes, cudaMemcpyHostToDevice, s), "H2D b");
  st = merit_dev_run(plan, da, db, dout, daux, stream);
  if (st != MERIT_OK) {
    std::string msg = g_last_error;
    cudaStreamSynchronize(s);
    return fail(st, msg);
  }
  if (info.out_bytes > 0)
    MERIT_TRY(cudaMemcpyAsync(h_out, dout, info.out_bytes, cudaMemcpyDeviceToHost, s), "D2H out");
  if (info.aux_elems > 0)
    MERIT_TRY(cudaMemcpyAsync(h_aux, daux, info.aux_elems * 4, cudaMemcpyDeviceToHost, s), "D2H aux");
  MERIT_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
#undef MERIT_TRY
  return MERIT_OK;
}

// ------------------------------------------------------------ generators --
// SplitMix64 exactly as workloads.hpp:74-94.
namespace {
struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t s) : state(s) {}
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform(double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(next() >> 11) * 0x1.0p-53);
  }
  int64_t range(int64_t lo, int64_t hi) {
    return lo + static_cast<int64_t>(next() % static_cast<uint64_t>(hi - lo + 1));
  }
};
}  // namespace

void merit_gen_uniform_f32(float* out, int64_t n, uint64_t seed, double lo, double hi) {
  SplitMix64 rng(seed);  // fill_random, workloads.hpp:96-105
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng.uniform(lo, hi));
}

void merit_gen_range_i16(int16_t* out, int64_t n, uint64_t seed, int64_t lo, int64_t hi) {
  SplitMix64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<int16_t>(rng.range(lo, hi));
}

void merit_gen_normal_f32(float* out, int64_t n, uint64_t seed, double sigma) {
  // Box-Muller over SplitMix64 uniforms (SURVEY §8(d) C3/C4 weights).
  SplitMix64 rng(seed);
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; i += 2) {
    double u1 = rng.uniform(0.0, 1.0), u2 = rng.uniform(0.0, 1.0);
    if (u1 < 1e-300) u1 = 1e-300;
    double r = std::sqrt(-2.0 * std::log(u1));
    out[i] = static_cast<float>(sigma * r * std::cos(two_pi * u2));
    if (i + 1 < n) out[i + 1] = static_cast<float>(sigma * r * std::sin(two_pi * u2));
  }
}

void merit_gen_me_pair(uint8_t* cur, uint8_t* ref, int64_t h, int64_t w, int64_t blk,
                       int64_t max_shift, int64_t noise, uint64_t seed) {
  // ref = box5x5(uniform bytes); cur = per-block shifted ref + noise.
  SplitMix64 rng(seed);
  uint8_t* raw = new uint8_t[h * w];
  for (int64_t i = 0; i < h * w; ++i) raw[i] = static_cast<uint8_t>(rng.range(0, 255));
  auto cl = [](int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : v > hi ? hi : v; };
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      int64_t s = 0;
      for (int64_t dy = -2; dy <= 2; ++dy)
        for (int64_t dx = -2; dx <= 2; ++dx) s += raw[cl(y + dy, 0, h - 1) * w + cl(x + dx, 0, w - 1)];
      ref[y * w + x] = static_cast<uint8_t>((s + 12) / 25);  // round half up
    }
  delete[] raw;
  const int64_t by = (h + blk - 1) / blk, bx = (w + blk - 1) / blk;
  for (int64_t b = 0; b < by * bx; ++b) {
    const int64_t y0 = (b / bx) * blk, x0 = (b % bx) * blk;
    const int64_t sx = rng.range(-max_shift, max_shift), sy = rng.range(-max_shift, max_shift);
    for (int64_t i = 0; i < blk && y0 + i < h; ++i)
      for (int64_t j = 0; j < blk && x0 + j < w; ++j) {
        const int64_t y = y0 + i, x = x0 + j;
        int64_t v = ref[cl(y + sy, 0, h - 1) * w + cl(x + sx, 0, w - 1)] + rng.range(-noise, noise);
        cur[y * w + x] = static_cast<uint8_t>(cl(v, 0, 255));
      }
  }
}

void merit_f32_to_bf16(const float* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, &in[i], 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) {  // NaN stays NaN
      out[i] = static_cast<uint16_t>((u >> 16) | 0x40);
      continue;
    }
    u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
    out[i] = static_cast<uint16_t>(u >> 16);
  }
}

}  // extern "C"
