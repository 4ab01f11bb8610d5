// merit_dev_measure_traffic: the measured counterpart of run_tiled's
// TrafficReport (engine.hpp:72-80).  The reference counts the words its
// scratchpad loads pass by pass (engine.hpp:233-241); the device run's real
// traffic is what the HBM controllers move, read here from the GPU's
// performance counters with the CUPTI range profiler (one user range around
// the run, user replay: the run repeats once per counter pass; an auto range
// per kernel does not see launches issued through this library's statically
// linked runtime): dram__bytes_read.sum, dram__bytes_write.sum and
// gpu__time_duration.sum of the range.  L2 is flushed before the run so the reads are the run's own
// (a preceding H2D copy would otherwise leave the sources in L2); dirty
// output lines still resident in L2 when the last kernel ends are not DRAM
// writes yet, and the report says so (dram_write_bytes is a lower bound).
//
// CUPTI is loaded with dlopen at the first call: the library itself has no
// link-time dependency on it, and without it (or without profiling
// permission) the call fails with MERIT_E_UNSUPPORTED_PROGRAM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>
#include <dlfcn.h>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace merit_dev {
namespace {

struct Cupti {
  bool ok = false;
  std::string why;
#define MERIT_CUPTI_FN(name) decltype(&::name) name = nullptr;
  MERIT_CUPTI_FN(cuptiProfilerInitialize)
  MERIT_CUPTI_FN(cuptiDeviceGetChipName)
  MERIT_CUPTI_FN(cuptiProfilerGetCounterAvailability)
  MERIT_CUPTI_FN(cuptiProfilerHostInitialize)
  MERIT_CUPTI_FN(cuptiProfilerHostDeinitialize)
  MERIT_CUPTI_FN(cuptiProfilerHostConfigAddMetrics)
  MERIT_CUPTI_FN(cuptiProfilerHostGetConfigImageSize)
  MERIT_CUPTI_FN(cuptiProfilerHostGetConfigImage)
  MERIT_CUPTI_FN(cuptiProfilerHostGetNumOfPasses)
  MERIT_CUPTI_FN(cuptiProfilerHostEvaluateToGpuValues)
  MERIT_CUPTI_FN(cuptiRangeProfilerEnable)
  MERIT_CUPTI_FN(cuptiRangeProfilerDisable)
  MERIT_CUPTI_FN(cuptiRangeProfilerGetCounterDataSize)
  MERIT_CUPTI_FN(cuptiRangeProfilerCounterDataImageInitialize)
  MERIT_CUPTI_FN(cuptiRangeProfilerSetConfig)
  MERIT_CUPTI_FN(cuptiRangeProfilerStart)
  MERIT_CUPTI_FN(cuptiRangeProfilerStop)
  MERIT_CUPTI_FN(cuptiRangeProfilerPushRange)
  MERIT_CUPTI_FN(cuptiRangeProfilerPopRange)
  MERIT_CUPTI_FN(cuptiRangeProfilerDecodeData)
  MERIT_CUPTI_FN(cuptiRangeProfilerGetCounterDataInfo)
#undef MERIT_CUPTI_FN
};

Cupti& cupti() {
  static Cupti c;
  static std::once_flag once;
  std::call_once(once, [] {
    // a CUPTI already in the process (e.g. the copy PyTorch loads at import)
    // must be the one used: a second instance does not see the launches
    void* h = dlopen("libcupti.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcupti.so", RTLD_NOW | RTLD_NOLOAD);
    for (const char* n : {"libcupti.so.12", "libcupti.so", "/usr/local/cuda/lib64/libcupti.so"})
      if (!h) h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      c.why = "libcupti.so not found";
      return;
    }
    bool all = true;
#define MERIT_CUPTI_LOAD(name)                                          \
  c.name = reinterpret_cast<decltype(c.name)>(dlsym(h, #name));        \
  if (!c.name) all = false;
    MERIT_CUPTI_LOAD(cuptiProfilerInitialize)
    MERIT_CUPTI_LOAD(cuptiDeviceGetChipName)
    MERIT_CUPTI_LOAD(cuptiProfilerGetCounterAvailability)
    MERIT_CUPTI_LOAD(cuptiProfilerHostInitialize)
    MERIT_CUPTI_LOAD(cuptiProfilerHostDeinitialize)
    MERIT_CUPTI_LOAD(cuptiProfilerHostConfigAddMetrics)
    MERIT_CUPTI_LOAD(cuptiProfilerHostGetConfigImageSize)
    MERIT_CUPTI_LOAD(cuptiProfilerHostGetConfigImage)
    MERIT_CUPTI_LOAD(cuptiProfilerHostGetNumOfPasses)
    MERIT_CUPTI_LOAD(cuptiProfilerHostEvaluateToGpuValues)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerEnable)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerDisable)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerGetCounterDataSize)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerCounterDataImageInitialize)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerSetConfig)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerStart)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerStop)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerPushRange)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerPopRange)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerDecodeData)
    MERIT_CUPTI_LOAD(cuptiRangeProfilerGetCounterDataInfo)
#undef MERIT_CUPTI_LOAD
    if (!all) {
      c.why = "libcupti.so lacks the range profiler API";
      return;
    }
    CUpti_Profiler_Initialize_Params ip = {CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    if (c.cuptiProfilerInitialize(&ip) != CUPTI_SUCCESS) {
      c.why = "cuptiProfilerInitialize failed";
      return;
    }
    c.ok = true;
  });
  return c;
}

// Read-only L2 flush: a read pass over twice the L2 evicts whatever a
// preceding copy or kernel left there (dirty lines are written back during
// the flush, outside the profiled run) and leaves only clean lines, whose
// eviction costs the measured run no DRAM writes.
__global__ void l2_flush_kernel(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);  // keeps the loads live
}

const char* const kMetrics[] = {"dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"};
constexpr size_t kNumMetrics = 3;

}  // namespace
}  // namespace merit_dev

using namespace merit_dev;

// The profiler refused (no CUPTI, no permission, counters held by another
// client of this GPU, ...): one recognisable message prefix, so callers can
// tell "this system cannot measure" from a failure of the run itself.
static merit_status unavailable(const std::string& what) {
  return fail(MERIT_E_UNSUPPORTED_PROGRAM, "measure_traffic unavailable on this system: " + what);
}

extern "C" merit_status merit_dev_measure_traffic(const merit_plan* plan, const void* d_a, const void* d_b,
                                                  void* d_out, void* d_aux, void* stream,
                                                  merit_measured_traffic* report) {
  if (!plan || !report) return fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  static std::mutex mu;  // one profiling session per process at a time
  std::lock_guard<std::mutex> lk(mu);
  Cupti& c = cupti();
  if (!c.ok) return unavailable(c.why);
  merit_status st = cuda_check(cudaFree(nullptr), "cudaFree(0)");
  if (st != MERIT_OK) return st;
  int dev = 0;
  if ((st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) != MERIT_OK) return st;
  // cuCtxGetCurrent through the runtime's driver entry point (no libcuda
  // link-time dependency: the library must load on hosts without a driver)
  CUcontext ctx = nullptr;
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(MERIT_E_CUDA, "cuCtxGetCurrent entry point");
    if (reinterpret_cast<CUresult (*)(CUcontext*)>(fn)(&ctx) != CUDA_SUCCESS || !ctx)
      return fail(MERIT_E_CUDA, "no current CUDA context");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);

  // host side: config image for the three metrics on this chip
  CUpti_Device_GetChipName_Params cn = {CUpti_Device_GetChipName_Params_STRUCT_SIZE};
  cn.deviceIndex = static_cast<size_t>(dev);
  if (c.cuptiDeviceGetChipName(&cn) != CUPTI_SUCCESS) return unavailable("cuptiDeviceGetChipName");
  CUpti_Profiler_GetCounterAvailability_Params ca = {CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
  ca.ctx = ctx;
  if (c.cuptiProfilerGetCounterAvailability(&ca) != CUPTI_SUCCESS)
    return unavailable("counter availability (profiling not permitted?)");
  std::vector<uint8_t> avail(ca.counterAvailabilityImageSize);
  ca.pCounterAvailabilityImage = avail.data();
  if (c.cuptiProfilerGetCounterAvailability(&ca) != CUPTI_SUCCESS)
    return unavailable("counter availability image");
  CUpti_Profiler_Host_Initialize_Params hi = {CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
  hi.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
  hi.pChipName = cn.pChipName;
  hi.pCounterAvailabilityImage = avail.data();
  if (c.cuptiProfilerHostInitialize(&hi) != CUPTI_SUCCESS) return unavailable("host initialize");
  CUpti_Profiler_Host_Object* host = hi.pHostObject;
  auto host_done = [&] {
    CUpti_Profiler_Host_Deinitialize_Params hd = {CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
    hd.pHostObject = host;
    c.cuptiProfilerHostDeinitialize(&hd);
  };
  const char* names[kNumMetrics] = {kMetrics[0], kMetrics[1], kMetrics[2]};
  CUpti_Profiler_Host_ConfigAddMetrics_Params am = {CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
  am.pHostObject = host;
  am.ppMetricNames = names;
  am.numMetrics = kNumMetrics;
  CUpti_Profiler_Host_GetConfigImageSize_Params cs = {CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
  cs.pHostObject = host;
  if (c.cuptiProfilerHostConfigAddMetrics(&am) != CUPTI_SUCCESS || c.cuptiProfilerHostGetConfigImageSize(&cs) != CUPTI_SUCCESS) {
    host_done();
    return unavailable("metric configuration");
  }
  std::vector<uint8_t> config(cs.configImageSize);
  CUpti_Profiler_Host_GetConfigImage_Params ci = {CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
  ci.pHostObject = host;
  ci.configImageSize = config.size();
  ci.pConfigImage = config.data();
  CUpti_Profiler_Host_GetNumOfPasses_Params np = {CUpti_Profiler_Host_GetNumOfPasses_Params_STRUCT_SIZE};
  np.configImageSize = config.size();
  np.pConfigImage = config.data();
  if (c.cuptiProfilerHostGetConfigImage(&ci) != CUPTI_SUCCESS || c.cuptiProfilerHostGetNumOfPasses(&np) != CUPTI_SUCCESS) {
    host_done();
    return unavailable("config image");
  }

  // L2 flush: a write pass over twice the L2 evicts the sources a preceding
  // copy may have left there (outside the profiled session)
  static void* flush = nullptr;
  static size_t flush_bytes = 0;
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  const size_t want = 2 * static_cast<size_t>(l2 > 0 ? l2 : (128 << 20));
  if (flush_bytes < want) {
    if (flush) cudaFree(flush);
    flush = nullptr;
    if ((st = cuda_check(cudaMalloc(&flush, want + 64), "cudaMalloc(L2 flush)")) != MERIT_OK ||
        (st = cuda_check(cudaMemset(flush, 0x5a, want + 64), "memset(L2 flush)")) != MERIT_OK) {
      host_done();
      return st;
    }
    flush_bytes = want;
  }
  // target side: range profiler on the context, one auto range per kernel
  CUpti_RangeProfiler_Enable_Params en = {CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
  en.ctx = ctx;
  if (c.cuptiRangeProfilerEnable(&en) != CUPTI_SUCCESS) {
    host_done();
    return unavailable("range profiler enable (profiling not permitted?)");
  }
  CUpti_RangeProfiler_Object* obj = en.pRangeProfilerObject;
  auto target_done = [&] {
    CUpti_RangeProfiler_Disable_Params di = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
    di.pRangeProfilerObject = obj;
    c.cuptiRangeProfilerDisable(&di);
  };
  const size_t max_ranges = 64;
  CUpti_RangeProfiler_GetCounterDataSize_Params ds = {CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
  ds.pRangeProfilerObject = obj;
  ds.pMetricNames = names;
  ds.numMetrics = kNumMetrics;
  ds.maxNumOfRanges = max_ranges;
  ds.maxNumRangeTreeNodes = static_cast<uint32_t>(max_ranges);
  if (c.cuptiRangeProfilerGetCounterDataSize(&ds) != CUPTI_SUCCESS) {
    target_done();
    host_done();
    return unavailable("counter data size");
  }
  std::vector<uint8_t> counters(ds.counterDataSize);
  CUpti_RangeProfiler_CounterDataImage_Initialize_Params cdi = {
      CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  cdi.pRangeProfilerObject = obj;
  cdi.counterDataSize = counters.size();
  cdi.pCounterData = counters.data();
  CUpti_RangeProfiler_SetConfig_Params sc = {CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
  sc.pRangeProfilerObject = obj;
  sc.configSize = config.size();
  sc.pConfig = config.data();
  sc.counterDataImageSize = counters.size();
  sc.pCounterDataImage = counters.data();
  // one user range around the whole run (every launch of the plan, whatever
  // API issues it), user replay: the run is repeated once per pass
  sc.range = CUPTI_UserRange;
  sc.replayMode = CUPTI_UserReplay;
  sc.maxRangesPerPass = max_ranges;
  sc.numNestingLevels = 1;
  sc.minNestingLevel = 1;
  sc.passIndex = 0;
  sc.targetNestingLevel = 1;
  if (c.cuptiRangeProfilerCounterDataImageInitialize(&cdi) != CUPTI_SUCCESS ||
      c.cuptiRangeProfilerSetConfig(&sc) != CUPTI_SUCCESS) {
    target_done();
    host_done();
    return unavailable("range profiler configuration");
  }
  const int64_t l0 = merit_dev_launch_count();
  int npass = 0;
  CUpti_RangeProfiler_Stop_Params so = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
  std::string run_err;
  for (;;) {
    // L2 flush before every pass (outside the range)
    l2_flush_kernel<<<4 * num_sms(), 512, 0, s>>>(static_cast<const uint4*>(flush), flush_bytes / 16,
                                                   reinterpret_cast<unsigned*>(static_cast<char*>(flush) + flush_bytes));
    if ((st = cuda_check(cudaGetLastError(), "L2 flush")) == MERIT_OK) st = cuda_check(cudaStreamSynchronize(s), "sync");
    CUpti_RangeProfiler_Start_Params sp = {CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    sp.pRangeProfilerObject = obj;
    CUpti_RangeProfiler_PushRange_Params pr = {CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pr.pRangeProfilerObject = obj;
    pr.pRangeName = "merit_dev_run";
    CUpti_RangeProfiler_PopRange_Params po = {CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
    po.pRangeProfilerObject = obj;
    CUptiResult rc_start = CUPTI_SUCCESS, rc_push = CUPTI_SUCCESS;
    if (st != MERIT_OK || (rc_start = c.cuptiRangeProfilerStart(&sp)) != CUPTI_SUCCESS ||
        (rc_push = c.cuptiRangeProfilerPushRange(&pr)) != CUPTI_SUCCESS) {
      if (st == MERIT_OK)
        st = unavailable("range profiler start (CUPTI result: start " + std::to_string(int(rc_start)) +
                                                   ", push " + std::to_string(int(rc_push)) + ")");
      break;
    }
    st = merit_dev_run(plan, d_a, d_b, d_out, d_aux, stream);
    if (st != MERIT_OK) run_err = merit_dev_last_error();
    cudaStreamSynchronize(s);
    so = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
    so.pRangeProfilerObject = obj;
    const CUptiResult rc_pop = c.cuptiRangeProfilerPopRange(&po);
    const CUptiResult rc_stop = c.cuptiRangeProfilerStop(&so);
    const bool stopped = rc_pop == CUPTI_SUCCESS && rc_stop == CUPTI_SUCCESS;
    ++npass;
    if (st != MERIT_OK) break;
    if (!stopped) {
      st = unavailable("range profiler stop (CUPTI result: pop " + std::to_string(int(rc_pop)) +
                                                 ", stop " + std::to_string(int(rc_stop)) + ", pass " +
                                                 std::to_string(npass) + ")");
      break;
    }
    if (so.isAllPassSubmitted || npass > 64) break;
  }
  CUpti_RangeProfiler_DecodeData_Params dd = {CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
  dd.pRangeProfilerObject = obj;
  if (st == MERIT_OK && c.cuptiRangeProfilerDecodeData(&dd) != CUPTI_SUCCESS)
    st = unavailable("range profiler decode");
  if (st != MERIT_OK) {
    const std::string msg = run_err.empty() ? std::string(merit_dev_last_error()) : run_err;
    target_done();
    host_done();
    return fail(st, msg);
  }
  CUpti_RangeProfiler_GetCounterDataInfo_Params gi = {CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
  gi.pCounterDataImage = counters.data();
  gi.counterDataImageSize = counters.size();
  if (c.cuptiRangeProfilerGetCounterDataInfo(&gi) != CUPTI_SUCCESS) {
    target_done();
    host_done();
    return unavailable("counter data info");
  }
  merit_measured_traffic r{};
  for (size_t i = 0; i < gi.numTotalRanges; ++i) {
    double v[kNumMetrics] = {0, 0, 0};
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = host;
    ev.pCounterDataImage = counters.data();
    ev.counterDataImageSize = counters.size();
    ev.rangeIndex = i;
    ev.ppMetricNames = names;
    ev.numMetrics = kNumMetrics;
    ev.pMetricValues = v;
    if (c.cuptiProfilerHostEvaluateToGpuValues(&ev) != CUPTI_SUCCESS) continue;
    r.dram_read_bytes += v[0];
    r.dram_write_bytes += v[1];
    r.range_time_ns += v[2];
  }
  r.ranges = static_cast<int64_t>(gi.numTotalRanges);
  if (r.ranges == 0) {
    target_done();
    host_done();
    return fail(MERIT_E_UNSUPPORTED_PROGRAM,
                "measure_traffic: no kernel ranges collected (dropped " + std::to_string(dd.numOfRangeDropped) +
                    ", all passes submitted " + std::to_string(int(so.isAllPassSubmitted)) + ", passes " +
                    std::to_string(np.numOfPasses) + ")");
  }
  r.launches = (merit_dev_launch_count() - l0) / (npass > 0 ? npass : 1);
  r.passes = npass;
  target_done();
  host_done();
  *report = r;
  return MERIT_OK;
}

extern "C" merit_status merit_dev_measure_traffic_host(const merit_plan* plan, const void* h_a, const void* h_b,
                                                       merit_measured_traffic* report) {
  if (!plan || !report) return fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  const merit_plan_info& in = plan->info;
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  const size_t bytes[4] = {static_cast<size_t>(in.src_a_bytes), static_cast<size_t>(in.src_b_bytes),
                           static_cast<size_t>(in.out_bytes > 0 ? in.out_bytes : 4),
                           static_cast<size_t>(in.aux_elems > 0 ? in.aux_elems * 4 : 4)};
  merit_status st = MERIT_OK;
  for (int i = 0; i < 4 && st == MERIT_OK; ++i) st = cuda_check(cudaMalloc(&buf[i], bytes[i] ? bytes[i] : 4), "cudaMalloc");
  if (st == MERIT_OK && h_a) st = cuda_check(cudaMemcpy(buf[0], h_a, bytes[0], cudaMemcpyHostToDevice), "H2D a");
  if (st == MERIT_OK && h_b) st = cuda_check(cudaMemcpy(buf[1], h_b, bytes[1], cudaMemcpyHostToDevice), "H2D b");
  if (st == MERIT_OK) st = merit_dev_measure_traffic(plan, buf[0], buf[1], buf[2], in.aux_elems > 0 ? buf[3] : nullptr,
                                                    nullptr, report);
  const std::string msg = st != MERIT_OK ? std::string(merit_dev_last_error()) : std::string();
  for (void* p : buf)
    if (p) cudaFree(p);
  return st == MERIT_OK ? st : fail(st, msg);
}
