// Drop-in check for include/merit/device.hpp: the reference's own workloads
// (merit::build_template + merit::fill_random, as in the reference's
// tests/test_workloads.cpp) run through the UNMODIFIED reference engine
// merit::run_full and through merit::device::run_full; results must agree
// bit for bit (exact interpreter, max-pool) or within the conv tolerance.
// Built by oracle/build.py against /root/reference/proj/include (this
// container) into oracle/_ref/test_device_header; run by
// tests/test_cpp_dropin.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "merit/device.hpp"
#include "merit/workloads.hpp"

using namespace merit;

static int failures = 0;

static void check(const std::string& name, const Params& prm, uint64_t seed, uint32_t flags = 0) {
  Workload w = build_template(name, prm);
  fill_random(w.src_a, 2 * seed + 1);
  fill_random(w.src_b, 2 * seed + 2);
  if (template_shares_input(name)) w.src_b = w.src_a;
  const Tensor want = run_full(w);
  const int kern = device::lowered_kernel(w, flags);
  const Tensor got = device::run_full(w, flags);
  bool ok = got.shape == want.shape && got.dtype == want.dtype;
  double worst = 0;
  if (ok && got.dtype == Dtype::Fix16) {
    ok = got.qdata == want.qdata;
  } else if (ok) {
    if (kern == MERIT_KERNEL_CONV_TC) {
      for (size_t i = 0; i < got.fdata.size(); ++i)
        worst = std::max(worst, std::abs(double(got.fdata[i]) - want.fdata[i]) / (1.0 + std::abs(want.fdata[i])));
      ok = worst <= 1e-4;
    } else {
      ok = std::memcmp(got.fdata.data(), want.fdata.data(), got.fdata.size() * 4) == 0;
    }
  }
  std::printf("%s %-18s kernel=%d seed=%llu worst=%.3g\n", ok ? "PASS" : "FAIL", name.c_str(), kern,
              (unsigned long long)seed, worst);
  if (!ok) ++failures;
}

int main() {
  SplitMix64 rng{12};
  for (int t = 0; t < 12; ++t) {
    Params prm{{"h", double(rng.range(5, 12))}, {"w", double(rng.range(5, 12))},
               {"k", double(rng.range(1, 3))}, {"stride", double(rng.range(1, 2))},
               {"cin", double(rng.range(1, 2))}, {"cout", double(rng.range(1, 3))}};
    if (t % 3 == 1) prm["fix"] = 1, prm["frac"] = double(rng.range(4, 10));
    check(t % 3 == 2 ? "relu_fused_conv" : "conv2d", prm, 2000 + t);
  }
  check("conv2d", {{"h", 20}, {"w", 20}, {"cin", 16}, {"cout", 32}}, 11);                 // tensor cores
  check("conv2d", {{"h", 17}, {"w", 14}, {"cin", 64}, {"cout", 48}, {"stride", 2}}, 12);  // tensor cores
  check("conv2d", {{"h", 17}, {"w", 14}, {"cin", 64}, {"cout", 48}, {"stride", 2}}, 13, MERIT_FLAG_EXACT);
  check("alexnet_conv1", {{"h", 47}, {"w", 47}}, 14);
  check("gemm", {{"m", 9}, {"n", 7}, {"k", 11}}, 15);
  check("gemm", {{"m", 5}, {"n", 6}, {"k", 7}, {"fix", 1}, {"frac", 6}}, 16);
  check("correlation", {{"c", 3}, {"h", 8}, {"w", 7}, {"d", 3}}, 17);
  check("motion_estimation", {{"h", 16}, {"w", 24}, {"blk", 4}, {"win", 5}}, 18);
  // REAL32 frames holding 8-bit pixels (the reference Tensor's only float
  // type): the header swap reaches the byte-SIMD SAD kernel (K2)
  {
    for (const auto& [blk, win] : {std::pair<int, int>{16, 33}, {8, 65}}) {
      Workload w = build_template("motion_estimation", {{"h", 64}, {"w", 96}, {"blk", double(blk)}, {"win", double(win)}});
      SplitMix64 r{77u + uint64_t(blk)};
      for (float& v : w.src_a.fdata) v = float(r.range(0, 255));
      for (size_t i = 0; i < w.src_b.fdata.size(); ++i) w.src_b.fdata[i] = float(r.range(0, 255));
      const Tensor want = run_full(w);
      const int kern = device::lowered_kernel(w);
      const Tensor got = device::run_full(w);
      const bool ok = kern == MERIT_KERNEL_SAD && got.shape == want.shape &&
                      std::memcmp(got.fdata.data(), want.fdata.data(), got.fdata.size() * 4) == 0;
      std::printf("%s motion_estimation-u8-valued blk=%d kernel=%d\n", ok ? "PASS" : "FAIL", blk, kern);
      if (!ok) ++failures;
    }
  }
  check("motion_estimation", {{"h", 8}, {"w", 8}, {"blk", 4}, {"win", 3}, {"fix", 1}}, 19);
  check("bilateral", {{"h", 9}, {"w", 8}, {"k", 5}}, 20);
  check("maxpool", {{"h", 9}, {"w", 11}, {"k", 3}, {"stride", 2}}, 21);
  check("maxpool", {{"h", 8}, {"w", 8}, {"k", 2}, {"fix", 1}}, 22);
  check("dilated", {{"h", 12}, {"w", 10}, {"k", 3}}, 23);
  // error behaviour: REJECT gather outside the source -> OutOfRange, like the reference
  {
    Workload w = build_template("maxpool", {{"h", 4}, {"w", 4}, {"k", 2}});
    w.view_a.terms[1].offset = -1;
    bool ref_threw = false, dev_threw = false;
    ErrorCode rc{}, dc{};
    try { run_full(w); } catch (const Error& e) { ref_threw = true; rc = e.code; }
    try { device::run_full(w); } catch (const Error& e) { dev_threw = true; dc = e.code; }
    const bool ok = ref_threw && dev_threw && rc == dc;
    std::printf("%s reject-error-code ref=%d dev=%d\n", ok ? "PASS" : "FAIL", int(rc), int(dc));
    if (!ok) ++failures;
  }
  // run_tiled (engine.hpp:289-295): same output as the reference's tiled run
  // and the identical TrafficReport (tests/test_engine.cpp:91-107's KAT plan)
  {
    Workload w = build_template("conv2d", {{"h", 68}, {"w", 68}, {"k", 5}, {"pad", 0}});
    fill_random(w.src_a, 1);
    fill_random(w.src_b, 2);
    TilingPlan plan{{16, 8}, {5, 5}};
    EngineConfig cfg;
    auto [want, wrep] = run_tiled(w, plan, cfg);
    auto [got, grep] = device::run_tiled(w, plan, cfg);
    double worst = 0;
    for (size_t i = 0; i < got.fdata.size(); ++i)
      worst = std::max(worst, std::abs(double(got.fdata[i]) - want.fdata[i]) / (1.0 + std::abs(want.fdata[i])));
    const bool same = wrep.dram_read_words_a == grep.dram_read_words_a &&
                      wrep.dram_read_words_b == grep.dram_read_words_b &&
                      wrep.dram_write_words == grep.dram_write_words &&
                      wrep.scratchpad_peak_words_a == grep.scratchpad_peak_words_a &&
                      wrep.scratchpad_peak_words_b == grep.scratchpad_peak_words_b &&
                      wrep.passes == grep.passes && wrep.macs == grep.macs;
    const bool ok = same && got.shape == want.shape && worst <= 1e-4 && grep.scratchpad_peak_words_a == 240;
    std::printf("%s run_tiled conv2d 5x5 plan {16,8}x{5,5}: peak_a=%llu passes=%llu worst=%.3g\n",
                ok ? "PASS" : "FAIL", (unsigned long long)grep.scratchpad_peak_words_a,
                (unsigned long long)grep.passes, worst);
    if (!ok) ++failures;
    // measured counterpart (GPU counters): the device reads the image once,
    // the reference's plan charges every tile its 20 x 12 footprint box
    // (on a 516 x 516 image: below ~1 MB the counters' fixed noise dominates)
    Workload big = build_template("conv2d", {{"h", 516}, {"w", 516}, {"k", 5}, {"pad", 0}});
    fill_random(big.src_a, 3);
    fill_random(big.src_b, 4);
    auto [bout, brep] = run_tiled(big, plan, cfg);
    (void)bout;
    try {
      const merit_measured_traffic m = device::measure_traffic(big);
      const double words = m.dram_read_bytes / 4.0;
      const bool okm = m.ranges == 1 && words < double(brep.dram_read_words_a) && words >= 0.85 * double(big.src_a.size());
      std::printf("%s measured DRAM read words %.0f vs reference tiled count %llu (image %zu words)\n",
                  okm ? "PASS" : "FAIL", words, (unsigned long long)brep.dram_read_words_a, big.src_a.size());
      if (!okm) ++failures;
    } catch (const Error& e) {
      // a host that refuses a CUPTI profiling session has nothing to measure
      // (merit_dev.h: fixed message prefix); anything else is a failure
      const bool refused = std::string(e.what()).find("measure_traffic unavailable on this system") != std::string::npos;
      std::printf("%s measured DRAM traffic: %s\n", refused ? "SKIP" : "FAIL", e.what());
      if (!refused) ++failures;
    }
    // an invalid plan fails with the reference's error code
    TilingPlan bad{{16, 8}, {5, 4}};
    bool rt = false, dt = false;
    ErrorCode rc{}, dc{};
    try { run_tiled(w, bad, cfg); } catch (const Error& e) { rt = true; rc = e.code; }
    try { device::run_tiled(w, bad, cfg); } catch (const Error& e) { dt = true; dc = e.code; }
    const bool ok2 = rt && dt && rc == dc;
    std::printf("%s run_tiled-bad-plan ref=%d dev=%d\n", ok2 ? "PASS" : "FAIL", int(rc), int(dc));
    if (!ok2) ++failures;
  }
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
