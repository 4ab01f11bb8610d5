// merit_dev_tiled_traffic: the reference's run_tiled TrafficReport
// (engine.hpp:72-80 and the pass loop of run_tiled_typed, :189-278) computed
// in closed form for the device path's run_tiled.
//
// run_tiled charges every pass (p-tile x a-tile) the Eq. 6 footprint box of
// each view for that pass's tile extents (footprint(), view.hpp:121-133);
// the box size depends only on the extents, which along each dimension are
// either the plan extent (full tiles) or the remainder (the last tile).  So
// the sums run over at most 2^(p_rank + a_rank) extent combinations weighted
// by how many passes have them, instead of over the passes themselves.
#include <algorithm>
#include <string>
#include <vector>

#include "plan.hpp"

namespace merit_dev {
namespace {

// Eq. 6 box words of one view for a tile with the given k extents.
bool box_words(const merit_view_spec& v, const std::vector<int64_t>& tile, uint64_t& words) {
  int64_t ext[MERIT_MAX_RANK];
  for (int i = 0; i < v.src_rank; ++i) ext[i] = 1;
  for (int t = 0; t < v.n_terms; ++t) {
    const merit_view_term& term = v.terms[t];
    if (term.stride < 0) return false;
    ext[term.axis] += (tile[term.component] - 1) * term.stride;
  }
  uint64_t w = 1;
  for (int i = 0; i < v.src_rank; ++i) w *= static_cast<uint64_t>(ext[i]);
  words = w;
  return true;
}

}  // namespace
}  // namespace merit_dev

extern "C" merit_status merit_dev_tiled_traffic(const merit_plan* plan, const int64_t* t_p, const int64_t* t_a,
                                                merit_traffic_report* report) {
  using namespace merit_dev;
  if (!plan || !t_p || !t_a || !report) return fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  if (!plan->members.empty()) return fail(MERIT_E_INVALID_ARGUMENT, "run_tiled takes a single-workload plan");
  const merit_view_spec& va = plan->desc.view_a;
  const merit_view_spec& vb = plan->desc.view_b;
  const int pr = va.p_rank, ar = va.a_rank;
  // TilingPlan::validate (engine.hpp:50-63)
  for (int i = 0; i < pr; ++i)
    if (t_p[i] < 1 || t_p[i] > va.p_shape[i]) return fail(MERIT_E_BAD_PARAMS, "p tile extent out of range");
  for (int i = 0; i < ar; ++i)
    if (t_a[i] < 1 || t_a[i] > va.a_shape[i]) return fail(MERIT_E_BAD_PARAMS, "a tile extent out of range");
  for (int i = 1; i < ar; ++i)
    if (t_a[i] != va.a_shape[i]) return fail(MERIT_E_BAD_PARAMS, "only the outermost a dimension may be tiled");
  // per k dimension: (extent, number of tiles with it) for full and last tiles
  const int kr = pr + ar;
  std::vector<int64_t> full_ext(kr), full_cnt(kr), rem_ext(kr), rem_cnt(kr);
  uint64_t p_vol = 1, a_vol = 1;
  for (int i = 0; i < kr; ++i) {
    const int64_t n = i < pr ? va.p_shape[i] : va.a_shape[i - pr];
    const int64_t t = i < pr ? t_p[i] : t_a[i - pr];
    full_ext[i] = t;
    full_cnt[i] = n / t;
    rem_ext[i] = n % t;
    rem_cnt[i] = rem_ext[i] ? 1 : 0;
    (i < pr ? p_vol : a_vol) *= static_cast<uint64_t>(n);
  }
  merit_traffic_report r{};
  std::vector<int64_t> tile(kr);
  for (uint32_t mask = 0; mask < (1u << kr); ++mask) {  // bit i: dimension i takes the last (partial) tile
    uint64_t count = 1;
    for (int i = 0; i < kr && count; ++i) {
      const bool last = (mask >> i) & 1u;
      count *= static_cast<uint64_t>(last ? rem_cnt[i] : full_cnt[i]);
      tile[i] = last ? rem_ext[i] : full_ext[i];
    }
    if (!count) continue;
    uint64_t wa = 0, wb = 0;
    if (!box_words(va, tile, wa) || !box_words(vb, tile, wb))
      return fail(MERIT_E_NEGATIVE_STRIDE, "footprint undefined for negative strides");
    r.dram_read_words_a += wa * count;
    r.dram_read_words_b += wb * count;
    r.scratchpad_peak_words_a = std::max(r.scratchpad_peak_words_a, wa);
    r.scratchpad_peak_words_b = std::max(r.scratchpad_peak_words_b, wb);
    r.passes += count;
  }
  r.macs = p_vol * a_vol;
  r.dram_write_words = p_vol * static_cast<uint64_t>(plan->desc.program.outputs);
  *report = r;
  return MERIT_OK;
}
