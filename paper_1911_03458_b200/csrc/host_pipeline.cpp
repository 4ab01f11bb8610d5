// Pipelined host-buffer runs (merit_dev_run_host).
//
// The reference's calling convention hands the engine host tensors and takes
// a host tensor back (engine.hpp:282-287).  On the device side that is
// H2D -> kernel -> D2H, and for every config here the PCIe transfers dominate
// (C2: 39 MB moved against a 55 us kernel).  PCIe is full duplex, so the run
// is cut along the outermost independent axis of the plan into slices:
//   max-pool  -> planes (the N*C leading extents),
//   conv      -> images (N, NCHW layouts only),
//   SAD       -> frame pairs, or block-row bands of a single pair (the
//                reference window of a band reaches into its neighbours'
//                rows; the band kernel reads the whole frame and zero-pads
//                only at the true frame edges, SadParams::by_begin/by_count),
// and slice k's H2D (stream 0), kernel (the caller's stream) and D2H
// (stream 1) are chained with events, so the D2H of slice k overlaps the H2D
// and kernel of slice k+1.  Every slice's kernel is the plan's own kernel on
// a sub-range; results are identical to the single-shot run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "plan.hpp"

namespace merit_dev {

namespace {

// Slice count: one per ~6 MB of transfers, at most 16, at most one per unit
// (measured: every slice costs ~8 us of copy-engine gaps, so a few large
// slices beat many small ones).  MERIT_HOST_CHUNKS=n forces n (1 = the
// unpipelined path).
int64_t slice_count(const merit_plan& plan, int64_t units) {
  const merit_plan_info& in = plan.info;
  const int64_t total = in.src_a_bytes + in.src_b_bytes + in.out_bytes + in.aux_elems * 4;
  int64_t k = std::max<int64_t>(1, std::min<int64_t>(16, total / (6 << 20)));
  if (const char* e = getenv("MERIT_HOST_CHUNKS")) k = std::max(1, atoi(e));
  return std::min(k, units);
}

merit_plan* clone_params(const merit_plan& p) {
  merit_plan* s = new merit_plan();
  s->kernel = p.kernel;
  s->info = p.info;
  s->mp = p.mp;
  s->sad = p.sad;
  s->conv = p.conv;
  s->conv_swapped = p.conv_swapped;
  return s;
}

// Units [u0, u1) of slice i of k over n units, triangular weights
// 1, 2, .., m, .., 2, 1: the first slice (whose H2D + kernel precede every
// D2H) and the last one (whose kernel + D2H follow every H2D) are the
// smallest, so the pipeline fills and drains in a fraction of a uniform
// slice.  MERIT_HOST_RAMP=0 gives uniform slices.
int64_t ramp_weight_sum(int64_t k, int64_t i) {  // sum of the first i weights
  static const int ramp = [] {
    const char* e = getenv("MERIT_HOST_RAMP");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  if (!ramp) return i;
  int64_t s = 0;
  for (int64_t j = 0; j < i; ++j) s += std::min(j + 1, k - j);
  return s;
}
void split(int64_t n, int64_t k, int64_t i, int64_t& u0, int64_t& u1) {
  const int64_t tot = ramp_weight_sum(k, k);
  if (n < tot) {  // too few units for the ramp: uniform (no empty slices)
    u0 = n * i / k;
    u1 = n * (i + 1) / k;
    return;
  }
  u0 = n * ramp_weight_sum(k, i) / tot;
  u1 = n * ramp_weight_sum(k, i + 1) / tot;
}

}  // namespace

void build_slices(const merit_plan& plan) {
  plan.slices_built = true;
  const merit_plan_info& in = plan.info;
  const int64_t out_b = in.out_bytes, aux_b = in.aux_elems * 4;
  std::vector<HostSlice> v;
  if (plan.kernel == MERIT_KERNEL_MAXPOOL) {
    const int64_t n = plan.mp.planes;
    if (n < 2 || in.src_a_bytes % n || out_b % n) return;
    const int64_t k = slice_count(plan, n);
    const int64_t au = in.src_a_bytes / n, ou = out_b / n;
    for (int64_t i = 0; i < k; ++i) {
      int64_t u0, u1;
      split(n, k, i, u0, u1);
      if (u1 == u0) continue;
      HostSlice s;
      s.sub = clone_params(plan);
      s.sub->mp.planes = u1 - u0;
      s.a_off = u0 * au;
      s.a_need = u1 * au;
      s.b_need = in.src_b_bytes;  // port B is not read; copied with the first slice
      s.out_off = s.out_lo = u0 * ou;
      s.out_hi = u1 * ou;
      v.push_back(s);
    }
  } else if (plan.kernel == MERIT_KERNEL_CONV_TC) {
    const ConvParams& c = plan.conv;
    const int64_t n = c.N;
    const int64_t esz = c.in_bf16 ? 2 : 4;
    const int64_t in_bytes = plan.conv_swapped ? in.src_b_bytes : in.src_a_bytes;
    const int64_t w_bytes = plan.conv_swapped ? in.src_a_bytes : in.src_b_bytes;
    if (c.gemm || n < 2 || c.a_sn != (int64_t)c.Cin * c.H * c.W || in_bytes != n * c.a_sn * esz ||
        c.o_sn != (int64_t)c.Cout * c.Ho * c.Wo || out_b % n)
      return;
    const int64_t k = slice_count(plan, n);
    const int64_t iu = c.a_sn * esz, ou = out_b / n;
    for (int64_t i = 0; i < k; ++i) {
      int64_t u0, u1;
      split(n, k, i, u0, u1);
      if (u1 == u0) continue;
      HostSlice s;
      s.sub = clone_params(plan);
      s.sub->conv.N = static_cast<int32_t>(u1 - u0);
      s.sub->conv.npix = (u1 - u0) * c.Ho * c.Wo;
      (plan.conv_swapped ? s.b_off : s.a_off) = u0 * iu;
      (plan.conv_swapped ? s.b_need : s.a_need) = u1 * iu;
      (plan.conv_swapped ? s.a_need : s.b_need) = w_bytes;  // weights with the first slice
      s.out_off = s.out_lo = u0 * ou;
      s.out_hi = u1 * ou;
      v.push_back(s);
    }
  } else if (plan.kernel == MERIT_KERNEL_SAD && !plan.sad.narrow) {  // narrowed plans run unsliced
    const SadParams& q = plan.sad;
    const int64_t cur_bytes = q.ref_is_b ? in.src_a_bytes : in.src_b_bytes;
    const int64_t ref_bytes = q.ref_is_b ? in.src_b_bytes : in.src_a_bytes;
    if (q.pairs >= 2) {
      const int64_t n = q.pairs;
      // fused plans: the fine level's records at fused_aux_off, the coarse
      // level's at fused_aux_off + aux2_delta (int32 elements), per pair each
      const int64_t x8 = q.fuse2 ? 12 * (int64_t)q.BY * q.BX : 0, x16 = q.fuse2 ? 12 * (int64_t)q.BY2 * q.BX2 : 0;
      if (cur_bytes % n || ref_bytes % n || out_b % n || (!q.fuse2 && aux_b % n)) return;
      if (q.fuse2 && aux_b != n * (x8 + x16)) return;
      const int64_t k = slice_count(plan, n);
      const int64_t cu = cur_bytes / n, ru = ref_bytes / n, ou = out_b / n, xu = q.fuse2 ? x8 : aux_b / n;
      const int64_t base8 = q.fuse2 ? 4 * plan.fused_aux_off : 0, base16 = q.fuse2 ? base8 + 4 * q.aux2_delta : 0;
      for (int64_t i = 0; i < k; ++i) {
        int64_t u0, u1;
        split(n, k, i, u0, u1);
        if (u1 == u0) continue;
        HostSlice s;
        s.sub = clone_params(plan);
        s.sub->sad.pairs = u1 - u0;
        (q.ref_is_b ? s.a_off : s.b_off) = u0 * cu;
        (q.ref_is_b ? s.b_off : s.a_off) = u0 * ru;
        (q.ref_is_b ? s.a_need : s.b_need) = u1 * cu;
        (q.ref_is_b ? s.b_need : s.a_need) = u1 * ru;
        s.out_off = s.out_lo = u0 * ou;
        s.out_hi = u1 * ou;
        s.aux_off = s.aux_lo = base8 + u0 * xu;
        s.aux_hi = base8 + u1 * xu;
        if (q.fuse2) {
          s.aux2_lo = base16 + u0 * x16;
          s.aux2_hi = base16 + u1 * x16;
          s.sub->sad.aux2_delta = (s.aux2_lo - s.aux_lo) / 4;
        }
        v.push_back(s);
      }
    } else {
      // block-row bands of the single pair; pointers are not offset (the
      // kernel writes global block indices)
      if (q.fuse2) return;  // a fused single pair runs unsliced
      const int64_t n = q.BY;
      if (n < 2 || cur_bytes % q.Hc || ref_bytes % q.Hr || out_b % n || aux_b % n) return;
      const int64_t k = slice_count(plan, n);
      const int64_t crow = cur_bytes / q.Hc, rrow = ref_bytes / q.Hr, ou = out_b / n, xu = aux_b / n;
      for (int64_t i = 0; i < k; ++i) {
        int64_t u0, u1;
        split(n, k, i, u0, u1);
        if (u1 == u0) continue;
        HostSlice s;
        s.sub = clone_params(plan);
        s.sub->sad.by_begin = static_cast<int32_t>(u0);
        s.sub->sad.by_count = static_cast<int32_t>(u1 - u0);
        // rows the band's tiles stage (one block row of margin for the
        // staged-window overshoot and 8x8 two-row tiles)
        const int64_t cur_rows = std::min<int64_t>(q.Hc, (u1 + 1) * q.BH + q.cy);
        const int64_t ref_rows = std::min<int64_t>(q.Hr, (u1 + 1) * q.BH + q.oy + q.WY + q.BH);
        (q.ref_is_b ? s.a_need : s.b_need) = std::max<int64_t>(0, cur_rows) * crow;
        (q.ref_is_b ? s.b_need : s.a_need) = std::max<int64_t>(0, ref_rows) * rrow;
        s.out_lo = u0 * ou;
        s.out_hi = u1 * ou;
        s.aux_lo = u0 * xu;
        s.aux_hi = u1 * xu;
        v.push_back(s);
      }
    }
  }
  if (v.size() < 2) {
    for (HostSlice& s : v) delete s.sub;
    return;
  }
  // the last slice needs every source byte (covers rounding in the row margins)
  v.back().a_need = in.src_a_bytes;
  v.back().b_need = in.src_b_bytes;
  plan.slices = std::move(v);
}

namespace {

merit_status launch_slice(const merit_plan& sub, const void* a, const void* b, void* out, void* aux,
                          void* stream) {
  switch (sub.kernel) {
    case MERIT_KERNEL_MAXPOOL: return launch_maxpool(sub, a, out, stream);
    case MERIT_KERNEL_SAD: return launch_sad(sub, a, b, out, aux, stream);
    case MERIT_KERNEL_CONV_TC: return launch_conv(sub, sub.conv_swapped ? b : a, sub.d_packed_b, out, stream);
    default: return fail(MERIT_E_INVALID_ARGUMENT, "plan kind does not slice");
  }
}

bool in_out_missing(const merit_plan& plan, const void* h_out, const void* h_aux) {
  return (plan.info.out_bytes > 0 && !h_out) || (plan.info.aux_elems > 0 && !h_aux);
}

}  // namespace

void release_host_pipeline(const merit_plan& plan) {
  for (void*& e : plan.copy_events)
    if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  plan.copy_events.clear();
  for (void*& s : plan.copy_stream) {
    if (s) cudaStreamDestroy(static_cast<cudaStream_t>(s));
    s = nullptr;
  }
}

merit_status run_host_pipelined(const merit_plan& plan, void* da, void* db, void* dout, void* daux,
                                const void* h_a, const void* h_b, void* h_out, void* h_aux, bool need_b,
                                void* stream) {
  if (!plan.slices_built) build_slices(plan);
  if (plan.slices.empty()) return MERIT_E_UNSUPPORTED_VIEW;
  // anything the single-shot path would reject is left to it (same errors)
  if (!da || !h_a || (plan.kernel == MERIT_KERNEL_SAD && (!db || !need_b))) return MERIT_E_UNSUPPORTED_VIEW;
  if (plan.kernel == MERIT_KERNEL_CONV_TC && !plan.packed_valid && !plan.conv_swapped && !need_b)
    return MERIT_E_UNSUPPORTED_VIEW;
  if ((in_out_missing(plan, h_out, h_aux))) return MERIT_E_UNSUPPORTED_VIEW;
  merit_status st = ensure_device_state(plan);
  if (st != MERIT_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t k = plan.slices.size();
  // weights packed on the fly: hold the plan's pack lock for the whole run
  // (it drains its streams before returning) and wait for earlier readers
  const bool packs = plan.kernel == MERIT_KERNEL_CONV_TC && !plan.packed_valid;
  std::unique_lock<std::mutex> pack_lock(plan.pack_mu, std::defer_lock);
  if (packs) {
    pack_lock.lock();
    if ((st = pack_wait(plan, stream)) != MERIT_OK) return st;
  }
  for (void*& cs : plan.copy_stream)
    if (!cs) {
      cudaStream_t t;
      if ((st = cuda_check(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking), "cudaStreamCreate")) != MERIT_OK)
        return st;
      cs = t;
    }
  while (plan.copy_events.size() < 2 * k + 2) {
    cudaEvent_t e;
    if ((st = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate")) != MERIT_OK)
      return st;
    plan.copy_events.push_back(e);
  }
  cudaStream_t h2d = static_cast<cudaStream_t>(plan.copy_stream[0]);
  cudaStream_t d2h = static_cast<cudaStream_t>(plan.copy_stream[1]);
  auto ev = [&](size_t i) { return static_cast<cudaEvent_t>(plan.copy_events[i]); };
  auto* ha = static_cast<const char*>(h_a);
  auto* hb = static_cast<const char*>(h_b);
  auto* ca = static_cast<char*>(da);
  auto* cb = static_cast<char*>(db);
  auto* co = static_cast<char*>(dout);
  auto* cx = static_cast<char*>(daux);
  auto* ho = static_cast<char*>(h_out);
  auto* hx = static_cast<char*>(h_aux);
  const merit_plan_info& in = plan.info;
  // caller's prior work on `stream` before our first H2D (it may produce the host inputs)
  cudaError_t e = cudaEventRecord(ev(0), s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h2d, ev(0), 0);
  int64_t a_done = 0, b_done = 0;
  for (size_t i = 0; i < k && e == cudaSuccess && st == MERIT_OK; ++i) {
    const HostSlice& sl = plan.slices[i];
    const int64_t a_need = std::min<int64_t>(sl.a_need, in.src_a_bytes);
    const int64_t b_need = need_b ? std::min<int64_t>(sl.b_need, in.src_b_bytes) : 0;
    if (a_need > a_done && e == cudaSuccess) {
      e = cudaMemcpyAsync(ca + a_done, ha + a_done, a_need - a_done, cudaMemcpyHostToDevice, h2d);
      a_done = a_need;
    }
    if (b_need > b_done && e == cudaSuccess) {
      e = cudaMemcpyAsync(cb + b_done, hb + b_done, b_need - b_done, cudaMemcpyHostToDevice, h2d);
      b_done = b_need;
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev(2 + 2 * i), h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev(2 + 2 * i), 0);
    if (e != cudaSuccess) break;
    if (i == 0 && plan.kernel == MERIT_KERNEL_CONV_TC && !plan.packed_valid) {
      st = launch_conv_pack(plan, plan.conv_swapped ? da : db, plan.d_packed_b, stream);
      if (st != MERIT_OK) break;
    }
    sl.sub->d_packed_b = plan.d_packed_b;
    st = launch_slice(*sl.sub, ca ? ca + sl.a_off : nullptr, cb ? cb + sl.b_off : nullptr,
                      co ? co + sl.out_off : nullptr, cx ? cx + sl.aux_off : nullptr, stream);
    if (st != MERIT_OK) break;
    e = cudaEventRecord(ev(3 + 2 * i), s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, ev(3 + 2 * i), 0);
    if (e == cudaSuccess && in.out_bytes > 0 && sl.out_hi > sl.out_lo)
      e = cudaMemcpyAsync(ho + sl.out_lo, co + sl.out_lo, sl.out_hi - sl.out_lo, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess && in.aux_elems > 0 && sl.aux_hi > sl.aux_lo)
      e = cudaMemcpyAsync(hx + sl.aux_lo, cx + sl.aux_lo, sl.aux_hi - sl.aux_lo, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess && in.aux_elems > 0 && sl.aux2_hi > sl.aux2_lo)
      e = cudaMemcpyAsync(hx + sl.aux2_lo, cx + sl.aux2_lo, sl.aux2_hi - sl.aux2_lo, cudaMemcpyDeviceToHost, d2h);
  }
  if (e == cudaSuccess && st == MERIT_OK) e = cudaEventRecord(ev(1), d2h);
  if (e == cudaSuccess && st == MERIT_OK) e = cudaStreamWaitEvent(s, ev(1), 0);
  // drain all three streams before returning (success or not)
  const std::string msg = st != MERIT_OK ? std::string(merit_dev_last_error()) : std::string();
  cudaStreamSynchronize(h2d);
  cudaStreamSynchronize(d2h);
  const cudaError_t se = cudaStreamSynchronize(s);
  if (st != MERIT_OK) return fail(st, msg);
  if (e != cudaSuccess) return cuda_check(e, "pipelined host run");
  return cuda_check(se, "cudaStreamSynchronize");
}

}  // namespace merit_dev

extern "C" merit_status merit_dev_plan_slices(const merit_plan* plan, merit_host_slice* out, int64_t cap,
                                              int64_t* n_slices) {
  if (!plan || !n_slices || (cap > 0 && !out)) return merit_dev::fail(MERIT_E_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(plan->host_mu);
  if (!plan->slices_built) merit_dev::build_slices(*plan);
  *n_slices = static_cast<int64_t>(plan->slices.size());
  for (int64_t i = 0; i < cap && i < *n_slices; ++i) {
    const merit_dev::HostSlice& s = plan->slices[i];
    out[i] = {std::min<int64_t>(s.a_need, plan->info.src_a_bytes), std::min<int64_t>(s.b_need, plan->info.src_b_bytes),
              s.out_lo, s.out_hi, s.aux_lo, s.aux_hi, s.aux2_lo, s.aux2_hi};
  }
  return MERIT_OK;
}

merit_plan::~merit_plan() {
  for (merit_dev::HostSlice& s : slices) delete s.sub;
  for (merit_plan* m : members) merit_dev_plan_destroy(m);
}
