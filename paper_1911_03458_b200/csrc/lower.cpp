// Validation and lowering of a MERIT workload descriptor to a device plan.
//
// Mirrors Workload::validate (engine.hpp:30-38) and StrategyProgram::validate
// (rip.hpp:96-106), then pattern-matches the program skeleton
// (workloads.hpp:47-68 mac/sad programs, :376-385 max-pool program) and the
// affine structure of the two ViewSpecs (view.hpp:24-49, Eq. 5) to pick a
// specialised kernel.  Anything that is not recognised goes to the exact
// generic interpreter (still a device kernel — there is no CPU path), unless
// a dtype makes that impossible, in which case plan creation fails.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "plan.hpp"

namespace merit_dev {
namespace {

int64_t vol(const int64_t* s, int n) {
  int64_t v = 1;
  for (int i = 0; i < n; ++i) v *= s[i];
  return v;
}

bool same_shape(const int64_t* a, int na, const int64_t* b, int nb) {
  if (na != nb) return false;
  for (int i = 0; i < na; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

merit_status check_view(const merit_view_spec& v, const char* name) {
  if (v.src_rank < 1 || v.src_rank > kMaxRank || v.p_rank < 0 || v.p_rank > kMaxRank ||
      v.a_rank < 0 || v.a_rank > kMaxRank || v.n_terms < 0 || v.n_terms > MERIT_MAX_TERMS)
    return fail(MERIT_E_INVALID_ARGUMENT, std::string(name) + ": rank or term count out of range");
  for (int i = 0; i < v.src_rank; ++i)
    if (v.src_shape[i] < 1)
      return fail(MERIT_E_BAD_PARAMS, std::string(name) + ": extents must be >= 1");
  if (v.boundary < MERIT_ZERO_PAD || v.boundary > MERIT_REJECT)
    return fail(MERIT_E_INVALID_ARGUMENT, std::string(name) + ": bad boundary");
  const int kr = v.p_rank + v.a_rank;
  for (int t = 0; t < v.n_terms; ++t) {
    const auto& tm = v.terms[t];
    // The reference indexes x[t.axis] / k[t.component] unchecked
    // (view.hpp:37-42); validate_spec (view.hpp:156-175) reports these as
    // AXIS_OUT_OF_RANGE / COMPONENT_OUT_OF_RANGE.  Reject them here.
    if (tm.axis < 0 || tm.axis >= v.src_rank)
      return fail(MERIT_E_BAD_PARAMS, std::string(name) + ": term axis out of range");
    if (tm.component < 0 || tm.component >= kr)
      return fail(MERIT_E_BAD_PARAMS, std::string(name) + ": term component out of range");
  }
  return MERIT_OK;
}

void affine_of(const merit_view_spec& v, ViewAffine& f) {
  std::memset(&f, 0, sizeof(f));
  f.src_rank = v.src_rank;
  f.k_rank = v.p_rank + v.a_rank;
  f.boundary = v.boundary;
  for (int i = 0; i < v.src_rank; ++i) f.src_shape[i] = v.src_shape[i];
  for (int t = 0; t < v.n_terms; ++t) {
    const auto& tm = v.terms[t];
    f.coef[tm.axis][tm.component] += tm.stride;
    f.off[tm.axis] += tm.offset;
  }
}

// Interval of source axis i over the whole (p, a) index box.
void axis_range(const ViewAffine& f, const int64_t* kshape, int i, int64_t& lo, int64_t& hi) {
  lo = hi = f.off[i];
  for (int j = 0; j < f.k_rank; ++j) {
    int64_t c = f.coef[i][j] * (kshape[j] - 1);
    if (c < 0) lo += c; else hi += c;
  }
}

bool view_in_range(const ViewAffine& f, const int64_t* kshape) {
  for (int i = 0; i < f.src_rank; ++i) {
    int64_t lo, hi;
    axis_range(f, kshape, i, lo, hi);
    if (lo < 0 || hi >= f.src_shape[i]) return false;
  }
  return true;
}

// ---------------------------------------------------------------- program --
struct Seg {
  const merit_alu_instr* ins;
  int n;
};

bool opnd(const merit_alu_instr& in, char which, int kind, int reg = -1) {
  int k = which == 'a' ? in.a_kind : which == 'b' ? in.b_kind : in.c_kind;
  int r = which == 'a' ? in.a_reg : which == 'b' ? in.b_reg : in.c_reg;
  if (k != kind) return false;
  if (kind == MERIT_OPND_REG && reg >= 0 && r != reg) return false;
  return true;
}

// Pre_1 = r <- 0 (ADD of zeros, workloads.hpp:51-53).
bool is_clear(const merit_alu_instr& in, int& reg) {
  if (in.op != MERIT_OP_ADD || in.dst_out) return false;
  if (!opnd(in, 'a', MERIT_OPND_ZERO) || !opnd(in, 'b', MERIT_OPND_ZERO) ||
      !opnd(in, 'c', MERIT_OPND_ZERO))
    return false;
  reg = in.dst_reg;
  return true;
}

// Post_1 = emit r (+0.0f) or emit max(r, 0) (relu_fused_conv, workloads.hpp:197-202).
bool is_emit(const merit_alu_instr& in, int reg, int32_t& post) {
  if (!in.dst_out) return false;
  if (in.op == MERIT_OP_ADD && opnd(in, 'a', MERIT_OPND_REG, reg) &&
      opnd(in, 'b', MERIT_OPND_ZERO) && opnd(in, 'c', MERIT_OPND_ZERO)) {
    post = POST_ADD_ZERO;
    return true;
  }
  if (in.op == MERIT_OP_MAX && opnd(in, 'a', MERIT_OPND_REG, reg) &&
      opnd(in, 'b', MERIT_OPND_ZERO)) {
    post = POST_RELU;
    return true;
  }
  return false;
}

enum Skeleton { SK_NONE, SK_MAC, SK_L1, SK_MAX };

// Recognise the three reduction skeletons.  Only Pre_1, Body and Post_1 may
// be non-empty; everything else is the generic interpreter's business.
Skeleton classify(const merit_workload_desc& d, const ProgramImage& pi, int32_t& post,
                  float& init) {
  const int D = pi.depth;
  auto seg = [&](int s) { return Seg{pi.instrs + pi.seg_start[s], pi.seg_len[s]}; };
  for (int s = 0; s < pi.n_segments; ++s) {
    if (s == 0 || s == D || s == 2 * D) continue;
    if (pi.seg_len[s] != 0) return SK_NONE;
  }
  if (D < 1 || pi.outputs != 1) return SK_NONE;
  Seg pre = seg(0), body = seg(D), postS = seg(2 * D);
  if (pre.n != 1 || body.n != 1 || postS.n != 1) return SK_NONE;
  const merit_alu_instr& b = body.ins[0];
  if (b.dst_out) return SK_NONE;
  const int r = b.dst_reg;
  if (!is_emit(postS.ins[0], r, post)) return SK_NONE;
  int creg = -1;
  if (b.op == MERIT_OP_MAC || b.op == MERIT_OP_L1) {
    if (!is_clear(pre.ins[0], creg) || creg != r) return SK_NONE;
    if (b.shift != 0 || !opnd(b, 'a', MERIT_OPND_REG, r)) return SK_NONE;
    bool ab = opnd(b, 'b', MERIT_OPND_PORT_A) && opnd(b, 'c', MERIT_OPND_PORT_B);
    bool ba = opnd(b, 'b', MERIT_OPND_PORT_B) && opnd(b, 'c', MERIT_OPND_PORT_A);
    if (!ab && !ba) return SK_NONE;
    return b.op == MERIT_OP_MAC ? SK_MAC : SK_L1;
  }
  if (b.op == MERIT_OP_MAX) {
    const merit_alu_instr& p = pre.ins[0];
    if (p.op != MERIT_OP_MOVC || p.dst_out || p.dst_reg != r) return SK_NONE;
    if (p.aux < 0 || p.aux >= pi.n_constants) return SK_NONE;
    // MAX r <- max(r, A): a = r, b = port A (std::max(a, b), rip.hpp:175-176).
    if (!opnd(b, 'a', MERIT_OPND_REG, r) || !opnd(b, 'b', MERIT_OPND_PORT_A)) return SK_NONE;
    if (post != POST_ADD_ZERO) return SK_NONE;
    init = static_cast<float>(pi.constants[p.aux]);
    (void)d;
    return SK_MAX;
  }
  return SK_NONE;
}

bool program_uses_port(const ProgramImage& pi, int port) {
  for (int i = 0; i < pi.n_instrs; ++i) {
    const auto& in = pi.instrs[i];
    if (in.a_kind == port || in.b_kind == port || in.c_kind == port) return true;
  }
  return false;
}

// ------------------------------------------------------------ view shapes --
// Does source axis i of view f equal exactly one component `c` with stride s
// and no other component?
bool axis_single(const ViewAffine& f, int i, int c, int64_t s) {
  for (int j = 0; j < f.k_rank; ++j)
    if (f.coef[i][j] != (j == c ? s : 0)) return false;
  return true;
}

// Components with nonzero coefficient on axis i.
int axis_comps(const ViewAffine& f, int i, int* comps) {
  int n = 0;
  for (int j = 0; j < f.k_rank; ++j)
    if (f.coef[i][j] != 0) comps[n++] = j;
  return n;
}

bool comp_unused(const ViewAffine& f, int c) {
  for (int i = 0; i < f.src_rank; ++i)
    if (f.coef[i][c] != 0) return false;
  return true;
}

// ---------------------------------------------------------------- maxpool --
bool lower_maxpool(const merit_workload_desc& d, const ViewAffine& va, const ViewAffine& vb, float init,
                   int32_t post, MaxpoolParams& mp) {
  const merit_view_spec& v = d.view_a;
  if (d.dtype_a != MERIT_F32 || d.dtype_out != MERIT_F32) return false;
  const int R = v.src_rank, P = v.p_rank;
  if (R < 2 || P != R || v.a_rank != 2) return false;
  // Leading axes: one p component each, stride 1, no offset.
  for (int i = 0; i < R - 2; ++i) {
    if (!axis_single(va, i, i, 1) || va.off[i] != 0) return false;
    if (v.p_shape[i] != v.src_shape[i]) return false;
  }
  const int cy = P - 2, cx = P - 1, ky = P, kx = P + 1;
  int comps[kMaxK];
  if (axis_comps(va, R - 2, comps) != 2 || comps[0] != cy || comps[1] != ky) return false;
  if (axis_comps(va, R - 1, comps) != 2 || comps[0] != cx || comps[1] != kx) return false;
  const int64_t sy = va.coef[R - 2][cy], dy = va.coef[R - 2][ky];
  const int64_t sx = va.coef[R - 1][cx], dx = va.coef[R - 1][kx];
  if (sy < 1 || sx < 1 || dy < 1 || dx < 1) return false;
  int64_t kshape[kMaxK];
  for (int j = 0; j < P; ++j) kshape[j] = v.p_shape[j];
  kshape[P] = v.a_shape[0];
  kshape[P + 1] = v.a_shape[1];
  if (v.boundary == MERIT_REJECT && !view_in_range(va, kshape)) return false;  // error path
  // run_full gathers port B at every step even though the max program never
  // reads it (engine.hpp:128-133): an out-of-range REJECT view_b must raise
  // OutOfRange, so it goes to the interpreter's error path
  if (d.view_b.boundary == MERIT_REJECT && !view_in_range(vb, kshape)) return false;
  const int64_t H = v.src_shape[R - 2], W = v.src_shape[R - 1];
  if (H > (1 << 30) || W > (1 << 30)) return false;
  mp.planes = 1;
  for (int i = 0; i < R - 2; ++i) mp.planes *= v.src_shape[i];
  mp.H = (int32_t)H; mp.W = (int32_t)W;
  mp.Ho = (int32_t)v.p_shape[cy]; mp.Wo = (int32_t)v.p_shape[cx];
  mp.KH = (int32_t)v.a_shape[0]; mp.KW = (int32_t)v.a_shape[1];
  mp.sy = (int32_t)sy; mp.sx = (int32_t)sx; mp.dy = (int32_t)dy; mp.dx = (int32_t)dx;
  mp.oy = (int32_t)va.off[R - 2]; mp.ox = (int32_t)va.off[R - 1];
  // REJECT in range behaves like CLAMP (no clamping ever happens).
  mp.boundary = v.boundary == MERIT_ZERO_PAD ? MERIT_ZERO_PAD : MERIT_CLAMP;
  mp.post = post;
  mp.init = init;
  mp.fast = (mp.KH == 3 && mp.KW == 3 && mp.sy == 2 && mp.sx == 2 && mp.dy == 1 && mp.dx == 1 &&
             mp.oy == -1 && mp.ox == -1 && mp.boundary == MERIT_CLAMP && (mp.W % 4) == 0 &&
             mp.Wo == mp.W / 2 && mp.Ho == mp.H / 2)
                ? 1 : 0;
  return true;
}

// -------------------------------------------------------------------- SAD --
// Current view:   [P]: pair; H: by*BH + i; W: bx*BW + j
// Reference view: [P]: pair; H: by*BH + dy + i + oy; W: bx*BW + dx + j + ox
bool match_sad_views(const merit_view_spec& vc, const ViewAffine& fc,
                     const merit_view_spec& vr, const ViewAffine& fr, SadParams& sp) {
  const int R = vc.src_rank;
  if (R != vr.src_rank || (R != 2 && R != 3)) return false;
  const int lead = R - 2;
  const int P = vc.p_rank;
  if (P != lead + 4 || vc.a_rank != 2) return false;
  const int c_by = lead, c_bx = lead + 1, c_dy = lead + 2, c_dx = lead + 3;
  const int c_i = P, c_j = P + 1;
  if (lead == 1) {
    if (!axis_single(fc, 0, 0, 1) || fc.off[0] != 0) return false;
    if (!axis_single(fr, 0, 0, 1) || fr.off[0] != 0) return false;
    if (vc.src_shape[0] != vr.src_shape[0] || vc.p_shape[0] != vc.src_shape[0]) return false;
  }
  const int64_t BH = vc.a_shape[0], BW = vc.a_shape[1];
  // current view rows / cols
  for (int ax = 0; ax < 2; ++ax) {
    const int i = lead + ax;
    const int cb = ax == 0 ? c_by : c_bx, ca = ax == 0 ? c_i : c_j;
    const int64_t B = ax == 0 ? BH : BW;
    for (int j = 0; j < fc.k_rank; ++j) {
      int64_t want = j == cb ? B : j == ca ? 1 : 0;
      if (fc.coef[i][j] != want) return false;
    }
    const int cdisp = ax == 0 ? c_dy : c_dx;
    for (int j = 0; j < fr.k_rank; ++j) {
      int64_t want = j == cb ? B : (j == ca || j == cdisp) ? 1 : 0;
      if (fr.coef[i][j] != want) return false;
    }
  }
  if (!comp_unused(fc, c_dy) || !comp_unused(fc, c_dx)) return false;
  if (!((BH == 16 && BW == 16) || (BH == 8 && BW == 8))) return false;
  sp.pairs = lead ? vc.src_shape[0] : 1;
  sp.Hc = (int32_t)vc.src_shape[lead]; sp.Wc = (int32_t)vc.src_shape[lead + 1];
  sp.Hr = (int32_t)vr.src_shape[lead]; sp.Wr = (int32_t)vr.src_shape[lead + 1];
  sp.BY = (int32_t)vc.p_shape[c_by]; sp.BX = (int32_t)vc.p_shape[c_bx];
  sp.WY = (int32_t)vc.p_shape[c_dy]; sp.WX = (int32_t)vc.p_shape[c_dx];
  sp.BH = (int32_t)BH; sp.BW = (int32_t)BW;
  sp.cy = (int32_t)fc.off[lead]; sp.cx = (int32_t)fc.off[lead + 1];
  sp.oy = (int32_t)fr.off[lead]; sp.ox = (int32_t)fr.off[lead + 1];
  // The current block must be inside its frame (the kernel stages it raw).
  int64_t kshape[kMaxK];
  for (int j = 0; j < P; ++j) kshape[j] = vc.p_shape[j];
  kshape[P] = BH;
  kshape[P + 1] = BW;
  if (!view_in_range(fc, kshape)) return false;
  if (sp.WY < 1 || sp.WX < 1 || sp.WY > 256 || sp.WX > 256) return false;
  if (sad_rows_per_thread(sp.BH, sp.WY, sp.WX) == 0) return false;
  if (vr.boundary == MERIT_REJECT && !view_in_range(fr, kshape)) return false;  // -> generic error
  sp.boundary = vr.boundary == MERIT_REJECT ? MERIT_ZERO_PAD : vr.boundary;
  return true;
}

bool lower_sad(const merit_workload_desc& d, const ViewAffine& fa, const ViewAffine& fb,
               int32_t post, SadParams& sp) {
  if (post != POST_ADD_ZERO) return false;
  // 8-bit frames, or REAL32 frames (what the reference's Tensor holds,
  // tensor.hpp:67) narrowed on the device with an exact fallback; argmin
  // records need the 8-bit path (the fallback interpreter writes maps only)
  const bool narrow = d.dtype_a == MERIT_F32 && d.dtype_b == MERIT_F32 && d.dtype_out == MERIT_F32 &&
                      !(d.flags & (MERIT_FLAG_ARGMIN | MERIT_FLAG_NO_MAP));
  if (!narrow && (d.dtype_a != MERIT_U8 || d.dtype_b != MERIT_U8)) return false;
  if (d.dtype_out != MERIT_I32 && d.dtype_out != MERIT_F32 && d.dtype_out != MERIT_U16) return false;
  if (!same_shape(d.view_a.p_shape, d.view_a.p_rank, d.view_b.p_shape, d.view_b.p_rank))
    return false;
  if (match_sad_views(d.view_a, fa, d.view_b, fb, sp)) {
    sp.ref_is_b = 1;
  } else if (match_sad_views(d.view_b, fb, d.view_a, fa, sp)) {
    sp.ref_is_b = 0;
  } else {
    return false;
  }
  sp.argmin = (d.flags & MERIT_FLAG_ARGMIN) ? 1 : 0;
  sp.write_map = (sp.argmin && (d.flags & MERIT_FLAG_NO_MAP)) ? 0 : 1;
  sp.out_f32 = d.dtype_out == MERIT_F32;
  sp.out_u16 = d.dtype_out == MERIT_U16;  // exact: 8-bit 8x8 / 16x16 SADs are <= 65,280
  sp.narrow = narrow ? 1 : 0;
  return true;
}

// ------------------------------------------------------------------- conv --
// Input view:  [N]: n; C: ci; H: y*sy + ky*dy + oy; W: x*sx + kx*dx + ox
// Weight view: (Cout, Cin, KH, KW) <- (co, ci, ky, kx)
// p = ([n,] co, y, x), a = (ci, ky, kx).
bool finish_conv(const merit_workload_desc& d, int32_t post, ConvParams& cp);

bool lower_conv(const merit_workload_desc& d, const ViewAffine& fa, const ViewAffine& fb,
                int32_t post, ConvParams& cp, bool& swapped) {
  if (d.dtype_out != MERIT_F32) return false;
  auto try_one = [&](const merit_view_spec& vi, const ViewAffine& fi, int dti,
                     const merit_view_spec& vw, const ViewAffine& fw, int dtw) -> bool {
    if (dti != MERIT_F32 && dti != MERIT_BF16) return false;
    if (dtw != MERIT_F32 && dtw != MERIT_BF16) return false;
    const int R = vi.src_rank;
    if (R != 3 && R != 4) return false;
    const int lead = R - 3;  // batch axis present?
    const int P = vi.p_rank;
    if (P != lead + 3 || vi.a_rank != 3 || vw.src_rank != 4) return false;
    const int c_n = 0, c_co = lead, c_y = lead + 1, c_x = lead + 2;
    const int c_ci = P, c_ky = P + 1, c_kx = P + 2;
    if (lead) {
      if (!axis_single(fi, 0, c_n, 1) || fi.off[0] != 0) return false;
      if (vi.p_shape[c_n] != vi.src_shape[0]) return false;
    }
    if (!axis_single(fi, lead, c_ci, 1) || fi.off[lead] != 0) return false;
    int comps[kMaxK];
    if (axis_comps(fi, lead + 1, comps) != 2 || comps[0] != c_y || comps[1] != c_ky) return false;
    if (axis_comps(fi, lead + 2, comps) != 2 || comps[0] != c_x || comps[1] != c_kx) return false;
    if (!comp_unused(fi, c_co)) return false;
    // weights
    if (!axis_single(fw, 0, c_co, 1) || !axis_single(fw, 1, c_ci, 1) ||
        !axis_single(fw, 2, c_ky, 1) || !axis_single(fw, 3, c_kx, 1))
      return false;
    for (int i = 0; i < 4; ++i)
      if (fw.off[i] != 0) return false;
    if (vw.src_shape[0] != vi.p_shape[c_co] || vw.src_shape[1] != vi.a_shape[0] ||
        vw.src_shape[2] != vi.a_shape[1] || vw.src_shape[3] != vi.a_shape[2])
      return false;
    if (vi.src_shape[lead] != vi.a_shape[0]) return false;  // Cin matches
    const int64_t sy = fi.coef[lead + 1][c_y], dy = fi.coef[lead + 1][c_ky];
    const int64_t sx = fi.coef[lead + 2][c_x], dx = fi.coef[lead + 2][c_kx];
    if (sy < 1 || sx < 1 || dy < 1 || dx < 1) return false;
    int64_t kshape[kMaxK];
    for (int j = 0; j < P; ++j) kshape[j] = vi.p_shape[j];
    for (int j = 0; j < 3; ++j) kshape[P + j] = vi.a_shape[j];
    if (vi.boundary == MERIT_CLAMP && !view_in_range(fi, kshape)) return false;
    if (vi.boundary == MERIT_REJECT && !view_in_range(fi, kshape)) return false;
    cp.N = lead ? (int32_t)vi.src_shape[0] : 1;
    cp.Cin = (int32_t)vi.src_shape[lead];
    cp.H = (int32_t)vi.src_shape[lead + 1];
    cp.W = (int32_t)vi.src_shape[lead + 2];
    cp.Cout = (int32_t)vi.p_shape[c_co];
    cp.Ho = (int32_t)vi.p_shape[c_y];
    cp.Wo = (int32_t)vi.p_shape[c_x];
    cp.KH = (int32_t)vi.a_shape[1];
    cp.KW = (int32_t)vi.a_shape[2];
    cp.sy = (int32_t)sy; cp.sx = (int32_t)sx; cp.dy = (int32_t)dy; cp.dx = (int32_t)dx;
    cp.oy = (int32_t)fi.off[lead + 1];
    cp.ox = (int32_t)fi.off[lead + 2];
    cp.in_bf16 = dti == MERIT_BF16;
    cp.w_bf16 = dtw == MERIT_BF16;
    // NCHW input / OIHW weights / NCHW output
    cp.a_sx = 1;
    cp.a_sy = cp.W;
    cp.a_sc = (int64_t)cp.H * cp.W;
    cp.a_sn = (int64_t)cp.Cin * cp.a_sc;
    cp.o_sp = 1;
    cp.o_sc = (int64_t)cp.Ho * cp.Wo;
    cp.o_sn = (int64_t)cp.Cout * cp.o_sc;
    cp.w_si = (int64_t)cp.KH * cp.KW;
    cp.w_so = (int64_t)cp.Cin * cp.w_si;
    cp.gemm = 0;
    return true;
  };
  swapped = false;
  if (!try_one(d.view_a, fa, d.dtype_a, d.view_b, fb, d.dtype_b)) {
    if (!try_one(d.view_b, fb, d.dtype_b, d.view_a, fa, d.dtype_a)) return false;
    swapped = true;
  }
  return finish_conv(d, post, cp);
}

// GEMM view (workloads.hpp:122-136): C[i,j] = sum_t A[i,t] B[t,j], p = (m, n),
// a = (k).  It runs on the general tensor-core kernel as a 1x1 "convolution"
// of one image of M x 1 pixels with K input and N output channels, through
// operand strides: A rows are pixels (channel stride 1, row stride K), B is
// [K][N] (output-channel stride 1, input-channel stride N), C is [M][N].
bool lower_gemm(const merit_workload_desc& d, const ViewAffine& fa, const ViewAffine& fb, int32_t post,
                ConvParams& cp, bool& swapped) {
  if (d.dtype_out != MERIT_F32) return false;
  auto try_one = [&](const merit_view_spec& va, const ViewAffine& xa, int dta, const merit_view_spec& vb,
                     const ViewAffine& xb, int dtb) -> bool {
    if ((dta != MERIT_F32 && dta != MERIT_BF16) || (dtb != MERIT_F32 && dtb != MERIT_BF16)) return false;
    if (va.src_rank != 2 || vb.src_rank != 2 || va.p_rank != 2 || va.a_rank != 1) return false;
    // A[i, t]: axis 0 <- p0, axis 1 <- a0;  B[t, j]: axis 0 <- a0, axis 1 <- p1
    if (!axis_single(xa, 0, 0, 1) || !axis_single(xa, 1, 2, 1) || !comp_unused(xa, 1)) return false;
    if (!axis_single(xb, 0, 2, 1) || !axis_single(xb, 1, 1, 1) || !comp_unused(xb, 0)) return false;
    if (xa.off[0] || xa.off[1] || xb.off[0] || xb.off[1]) return false;
    const int64_t M = va.p_shape[0], N = va.p_shape[1], K = va.a_shape[0];
    if (va.src_shape[0] != M || va.src_shape[1] != K || vb.src_shape[0] != K || vb.src_shape[1] != N)
      return false;
    cp = ConvParams{};
    cp.N = 1;
    cp.Cin = (int32_t)K;
    cp.H = cp.Ho = (int32_t)M;
    cp.W = cp.Wo = 1;
    cp.Cout = (int32_t)N;
    cp.KH = cp.KW = 1;
    cp.in_bf16 = dta == MERIT_BF16;
    cp.w_bf16 = dtb == MERIT_BF16;
    cp.a_sc = 1;
    cp.a_sy = K;
    cp.o_sc = 1;
    cp.o_sp = N;
    cp.w_so = 1;
    cp.w_si = N;
    cp.gemm = 1;
    return true;
  };
  swapped = false;
  if (!try_one(d.view_a, fa, d.dtype_a, d.view_b, fb, d.dtype_b)) {
    if (!try_one(d.view_b, fb, d.dtype_b, d.view_a, fa, d.dtype_a)) return false;
    swapped = true;
  }
  return finish_conv(d, post, cp);
}

// Correlation views (workloads.hpp:230-251): A = (a0, p0 + ay, p1 + ax),
// B = (a0, p0 + p2 + by, p1 + p3 + bx), p = (y, x, dy, dx), a = (c), both
// REAL32 [C][H][W]; either port may carry the displaced view.  ZERO_PAD (or a
// view provably inside its source) so the kernel's zero fill is the view's.
bool lower_corr(const merit_workload_desc& d, const ViewAffine& fa, const ViewAffine& fb, int32_t post,
                CorrParams& cr, bool& swapped) {
  if (d.dtype_a != MERIT_F32 || d.dtype_b != MERIT_F32 || d.dtype_out != MERIT_F32) return false;
  auto try_one = [&](const merit_view_spec& v1, const ViewAffine& f1, const merit_view_spec& v2,
                     const ViewAffine& f2) -> bool {
    if (v1.src_rank != 3 || v2.src_rank != 3 || v1.p_rank != 4 || v1.a_rank != 1) return false;
    const int cy = 0, cx = 1, cdy = 2, cdx = 3, cc = 4;
    if (!axis_single(f1, 0, cc, 1) || f1.off[0] != 0 || !axis_single(f2, 0, cc, 1) || f2.off[0] != 0)
      return false;
    if (!axis_single(f1, 1, cy, 1) || !axis_single(f1, 2, cx, 1)) return false;
    for (int i = 0; i < 3; ++i)
      if (f2.coef[i][cy] != (i == 1) || f2.coef[i][cdy] != (i == 1) || f2.coef[i][cx] != (i == 2) ||
          f2.coef[i][cdx] != (i == 2))
        return false;
    if (v1.src_shape[0] != v1.a_shape[0] || v2.src_shape[0] != v1.a_shape[0]) return false;
    int64_t kshape[kMaxK];
    for (int j = 0; j < 4; ++j) kshape[j] = v1.p_shape[j];
    kshape[4] = v1.a_shape[0];
    if (v1.boundary != MERIT_ZERO_PAD && !view_in_range(f1, kshape)) return false;
    if (v2.boundary != MERIT_ZERO_PAD && !view_in_range(f2, kshape)) return false;
    for (int j = 0; j < 4; ++j)
      if (v1.p_shape[j] > (1 << 20)) return false;
    if (corr_threads_per_column_quad((int)v1.p_shape[cdy], (int)v1.p_shape[cdx]) == 0) return false;
    cr.C = (int32_t)v1.a_shape[0];
    cr.Ha = (int32_t)v1.src_shape[1]; cr.Wa = (int32_t)v1.src_shape[2];
    cr.Hb = (int32_t)v2.src_shape[1]; cr.Wb = (int32_t)v2.src_shape[2];
    cr.Ho = (int32_t)v1.p_shape[cy]; cr.Wo = (int32_t)v1.p_shape[cx];
    cr.DY = (int32_t)v1.p_shape[cdy]; cr.DX = (int32_t)v1.p_shape[cdx];
    cr.ay = (int32_t)f1.off[1]; cr.ax = (int32_t)f1.off[2];
    cr.by = (int32_t)f2.off[1]; cr.bx = (int32_t)f2.off[2];
    cr.post = post;
    return true;
  };
  swapped = false;
  if (try_one(d.view_a, fa, d.view_b, fb)) return true;
  swapped = true;
  return try_one(d.view_b, fb, d.view_a, fa);
}

bool finish_conv(const merit_workload_desc& d, int32_t post, ConvParams& cp) {
  const bool both_bf16 = cp.in_bf16 && cp.w_bf16;
  cp.split = (both_bf16 || (d.flags & MERIT_FLAG_FAST_BF16)) ? 1 : 3;
  cp.post = post;
  const int cout16 = (cp.Cout + 15) / 16 * 16;
  cp.n_tiles_n = (cout16 + 255) / 256;
  cp.BN = (cout16 + cp.n_tiles_n - 1) / cp.n_tiles_n;
  cp.BN = (cp.BN + 15) / 16 * 16;
  cp.CB = (cp.Cin + 63) / 64;
  cp.n_kb = cp.KH * cp.KW * cp.CB;
  cp.npix = (int64_t)cp.N * cp.Ho * cp.Wo;
  const int planes_b = cp.split == 1 ? 1 : 2;
  cp.packed_b_bytes = (int64_t)cp.n_tiles_n * cp.n_kb * planes_b * cp.BN * 128;
  if (cp.npix >= (int64_t(1) << 31)) return false;
  return true;
}

}  // namespace

int64_t elem_size(int dtype) {
  switch (dtype) {
    case MERIT_F32: return 4;
    case MERIT_I16: return 2;
    case MERIT_BF16: return 2;
    case MERIT_U8: return 1;
    case MERIT_I32: return 4;
    case MERIT_U16: return 2;
    default: return 0;
  }
}

merit_status lower(const merit_workload_desc& d, merit_plan& plan) {
  merit_status st;
  if ((st = check_view(d.view_a, "view_a")) != MERIT_OK) return st;
  if ((st = check_view(d.view_b, "view_b")) != MERIT_OK) return st;
  for (int dt : {d.dtype_a, d.dtype_b, d.dtype_out})
    if (elem_size(dt) == 0) return fail(MERIT_E_UNKNOWN_DTYPE, "unknown dtype code");
  // Workload::validate (engine.hpp:30-38)
  if (!same_shape(d.view_a.p_shape, d.view_a.p_rank, d.view_b.p_shape, d.view_b.p_rank) ||
      !same_shape(d.view_a.a_shape, d.view_a.a_rank, d.view_b.a_shape, d.view_b.a_rank))
    return fail(MERIT_E_BAD_PARAMS, "views must share p and a shapes");
  const merit_program& pg = d.program;
  if (pg.depth != d.view_a.a_rank)
    return fail(MERIT_E_BAD_PARAMS, "program depth must match |a|");
  // StrategyProgram::validate (rip.hpp:96-106)
  if (pg.n_segments != 2 * pg.depth + 1)
    return fail(MERIT_E_BAD_PARAMS, "program needs 2*depth+1 segments");
  if (pg.n_segments > 0 && (!pg.seg_len))
    return fail(MERIT_E_INVALID_ARGUMENT, "program segment lengths missing");
  ProgramImage& pi = plan.prog;
  std::memset(&pi, 0, sizeof(pi));
  pi.depth = pg.depth;
  pi.outputs = pg.outputs;
  pi.n_segments = pg.n_segments;
  int total = 0;
  for (int s = 0; s < pg.n_segments; ++s) {
    if (pg.seg_len[s] < 0) return fail(MERIT_E_INVALID_ARGUMENT, "negative segment length");
    pi.seg_start[s] = total;
    pi.seg_len[s] = pg.seg_len[s];
    total += pg.seg_len[s];
  }
  if (total > MERIT_MAX_INSTRS) return fail(MERIT_E_INVALID_ARGUMENT, "program too long");
  if (total > 0 && !pg.instrs) return fail(MERIT_E_INVALID_ARGUMENT, "program instrs missing");
  pi.n_instrs = total;
  for (int i = 0; i < total; ++i) {
    const merit_alu_instr& in = pg.instrs[i];
    if (!in.dst_out && (in.dst_reg < 0 || in.dst_reg >= 16))
      return fail(MERIT_E_BAD_PARAMS, "register id must be < 16");
    if (in.shift < 0 || in.shift > 15) return fail(MERIT_E_BAD_PARAMS, "shift must be 0..15");
    if (in.op < MERIT_OP_ADD || in.op > MERIT_OP_DIV)
      return fail(MERIT_E_INVALID_ARGUMENT, "unknown op");
    const int kinds[3] = {in.a_kind, in.b_kind, in.c_kind};
    const int regs[3] = {in.a_reg, in.b_reg, in.c_reg};
    for (int q = 0; q < 3; ++q) {
      if (kinds[q] < MERIT_OPND_REG || kinds[q] > MERIT_OPND_ZERO)
        return fail(MERIT_E_INVALID_ARGUMENT, "unknown operand kind");
      if (kinds[q] == MERIT_OPND_REG && (regs[q] < 0 || regs[q] >= 16))
        return fail(MERIT_E_BAD_PARAMS, "operand register id must be < 16");
    }
    pi.instrs[i] = in;
  }
  if (pg.n_constants < 0 || pg.n_constants > MERIT_MAX_CONSTANTS)
    return fail(MERIT_E_INVALID_ARGUMENT, "too many constants");
  pi.n_constants = pg.n_constants;
  for (int i = 0; i < pg.n_constants; ++i) pi.constants[i] = pg.constants[i];
  if (pg.n_tables < 0 || pg.n_tables > MERIT_MAX_TABLES)
    return fail(MERIT_E_INVALID_ARGUMENT, "too many tables");
  pi.n_tables = pg.n_tables;
  int so = 0;
  for (int t = 0; t < pg.n_tables; ++t) {
    const merit_lookup_table& tb = pg.tables[t];
    if (tb.n_samples < 1 || tb.n_samples > MERIT_MAX_TABLE_SAMPLES || !tb.samples)
      return fail(MERIT_E_INVALID_ARGUMENT, "bad lookup table");
    pi.tab_lo[t] = tb.lo;
    pi.tab_hi[t] = tb.hi;
    pi.tab_n[t] = tb.n_samples;
    pi.tab_clamp[t] = tb.clamp;
    pi.tab_off[t] = so;
    for (int i = 0; i < tb.n_samples; ++i) pi.table_samples[so + i] = tb.samples[i];
    so += tb.n_samples;
  }
  pi.n_table_samples = so;

  const merit_view_spec& v = d.view_a;
  // Tensor::real(output_shape()) rejects rank 0 and extents < 1 (tensor.hpp:166-170).
  if (v.p_rank == 0 && pg.outputs <= 1) return fail(MERIT_E_BAD_PARAMS, "rank must be >= 1");
  if (pg.outputs < 1) return fail(MERIT_E_BAD_PARAMS, "extents must be >= 1");
  for (int i = 0; i < v.p_rank; ++i)
    if (v.p_shape[i] < 1) return fail(MERIT_E_BAD_PARAMS, "extents must be >= 1");
  for (int i = 0; i < v.a_rank; ++i)  // phase_range throws on an empty a extent
    if (v.a_shape[i] < 1) return fail(MERIT_E_OUT_OF_RANGE, "phase index out of range");

  ViewAffine fa, fb;
  affine_of(d.view_a, fa);
  affine_of(d.view_b, fb);

  // Mode is decided by src_a's dtype like run_full (engine.hpp:282-287).
  const bool fix16 = d.dtype_a == MERIT_I16;
  if (fix16 != (d.dtype_b == MERIT_I16))
    return fail(MERIT_E_BAD_PARAMS, "both sources must be FIX16 or neither");
  if (fix16 && d.dtype_out != MERIT_I16)
    return fail(MERIT_E_BAD_PARAMS, "FIX16 workloads produce FIX16 outputs");

  merit_plan_info& info = plan.info;
  std::memset(&info, 0, sizeof(info));
  info.out_rank = v.p_rank + (pg.outputs > 1 ? 1 : 0);
  for (int i = 0; i < v.p_rank; ++i) info.out_shape[i] = v.p_shape[i];
  if (pg.outputs > 1) info.out_shape[v.p_rank] = pg.outputs;
  info.n_outputs = vol(v.p_shape, v.p_rank);
  info.out_elems = info.n_outputs * pg.outputs;
  info.src_a_bytes = vol(d.view_a.src_shape, d.view_a.src_rank) * elem_size(d.dtype_a);
  info.src_b_bytes = vol(d.view_b.src_shape, d.view_b.src_rank) * elem_size(d.dtype_b);
  info.launches_per_run = 1;

  int32_t post = POST_ADD_ZERO;
  float init = 0.f;
  Skeleton sk = (d.flags & MERIT_FLAG_EXACT) || fix16 ? SK_NONE : classify(d, pi, post, init);
  const int64_t avol = vol(v.a_shape, v.a_rank);

  if (sk == SK_MAX && lower_maxpool(d, fa, fb, init, post, plan.mp)) {
    plan.kernel = MERIT_KERNEL_MAXPOOL;
    const auto& mp = plan.mp;
    info.algorithmic_ops = (double)info.n_outputs * avol;
    info.algorithmic_bytes = (double)info.src_a_bytes + (double)info.out_elems * 4;
    std::snprintf(info.description, sizeof(info.description),
                  "maxpool planes=%lld %dx%d -> %dx%d k=%dx%d s=%d,%d o=%d,%d %s%s",
                  (long long)mp.planes, mp.H, mp.W, mp.Ho, mp.Wo, mp.KH, mp.KW, mp.sy, mp.sx,
                  mp.oy, mp.ox, mp.boundary == MERIT_CLAMP ? "clamp" : "zero",
                  mp.fast ? " fast3x3s2" : "");
  } else if (sk == SK_L1 && lower_sad(d, fa, fb, post, plan.sad)) {
    plan.kernel = MERIT_KERNEL_SAD;
    const auto& sp = plan.sad;
    const int64_t blocks = sp.pairs * sp.BY * sp.BX;
    if (!sp.write_map) info.out_elems = 0;
    info.aux_elems = sp.argmin ? blocks * 3 : 0;
    info.algorithmic_ops = (double)info.n_outputs * avol;
    info.algorithmic_bytes = (double)info.src_a_bytes + (double)info.src_b_bytes +
                             (double)info.out_elems * elem_size(d.dtype_out) + (double)info.aux_elems * 4;
    std::snprintf(info.description, sizeof(info.description),
                  "sad pairs=%lld frame=%dx%d blocks=%dx%d blk=%dx%d window=%dx%d off=%d,%d %s%s%s",
                  (long long)sp.pairs, sp.Hc, sp.Wc, sp.BY, sp.BX, sp.BH, sp.BW, sp.WY, sp.WX,
                  sp.oy, sp.ox, sp.boundary == MERIT_CLAMP ? "clamp" : "zero",
                  sp.argmin ? " +argmin" : "", sp.write_map ? "" : " (no map)");
  } else if (sk == SK_MAC) {
    bool swapped = false;
    if (lower_conv(d, fa, fb, post, plan.conv, swapped) || lower_gemm(d, fa, fb, post, plan.conv, swapped)) {
      plan.kernel = MERIT_KERNEL_CONV_TC;
      const auto& cp = plan.conv;
      info.algorithmic_ops = (double)info.n_outputs * avol;  // MACs
      const int64_t in_bytes = swapped ? info.src_b_bytes : info.src_a_bytes;
      const int64_t w_bytes = swapped ? info.src_a_bytes : info.src_b_bytes;
      info.algorithmic_bytes = (double)in_bytes + (double)w_bytes + (double)info.out_elems * 4;
      if (cp.gemm)
        std::snprintf(info.description, sizeof(info.description),
                      "conv_tc gemm M=%d N=%d K=%d %s split=%d BN=%d kb=%d%s", cp.H, cp.Cout, cp.Cin,
                      cp.in_bf16 ? "bf16" : "f32", cp.split, cp.BN, cp.n_kb, cp.post == POST_RELU ? " relu" : "");
      else
        std::snprintf(info.description, sizeof(info.description),
                      "conv_tc N=%d Cin=%d %dx%d -> Cout=%d %dx%d k=%dx%d s=%d,%d d=%d,%d o=%d,%d "
                      "%s split=%d BN=%d kb=%d%s",
                      cp.N, cp.Cin, cp.H, cp.W, cp.Cout, cp.Ho, cp.Wo, cp.KH, cp.KW, cp.sy, cp.sx,
                      cp.dy, cp.dx, cp.oy, cp.ox, cp.in_bf16 ? "bf16" : "f32", cp.split, cp.BN,
                      cp.n_kb, cp.post == POST_RELU ? " relu" : "");
      plan.conv_swapped = swapped;
    } else if (lower_corr(d, fa, fb, post, plan.corr, swapped)) {
      plan.kernel = MERIT_KERNEL_CORR;
      plan.corr_swapped = swapped;
      const auto& cr = plan.corr;
      info.algorithmic_ops = (double)info.n_outputs * avol;  // MACs
      info.algorithmic_bytes = (double)info.src_a_bytes + (double)info.src_b_bytes + (double)info.out_elems * 4;
      std::snprintf(info.description, sizeof(info.description),
                    "corr C=%d %dx%d displacements %dx%d off a=%d,%d b=%d,%d exact%s", cr.C, cr.Ho, cr.Wo, cr.DY,
                    cr.DX, cr.ay, cr.ax, cr.by, cr.bx, cr.post == POST_RELU ? " relu" : "");
    }
  }
  if (plan.kernel != MERIT_KERNEL_SAD && (d.flags & (MERIT_FLAG_ARGMIN | MERIT_FLAG_NO_MAP)))
    return fail(MERIT_E_UNSUPPORTED_PROGRAM,
                "argmin is only available for L1 block-matching workloads on the SAD kernel");
  if (plan.kernel == MERIT_KERNEL_GENERIC || (plan.kernel == MERIT_KERNEL_SAD && plan.sad.narrow)) {
    // Exact interpreter (also the fallback of a narrowed SAD plan).  Any
    // storage dtype widens to the mode's value type.
    if (!fix16 && d.dtype_out != MERIT_F32)
      return fail(MERIT_E_UNSUPPORTED_PROGRAM, "REAL32 generic execution writes f32 outputs");
    GenericParams& g = plan.gen;
    g.fix16 = fix16;
    g.p_rank = v.p_rank;
    g.a_rank = v.a_rank;
    for (int i = 0; i < v.p_rank; ++i) g.p_shape[i] = v.p_shape[i];
    for (int i = 0; i < v.a_rank; ++i) g.a_shape[i] = v.a_shape[i];
    g.rows = info.n_outputs;
    g.a_vol = avol;
    g.dtype_a = d.dtype_a;
    g.dtype_b = d.dtype_b;
    g.dtype_out = d.dtype_out;
    g.uses_a = 1;  // gathers happen (and may throw) whether or not a port is read
    g.uses_b = 1;
    g.va = fa;
    g.vb = fb;
    if (plan.kernel == MERIT_KERNEL_GENERIC) {
      info.algorithmic_ops = (double)info.n_outputs * avol;
      info.algorithmic_bytes = (double)info.src_a_bytes + (double)info.src_b_bytes +
                               (double)info.out_elems * elem_size(d.dtype_out);
      std::snprintf(info.description, sizeof(info.description),
                    "generic %s rows=%lld a_vol=%lld outputs=%d", fix16 ? "fix16" : "real32",
                    (long long)g.rows, (long long)avol, pg.outputs);
    } else {
      const size_t n = std::strlen(info.description);
      std::snprintf(info.description + n, sizeof(info.description) - n,
                    " (f32 frames narrowed to u8 on device, exact fallback)");
    }
    (void)program_uses_port;
  }
  info.kernel = plan.kernel;
  info.out_bytes = info.out_elems * elem_size(d.dtype_out);
  info.executed_ops = info.algorithmic_ops;
  if (plan.kernel == MERIT_KERNEL_SAD && plan.sad.narrow) info.launches_per_run = 3;
  if (plan.kernel == MERIT_KERNEL_CONV_TC) info.launches_per_run = 1;
  return MERIT_OK;
}

}  // namespace merit_dev
