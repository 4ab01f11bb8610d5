/*
 * oracle.c — CPU restatement of the reference's MERIT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.  The device library
 * (paper_1911_03458_b200/libmerit_dev.so) never links or calls it.
 *
 * Parity is pinned two ways (tests/test_oracle_golden.py):
 *  - against golden vectors produced by the reference itself
 *    (tests/golden/make_golden.py runs oracle/_ref/libmerit_ref.so, which is
 *    compiled from /root/reference/proj/include by oracle/build_ref.sh), and
 *  - against the reference tests' known-answer cases
 *    (tests/test_workloads.cpp:60-69, :95-104, :115-121 of the reference).
 *
 * Every function cites the reference code it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "merit_dev.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* SplitMix64 and fill_random — workloads.hpp:74-105                          */
typedef struct { uint64_t state; } sm64;

static uint64_t sm64_next(sm64* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double sm64_uniform(sm64* r, double lo, double hi) {
  return lo + (hi - lo) * ((double)(sm64_next(r) >> 11) * 0x1.0p-53);
}
static int64_t sm64_range(sm64* r, int64_t lo, int64_t hi) {
  return lo + (int64_t)(sm64_next(r) % (uint64_t)(hi - lo + 1));
}

void oracle_fill_uniform_f32(float* out, int64_t n, uint64_t seed, double lo, double hi) {
  sm64 r = {seed};
  for (int64_t i = 0; i < n; ++i) out[i] = (float)sm64_uniform(&r, lo, hi);
}
void oracle_fill_range_i16(int16_t* out, int64_t n, uint64_t seed, int64_t lo, int64_t hi) {
  sm64 r = {seed};
  for (int64_t i = 0; i < n; ++i) out[i] = (int16_t)sm64_range(&r, lo, hi);
}
/* Seeded synthetic inputs of SURVEY §8(d), restated here so that the CPU
 * baseline arms of bench.py never load the device library:
 * normal(0, sigma) by Box-Muller over SplitMix64 uniforms (C3/C4 weights),
 * fp32 -> bf16 round-to-nearest-even (C4 activations), and the motion
 * estimation frame pair (ref = 5x5 box filter of uniform bytes, clamped
 * border, round half up; cur = ref shifted per blk x blk block by
 * range(-max_shift, max_shift) plus range(-noise, noise), clamped).
 * tests/test_oracle_golden.py checks them byte-for-byte against the device
 * library's merit_gen_* (the generators the GPU arm uses). */
void oracle_gen_normal_f32(float* out, int64_t n, uint64_t seed, double sigma) {
  sm64 r = {seed};
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; i += 2) {
    double u1 = sm64_uniform(&r, 0.0, 1.0), u2 = sm64_uniform(&r, 0.0, 1.0);
    if (u1 < 1e-300) u1 = 1e-300;
    const double rad = sqrt(-2.0 * log(u1));
    out[i] = (float)(sigma * rad * cos(two_pi * u2));
    if (i + 1 < n) out[i + 1] = (float)(sigma * rad * sin(two_pi * u2));
  }
}

void oracle_f32_to_bf16(const float* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, &in[i], 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) {
      out[i] = (uint16_t)((u >> 16) | 0x40);
      continue;
    }
    u += 0x7fffu + ((u >> 16) & 1u);
    out[i] = (uint16_t)(u >> 16);
  }
}

static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : v > hi ? hi : v; }

void oracle_gen_me_pair(uint8_t* cur, uint8_t* ref, int64_t h, int64_t w, int64_t blk, int64_t max_shift,
                        int64_t noise, uint64_t seed) {
  sm64 r = {seed};
  uint8_t* raw = (uint8_t*)malloc((size_t)(h * w));
  for (int64_t i = 0; i < h * w; ++i) raw[i] = (uint8_t)sm64_range(&r, 0, 255);
  for (int64_t y = 0; y < h; ++y)
    for (int64_t x = 0; x < w; ++x) {
      int64_t s = 0;
      for (int64_t dy = -2; dy <= 2; ++dy)
        for (int64_t dx = -2; dx <= 2; ++dx) s += raw[clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
      ref[y * w + x] = (uint8_t)((s + 12) / 25);
    }
  free(raw);
  const int64_t by = (h + blk - 1) / blk, bx = (w + blk - 1) / blk;
  for (int64_t b = 0; b < by * bx; ++b) {
    const int64_t y0 = (b / bx) * blk, x0 = (b % bx) * blk;
    const int64_t sx = sm64_range(&r, -max_shift, max_shift), sy = sm64_range(&r, -max_shift, max_shift);
    for (int64_t i = 0; i < blk && y0 + i < h; ++i)
      for (int64_t j = 0; j < blk && x0 + j < w; ++j) {
        const int64_t y = y0 + i, x = x0 + j;
        const int64_t v = ref[clampi(y + sy, 0, h - 1) * w + clampi(x + sx, 0, w - 1)] + sm64_range(&r, -noise, noise);
        cur[y * w + x] = (uint8_t)clampi(v, 0, 255);
      }
  }
}

uint64_t oracle_splitmix_next(uint64_t* state) {
  sm64 r = {*state};
  uint64_t v = sm64_next(&r);
  *state = r.state;
  return v;
}

/* ------------------------------------------------------------------------ */
/* Max-pool with the ENGINE's semantics: the max-pool program
 * (workloads.hpp:376-385) run by run_full_typed (engine.hpp:120-143):
 * r = MOVC init; r = std::max(r, v) == (r < v) ? v : r in row-major (ky, kx)
 * order (rip.hpp:175-176); emit r + 0.0f (rip.hpp:167-168).  CLAMP clamps
 * each coordinate (view.hpp:73-76), ZERO_PAD reads 0 (view.hpp:71-72).
 * For CLAMP this equals oracle_maxpool (workloads.hpp:642-671) extended with
 * -inf padding (verified in SURVEY §8(c)). */
void oracle_maxpool(const float* in, float* out, int64_t planes, int H, int W, int Ho, int Wo,
                    int KH, int KW, int sy, int sx, int dy, int dx, int oy, int ox, int clamp,
                    float init, int relu) {
#pragma omp parallel for schedule(static)
  for (int64_t pl = 0; pl < planes; ++pl) {
    const float* src = in + pl * (int64_t)H * W;
    float* dst = out + pl * (int64_t)Ho * Wo;
    for (int y = 0; y < Ho; ++y)
      for (int x = 0; x < Wo; ++x) {
        float r = init;
        for (int ky = 0; ky < KH; ++ky)
          for (int kx = 0; kx < KW; ++kx) {
            int iy = y * sy + ky * dy + oy, ix = x * sx + kx * dx + ox;
            float v;
            if (iy < 0 || iy >= H || ix < 0 || ix >= W) {
              if (clamp) {
                iy = iy < 0 ? 0 : (iy >= H ? H - 1 : iy);
                ix = ix < 0 ? 0 : (ix >= W ? W - 1 : ix);
                v = src[(int64_t)iy * W + ix];
              } else {
                v = 0.0f;
              }
            } else {
              v = src[(int64_t)iy * W + ix];
            }
            r = (r < v) ? v : r;
          }
        dst[(int64_t)y * Wo + x] = relu ? ((r < 0.0f) ? 0.0f : r) : (r + 0.0f);
      }
  }
}

/* ------------------------------------------------------------------------ */
/* Convolution — oracle_conv2d (workloads.hpp:458-499) with a batch axis:
 * plain nested loops, ZERO_PAD, accumulation in double, one rounding to
 * float at the end (workloads.hpp:487, :495).  Weights (co, ci, ky, kx).
 * in/w are f32 (the fp32 originals for the bf16 config). */
void oracle_conv2d_nchw(const float* in, const float* w, float* out, int N, int Cin, int H, int W,
                        int Cout, int Ho, int Wo, int KH, int KW, int sy, int sx, int dy, int dx,
                        int oy, int ox, int relu) {
  const int64_t total = (int64_t)N * Cout * Ho;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < total; ++t) {
    const int y = (int)(t % Ho);
    const int co = (int)((t / Ho) % Cout);
    const int n = (int)(t / ((int64_t)Ho * Cout));
    const float* img = in + (int64_t)n * Cin * H * W;
    float* dst = out + (((int64_t)n * Cout + co) * Ho + y) * Wo;
    for (int x = 0; x < Wo; ++x) {
      double s = 0.0;
      for (int ci = 0; ci < Cin; ++ci)
        for (int ky = 0; ky < KH; ++ky) {
          const int iy = y * sy + ky * dy + oy;
          if (iy < 0 || iy >= H) continue; /* iv = 0 contributes exactly 0 */
          for (int kx = 0; kx < KW; ++kx) {
            const int ix = x * sx + kx * dx + ox;
            if (ix < 0 || ix >= W) continue;
            s += (double)img[((int64_t)ci * H + iy) * W + ix] *
                 (double)w[(((int64_t)co * Cin + ci) * KH + ky) * KW + kx];
          }
        }
      if (relu && s < 0.0) s = 0.0;
      dst[x] = (float)s;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Block-matching SAD — oracle_motion_estimation (workloads.hpp:548-585),
 * REAL32 branch, on 8-bit frames: s += |cur - ref|, ref = 0 outside the
 * frame (ZERO_PAD, :569-576) or the clamped pixel (CLAMP).  All partial
 * sums are integers < 2^24, so int32 is exact.  Block grid by x bx is given
 * (the oracle floors h/blk, :556); (oy, ox) is the reference offset at
 * displacement 0 (= -win/2 in the template).  Optional leading pair axis. */
void oracle_me_sad(const uint8_t* cur, const uint8_t* ref, int32_t* out, int64_t pairs, int H,
                   int W, int BY, int BX, int BH, int BW, int WY, int WX, int oy, int ox,
                   int clamp) {
  const int64_t jobs = pairs * BY * BX;
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t jb = 0; jb < jobs; ++jb) {
    const int bx = (int)(jb % BX);
    const int by = (int)((jb / BX) % BY);
    const int64_t pr = jb / ((int64_t)BX * BY);
    const uint8_t* c = cur + pr * (int64_t)H * W;
    const uint8_t* r = ref + pr * (int64_t)H * W;
    int32_t* o = out + jb * (int64_t)WY * WX;
    for (int dy = 0; dy < WY; ++dy)
      for (int dx = 0; dx < WX; ++dx) {
        int32_t s = 0;
        for (int i = 0; i < BH; ++i)
          for (int j = 0; j < BW; ++j) {
            const int cy = by * BH + i, cx = bx * BW + j;
            int ry = cy + dy + oy, rx = cx + dx + ox;
            int rv;
            if (ry >= 0 && ry < H && rx >= 0 && rx < W) {
              rv = r[(int64_t)ry * W + rx];
            } else if (clamp) {
              ry = ry < 0 ? 0 : (ry >= H ? H - 1 : ry);
              rx = rx < 0 ? 0 : (rx >= W ? W - 1 : rx);
              rv = r[(int64_t)ry * W + rx];
            } else {
              rv = 0;
            }
            const int d = (int)c[(int64_t)cy * W + cx] - rv;
            s += d < 0 ? -d : d;
          }
        o[dy * WX + dx] = s;
      }
  }
}

/* Caller-side argmin over a SAD map (not in the reference: SPEC.md:562,576
 * leave it to callers).  Lowest SAD, ties to the lowest raster index
 * dy*WX + dx.  Writes (dy + oy, dx + ox, sad) per block. */
void oracle_me_argmin(const int32_t* sad, int32_t* mv, int64_t blocks, int WY, int WX, int oy,
                      int ox) {
  for (int64_t b = 0; b < blocks; ++b) {
    const int32_t* s = sad + b * (int64_t)WY * WX;
    int best = 0;
    for (int i = 1; i < WY * WX; ++i)
      if (s[i] < s[best]) best = i;
    mv[3 * b + 0] = best / WX + oy;
    mv[3 * b + 1] = best % WX + ox;
    mv[3 * b + 2] = s[best];
  }
}

/* ------------------------------------------------------------------------ */
/* Generic engine restatement: run_full (engine.hpp:282-287) =
 * run_full_typed (engine.hpp:120-143) over view_gather (view.hpp:68-84),
 * phase_range (rip.hpp:112-126) and RipState::exec (rip.hpp:221-262) with
 * the Real32Mode / Fix16Mode ALU (rip.hpp:130-200).  Single-threaded, for
 * small workloads.  Returns 0 or a merit_status code (the reference throws). */
static int32_t sat16(int64_t v) { return v < -32768 ? -32768 : v > 32767 ? 32767 : (int32_t)v; }

typedef struct {
  int src_rank, k_rank, boundary;
  int64_t shape[MERIT_MAX_RANK];
  int64_t coef[MERIT_MAX_RANK][2 * MERIT_MAX_RANK];
  int64_t off[MERIT_MAX_RANK];
} affine_t;

static void mk_affine(const merit_view_spec* v, affine_t* f) {
  memset(f, 0, sizeof(*f));
  f->src_rank = v->src_rank;
  f->k_rank = v->p_rank + v->a_rank;
  f->boundary = v->boundary;
  for (int i = 0; i < v->src_rank; ++i) f->shape[i] = v->src_shape[i];
  for (int t = 0; t < v->n_terms; ++t) {
    f->coef[v->terms[t].axis][v->terms[t].component] += v->terms[t].stride;
    f->off[v->terms[t].axis] += v->terms[t].offset;
  }
}

static int gather(const affine_t* f, const int64_t* k, const void* src, int dtype, double* val) {
  int64_t flat = 0;
  int zero = 0;
  for (int i = 0; i < f->src_rank; ++i) {
    int64_t x = f->off[i];
    for (int j = 0; j < f->k_rank; ++j) x += f->coef[i][j] * k[j];
    if (x < 0 || x >= f->shape[i]) {
      if (f->boundary == MERIT_ZERO_PAD) zero = 1;
      else if (f->boundary == MERIT_CLAMP) x = x < 0 ? 0 : f->shape[i] - 1;
      else return MERIT_E_OUT_OF_RANGE;
    }
    flat = flat * f->shape[i] + x;
  }
  if (zero) { *val = 0.0; return 0; }
  switch (dtype) {
    case MERIT_F32: *val = ((const float*)src)[flat]; break;
    case MERIT_I16: *val = ((const int16_t*)src)[flat]; break;
    case MERIT_U8: *val = ((const uint8_t*)src)[flat]; break;
    case MERIT_I32: *val = ((const int32_t*)src)[flat]; break;
    case MERIT_BF16: {
      uint32_t u = (uint32_t)((const uint16_t*)src)[flat] << 16;
      float f32;
      memcpy(&f32, &u, 4);
      *val = f32;
      break;
    }
    default: return MERIT_E_UNKNOWN_DTYPE;
  }
  return 0;
}

static double table_lookup(const merit_lookup_table* t, double x, int* err) {
  if (x < t->lo || x > t->hi) {
    if (!t->clamp) { *err = MERIT_E_LUT_RANGE; return 0; }
    x = x < t->lo ? t->lo : t->hi;
  }
  if (t->n_samples == 1) return t->samples[0];
  double tt = (x - t->lo) / (t->hi - t->lo) * (double)(t->n_samples - 1);
  size_t i = (size_t)tt;
  if (i >= (size_t)(t->n_samples - 1)) return t->samples[t->n_samples - 1];
  double fr = tt - (double)i;
  return t->samples[i] * (1.0 - fr) + t->samples[i + 1] * fr;
}

int oracle_run_full(const merit_workload_desc* d, const void* a, const void* b, void* out) {
  affine_t fa, fb;
  mk_affine(&d->view_a, &fa);
  mk_affine(&d->view_b, &fb);
  const merit_program* P = &d->program;
  const int fix = d->dtype_a == MERIT_I16;
  const int pr = d->view_a.p_rank, D = d->view_a.a_rank, kr = pr + D;
  int seg_start[2 * MERIT_MAX_RANK + 2];
  int acc = 0;
  for (int s = 0; s < P->n_segments; ++s) { seg_start[s] = acc; acc += P->seg_len[s]; }
  int64_t rows = 1;
  for (int i = 0; i < pr; ++i) rows *= d->view_a.p_shape[i];
  for (int64_t row = 0; row < rows; ++row) {
    int64_t k[2 * MERIT_MAX_RANK];
    int64_t rr = row;
    for (int i = pr - 1; i >= 0; --i) { k[i] = rr % d->view_a.p_shape[i]; rr /= d->view_a.p_shape[i]; }
    for (int i = 0; i < D; ++i) k[pr + i] = 0;
    float fr[16] = {0};
    int32_t qr[16] = {0};
    int emitted = 0;
    for (;;) {
      int zeros = 0, maxed = 0;
      while (zeros < D && k[pr + D - 1 - zeros] == 0) ++zeros;
      while (maxed < D && k[pr + D - 1 - maxed] == d->view_a.a_shape[D - 1 - maxed] - 1) ++maxed;
      const int first = zeros > 0 ? D - zeros : D, last = maxed > 0 ? D + maxed : D;
      double va, vb;
      int e;
      if ((e = gather(&fa, k, a, d->dtype_a, &va))) return e;
      if ((e = gather(&fb, k, b, d->dtype_b, &vb))) return e;
      for (int seg = first; seg <= last; ++seg)
        for (int q = 0; q < P->seg_len[seg]; ++q) {
          const merit_alu_instr* in = &P->instrs[seg_start[seg] + q];
          const int kinds[3] = {in->a_kind, in->b_kind, in->c_kind};
          const int regs[3] = {in->a_reg, in->b_reg, in->c_reg};
          if (!fix) {
            float o[3];
            for (int z = 0; z < 3; ++z)
              o[z] = kinds[z] == MERIT_OPND_REG ? fr[regs[z]] : kinds[z] == MERIT_OPND_PORT_A ? (float)va
                     : kinds[z] == MERIT_OPND_PORT_B ? (float)vb : 0.0f;
            const float A = o[0], B = o[1], Cc = o[2];
            float res = 0;
            int err = 0;
            switch (in->op) {
              case MERIT_OP_ADD: res = A + (float)ldexp((double)B + Cc, -in->shift); break;
              case MERIT_OP_SUB: res = A + (float)ldexp((double)B - Cc, -in->shift); break;
              case MERIT_OP_L1: res = A + (float)ldexp(fabs((double)B - Cc), -in->shift); break;
              case MERIT_OP_MAC: res = A + (float)ldexp((double)B * Cc, -in->shift); break;
              case MERIT_OP_MAX: res = (A < B) ? B : A; break;
              case MERIT_OP_MIN: res = (B < A) ? B : A; break;
              case MERIT_OP_SEL: res = A != 0.0f ? B : Cc; break;
              case MERIT_OP_BAND: res = (float)(llroundf(A) & llroundf(B)); break;
              case MERIT_OP_BOR: res = (float)(llroundf(A) | llroundf(B)); break;
              case MERIT_OP_BXOR: res = (float)(llroundf(A) ^ llroundf(B)); break;
              case MERIT_OP_BNOT: res = (float)(~llroundf(A)); break;
              case MERIT_OP_IDX: res = (float)k[in->aux]; break;
              case MERIT_OP_LUT: res = (float)table_lookup(&P->tables[in->aux], (double)A, &err); break;
              case MERIT_OP_MOVC: res = (float)P->constants[in->aux]; break;
              case MERIT_OP_DIV:
                if (B == 0.0f) return MERIT_E_DIV_BY_ZERO;
                res = (float)((double)A / (double)B);
                break;
              default: return MERIT_E_BAD_PARAMS;
            }
            if (err) return err;
            if (in->dst_out) {
              if (emitted < P->outputs) ((float*)out)[row * P->outputs + emitted] = res;
              ++emitted;
            } else {
              fr[in->dst_reg] = res;
            }
          } else {
            int32_t o[3];
            for (int z = 0; z < 3; ++z)
              o[z] = kinds[z] == MERIT_OPND_REG ? qr[regs[z]] : kinds[z] == MERIT_OPND_PORT_A ? (int32_t)va
                     : kinds[z] == MERIT_OPND_PORT_B ? (int32_t)vb : 0;
            const int32_t A = o[0], B = o[1], Cc = o[2];
            const int s = in->shift;
            int32_t res = 0;
            int err = 0;
            switch (in->op) {
              case MERIT_OP_ADD: res = sat16((int64_t)(A + (int32_t)(((int64_t)B + Cc) >> s))); break;
              case MERIT_OP_SUB: res = sat16((int64_t)(A + (int32_t)(((int64_t)B - Cc) >> s))); break;
              case MERIT_OP_L1: {
                int64_t dd = (int64_t)B - Cc;
                res = sat16((int64_t)(A + (int32_t)((dd < 0 ? -dd : dd) >> s)));
                break;
              }
              case MERIT_OP_MAC: res = sat16((int64_t)(A + (int32_t)(((int64_t)B * Cc) >> s))); break;
              case MERIT_OP_MAX: res = sat16(A < B ? B : A); break;
              case MERIT_OP_MIN: res = sat16(B < A ? B : A); break;
              case MERIT_OP_SEL: res = A != 0 ? B : Cc; break;
              case MERIT_OP_BAND: res = sat16((int64_t)A & (int64_t)B); break;
              case MERIT_OP_BOR: res = sat16((int64_t)A | (int64_t)B); break;
              case MERIT_OP_BXOR: res = sat16((int64_t)A ^ (int64_t)B); break;
              case MERIT_OP_BNOT: res = sat16(~(int64_t)A); break;
              case MERIT_OP_IDX: res = sat16(k[in->aux]); break;
              case MERIT_OP_LUT: res = sat16(llround(table_lookup(&P->tables[in->aux], (double)A, &err))); break;
              case MERIT_OP_MOVC: res = sat16(llround(P->constants[in->aux])); break;
              default: return MERIT_E_BAD_PARAMS;
            }
            if (err) return err;
            if (in->dst_out) {
              if (emitted < P->outputs) ((int16_t*)out)[row * P->outputs + emitted] = (int16_t)sat16(res);
              ++emitted;
            } else {
              qr[in->dst_reg] = res;
            }
          }
        }
      int i = D - 1;
      for (; i >= 0; --i) {
        if (++k[pr + i] < d->view_a.a_shape[i]) break;
        k[pr + i] = 0;
      }
      if (i < 0) break;
    }
    if (emitted != P->outputs) return MERIT_E_BAD_PARAMS;
  }
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
