// K0 — exact device interpreter of a MERIT workload.
//
// One thread per output row p (engine.hpp:120-143 run_full_typed): a fresh
// 16-register file (rip.hpp:215-217), the accumulation index a walked in
// row-major order (tensor.hpp:59-65 next_index), the phase segment range from
// the trailing-zero / trailing-max counts of a (rip.hpp:112-126), both ports
// gathered through the affine view with its boundary rule (view.hpp:68-84),
// and every ALU op evaluated with the reference's exact scalar semantics for
// Real32Mode (float values, double intermediates, rip.hpp:130-142) or
// Fix16Mode (int32 values saturated to int16, rip.hpp:144-158).
// It is bit-exact with the reference engine and serves every program the
// specialised kernels do not recognise (gemm, correlation, bilateral, FIX16,
// dilated/strided convolutions when exactness is requested).
#include <cmath>

#include "common.cuh"

namespace merit_dev {
namespace {

struct GenArgs {
  GenericParams g;
  const ProgramImage* prog;
  const void* a;
  const void* b;
  void* out;
  int32_t* err;
  const int32_t* run_if;  // non-null: run only if *run_if != 0 (fallback of a narrowed SAD plan)
};

__device__ __forceinline__ void raise_err(int32_t* err, int code) { atomicCAS(err, 0, code); }

__device__ __forceinline__ int32_t sat16(long long v) {
  return v < -32768 ? -32768 : v > 32767 ? 32767 : static_cast<int32_t>(v);
}

// Gather one element (view_gather, view.hpp:68-84).  Returns false and raises
// OutOfRange for REJECT.
__device__ bool gather(const ViewAffine& f, const long long* k, int krank, const void* src,
                       int dtype, double& val, int32_t* err) {
  long long flat = 0;
  bool zero = false;
  for (int i = 0; i < f.src_rank; ++i) {
    long long x = f.off[i];
    for (int j = 0; j < krank; ++j) x += f.coef[i][j] * k[j];
    const long long n = f.src_shape[i];
    if (x < 0 || x >= n) {
      if (f.boundary == MERIT_ZERO_PAD) {
        zero = true;
      } else if (f.boundary == MERIT_CLAMP) {
        x = x < 0 ? 0 : n - 1;
      } else {
        raise_err(err, MERIT_E_OUT_OF_RANGE);
        return false;
      }
    }
    flat = flat * n + x;
  }
  if (zero) {
    val = 0.0;
    return true;
  }
  switch (dtype) {
    case MERIT_F32: val = static_cast<const float*>(src)[flat]; break;
    case MERIT_I16: val = static_cast<const int16_t*>(src)[flat]; break;
    case MERIT_U8: val = static_cast<const uint8_t*>(src)[flat]; break;
    case MERIT_I32: val = static_cast<const int32_t*>(src)[flat]; break;
    case MERIT_BF16: {
      uint32_t u = static_cast<uint32_t>(static_cast<const uint16_t*>(src)[flat]) << 16;
      val = __uint_as_float(u);
      break;
    }
    default: val = 0.0;
  }
  return true;
}

// LookupTable::lookup (rip.hpp:66-77).
__device__ bool lut(const ProgramImage& P, int t, double x, double& y, int32_t* err) {
  const double lo = P.tab_lo[t], hi = P.tab_hi[t];
  const int n = P.tab_n[t];
  const double* s = P.table_samples + P.tab_off[t];
  if (x < lo || x > hi) {
    if (!P.tab_clamp[t]) {
      raise_err(err, MERIT_E_LUT_RANGE);
      return false;
    }
    x = x < lo ? lo : hi;  // std::clamp
  }
  if (n == 1) {
    y = s[0];
    return true;
  }
  double tt = (x - lo) / (hi - lo) * static_cast<double>(n - 1);
  unsigned long long i = static_cast<unsigned long long>(tt);
  if (i >= static_cast<unsigned long long>(n - 1)) {
    y = s[n - 1];
    return true;
  }
  double fr = tt - static_cast<double>(i);
  y = s[i] * (1.0 - fr) + s[i + 1] * fr;
  return true;
}

// Real32Mode scalar ALU (rip.hpp:160-200 with Real32Mode).  The compiler
// must not contract products into FMAs here: every step is written with
// explicit round-to-nearest intrinsics.
__device__ __forceinline__ float r32_shift(double v, int s) {
  return __double2float_rn(ldexp(v, -s));
}

__global__ void generic_kernel(GenArgs A) {
  const GenericParams& g = A.g;
  const ProgramImage& P = *A.prog;
  const long long row = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  pdl_launch_dependents();
  pdl_wait();
  if (row >= g.rows) return;
  if (A.run_if && *A.run_if == 0) return;
  long long k[kMaxK];
  // p index of this row (row-major, tensor.hpp:59-65)
  long long r = row;
  for (int i = g.p_rank - 1; i >= 0; --i) {
    k[i] = r % g.p_shape[i];
    r /= g.p_shape[i];
  }
  const int D = g.a_rank;
  const int krank = g.p_rank + D;
  for (int i = 0; i < D; ++i) k[g.p_rank + i] = 0;
  const int outputs = P.outputs;
  int emitted = 0;
  float fr[16];
  int32_t qr[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    fr[i] = 0.f;
    qr[i] = 0;
  }
  for (;;) {
    // phase_range (rip.hpp:112-126)
    int zeros = 0;
    while (zeros < D && k[g.p_rank + D - 1 - zeros] == 0) ++zeros;
    int maxed = 0;
    while (maxed < D && k[g.p_rank + D - 1 - maxed] == g.a_shape[D - 1 - maxed] - 1) ++maxed;
    const int first = zeros > 0 ? D - zeros : D;
    const int last = maxed > 0 ? D + maxed : D;
    double va = 0.0, vb = 0.0;
    if (!gather(g.va, k, krank, A.a, g.dtype_a, va, A.err)) return;
    if (!gather(g.vb, k, krank, A.b, g.dtype_b, vb, A.err)) return;
    for (int seg = first; seg <= last; ++seg) {
      const int s0 = P.seg_start[seg], n = P.seg_len[seg];
      for (int q = 0; q < n; ++q) {
        const merit_alu_instr in = P.instrs[s0 + q];
        if (!g.fix16) {
          const float pa = static_cast<float>(va), pb = static_cast<float>(vb);
          auto rd = [&](int kind, int reg) -> float {
            return kind == MERIT_OPND_REG ? fr[reg]
                   : kind == MERIT_OPND_PORT_A ? pa
                   : kind == MERIT_OPND_PORT_B ? pb
                                               : 0.f;
          };
          const float a = rd(in.a_kind, in.a_reg), b = rd(in.b_kind, in.b_reg),
                      c = rd(in.c_kind, in.c_reg);
          float res = 0.f;
          switch (in.op) {
            case MERIT_OP_ADD: res = __fadd_rn(a, r32_shift(__dadd_rn((double)b, (double)c), in.shift)); break;
            case MERIT_OP_SUB: res = __fadd_rn(a, r32_shift(__dsub_rn((double)b, (double)c), in.shift)); break;
            case MERIT_OP_L1: res = __fadd_rn(a, r32_shift(fabs(__dsub_rn((double)b, (double)c)), in.shift)); break;
            case MERIT_OP_MAC: res = __fadd_rn(a, r32_shift(__dmul_rn((double)b, (double)c), in.shift)); break;
            case MERIT_OP_MAX: res = (a < b) ? b : a; break;
            case MERIT_OP_MIN: res = (b < a) ? b : a; break;
            case MERIT_OP_SEL: res = a != 0.f ? b : c; break;
            case MERIT_OP_BAND: res = static_cast<float>(llroundf(a) & llroundf(b)); break;
            case MERIT_OP_BOR: res = static_cast<float>(llroundf(a) | llroundf(b)); break;
            case MERIT_OP_BXOR: res = static_cast<float>(llroundf(a) ^ llroundf(b)); break;
            case MERIT_OP_BNOT: res = static_cast<float>(~llroundf(a)); break;
            case MERIT_OP_IDX:
              if (in.aux < 0 || in.aux >= krank) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              res = static_cast<float>(k[in.aux]);
              break;
            case MERIT_OP_LUT: {
              if (in.aux < 0 || in.aux >= P.n_tables) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              double y;
              if (!lut(P, in.aux, static_cast<double>(a), y, A.err)) return;
              res = static_cast<float>(y);
              break;
            }
            case MERIT_OP_MOVC:
              if (in.aux < 0 || in.aux >= P.n_constants) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              res = static_cast<float>(P.constants[in.aux]);
              break;
            case MERIT_OP_DIV:
              if (b == 0.f) { raise_err(A.err, MERIT_E_DIV_BY_ZERO); return; }
              res = __double2float_rn(__ddiv_rn((double)a, (double)b));
              break;
            default: raise_err(A.err, MERIT_E_BAD_PARAMS); return;
          }
          if (in.dst_out) {
            if (emitted < outputs) static_cast<float*>(A.out)[row * outputs + emitted] = res;
            ++emitted;
          } else {
            fr[in.dst_reg] = res;
          }
        } else {
          const int32_t pa = static_cast<int32_t>(va), pb = static_cast<int32_t>(vb);
          auto rd = [&](int kind, int reg) -> int32_t {
            return kind == MERIT_OPND_REG ? qr[reg]
                   : kind == MERIT_OPND_PORT_A ? pa
                   : kind == MERIT_OPND_PORT_B ? pb
                                               : 0;
          };
          const int32_t a = rd(in.a_kind, in.a_reg), b = rd(in.b_kind, in.b_reg),
                        c = rd(in.c_kind, in.c_reg);
          int32_t res = 0;
          const int s = in.shift;
          switch (in.op) {
            case MERIT_OP_ADD: res = sat16((long long)(a + static_cast<int32_t>(((long long)b + c) >> s))); break;
            case MERIT_OP_SUB: res = sat16((long long)(a + static_cast<int32_t>(((long long)b - c) >> s))); break;
            case MERIT_OP_L1: {
              long long d = (long long)b - c;
              d = d < 0 ? -d : d;
              res = sat16((long long)(a + static_cast<int32_t>(d >> s)));
              break;
            }
            case MERIT_OP_MAC: res = sat16((long long)(a + static_cast<int32_t>(((long long)b * c) >> s))); break;
            case MERIT_OP_MAX: res = sat16(a < b ? b : a); break;
            case MERIT_OP_MIN: res = sat16(b < a ? b : a); break;
            case MERIT_OP_SEL: res = a != 0 ? b : c; break;
            case MERIT_OP_BAND: res = sat16((long long)a & (long long)b); break;
            case MERIT_OP_BOR: res = sat16((long long)a | (long long)b); break;
            case MERIT_OP_BXOR: res = sat16((long long)a ^ (long long)b); break;
            case MERIT_OP_BNOT: res = sat16(~(long long)a); break;
            case MERIT_OP_IDX:
              if (in.aux < 0 || in.aux >= krank) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              res = sat16(k[in.aux]);
              break;
            case MERIT_OP_LUT: {
              if (in.aux < 0 || in.aux >= P.n_tables) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              double y;
              if (!lut(P, in.aux, static_cast<double>(a), y, A.err)) return;
              res = sat16(llround(y));
              break;
            }
            case MERIT_OP_MOVC:
              if (in.aux < 0 || in.aux >= P.n_constants) { raise_err(A.err, MERIT_E_BAD_PARAMS); return; }
              res = sat16(llround(P.constants[in.aux]));
              break;
            case MERIT_OP_DIV: raise_err(A.err, MERIT_E_BAD_PARAMS); return;  // REAL32-only
            default: raise_err(A.err, MERIT_E_BAD_PARAMS); return;
          }
          if (in.dst_out) {
            if (emitted < outputs)
              static_cast<int16_t*>(A.out)[row * outputs + emitted] = static_cast<int16_t>(sat16(res));
            ++emitted;
          } else {
            qr[in.dst_reg] = res;
          }
        }
      }
    }
    // next_index over a (tensor.hpp:59-65)
    int i = D - 1;
    for (; i >= 0; --i) {
      if (++k[g.p_rank + i] < g.a_shape[i]) break;
      k[g.p_rank + i] = 0;
    }
    if (i < 0) break;
  }
  if (emitted != outputs) raise_err(A.err, MERIT_E_BAD_PARAMS);
}

}  // namespace

merit_status launch_generic(const merit_plan& plan, const void* a, const void* b, void* out,
                            void* stream, const int32_t* run_if) {
  GenArgs args;
  args.run_if = run_if;
  args.g = plan.gen;
  args.prog = static_cast<const ProgramImage*>(plan.d_prog);
  args.a = a;
  args.b = b;
  args.out = out;
  args.err = static_cast<int32_t*>(plan.d_err);
  const int threads = 128;
  const long long blocks = (plan.gen.rows + threads - 1) / threads;
  if (blocks == 0) return MERIT_OK;
  if (blocks > 0x7fffffffLL) return fail(MERIT_E_INVALID_ARGUMENT, "too many rows");
  cudaError_t e = launch_pdl(generic_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0,
                             static_cast<cudaStream_t>(stream), 1, args);
  if (e != cudaSuccess) return cuda_check(e, "launch(generic)");
  return launch_status("generic_kernel");
}

}  // namespace merit_dev
