"""Workload templates and the five BASELINE configurations.

The template builders mirror the reference's (workloads.hpp:47-406: same
views, same programs) so that a reference caller's workload lowers onto the
device unchanged; the ``config_*`` builders are the batched custom ViewSpecs
of SURVEY.md §8(a) A1 (a leading batch / frame-pair p-axis added to the
single-image templates).  Inputs are synthesised by the library's SplitMix64
generators (workloads.hpp:74-105) so tests, the oracle and the benchmark see
identical bytes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Optional, Tuple

import numpy as np

from . import _capi
from .merit import (AluInstr, Boundary, Dst, Dtype, LookupTable, Op, Operand, StrategyProgram,
                    ViewSpec, ViewTerm, Workload, Error, ErrorCode)

Z = Operand.zero


# ---------------------------------------------------------------- programs --
def mac_program(depth: int, shift: int) -> StrategyProgram:
    """workloads.hpp:47-61: r0 <- 0 at Pre_1, r0 += (a*b)>>s, emit r0 at Post_1."""
    p = StrategyProgram(depth=depth, segments=[[] for _ in range(2 * depth + 1)])
    p.segments[p.pre(1)].append(AluInstr(Op.ADD, Dst.r(0), Z(), Z(), Z(), 0, 0))
    p.segments[p.body()].append(AluInstr(Op.MAC, Dst.r(0), Operand.r(0), Operand.a(),
                                         Operand.b(), shift, 0))
    p.segments[p.post(1)].append(AluInstr(Op.ADD, Dst.emit(), Operand.r(0), Z(), Z(), 0, 0))
    return p


def sad_program(depth: int) -> StrategyProgram:
    """workloads.hpp:64-68: the MAC skeleton with L1 as the product function."""
    p = mac_program(depth, 0)
    p.segments[p.body()][0].op = Op.L1
    return p


def maxpool_program(fix: bool = False) -> StrategyProgram:
    """workloads.hpp:376-385."""
    p = StrategyProgram(depth=2, segments=[[] for _ in range(5)])
    p.constants = [-32768.0 if fix else -3.0e38]
    p.segments[p.pre(1)] = [AluInstr(Op.MOVC, Dst.r(0), Z(), Z(), Z(), 0, 0)]
    p.segments[p.body()] = [AluInstr(Op.MAX, Dst.r(0), Operand.r(0), Operand.a(), Z(), 0, 0)]
    p.segments[p.post(1)] = [AluInstr(Op.ADD, Dst.emit(), Operand.r(0), Z(), Z(), 0, 0)]
    return p


def relu_post(p: StrategyProgram) -> StrategyProgram:
    """relu_fused_conv's Post_1 (workloads.hpp:197-202)."""
    p.segments[p.post(1)] = [AluInstr(Op.MAX, Dst.emit(), Operand.r(0), Z(), Z(), 0, 0)]
    return p


# --------------------------------------------------------------- templates --
def _iparam(prm: Dict[str, float], key: str, default: int) -> int:
    v = prm.get(key, default)
    if float(v) != int(v):
        raise Error(ErrorCode.BadParams, f"{key} must be an integer")
    return int(v)


def _ipos(prm, key, default):
    v = _iparam(prm, key, default)
    if v < 1:
        raise Error(ErrorCode.BadParams, f"{key} must be positive")
    return v


@dataclass
class ConvGeom:  # workloads.hpp:138-160
    cin: int
    cout: int
    h: int
    wd: int
    k: int
    stride: int
    dilation: int
    pad: int
    ho: int
    wo: int


def conv_geom(prm, def_dilation: int, def_pad_same: bool) -> ConvGeom:
    cin, cout = _ipos(prm, "cin", 1), _ipos(prm, "cout", 1)
    h, wd, k = _ipos(prm, "h", 32), _ipos(prm, "w", 32), _ipos(prm, "k", 3)
    stride = _ipos(prm, "stride", 1)
    dil = _ipos(prm, "dilation", def_dilation)
    pad = _iparam(prm, "pad", ((k - 1) * dil) // 2 if def_pad_same else 0)
    span = (k - 1) * dil + 1
    ho = (h + 2 * pad - span) // stride + 1
    wo = (wd + 2 * pad - span) // stride + 1
    if ho < 1 or wo < 1:
        raise Error(ErrorCode.BadParams, "kernel larger than padded image")
    return ConvGeom(cin, cout, h, wd, k, stride, dil, pad, ho, wo)


def _src(shape, fix):
    return np.zeros(shape, dtype=np.int16 if fix else np.float32)


def build_conv2d(g: ConvGeom, fix: bool = False, frac: int = 8, fuse_relu: bool = False) -> Workload:
    """workloads.hpp:164-204."""
    if g.cin == 1 and g.cout == 1:
        va = ViewSpec([g.h, g.wd], [g.ho, g.wo], [g.k, g.k],
                      [ViewTerm(0, 0, g.stride, 0), ViewTerm(2, 0, g.dilation, -g.pad),
                       ViewTerm(1, 1, g.stride, 0), ViewTerm(3, 1, g.dilation, -g.pad)])
        vb = ViewSpec([g.k, g.k], [g.ho, g.wo], [g.k, g.k], [ViewTerm(2, 0, 1, 0), ViewTerm(3, 1, 1, 0)])
        w = Workload(va, vb, _src([g.h, g.wd], fix), _src([g.k, g.k], fix), mac_program(2, frac if fix else 0))
    else:
        va = ViewSpec([g.cin, g.h, g.wd], [g.cout, g.ho, g.wo], [g.cin, g.k, g.k],
                      [ViewTerm(3, 0, 1, 0), ViewTerm(1, 1, g.stride, 0),
                       ViewTerm(4, 1, g.dilation, -g.pad), ViewTerm(2, 2, g.stride, 0),
                       ViewTerm(5, 2, g.dilation, -g.pad)])
        vb = ViewSpec([g.cout, g.cin, g.k, g.k], [g.cout, g.ho, g.wo], [g.cin, g.k, g.k],
                      [ViewTerm(0, 0, 1, 0), ViewTerm(3, 1, 1, 0), ViewTerm(4, 2, 1, 0),
                       ViewTerm(5, 3, 1, 0)])
        w = Workload(va, vb, _src([g.cin, g.h, g.wd], fix), _src([g.cout, g.cin, g.k, g.k], fix),
                     mac_program(3, frac if fix else 0))
    if fuse_relu:
        relu_post(w.program)
    if fix:
        w.frac_bits = frac
    return w


def build_gemm(prm) -> Workload:
    """workloads.hpp:122-136."""
    m, n, k = _ipos(prm, "m", 8), _ipos(prm, "n", 8), _ipos(prm, "k", 8)
    fix = _iparam(prm, "fix", 0) != 0
    frac = _iparam(prm, "frac", 8)
    va = ViewSpec([m, k], [m, n], [k], [ViewTerm(0, 0, 1, 0), ViewTerm(2, 1, 1, 0)])
    vb = ViewSpec([k, n], [m, n], [k], [ViewTerm(2, 0, 1, 0), ViewTerm(1, 1, 1, 0)])
    w = Workload(va, vb, _src([m, k], fix), _src([k, n], fix), mac_program(1, frac if fix else 0))
    w.frac_bits = frac if fix else 0
    return w


def build_alexnet_conv1(prm) -> Workload:
    """workloads.hpp:208-228."""
    h, wd = _ipos(prm, "h", 227), _ipos(prm, "w", 227)
    va = ViewSpec([3, h, wd], [48, 55, 55], [3, 11, 11],
                  [ViewTerm(3, 0, 1, 0), ViewTerm(1, 1, 4, 0), ViewTerm(4, 1, 1, -5),
                   ViewTerm(2, 2, 4, 0), ViewTerm(5, 2, 1, -5)])
    vb = ViewSpec([48, 3, 11, 11], [48, 55, 55], [3, 11, 11],
                  [ViewTerm(0, 0, 1, 0), ViewTerm(3, 1, 1, 0), ViewTerm(4, 2, 1, 0), ViewTerm(5, 3, 1, 0)])
    return Workload(va, vb, _src([3, h, wd], False), _src([48, 3, 11, 11], False), mac_program(3, 0))


def build_correlation(prm) -> Workload:
    """workloads.hpp:232-251."""
    c, h, wd, d = _ipos(prm, "c", 3), _ipos(prm, "h", 8), _ipos(prm, "w", 8), _ipos(prm, "d", 3)
    va = ViewSpec([c, h, wd], [h, wd, d, d], [c],
                  [ViewTerm(4, 0, 1, 0), ViewTerm(0, 1, 1, 0), ViewTerm(1, 2, 1, 0)])
    vb = ViewSpec([c, h, wd], [h, wd, d, d], [c],
                  [ViewTerm(4, 0, 1, 0), ViewTerm(0, 1, 1, 0), ViewTerm(2, 1, 1, 0),
                   ViewTerm(1, 2, 1, 0), ViewTerm(3, 2, 1, 0)])
    return Workload(va, vb, _src([c, h, wd], False), _src([c, h, wd], False), mac_program(1, 0))


def build_motion_estimation(prm) -> Workload:
    """workloads.hpp:255-279."""
    h, wd = _ipos(prm, "h", 16), _ipos(prm, "w", 16)
    blk, win = _ipos(prm, "blk", 4), _ipos(prm, "win", 3)
    fix = _iparam(prm, "fix", 0) != 0
    frac = _iparam(prm, "frac", 8)
    if h % blk or wd % blk:
        raise Error(ErrorCode.BadParams, "frame extents must be block multiples")
    by, bx = h // blk, wd // blk
    va = ViewSpec([h, wd], [by, bx, win, win], [blk, blk],
                  [ViewTerm(0, 0, blk, 0), ViewTerm(4, 0, 1, 0), ViewTerm(1, 1, blk, 0), ViewTerm(5, 1, 1, 0)])
    vb = ViewSpec([h, wd], [by, bx, win, win], [blk, blk],
                  [ViewTerm(0, 0, blk, 0), ViewTerm(2, 0, 1, -(win // 2)), ViewTerm(4, 0, 1, 0),
                   ViewTerm(1, 1, blk, 0), ViewTerm(3, 1, 1, -(win // 2)), ViewTerm(5, 1, 1, 0)])
    w = Workload(va, vb, _src([h, wd], fix), _src([h, wd], fix), sad_program(2))
    w.frac_bits = frac if fix else 0
    return w


def build_bilateral(prm) -> Workload:
    """workloads.hpp:285-349 (REAL32 only: uses LUT and DIV)."""
    import math
    if _iparam(prm, "fix", 0):
        raise Error(ErrorCode.BadParams, "bilateral is REAL32-only (uses DIV)")
    h, wd, k = _ipos(prm, "h", 16), _ipos(prm, "w", 16), _ipos(prm, "k", 5)
    sigma_r = float(prm.get("sigma_r", 0.5))
    sigma_s = float(prm.get("sigma_s", k / 3.0))
    rng_ = float(prm.get("range", 2.0))
    if sigma_r <= 0 or sigma_s <= 0 or rng_ <= 0:
        raise Error(ErrorCode.BadParams, "sigmas and range must be positive")
    va = ViewSpec([h, wd], [h, wd], [k, k],
                  [ViewTerm(0, 0, 1, 0), ViewTerm(2, 0, 1, -(k // 2)), ViewTerm(1, 1, 1, 0),
                   ViewTerm(3, 1, 1, -(k // 2))], Boundary.Clamp)
    vb = ViewSpec([h, wd], [h, wd], [k, k], [ViewTerm(0, 0, 1, 0), ViewTerm(1, 1, 1, 0)])
    rl = LookupTable(-rng_, rng_, [], True)
    for i in range(256):
        d = -rng_ + 2.0 * rng_ * i / 255.0
        rl.samples.append(math.exp(-d * d / (2.0 * sigma_r * sigma_r)))
    sl = LookupTable(0.0, float(k - 1), [], True)
    for i in range(k):
        d = float(i - k // 2)
        sl.samples.append(math.exp(-d * d / (2.0 * sigma_s * sigma_s)))
    p = StrategyProgram(depth=2, segments=[[] for _ in range(5)], tables=[rl, sl])
    r = Operand.r
    p.segments[p.pre(1)] = [AluInstr(Op.ADD, Dst.r(0), Z(), Z(), Z()),
                            AluInstr(Op.ADD, Dst.r(1), Z(), Z(), Z())]
    p.segments[p.body()] = [
        AluInstr(Op.SUB, Dst.r(2), Z(), Operand.b(), Operand.a()),
        AluInstr(Op.LUT, Dst.r(3), r(2), Z(), Z(), 0, 0),
        AluInstr(Op.IDX, Dst.r(4), Z(), Z(), Z(), 0, 2),
        AluInstr(Op.LUT, Dst.r(4), r(4), Z(), Z(), 0, 1),
        AluInstr(Op.IDX, Dst.r(5), Z(), Z(), Z(), 0, 3),
        AluInstr(Op.LUT, Dst.r(5), r(5), Z(), Z(), 0, 1),
        AluInstr(Op.MAC, Dst.r(6), Z(), r(3), r(4)),
        AluInstr(Op.MAC, Dst.r(6), Z(), r(6), r(5)),
        AluInstr(Op.ADD, Dst.r(0), r(0), r(6), Z()),
        AluInstr(Op.MAC, Dst.r(1), r(1), r(6), Operand.a()),
    ]
    p.segments[p.post(1)] = [AluInstr(Op.DIV, Dst.emit(), r(1), r(0), Z())]
    return Workload(va, vb, _src([h, wd], False), _src([h, wd], False), p)


def build_maxpool(prm) -> Workload:
    """workloads.hpp:353-387 (REJECT boundary, windows inside the image)."""
    h, wd, k = _ipos(prm, "h", 8), _ipos(prm, "w", 8), _ipos(prm, "k", 2)
    stride = _ipos(prm, "stride", k)
    fix = _iparam(prm, "fix", 0) != 0
    frac = _iparam(prm, "frac", 8)
    if h < k or wd < k:
        raise Error(ErrorCode.BadParams, "window larger than image")
    ho, wo = (h - k) // stride + 1, (wd - k) // stride + 1
    va = ViewSpec([h, wd], [ho, wo], [k, k],
                  [ViewTerm(0, 0, stride, 0), ViewTerm(2, 0, 1, 0), ViewTerm(1, 1, stride, 0),
                   ViewTerm(3, 1, 1, 0)], Boundary.Reject)
    vb = ViewSpec([1], [ho, wo], [k, k], [])
    w = Workload(va, vb, _src([h, wd], fix), _src([1], fix), maxpool_program(fix))
    w.frac_bits = frac if fix else 0
    return w


TEMPLATES = ("gemm", "conv2d", "dilated", "alexnet_conv1", "correlation", "bilateral",
             "motion_estimation", "maxpool", "relu_fused_conv")


def build_template(name: str, prm: Optional[Dict[str, float]] = None) -> Workload:
    """workloads.hpp:391-406."""
    prm = dict(prm or {})
    fix = _iparam(prm, "fix", 0) != 0
    frac = _iparam(prm, "frac", 8)
    if name == "gemm":
        return build_gemm(prm)
    if name == "conv2d":
        return build_conv2d(conv_geom(prm, 1, True), fix, frac, False)
    if name == "dilated":
        return build_conv2d(conv_geom(prm, 2, False), fix, frac, False)
    if name == "relu_fused_conv":
        return build_conv2d(conv_geom(prm, 1, True), fix, frac, True)
    if name == "alexnet_conv1":
        return build_alexnet_conv1(prm)
    if name == "correlation":
        return build_correlation(prm)
    if name == "motion_estimation":
        return build_motion_estimation(prm)
    if name == "bilateral":
        return build_bilateral(prm)
    if name == "maxpool":
        return build_maxpool(prm)
    raise Error(ErrorCode.UnknownTemplate, "unknown template " + name)


def template_shares_input(name: str) -> bool:  # workloads.hpp:109-111
    return name == "bilateral"


# ---------------------------------------------------- batched config views --
def maxpool_nchw_view(n, c, h, w, k=3, stride=2, pad=1) -> Workload:
    """C1: 2-D max-pool over NCHW with -inf padding expressed as CLAMP
    (CLAMP == -inf pad for max)."""
    ho = (h + 2 * pad - k) // stride + 1
    wo = (w + 2 * pad - k) // stride + 1
    va = ViewSpec([n, c, h, w], [n, c, ho, wo], [k, k],
                  [ViewTerm(0, 0, 1, 0), ViewTerm(1, 1, 1, 0), ViewTerm(2, 2, stride, -pad),
                   ViewTerm(4, 2, 1, 0), ViewTerm(3, 3, stride, -pad), ViewTerm(5, 3, 1, 0)],
                  Boundary.Clamp)
    vb = ViewSpec([1], [n, c, ho, wo], [k, k], [])
    return Workload(va, vb, None, np.zeros([1], np.float32), maxpool_program(False))


def me_view(h, w, blk, radius, pairs: Optional[int] = None) -> Workload:
    """C2/C5: block matching with floor(h/blk) block rows (oracle_motion_estimation
    semantics, workloads.hpp:556), ZERO_PAD reference; optional frame-pair axis."""
    by, bx, win = h // blk, w // blk, 2 * radius + 1
    lead = 1 if pairs is not None else 0
    src = ([pairs] if lead else []) + [h, w]
    p = ([pairs] if lead else []) + [by, bx, win, win]
    P = len(p)
    t_pair = [ViewTerm(0, 0, 1, 0)] if lead else []
    cy, cx, dy, dx, i, j = lead, lead + 1, lead + 2, lead + 3, P, P + 1
    va = ViewSpec(src, p, [blk, blk], t_pair + [
        ViewTerm(cy, lead, blk, 0), ViewTerm(i, lead, 1, 0),
        ViewTerm(cx, lead + 1, blk, 0), ViewTerm(j, lead + 1, 1, 0)])
    vb = ViewSpec(src, p, [blk, blk], t_pair + [
        ViewTerm(cy, lead, blk, 0), ViewTerm(dy, lead, 1, -radius), ViewTerm(i, lead, 1, 0),
        ViewTerm(cx, lead + 1, blk, 0), ViewTerm(dx, lead + 1, 1, -radius), ViewTerm(j, lead + 1, 1, 0)],
        Boundary.ZeroPad)
    return Workload(va, vb, None, None, sad_program(2), dtype_a=Dtype.U8, dtype_b=Dtype.U8,
                    dtype_out=Dtype.I32)


def conv_nchw_view(n, cin, h, w, cout, k=3, stride=1, pad=1, dilation=1, relu=False) -> Workload:
    """C3/C4: batched NCHW conv; p = (n, co, y, x), a = (ci, ky, kx)."""
    ho = (h + 2 * pad - ((k - 1) * dilation + 1)) // stride + 1
    wo = (w + 2 * pad - ((k - 1) * dilation + 1)) // stride + 1
    va = ViewSpec([n, cin, h, w], [n, cout, ho, wo], [cin, k, k],
                  [ViewTerm(0, 0, 1, 0), ViewTerm(4, 1, 1, 0),
                   ViewTerm(2, 2, stride, 0), ViewTerm(5, 2, dilation, -pad),
                   ViewTerm(3, 3, stride, 0), ViewTerm(6, 3, dilation, -pad)])
    vb = ViewSpec([cout, cin, k, k], [n, cout, ho, wo], [cin, k, k],
                  [ViewTerm(1, 0, 1, 0), ViewTerm(4, 1, 1, 0), ViewTerm(5, 2, 1, 0), ViewTerm(6, 3, 1, 0)])
    prog = mac_program(3, 0)
    if relu:
        relu_post(prog)
    return Workload(va, vb, None, None, prog)


# ------------------------------------------------------------- generators --
def gen_uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """fill_random (workloads.hpp:96-105) for REAL32."""
    out = np.empty(shape, dtype=np.float32)
    _capi.load().merit_gen_uniform_f32(out.ctypes.data_as(C.c_void_p), out.size, seed, lo, hi)
    return out


def gen_range_i16(shape, seed: int, lo: int = -256, hi: int = 256) -> np.ndarray:
    """fill_random (workloads.hpp:102-103) for FIX16."""
    out = np.empty(shape, dtype=np.int16)
    _capi.load().merit_gen_range_i16(out.ctypes.data_as(C.c_void_p), out.size, seed, lo, hi)
    return out


def fill_random(w: Workload, seed_a: int, seed_b: int):
    """The reference tests' fill_random(src_a, 2s+1), fill_random(src_b, 2s+2)."""
    for attr, seed in (("src_a", seed_a), ("src_b", seed_b)):
        src = getattr(w, attr)
        if src.dtype == np.int16:
            setattr(w, attr, gen_range_i16(src.shape, seed))
        else:
            setattr(w, attr, gen_uniform(src.shape, seed))
    return w


def gen_normal(shape, seed: int, sigma: float) -> np.ndarray:
    out = np.empty(shape, dtype=np.float32)
    _capi.load().merit_gen_normal_f32(out.ctypes.data_as(C.c_void_p), out.size, seed, sigma)
    return out


def gen_me_pair(h: int, w: int, seed: int, blk: int = 16, max_shift: int = 16,
                noise: int = 4) -> Tuple[np.ndarray, np.ndarray]:
    """SURVEY §8(d) C2 frame generator: (cur, ref) uint8 frames."""
    cur = np.empty((h, w), dtype=np.uint8)
    ref = np.empty((h, w), dtype=np.uint8)
    _capi.load().merit_gen_me_pair(cur.ctypes.data_as(C.c_void_p), ref.ctypes.data_as(C.c_void_p),
                                   h, w, blk, max_shift, noise, seed)
    return cur, ref


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) as uint16 bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    _capi.load().merit_f32_to_bf16(x.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), x.size)
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------- config inputs --
CONFIGS = {
    "C1": "maxpool 3x3 s2 p1 (-inf) fp32 NCHW (8,64,112,112)",
    "C2": "motion estimation 1920x1080 u8, 16x16 blocks, +/-16, SAD int32 + argmin",
    "C3": "conv fp32 NCHW (32,64,56,56) * (64,64,3,3) s1 p1",
    "C4": "conv bf16 NCHW (256,128,56,56) * (256,128,3,3) s2 p1, fp32 accumulate",
    "C5": "motion estimation 3840x2160 u8 x64 pairs, 8x8 and 16x16 blocks, +/-32",
}


def config_workload(name: str, scale: int = 1, seed_offset: int = 0, with_inputs: bool = True,
                    pairs: Optional[int] = None, blk: int = 16):
    """Build config C1..C5.  ``scale`` divides the batch (for
    shards / small parity runs); inputs are generated with the survey's seeds."""
    if name == "C1":
        n = max(1, 8 // scale)
        w = maxpool_nchw_view(n, 64, 112, 112)
        if with_inputs:
            w.src_a = gen_uniform([n, 64, 112, 112], 1 + seed_offset)
        return w
    if name == "C2":
        w = me_view(1080, 1920, 16, 16)
        if with_inputs:
            cur, ref = gen_me_pair(1080, 1920, 2 + seed_offset)
            w.src_a, w.src_b = cur, ref
        return w
    if name == "C3":
        n = max(1, 32 // scale)
        w = conv_nchw_view(n, 64, 56, 56, 64, 3, 1, 1)
        if with_inputs:
            w.src_a = gen_uniform([n, 64, 56, 56], 3 + seed_offset)
            w.src_b = gen_normal([64, 64, 3, 3], 1003 + seed_offset, (2.0 / 576) ** 0.5)
        return w
    if name == "C4":
        n = max(1, 256 // scale)
        w = conv_nchw_view(n, 128, 56, 56, 256, 3, 2, 1)
        w.dtype_a = Dtype.BF16
        w.dtype_b = Dtype.BF16
        if with_inputs:
            x = gen_uniform([n, 128, 56, 56], 4 + seed_offset)
            wt = gen_normal([256, 128, 3, 3], 1004 + seed_offset, (2.0 / 1152) ** 0.5)
            w.src_a, w.src_b = to_bf16_bits(x), to_bf16_bits(wt)
            w.fp32_inputs = (x, wt)
        return w
    if name == "C5":
        npairs = pairs if pairs is not None else max(1, 64 // scale)
        w = me_view(2160, 3840, blk, 32, pairs=npairs)
        if with_inputs:
            cur = np.empty((npairs, 2160, 3840), np.uint8)
            ref = np.empty((npairs, 2160, 3840), np.uint8)
            for i in range(npairs):
                cur[i], ref[i] = gen_me_pair(2160, 3840, 5 + i + seed_offset, 16, 16, 4)
            w.src_a, w.src_b = cur, ref
        return w
    raise KeyError(name)
