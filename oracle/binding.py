"""ctypes binding of the test-only checkers (oracle.c and oracle/_ref).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_lib = None
_ref = None


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def lib():
    global _lib
    if _lib is None:
        from . import build as _b
        path = _b.LIB
        if not path.exists():
            _b.build_oracle()
        L = C.CDLL(str(path))
        L.oracle_fill_uniform_f32.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_double]
        L.oracle_fill_range_i16.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int64, C.c_int64]
        L.oracle_gen_normal_f32.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_double]
        L.oracle_f32_to_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_gen_me_pair.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int64] * 5 + [C.c_uint64]
        L.oracle_maxpool.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_int] * 13 + [C.c_float, C.c_int]
        L.oracle_conv2d_nchw.argtypes = [C.c_void_p] * 3 + [C.c_int] * 16
        L.oracle_me_sad.argtypes = [C.c_void_p] * 3 + [C.c_int64] + [C.c_int] * 11
        L.oracle_me_argmin.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_int] * 4
        L.oracle_run_full.argtypes = [C.c_void_p] * 4
        L.oracle_run_full.restype = C.c_int
        L.oracle_num_threads.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    from . import build as _b
    return _b.REF_LIB.exists() or (_b.REF_INCLUDE / "merit" / "engine.hpp").exists()


def ref():
    """The reference itself (oracle/_ref/libmerit_ref.so)."""
    global _ref
    if _ref is None:
        from . import build as _b
        path = _b.build_ref()
        if path is None or not Path(path).exists():
            raise RuntimeError("oracle/_ref/libmerit_ref.so is not built and /root/reference is absent")
        L = C.CDLL(str(path))
        L.ref_run_full.argtypes = [C.c_void_p] * 4
        L.ref_run_full.restype = C.c_int
        L.ref_run_tiled.argtypes = [C.c_void_p] * 3 + [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_run_tiled.restype = C.c_int
        L.ref_run_tiled_caps.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.ref_run_tiled_caps.restype = C.c_int
        L.ref_mrt1_write.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_mrt1_write.restype = C.c_int64
        L.ref_mrt1_read.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_mrt1_read.restype = C.c_int
        L.ref_fill_random_f32.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_double]
        L.ref_fill_random_i16.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        L.ref_template_case.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_void_p,
                                        C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int64),
                                        C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_int64]
        L.ref_template_case.restype = C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_bench_load_frames.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
        L.ref_sample_me.argtypes = [C.c_int64] * 5 + [C.c_int]
        L.ref_sample_me.restype = C.c_int64
        L.ref_bench_load_images.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64]
        L.ref_sample_maxpool.argtypes = [C.c_int]
        L.ref_sample_maxpool.restype = C.c_int64
        L.ref_sample_conv.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int]
        L.ref_sample_conv.restype = C.c_int64
        _ref = L
    return _ref


# ---------------------------------------------------------------- oracle ---
def fill_uniform(n, seed, lo=-1.0, hi=1.0):
    out = np.empty(n, np.float32)
    lib().oracle_fill_uniform_f32(_p(out), n, seed, lo, hi)
    return out


def gen_uniform(shape, seed, lo=-1.0, hi=1.0):
    out = np.empty(shape, np.float32)
    lib().oracle_fill_uniform_f32(_p(out), out.size, seed, lo, hi)
    return out


def gen_normal(shape, seed, sigma):
    out = np.empty(shape, np.float32)
    lib().oracle_gen_normal_f32(_p(out), out.size, seed, sigma)
    return out


def to_bf16_bits(x):
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    lib().oracle_f32_to_bf16(_p(x), _p(out), x.size)
    return out


def gen_me_pair(h, w, seed, blk=16, max_shift=16, noise=4):
    cur = np.empty((h, w), np.uint8)
    ref_ = np.empty((h, w), np.uint8)
    lib().oracle_gen_me_pair(_p(cur), _p(ref_), h, w, blk, max_shift, noise, seed)
    return cur, ref_


def fill_range_i16(n, seed, lo=-256, hi=256):
    out = np.empty(n, np.int16)
    lib().oracle_fill_range_i16(_p(out), n, seed, lo, hi)
    return out


def maxpool(x, Ho, Wo, k=3, stride=2, pad=1, clamp=True, init=-3.0e38, relu=False, KW=None,
            sx=None, ox=None, dil=1):
    x = np.ascontiguousarray(x, np.float32)
    H, W = x.shape[-2:]
    planes = int(np.prod(x.shape[:-2]))
    out = np.empty(x.shape[:-2] + (Ho, Wo), np.float32)
    KW = k if KW is None else KW
    sx = stride if sx is None else sx
    ox = -pad if ox is None else ox
    lib().oracle_maxpool(_p(x), _p(out), planes, H, W, Ho, Wo, k, KW, stride, sx, dil, dil, -pad, ox,
                         int(clamp), C.c_float(init), int(relu))
    return out


def conv2d(x, w, stride=1, pad=1, dilation=1, relu=False, Ho=None, Wo=None):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    N, Cin, H, W = x.shape
    Cout, _, KH, KW = w.shape
    if Ho is None:
        Ho = (H + 2 * pad - ((KH - 1) * dilation + 1)) // stride + 1
        Wo = (W + 2 * pad - ((KW - 1) * dilation + 1)) // stride + 1
    out = np.empty((N, Cout, Ho, Wo), np.float32)
    lib().oracle_conv2d_nchw(_p(x), _p(w), _p(out), N, Cin, H, W, Cout, Ho, Wo, KH, KW, stride,
                             stride, dilation, dilation, -pad, -pad, int(relu))
    return out


def me_sad(cur, ref_, blk, radius, clamp=False):
    cur = np.ascontiguousarray(cur, np.uint8)
    ref_ = np.ascontiguousarray(ref_, np.uint8)
    pairs = 1 if cur.ndim == 2 else cur.shape[0]
    H, W = cur.shape[-2:]
    BY, BX, win = H // blk, W // blk, 2 * radius + 1
    out = np.empty(((pairs,) if cur.ndim == 3 else ()) + (BY, BX, win, win), np.int32)
    lib().oracle_me_sad(_p(cur), _p(ref_), _p(out), pairs, H, W, BY, BX, blk, blk, win, win,
                        -radius, -radius, int(clamp))
    return out


def me_argmin(sad, radius):
    win = sad.shape[-1]
    blocks = int(np.prod(sad.shape[:-2]))
    mv = np.empty((blocks, 3), np.int32)
    lib().oracle_me_argmin(_p(np.ascontiguousarray(sad, np.int32)), _p(mv), blocks, win, win,
                           -radius, -radius)
    return mv


def run_full(w, out_dtype=None):
    """Generic engine restatement on a paper_1911_03458_b200.Workload."""
    from paper_1911_03458_b200.merit import _DescHolder, _host, Error, Dtype
    h = _DescHolder(w, 0)
    da, db, do = h.dtypes
    shape = w.output_shape()
    out = np.empty(shape, np.int16 if do == Dtype.Fix16 else np.float32)
    a = np.ascontiguousarray(_host(w.src_a))
    b = np.ascontiguousarray(_host(w.src_b))
    st = lib().oracle_run_full(C.byref(h.desc), _p(a), _p(b), _p(out))
    if st:
        raise Error(st, "oracle_run_full failed")
    return out


def ref_run_full(w):
    """The reference engine (merit::run_full) on a Workload."""
    from paper_1911_03458_b200.merit import _DescHolder, _host, Error, Dtype
    h = _DescHolder(w, 0)
    da, db, do = h.dtypes
    out = np.empty(w.output_shape(), np.int16 if da == Dtype.Fix16 else np.float32)
    a = np.ascontiguousarray(_host(w.src_a))
    b = np.ascontiguousarray(_host(w.src_b))
    st = ref().ref_run_full(C.byref(h.desc), _p(a), _p(b), _p(out))
    if st:
        raise Error(st, ref().ref_last_error().decode())
    return out


def ref_run_tiled(w, t_p, t_a, caps=(1 << 40, 1 << 40)):
    """merit::run_tiled with EngineConfig{scratch_words_a, scratch_words_b} = caps."""
    from paper_1911_03458_b200.merit import _DescHolder, _host, Error, Dtype
    h = _DescHolder(w, 0)
    da, _, _ = h.dtypes
    out = np.empty(w.output_shape(), np.int16 if da == Dtype.Fix16 else np.float32)
    a = np.ascontiguousarray(_host(w.src_a))
    b = np.ascontiguousarray(_host(w.src_b))
    tp = np.asarray(t_p, np.int64)
    ta = np.asarray(t_a, np.int64)
    traffic = np.zeros(7, np.uint64)
    st = ref().ref_run_tiled_caps(C.byref(h.desc), _p(a), _p(b), _p(tp), _p(ta), int(caps[0]), int(caps[1]),
                                  _p(out), _p(traffic))
    if st:
        raise Error(st, ref().ref_last_error().decode())
    return out, traffic


def ref_mrt1_bytes(arr, frac_bits=0) -> bytes:
    """merit::Tensor::write of a float32 / int16 array (the reference's bytes)."""
    a = np.ascontiguousarray(arr)
    shape = np.asarray(a.shape, np.int64)
    cap = 8 + 4 * a.ndim + a.nbytes
    buf = np.empty(cap, np.uint8)
    n = ref().ref_mrt1_write(0 if a.dtype == np.float32 else 1, frac_bits, _p(shape), a.ndim, _p(a), _p(buf), cap)
    if n < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return buf[:n].tobytes()


def ref_mrt1_parse(data: bytes):
    """merit::Tensor::read: (array, frac_bits) or raises Error(code)."""
    from paper_1911_03458_b200.merit import Error
    raw = np.frombuffer(data, np.uint8)
    dt, fb, rk = C.c_int(), C.c_int(), C.c_int()
    shape = np.zeros(16, np.int64)
    cap = max(len(data), 16)
    payload = np.empty(cap, np.uint8)
    st = ref().ref_mrt1_read(_p(np.ascontiguousarray(raw)), len(data), C.byref(dt), C.byref(fb), C.byref(rk),
                             _p(shape), _p(payload), cap)
    if st:
        raise Error(st, ref().ref_last_error().decode())
    shp = tuple(int(x) for x in shape[:rk.value])
    n = int(np.prod(shp))
    arr = payload[:n * (4 if dt.value == 0 else 2)].view(np.float32 if dt.value == 0 else np.int16).reshape(shp)
    return arr.copy(), fb.value


def ref_template_case(name, params: dict, seed: int, cap=1 << 22):
    """build_template + fill_random(2s+1, 2s+2) + run_full + oracle, all in the
    reference.  Returns dict(src_a, src_b, engine, oracle, fix)."""
    ps = ",".join(f"{k}={v}" for k, v in params.items()).encode()
    fix = bool(params.get("fix", 0))
    dt = np.int16 if fix else np.float32
    bufs = [np.empty(cap, dt) for _ in range(4)]
    na, nb, no = C.c_int64(), C.c_int64(), C.c_int64()
    st = ref().ref_template_case(name.encode(), ps, seed, _p(bufs[0]), C.byref(na), _p(bufs[1]),
                                 C.byref(nb), _p(bufs[2]), _p(bufs[3]), C.byref(no), cap)
    if st:
        from paper_1911_03458_b200.merit import Error
        raise Error(st, ref().ref_last_error().decode())
    return dict(src_a=bufs[0][:na.value].copy(), src_b=bufs[1][:nb.value].copy(),
                engine=bufs[2][:no.value].copy(), oracle=bufs[3][:no.value].copy(), fix=fix)
