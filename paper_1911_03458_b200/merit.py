"""Python mirror of the reference's operator API, executed on the B200.

Same names and argument meaning as the reference's C++ headers so that parity
tests read like the reference's own tests:

* ``ViewTerm`` / ``ViewSpec`` / ``Boundary``  — view.hpp:11-49
* ``Op`` / ``Operand`` / ``Dst`` / ``AluInstr`` / ``LookupTable`` /
  ``StrategyProgram``                          — rip.hpp:15-107
* ``Workload``                                 — engine.hpp:16-39
* ``run_full(w)``                              — engine.hpp:282-287
* ``Error`` / ``ErrorCode``                    — tensor.hpp:15-34

Everything below lowers the workload to the C ABI (include/merit_dev.h) and
runs it on the GPU.  There is no CPU execution path: with no CUDA device,
``run_full`` raises.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi


class ErrorCode(enum.IntEnum):  # tensor.hpp:15-29, +1 so that 0 means OK
    OutOfRange = 1
    BadMagic = 2
    TruncatedPayload = 3
    UnknownDtype = 4
    NegativeStride = 5
    LutRange = 6
    DivByZero = 7
    ScratchpadOverflow = 8
    OutOfFootprint = 9
    Indivisible = 10
    UnknownTemplate = 11
    BadParams = 12
    Usage = 13
    UnsupportedProgram = 100
    UnsupportedView = 101
    Cuda = 102
    InvalidArgument = 103


class Error(RuntimeError):
    """merit::Error (tensor.hpp:31-34): a RuntimeError carrying an ErrorCode."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        try:
            self.code = ErrorCode(code)
        except ValueError:
            self.code = code


class Boundary(enum.IntEnum):  # view.hpp:11
    ZeroPad = 0
    Clamp = 1
    Reject = 2


class Dtype(enum.IntEnum):  # merit_dtype (tensor.hpp:67 + device storage types)
    Real32 = 0   # MERIT_F32
    Fix16 = 1    # MERIT_I16
    BF16 = 2
    U8 = 3
    I32 = 4
    U16 = 5      # exact SAD map of 8-bit 8x8 / 16x16 blocks (half the bytes of I32)


class Op(enum.IntEnum):  # rip.hpp:15-31
    ADD = 0
    SUB = 1
    L1 = 2
    MAC = 3
    MAX = 4
    MIN = 5
    SEL = 6
    BAND = 7
    BOR = 8
    BXOR = 9
    BNOT = 10
    IDX = 11
    LUT = 12
    MOVC = 13
    DIV = 14


class Kernel(enum.IntEnum):  # merit_kernel_kind
    GENERIC = 0
    MAXPOOL = 1
    SAD = 2
    CONV_TC = 3
    CORR = 4
    MULTI = 5


FLAG_EXACT = 1
FLAG_ARGMIN = 2
FLAG_NO_MAP = 4
FLAG_FAST_BF16 = 8


@dataclass
class ViewTerm:  # view.hpp:15-20
    component: int = 0
    axis: int = 0
    stride: int = 1
    offset: int = 0


@dataclass
class ViewSpec:  # view.hpp:24-49
    source_shape: List[int]
    p_shape: List[int]
    a_shape: List[int]
    terms: List[ViewTerm] = field(default_factory=list)
    boundary: Boundary = Boundary.ZeroPad

    def k_rank(self) -> int:
        return len(self.p_shape) + len(self.a_shape)

    def source_index(self, k: Sequence[int]) -> List[int]:
        """Eq. 5 (view.hpp:37-42): raw source coordinates of index k."""
        x = [0] * len(self.source_shape)
        for t in self.terms:
            x[t.axis] += k[t.component] * t.stride + t.offset
        return x

    def in_range(self, x: Sequence[int]) -> bool:  # view.hpp:44-48
        return all(0 <= xi < n for xi, n in zip(x, self.source_shape))


class Operand:  # rip.hpp:33-41
    Reg, PortA, PortB, Zero = 0, 1, 2, 3

    def __init__(self, kind: int = 3, reg: int = 0):
        self.kind, self.reg = kind, reg

    @staticmethod
    def r(i: int) -> "Operand":
        return Operand(Operand.Reg, i)

    @staticmethod
    def a() -> "Operand":
        return Operand(Operand.PortA)

    @staticmethod
    def b() -> "Operand":
        return Operand(Operand.PortB)

    @staticmethod
    def zero() -> "Operand":
        return Operand(Operand.Zero)


class Dst:  # rip.hpp:43-49
    def __init__(self, out: bool = False, reg: int = 0):
        self.out, self.reg = out, reg

    @staticmethod
    def r(i: int) -> "Dst":
        return Dst(False, i)

    @staticmethod
    def emit() -> "Dst":
        return Dst(True, 0)


@dataclass
class AluInstr:  # rip.hpp:51-57
    op: Op
    dst: Dst
    a: Operand
    b: Operand
    c: Operand
    shift: int = 0
    aux: int = 0


@dataclass
class LookupTable:  # rip.hpp:61-78
    lo: float = 0.0
    hi: float = 1.0
    samples: List[float] = field(default_factory=list)
    clamp: bool = True


@dataclass
class StrategyProgram:  # rip.hpp:85-107
    depth: int = 1
    segments: List[List[AluInstr]] = field(default_factory=list)
    constants: List[float] = field(default_factory=list)
    tables: List[LookupTable] = field(default_factory=list)
    outputs: int = 1

    def body(self) -> int:
        return self.depth

    def pre(self, level: int) -> int:
        return level - 1

    def post(self, level: int) -> int:
        return 2 * self.depth + 1 - level


def _np_dtype_code(arr) -> int:
    if arr is None:
        return Dtype.Real32
    try:
        import torch
        if isinstance(arr, torch.Tensor):
            return {torch.float32: Dtype.Real32, torch.int16: Dtype.Fix16,
                    torch.bfloat16: Dtype.BF16, torch.uint8: Dtype.U8,
                    torch.int32: Dtype.I32}[arr.dtype]
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(arr)
    return {np.dtype(np.float32): Dtype.Real32, np.dtype(np.int16): Dtype.Fix16,
            np.dtype(np.uint8): Dtype.U8, np.dtype(np.int32): Dtype.I32}[a.dtype]


@dataclass
class Workload:  # engine.hpp:16-39
    view_a: ViewSpec
    view_b: ViewSpec
    src_a: object = None   # numpy / torch tensor of shape view_a.source_shape
    src_b: object = None
    program: StrategyProgram = field(default_factory=StrategyProgram)
    frac_bits: int = 0
    # Device storage types; default inferred from src_a/src_b (numpy has no bf16,
    # so bf16 sources are passed as uint16 bit patterns with dtype_a=Dtype.BF16).
    dtype_a: Optional[Dtype] = None
    dtype_b: Optional[Dtype] = None
    dtype_out: Optional[Dtype] = None

    def p_shape(self):
        return self.view_a.p_shape

    def a_shape(self):
        return self.view_a.a_shape

    def output_shape(self) -> List[int]:
        s = list(self.view_a.p_shape)
        if self.program.outputs > 1:
            s.append(self.program.outputs)
        return s

    def resolved_dtypes(self):
        da = self.dtype_a if self.dtype_a is not None else _np_dtype_code(self.src_a)
        db = self.dtype_b if self.dtype_b is not None else _np_dtype_code(self.src_b)
        if self.dtype_out is not None:
            do = self.dtype_out
        elif da == Dtype.Fix16:
            do = Dtype.Fix16
        else:
            do = Dtype.Real32
        return Dtype(da), Dtype(db), Dtype(do)


# ------------------------------------------------------------- lowering ----
def _view_c(v: ViewSpec) -> _capi.ViewSpecC:
    c = _capi.ViewSpecC()
    if len(v.source_shape) > _capi.MAX_RANK or len(v.p_shape) > _capi.MAX_RANK or \
            len(v.a_shape) > _capi.MAX_RANK or len(v.terms) > _capi.MAX_TERMS:
        raise Error(ErrorCode.InvalidArgument, "view rank or term count exceeds the ABI limits")
    c.src_rank, c.p_rank, c.a_rank, c.n_terms = (len(v.source_shape), len(v.p_shape),
                                                 len(v.a_shape), len(v.terms))
    for i, e in enumerate(v.source_shape):
        c.src_shape[i] = int(e)
    for i, e in enumerate(v.p_shape):
        c.p_shape[i] = int(e)
    for i, e in enumerate(v.a_shape):
        c.a_shape[i] = int(e)
    for i, t in enumerate(v.terms):
        c.terms[i] = _capi.ViewTermC(int(t.component), int(t.axis), int(t.stride), int(t.offset))
    c.boundary = int(v.boundary)
    return c


class _DescHolder:
    """Owns the C descriptor plus the arrays its pointers reference."""

    def __init__(self, w: Workload, flags: int):
        p = w.program
        da, db, do = w.resolved_dtypes()
        d = _capi.WorkloadDescC()
        d.view_a = _view_c(w.view_a)
        d.view_b = _view_c(w.view_b)
        d.dtype_a, d.dtype_b, d.dtype_out = int(da), int(db), int(do)
        d.frac_bits = int(w.frac_bits)
        d.flags = int(flags)
        seg_len = [len(s) for s in p.segments]
        instrs = [ins for s in p.segments for ins in s]
        if len(instrs) > _capi.MAX_INSTRS:
            raise Error(ErrorCode.InvalidArgument, "program too long for the ABI")
        self.seg_len = (C.c_int32 * max(1, len(seg_len)))(*seg_len)
        arr = (_capi.AluInstrC * max(1, len(instrs)))()
        for i, ins in enumerate(instrs):
            arr[i] = _capi.AluInstrC(int(ins.op), int(ins.dst.out), int(ins.dst.reg),
                                     ins.a.kind, ins.a.reg, ins.b.kind, ins.b.reg,
                                     ins.c.kind, ins.c.reg, int(ins.shift), int(ins.aux))
        self.instrs = arr
        self.consts = (C.c_double * max(1, len(p.constants)))(*p.constants)
        self.tab_samples = [(C.c_double * max(1, len(t.samples)))(*t.samples) for t in p.tables]
        self.tables = (_capi.LookupTableC * max(1, len(p.tables)))()
        for i, t in enumerate(p.tables):
            self.tables[i] = _capi.LookupTableC(float(t.lo), float(t.hi), len(t.samples),
                                                int(bool(t.clamp)),
                                                C.cast(self.tab_samples[i], C.POINTER(C.c_double)))
        pc = d.program
        pc.depth, pc.outputs, pc.n_segments = int(p.depth), int(p.outputs), len(seg_len)
        pc.n_constants, pc.n_tables = len(p.constants), len(p.tables)
        pc.seg_len = C.cast(self.seg_len, C.POINTER(C.c_int32))
        pc.instrs = C.cast(self.instrs, C.POINTER(_capi.AluInstrC))
        pc.constants = C.cast(self.consts, C.POINTER(C.c_double))
        pc.tables = C.cast(self.tables, C.POINTER(_capi.LookupTableC))
        self.desc = d
        self.dtypes = (da, db, do)


def _check(st: int):
    if st != 0:
        lib = _capi.load()
        raise Error(st, lib.merit_dev_last_error().decode(errors="replace"))


_NP_OF = {Dtype.Real32: np.float32, Dtype.Fix16: np.int16, Dtype.BF16: np.uint16,
          Dtype.U8: np.uint8, Dtype.I32: np.int32, Dtype.U16: np.uint16}


class Plan:
    """A lowered device plan (merit_dev_plan_create)."""

    def __init__(self, w: Workload, flags: int = 0):
        self.lib = _capi.load()
        self._holder = _DescHolder(w, flags)
        h = C.c_void_p()
        _check(self.lib.merit_dev_plan_create(C.byref(self._holder.desc), C.byref(h)))
        self.handle = h
        info = _capi.PlanInfoC()
        _check(self.lib.merit_dev_plan_query(self.handle, C.byref(info)))
        self.info = info
        self.kernel = Kernel(info.kernel)
        self.out_shape = tuple(info.out_shape[i] for i in range(info.out_rank))
        self.dtypes = self._holder.dtypes
        self.description = info.description.decode()

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.merit_dev_plan_destroy(self.handle)
                self.handle = None
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    # -- device buffers (torch CUDA tensors or raw pointers) ------------------
    @staticmethod
    def _ptr(x):
        if x is None:
            return None
        if isinstance(x, int):
            return C.c_void_p(x)
        return C.c_void_p(x.data_ptr())

    packed = False  # weights pre-packed on the device (src_b may then be omitted)

    def pack_b(self, d_src_b, stream=None):
        self._check_buf(d_src_b, self.info.src_b_bytes, "src_b")
        _check(self.lib.merit_dev_plan_pack_b(self.handle, self._ptr(d_src_b),
                                              C.c_void_p(stream or 0)))
        self.packed = True

    def _check_buf(self, x, need: int, what: str):
        """Device buffers given as tensors must be CUDA tensors of at least
        `need` bytes (raw integer pointers are the caller's responsibility)."""
        if x is None or isinstance(x, int) or need <= 0:
            return
        if not getattr(x, "is_cuda", False):
            raise Error(ErrorCode.BadParams, f"{what} must be a CUDA tensor (device buffers)")
        if not x.is_contiguous():
            raise Error(ErrorCode.BadParams, f"{what} must be contiguous")
        if x.numel() * x.element_size() < need:
            raise Error(ErrorCode.BadParams, f"{what} holds {x.numel() * x.element_size()} bytes, needs {need}")

    def run(self, d_src_a, d_src_b, d_out, d_aux=None, stream=None):
        """merit_dev_run on device buffers (torch CUDA tensors or raw pointers)."""
        i = self.info
        self._check_buf(d_src_a, i.src_a_bytes, "src_a")
        self._check_buf(d_src_b, i.src_b_bytes if not self.packed else 0, "src_b")
        self._check_buf(d_out, i.out_bytes, "out")
        self._check_buf(d_aux, i.aux_elems * 4, "aux")
        _check(self.lib.merit_dev_run(self.handle, self._ptr(d_src_a), self._ptr(d_src_b),
                                      self._ptr(d_out), self._ptr(d_aux), C.c_void_p(stream or 0)))

    def host_slices(self) -> list:
        """How run_host pipelines this plan: [{a_need, b_need, out_lo, out_hi,
        aux_lo, aux_hi}] per slice ([] = unsliced).  Host-only."""
        n = C.c_int64(0)
        _check(self.lib.merit_dev_plan_slices(self.handle, None, 0, C.byref(n)))
        arr = (_capi.HostSliceC * max(1, n.value))()
        _check(self.lib.merit_dev_plan_slices(self.handle, arr, n.value, C.byref(n)))
        return [{k: int(getattr(arr[i], k)) for k, _ in _capi.HostSliceC._fields_} for i in range(n.value)]

    def tiled_traffic(self, t_p, t_a) -> dict:
        """merit::run_tiled's TrafficReport (engine.hpp:72-80) for the tiling plan
        {t_p, t_a}: validated like TilingPlan::validate, Eq. 6 words per pass."""
        tp = np.ascontiguousarray(t_p, np.int64)
        ta = np.ascontiguousarray(t_a, np.int64)
        if tp.size != self._holder.desc.view_a.p_rank or ta.size != self._holder.desc.view_a.a_rank:
            raise Error(ErrorCode.BadParams, "tile rank mismatch")
        r = _capi.TrafficReportC()
        _check(self.lib.merit_dev_tiled_traffic(self.handle, tp.ctypes.data_as(C.c_void_p),
                                                ta.ctypes.data_as(C.c_void_p), C.byref(r)))
        return {k: int(getattr(r, k)) for k, _ in r._fields_}

    def measure_traffic(self, d_src_a, d_src_b, d_out=None, d_aux=None, stream=None) -> dict:
        """merit_dev_measure_traffic: one run on device buffers with the GPU's
        DRAM counters armed (CUPTI), after an L2 flush: the bytes HBM served
        and the kernel time, summed over the plan's launches."""
        r = _capi.MeasuredTrafficC()
        _check(self.lib.merit_dev_measure_traffic(self.handle, self._ptr(d_src_a), self._ptr(d_src_b),
                                                  self._ptr(d_out), self._ptr(d_aux), C.c_void_p(stream or 0),
                                                  C.byref(r)))
        return {k: (float(getattr(r, k)) if k.startswith(("dram", "range_time")) else int(getattr(r, k)))
                for k, _ in r._fields_ if k != "_pad"}

    # -- host buffers: the reference's run_full convention --------------------
    @staticmethod
    def _check_host(x, dtype, need: int, what: str):
        if not isinstance(x, np.ndarray):
            raise Error(ErrorCode.BadParams, f"{what} must be a numpy array")
        if x.dtype != np.dtype(dtype):
            raise Error(ErrorCode.BadParams, f"{what} has dtype {x.dtype}, needs {np.dtype(dtype)}")
        if not x.flags["C_CONTIGUOUS"] or not x.flags["WRITEABLE"]:
            raise Error(ErrorCode.BadParams, f"{what} must be a writeable C-contiguous array")
        if x.nbytes < need:
            raise Error(ErrorCode.BadParams, f"{what} holds {x.nbytes} bytes, needs {need}")

    def run_host(self, src_a, src_b, out: Optional[np.ndarray] = None,
                 aux: Optional[np.ndarray] = None, stream=None):
        a = np.ascontiguousarray(src_a)
        b = np.ascontiguousarray(src_b) if src_b is not None else None
        _, _, do = self.dtypes
        if out is None:
            out = np.empty(self.out_shape if self.info.out_elems else (0,), dtype=_NP_OF[do])
        if aux is None and self.info.aux_elems:
            aux = np.empty((self.info.aux_elems // 3, 3), dtype=np.int32)
        if a.nbytes != self.info.src_a_bytes:
            raise Error(ErrorCode.BadParams, "source shape mismatch (src_a)")
        if b is not None and b.nbytes != self.info.src_b_bytes:
            raise Error(ErrorCode.BadParams, "source shape mismatch (src_b)")
        # the C call copies out_bytes / aux_elems * 4 bytes into the raw host
        # pointers: caller-supplied arrays must be exactly right
        if self.info.out_elems:
            self._check_host(out, _NP_OF[do], self.info.out_bytes, "out")
        if self.info.aux_elems:
            self._check_host(aux, np.int32, self.info.aux_elems * 4, "aux")
        _check(self.lib.merit_dev_run_host(
            self.handle, a.ctypes.data_as(C.c_void_p),
            b.ctypes.data_as(C.c_void_p) if b is not None else None,
            out.ctypes.data_as(C.c_void_p) if out.size else None,
            aux.ctypes.data_as(C.c_void_p) if aux is not None else None,
            C.c_void_p(stream or 0)))
        return out, aux


class PlanGroup(Plan):
    """Several workloads over the same two sources as one plan
    (merit_dev_plan_create_multi): what a reference caller does with one
    run_full per workload.  Members the device computes in one pass are fused
    (the 8x8 + 16x16 block searches of C5); ``run`` takes the shared sources
    once and writes the members' outputs / argmin records back to back
    (``members[i]["out_offset"]`` bytes, ``["aux_offset"]`` int32 elements)."""

    def __init__(self, ws: Sequence[Workload], flags: int = 0):
        self.lib = _capi.load()
        ws = list(ws)
        if not ws:
            raise Error(ErrorCode.InvalidArgument, "empty workload list")
        self._holders = [_DescHolder(w, flags) for w in ws]
        self._holder = self._holders[0]
        arr = (_capi.WorkloadDescC * len(ws))(*[h.desc for h in self._holders])
        h = C.c_void_p()
        _check(self.lib.merit_dev_plan_create_multi(arr, len(ws), C.byref(h)))
        self.handle = h
        info = _capi.PlanInfoC()
        _check(self.lib.merit_dev_plan_query(self.handle, C.byref(info)))
        self.info = info
        self.kernel = Kernel(info.kernel)
        self.description = info.description.decode()
        self.dtypes = self._holder.dtypes
        self.out_shape = (int(info.out_elems),)
        self.members = []
        for i, w in enumerate(ws):
            mi = _capi.PlanInfoC()
            oo, ao = C.c_int64(), C.c_int64()
            _check(self.lib.merit_dev_plan_member(self.handle, i, C.byref(mi), C.byref(oo), C.byref(ao)))
            self.members.append({"info": mi, "out_offset": oo.value, "aux_offset": ao.value,
                                 "out_shape": tuple(mi.out_shape[k] for k in range(mi.out_rank)),
                                 "dtype_out": self._holders[i].dtypes[2]})

    def run_host(self, src_a, src_b, out=None, aux=None, stream=None):
        """merit_dev_run_host: [(out_i or None, aux_i or None) per member]."""
        a = np.ascontiguousarray(src_a)
        b = np.ascontiguousarray(src_b)
        if a.nbytes != self.info.src_a_bytes or b.nbytes != self.info.src_b_bytes:
            raise Error(ErrorCode.BadParams, "source shape mismatch")
        obuf = np.empty(max(1, int(self.info.out_bytes)), np.uint8)
        xbuf = np.empty(max(1, int(self.info.aux_elems)), np.int32)
        _check(self.lib.merit_dev_run_host(
            self.handle, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
            obuf.ctypes.data_as(C.c_void_p) if self.info.out_elems else None,
            xbuf.ctypes.data_as(C.c_void_p) if self.info.aux_elems else None, C.c_void_p(stream or 0)))
        res = []
        for m in self.members:
            mi = m["info"]
            o = None
            if mi.out_elems:
                o = obuf[m["out_offset"]:m["out_offset"] + mi.out_bytes].view(_NP_OF[m["dtype_out"]])
                o = o.reshape(m["out_shape"]).copy()
            x = xbuf[m["aux_offset"]:m["aux_offset"] + mi.aux_elems].reshape(-1, 3).copy() if mi.aux_elems else None
            res.append((o, x))
        return res


def run_full_many(ws: Sequence[Workload], flags: int = 0):
    """run_full (engine.hpp:282-287) of several workloads over the same two
    sources, as one device plan: [(output or None, argmin records or None)]."""
    ws = list(ws)
    for w in ws:
        _check_sources(w)
    g = PlanGroup(ws, flags)
    return g.run_host(_host(ws[0].src_a), _host(ws[0].src_b))


def run_full(w: Workload, flags: int = 0):
    """engine.hpp:282-287: run the workload on the device, return the host
    output tensor of shape ``w.output_shape()``."""
    _check_sources(w)
    plan = Plan(w, flags)
    out, _ = plan.run_host(_host(w.src_a), _host(w.src_b))
    return out


def run_tiled(w: Workload, t_p, t_a, flags: int = 0, scratch_words_a: int = 8192,
              scratch_words_b: int = 4096, measure: bool = False):
    """engine.hpp:289-295 on the device: the output of run_full (the device
    executes its own footprint-staged tiling) and the TilingPlan's
    TrafficReport as a dict.  EngineConfig's capacities (engine.hpp:82-87)
    keep their diagnostic meaning: a footprint box larger than
    scratch_words_a / _b raises ScratchpadOverflow (engine.hpp:154-155).
    measure=True adds ``rep["measured"]``: the DRAM bytes the device run
    actually moved, from the GPU's counters (Plan.measure_traffic)."""
    _check_sources(w)
    plan = Plan(w, flags)
    rep = plan.tiled_traffic(t_p, t_a)
    if rep["scratchpad_peak_words_a"] > scratch_words_a or rep["scratchpad_peak_words_b"] > scratch_words_b:
        raise Error(ErrorCode.ScratchpadOverflow, "tile exceeds scratchpad")
    if measure:
        import torch
        a = torch.from_numpy(np.ascontiguousarray(_host(w.src_a))).cuda()
        b = torch.from_numpy(np.ascontiguousarray(_host(w.src_b))).cuda()
        o = torch.empty(max(1, int(plan.info.out_bytes)), dtype=torch.uint8, device="cuda")
        x = torch.empty(max(1, int(plan.info.aux_elems)), dtype=torch.int32, device="cuda")
        rep["measured"] = plan.measure_traffic(a, b, o, x if plan.info.aux_elems else None)
        out = o[:int(plan.info.out_bytes)].cpu().numpy().view(_NP_OF[plan.dtypes[2]]).reshape(plan.out_shape)
        return out, rep
    out, _ = plan.run_host(_host(w.src_a), _host(w.src_b))
    return out, rep


def run_full_argmin(w: Workload, with_map: bool = True):
    """L1 block matching plus the per-block argmin (mv_y, mv_x, min SAD) with the
    lowest-raster tie-break.  Returns (sad_map or None, argmin[int32, (blocks, 3)])."""
    _check_sources(w)
    plan = Plan(w, FLAG_ARGMIN | (0 if with_map else FLAG_NO_MAP))
    out, aux = plan.run_host(_host(w.src_a), _host(w.src_b))
    return (out if with_map else None), aux


def _host(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            if x.dtype == torch.bfloat16:
                return x.detach().cpu().view(torch.int16).numpy().view(np.uint16)
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)


def _check_sources(w: Workload):
    # Workload::validate's source-shape check (engine.hpp:35-36).
    for src, v in ((w.src_a, w.view_a), (w.src_b, w.view_b)):
        if src is None:
            raise Error(ErrorCode.BadParams, "source shape mismatch")
        if tuple(np.shape(src) if not hasattr(src, "shape") else src.shape) != \
                tuple(v.source_shape):
            raise Error(ErrorCode.BadParams, "source shape mismatch")
