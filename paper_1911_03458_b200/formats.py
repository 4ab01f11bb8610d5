"""The reference's on-disk and wire formats for workloads.

* MRT1 tensors — ``Tensor::write / Tensor::read`` (tensor.hpp:123-163):
  ``"MRT1"``, u8 dtype (0 = REAL32, 1 = FIX16), u8 frac_bits, u16 rank, rank
  x u32 extents, then the payload (u32 float bits / u16 values), all
  little-endian.  Read errors carry the reference's codes: BadMagic,
  UnknownDtype, TruncatedPayload (short payload or rank 0), BadParams
  (an extent < 1, Tensor::check_shape).
* JSON manifests — ``{"view_a", "view_b", "program", "tensor_a", "tensor_b"
  [, "tiling"]}`` as read by the reference CLI's ``load_manifest``
  (tools/merit.cpp:102-118), with views and programs in the field layout of
  ``serialize.hpp:104-184`` (op names, operand strings ``rN`` / ``a`` / ``b``
  / ``_``, destinations ``out`` / ``rN``, boundary names).

Relative tensor paths resolve against the manifest's directory.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

from .merit import (AluInstr, Boundary, Dst, Error, ErrorCode, LookupTable, Op, Operand,
                    StrategyProgram, ViewSpec, ViewTerm, Workload)

_BOUNDARY_NAMES = {Boundary.ZeroPad: "ZERO_PAD", Boundary.Clamp: "CLAMP", Boundary.Reject: "REJECT"}


# ----------------------------------------------------------------- MRT1 ---
def write_mrt1(path, arr, frac_bits: int = 0) -> None:
    a = np.ascontiguousarray(arr)
    if a.dtype == np.float32:
        code = 0
    elif a.dtype == np.int16:
        code = 1
    else:
        raise Error(ErrorCode.UnknownDtype, f"MRT1 holds REAL32 or FIX16, not {a.dtype}")
    if a.ndim < 1 or any(e < 1 for e in a.shape):
        raise Error(ErrorCode.BadParams, "extents must be >= 1")
    head = b"MRT1" + struct.pack("<BBH", code, frac_bits if code else 0, a.ndim)
    head += struct.pack("<%dI" % a.ndim, *a.shape)
    Path(path).write_bytes(head + a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())


def read_mrt1(path) -> Tuple[np.ndarray, int]:
    """Returns (array, frac_bits)."""
    data = Path(path).read_bytes()
    if data[:4] != b"MRT1":
        raise Error(ErrorCode.BadMagic, "bad magic, expected MRT1")
    if len(data) < 8:
        raise Error(ErrorCode.TruncatedPayload, "unexpected EOF")
    code, frac, rank = struct.unpack_from("<BBH", data, 4)
    if code > 1:
        raise Error(ErrorCode.UnknownDtype, "unknown dtype code")
    if len(data) < 8 + 4 * rank:
        raise Error(ErrorCode.TruncatedPayload, "unexpected EOF")
    shape = struct.unpack_from("<%dI" % rank, data, 8)
    if rank < 1:
        raise Error(ErrorCode.TruncatedPayload, "rank must be >= 1")
    if any(e < 1 for e in shape):
        raise Error(ErrorCode.BadParams, "extents must be >= 1")
    dt = np.dtype("<f4") if code == 0 else np.dtype("<i2")
    n = int(np.prod(shape))
    off = 8 + 4 * rank
    if len(data) < off + n * dt.itemsize:
        raise Error(ErrorCode.TruncatedPayload, "unexpected EOF")
    arr = np.frombuffer(data, dt, n, off).astype(np.float32 if code == 0 else np.int16).reshape(shape)
    return arr, (frac if code else 0)


# ----------------------------------------------------------------- JSON ---
def _operand_str(o: Operand) -> str:
    return {Operand.Reg: f"r{o.reg}", Operand.PortA: "a", Operand.PortB: "b"}.get(o.kind, "_")


def _operand_from(s: str) -> Operand:
    if s == "a":
        return Operand.a()
    if s == "b":
        return Operand.b()
    if s == "_":
        return Operand.zero()
    if len(s) >= 2 and s[0] == "r" and s[1:].isdigit():
        i = int(s[1:])
        if not 0 <= i <= 15:
            raise Error(ErrorCode.BadParams, f"register id out of range: {s}")
        return Operand.r(i)
    raise Error(ErrorCode.BadParams, f"bad operand {s}")


def _dst_from(s: str) -> Dst:
    if s == "out":
        return Dst.emit()
    o = _operand_from(s)
    if o.kind != Operand.Reg:
        raise Error(ErrorCode.BadParams, f"bad destination {s}")
    return Dst.r(o.reg)


def view_to_json(v: ViewSpec) -> dict:  # serialize.hpp:104-117
    return {"source_shape": list(map(int, v.source_shape)), "p_shape": list(map(int, v.p_shape)),
            "a_shape": list(map(int, v.a_shape)),
            "terms": [{"component": t.component, "axis": t.axis, "stride": t.stride, "offset": t.offset}
                      for t in v.terms],
            "boundary": _BOUNDARY_NAMES[Boundary(v.boundary)]}


def view_from_json(j: dict) -> ViewSpec:  # serialize.hpp:119-131
    try:
        v = ViewSpec(list(j["source_shape"]), list(j["p_shape"]), list(j["a_shape"]),
                     [ViewTerm(int(t["component"]), int(t["axis"]), int(t["stride"]), int(t["offset"]))
                      for t in j["terms"]])
    except (KeyError, TypeError) as e:
        raise Error(ErrorCode.BadParams, f"bad view: {e}") from None
    if "boundary" in j:
        names = {n: b for b, n in _BOUNDARY_NAMES.items()}
        if j["boundary"] not in names:
            raise Error(ErrorCode.BadParams, f"unknown boundary {j['boundary']}")
        v.boundary = names[j["boundary"]]
    return v


def program_to_json(p: StrategyProgram) -> dict:  # serialize.hpp:133-158
    return {"depth": p.depth,
            "segments": [[{"op": Op(i.op).name, "dst": "out" if i.dst.out else f"r{i.dst.reg}",
                           "a": _operand_str(i.a), "b": _operand_str(i.b), "c": _operand_str(i.c),
                           "shift": i.shift, "aux": i.aux} for i in seg] for seg in p.segments],
            "constants": list(p.constants),
            "tables": [{"lo": t.lo, "hi": t.hi, "samples": list(t.samples), "clamp": t.clamp}
                       for t in p.tables],
            "outputs": p.outputs}


def program_from_json(j: dict) -> StrategyProgram:  # serialize.hpp:160-184
    try:
        segs = [[AluInstr(Op[i["op"]] if i["op"] in Op.__members__ else _bad_op(i["op"]),
                          _dst_from(i["dst"]), _operand_from(i["a"]), _operand_from(i["b"]),
                          _operand_from(i["c"]), int(i.get("shift", 0)), int(i.get("aux", 0)))
                 for i in seg] for seg in j["segments"]]
        p = StrategyProgram(int(j["depth"]), segs, [float(c) for c in j.get("constants", [])],
                            [LookupTable(float(t["lo"]), float(t["hi"]), [float(s) for s in t["samples"]],
                                         bool(t.get("clamp", True))) for t in j.get("tables", [])],
                            int(j.get("outputs", 1)))
    except (KeyError, TypeError) as e:
        raise Error(ErrorCode.BadParams, f"bad program: {e}") from None
    return p


def _bad_op(name):
    raise Error(ErrorCode.BadParams, f"unknown op {name}")


def traffic_to_json(rep: dict) -> dict:  # serialize.hpp:186-196
    keys = ["dram_read_words_a", "dram_read_words_b", "dram_write_words", "scratchpad_peak_words_a",
            "scratchpad_peak_words_b", "passes", "macs"]
    return {k: int(rep[k]) for k in keys}


# ------------------------------------------------------------- manifests ---
def write_manifest(directory, w: Workload, tiling: Optional[str] = None, stem: str = "workload") -> Path:
    """Write <stem>.json plus <stem>_a.mrt / <stem>_b.mrt (REAL32 / FIX16 sources)."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    write_mrt1(d / f"{stem}_a.mrt", w.src_a, w.frac_bits)
    write_mrt1(d / f"{stem}_b.mrt", w.src_b, w.frac_bits)
    m = {"view_a": view_to_json(w.view_a), "view_b": view_to_json(w.view_b),
         "program": program_to_json(w.program), "tensor_a": f"{stem}_a.mrt", "tensor_b": f"{stem}_b.mrt"}
    if tiling:
        m["tiling"] = tiling
    path = d / f"{stem}.json"
    path.write_text(json.dumps(m, indent=1) + "\n")
    return path


def load_manifest(path) -> Tuple[Workload, Optional[str]]:
    """tools/merit.cpp:102-118: (workload, tiling string or None)."""
    p = Path(path)
    try:
        j = json.loads(p.read_text())
    except OSError:
        raise Error(ErrorCode.Usage, f"cannot open {path}") from None
    except json.JSONDecodeError as e:
        raise Error(ErrorCode.BadParams, f"bad manifest JSON: {e}") from None
    w = Workload(view_from_json(j["view_a"]), view_from_json(j["view_b"]),
                 program=program_from_json(j["program"]))
    a, fa = read_mrt1(p.parent / j["tensor_a"])
    b, _ = read_mrt1(p.parent / j["tensor_b"])
    w.src_a, w.src_b, w.frac_bits = a, b, fa
    return w, j.get("tiling")
