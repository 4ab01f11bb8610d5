"""ctypes binding of the C ABI declared in include/merit_dev.h.

Loads the in-tree ``libmerit_dev.so`` (built by ``build.py``).  There is no
fallback: if the library is missing, importing the device API raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

MAX_RANK = 8
MAX_TERMS = 24
MAX_INSTRS = 64

import os

LIB_PATH = Path(__file__).resolve().parent / "libmerit_dev.so"
# MERIT_DEV_LIB selects another build of the same ABI (e.g. the diagnostic
# libmerit_dev_debug.so from `python -m paper_1911_03458_b200.build --debug`).
if os.environ.get("MERIT_DEV_LIB"):
    LIB_PATH = Path(os.environ["MERIT_DEV_LIB"]).resolve()


class ViewTermC(C.Structure):
    _fields_ = [("component", C.c_int32), ("axis", C.c_int32), ("stride", C.c_int64),
                ("offset", C.c_int64)]


class ViewSpecC(C.Structure):
    _fields_ = [("src_rank", C.c_int32), ("p_rank", C.c_int32), ("a_rank", C.c_int32),
                ("n_terms", C.c_int32), ("src_shape", C.c_int64 * MAX_RANK),
                ("p_shape", C.c_int64 * MAX_RANK), ("a_shape", C.c_int64 * MAX_RANK),
                ("terms", ViewTermC * MAX_TERMS), ("boundary", C.c_int32), ("_pad", C.c_int32)]


class AluInstrC(C.Structure):
    _fields_ = [("op", C.c_int32), ("dst_out", C.c_int32), ("dst_reg", C.c_int32),
                ("a_kind", C.c_int32), ("a_reg", C.c_int32), ("b_kind", C.c_int32),
                ("b_reg", C.c_int32), ("c_kind", C.c_int32), ("c_reg", C.c_int32),
                ("shift", C.c_int32), ("aux", C.c_int32)]


class LookupTableC(C.Structure):
    _fields_ = [("lo", C.c_double), ("hi", C.c_double), ("n_samples", C.c_int32),
                ("clamp", C.c_int32), ("samples", C.POINTER(C.c_double))]


class ProgramC(C.Structure):
    _fields_ = [("depth", C.c_int32), ("outputs", C.c_int32), ("n_segments", C.c_int32),
                ("n_constants", C.c_int32), ("n_tables", C.c_int32), ("_pad", C.c_int32),
                ("seg_len", C.POINTER(C.c_int32)), ("instrs", C.POINTER(AluInstrC)),
                ("constants", C.POINTER(C.c_double)), ("tables", C.POINTER(LookupTableC))]


class WorkloadDescC(C.Structure):
    _fields_ = [("view_a", ViewSpecC), ("view_b", ViewSpecC), ("dtype_a", C.c_int32),
                ("dtype_b", C.c_int32), ("dtype_out", C.c_int32), ("frac_bits", C.c_int32),
                ("flags", C.c_uint32), ("_pad", C.c_int32), ("program", ProgramC)]


class PlanInfoC(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("out_rank", C.c_int32),
                ("out_shape", C.c_int64 * (MAX_RANK + 1)), ("out_elems", C.c_int64),
                ("out_bytes", C.c_int64), ("aux_elems", C.c_int64), ("src_a_bytes", C.c_int64),
                ("src_b_bytes", C.c_int64), ("n_outputs", C.c_int64),
                ("algorithmic_ops", C.c_double), ("algorithmic_bytes", C.c_double),
                ("executed_ops", C.c_double),
                ("launches_per_run", C.c_int32), ("_pad", C.c_int32),
                ("description", C.c_char * 256)]


class TrafficReportC(C.Structure):  # merit_traffic_report (engine.hpp:72-80)
    _fields_ = [("dram_read_words_a", C.c_uint64), ("dram_read_words_b", C.c_uint64),
                ("dram_write_words", C.c_uint64), ("scratchpad_peak_words_a", C.c_uint64),
                ("scratchpad_peak_words_b", C.c_uint64), ("passes", C.c_uint64), ("macs", C.c_uint64)]


class HostSliceC(C.Structure):  # merit_host_slice (pipelined merit_dev_run_host)
    _fields_ = [("a_need", C.c_int64), ("b_need", C.c_int64), ("out_lo", C.c_int64), ("out_hi", C.c_int64),
                ("aux_lo", C.c_int64), ("aux_hi", C.c_int64), ("aux2_lo", C.c_int64), ("aux2_hi", C.c_int64)]


class MeasuredTrafficC(C.Structure):  # merit_measured_traffic
    _fields_ = [("dram_read_bytes", C.c_double), ("dram_write_bytes", C.c_double), ("range_time_ns", C.c_double),
                ("ranges", C.c_int64), ("launches", C.c_int64), ("passes", C.c_int32), ("_pad", C.c_int32)]


# Exported symbols and their prototypes (kept in sync with include/merit_dev.h;
# tests/test_capi_symbols.py checks every declared symbol is exported).
PROTOTYPES = {
    "merit_dev_abi_version": (C.c_int32, []),
    "merit_dev_build_info": (C.c_char_p, []),
    "merit_dev_last_error": (C.c_char_p, []),
    "merit_dev_plan_create": (C.c_int, [C.POINTER(WorkloadDescC), C.POINTER(C.c_void_p)]),
    "merit_dev_plan_destroy": (C.c_int, [C.c_void_p]),
    "merit_dev_plan_create_multi": (C.c_int, [C.POINTER(WorkloadDescC), C.c_int32, C.POINTER(C.c_void_p)]),
    "merit_dev_plan_member": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(PlanInfoC), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64)]),
    "merit_dev_plan_query": (C.c_int, [C.c_void_p, C.POINTER(PlanInfoC)]),
    "merit_dev_plan_pack_b": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "merit_dev_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "merit_dev_run_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "merit_gen_uniform_f32": (None, [C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_double]),
    "merit_gen_normal_f32": (None, [C.c_void_p, C.c_int64, C.c_uint64, C.c_double]),
    "merit_gen_range_i16": (None, [C.c_void_p, C.c_int64, C.c_uint64, C.c_int64, C.c_int64]),
    "merit_gen_me_pair": (None, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                 C.c_int64, C.c_int64, C.c_uint64]),
    "merit_f32_to_bf16": (None, [C.c_void_p, C.c_void_p, C.c_int64]),
    "merit_dev_launch_count": (C.c_int64, []),
    "merit_dev_last_kernel": (C.c_char_p, []),
    "merit_dev_tiled_traffic": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(TrafficReportC)]),
    "merit_dev_plan_slices": (C.c_int, [C.c_void_p, C.POINTER(HostSliceC), C.c_int64, C.POINTER(C.c_int64)]),
    "merit_dev_measure_traffic": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.POINTER(MeasuredTrafficC)]),
    "merit_dev_measure_traffic_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(MeasuredTrafficC)]),
}

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load libmerit_dev.so (building it in-tree if absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and build_if_missing:
        from . import build as _build
        _build.build()
    if not LIB_PATH.exists():
        raise RuntimeError(f"merit device library not found at {LIB_PATH}; run "
                           "`python -m paper_1911_03458_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
