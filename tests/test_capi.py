"""CPU tests of the C ABI boundary: the library loads, exports every symbol
include/merit_dev.h declares, its struct layouts match the Python mirror,
and plan creation (lowering) behaves like Workload::validate — no GPU needed."""
import ctypes as C
import re
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from paper_1911_03458_b200 import (FLAG_ARGMIN, FLAG_EXACT, FLAG_NO_MAP, Error, ErrorCode, Kernel,
                                   Plan, ViewTerm, _capi)
from paper_1911_03458_b200 import workloads as W

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "merit_dev.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s*\*?\s+)+\*?(merit_[a-z_0-9]+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(devlib):
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(devlib, n), f"{n} declared in merit_dev.h but not exported"
        assert n in _capi.PROTOTYPES, f"{n} missing from the ctypes prototypes"


def test_abi_version_and_build_info(devlib):
    assert devlib.merit_dev_abi_version() == 1
    assert b"sm_100a" in devlib.merit_dev_build_info()


def test_struct_layouts_match_c():
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "merit_dev.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(merit_view_term), sizeof(merit_view_spec),
  sizeof(merit_alu_instr), sizeof(merit_lookup_table), sizeof(merit_program),
  sizeof(merit_workload_desc), sizeof(merit_plan_info), offsetof(merit_workload_desc, program));
 return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        src = Path(d) / "s.c"
        src.write_text(prog)
        exe = Path(d) / "s"
        subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
        got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_capi.ViewTermC), C.sizeof(_capi.ViewSpecC), C.sizeof(_capi.AluInstrC),
            C.sizeof(_capi.LookupTableC), C.sizeof(_capi.ProgramC), C.sizeof(_capi.WorkloadDescC),
            C.sizeof(_capi.PlanInfoC), _capi.WorkloadDescC.program.offset]
    assert got == want


@pytest.mark.parametrize("cfg,kernel,flags", [
    ("C1", Kernel.MAXPOOL, 0), ("C2", Kernel.SAD, FLAG_ARGMIN), ("C3", Kernel.CONV_TC, 0),
    ("C4", Kernel.CONV_TC, 0)])
def test_configs_lower_to_specialised_kernels(cfg, kernel, flags):
    p = Plan(W.config_workload(cfg, with_inputs=False), flags)
    assert p.kernel == kernel
    assert p.info.launches_per_run == 1


def test_config_plan_accounting():
    # SURVEY §8(d) per-unit figures
    p = Plan(W.config_workload("C1", with_inputs=False))
    assert p.info.n_outputs == 1605632 and p.info.algorithmic_bytes == 32112640
    p = Plan(W.config_workload("C2", with_inputs=False), FLAG_ARGMIN)
    assert p.info.n_outputs == 8755560 and p.info.algorithmic_ops == 2241423360
    assert p.out_shape == (67, 120, 33, 33) and p.info.aux_elems == 8040 * 3
    p = Plan(W.config_workload("C3", with_inputs=False))
    assert 2 * p.info.algorithmic_ops == 7398752256
    p = Plan(W.config_workload("C4", with_inputs=False))
    assert 2 * p.info.algorithmic_ops == 118380036096 and p.info.algorithmic_bytes == 411631616
    p = Plan(W.config_workload("C5", with_inputs=False, pairs=64), FLAG_ARGMIN | FLAG_NO_MAP)
    assert p.info.out_elems == 0 and p.info.n_outputs * 256 == 64 * 35043840000


def test_templates_lower():
    kinds = {t: Plan(W.build_template(t, {})).kernel for t in W.TEMPLATES}
    assert kinds["maxpool"] == Kernel.MAXPOOL
    assert kinds["alexnet_conv1"] == Kernel.CONV_TC
    assert kinds["gemm"] == Kernel.CONV_TC  # through operand strides on the general kernel
    assert kinds["correlation"] == Kernel.CORR  # displacement correlation kernel (K4)
    for t in ("bilateral", "motion_estimation", "conv2d", "dilated"):
        assert kinds[t] == Kernel.GENERIC
    corr = {"c": 16, "h": 12, "w": 10, "d": 5}
    assert Plan(W.build_template("correlation", corr)).description.startswith("corr C=16 12x10 displacements 5x5")
    assert Plan(W.build_template("correlation", corr), FLAG_EXACT).kernel == Kernel.GENERIC
    # a window wider than one CTA's threads stays on the interpreter
    assert Plan(W.build_template("correlation", dict(corr, d=200))).kernel == Kernel.GENERIC
    assert Plan(W.build_template("conv2d", {"cin": 4, "cout": 8})).kernel == Kernel.CONV_TC
    assert Plan(W.build_template("relu_fused_conv", {"cin": 4, "cout": 8})).description.endswith("relu")
    # FIX16 always runs the exact interpreter
    assert Plan(W.build_template("maxpool", {"fix": 1})).kernel == Kernel.GENERIC
    assert Plan(W.build_template("conv2d", {"cin": 4, "cout": 8, "fix": 1})).kernel == Kernel.GENERIC
    # EXACT forces the interpreter
    assert Plan(W.config_workload("C3", with_inputs=False), FLAG_EXACT).kernel == Kernel.GENERIC


def test_validate_errors_mirror_reference():
    w = W.build_template("gemm", {})
    w.view_b.p_shape = [8, 9]
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # views must share p and a shapes
    w = W.build_template("gemm", {})
    w.program.depth = 2
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # depth must match |a|
    w = W.build_template("gemm", {})
    w.program.segments.append([])
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # 2*depth+1 segments
    w = W.build_template("gemm", {})
    w.program.segments[1][0].dst.reg = 16
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # register id < 16
    w = W.build_template("gemm", {})
    w.program.segments[1][0].shift = 16
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # shift 0..15
    w = W.build_template("gemm", {})
    w.view_a.terms.append(ViewTerm(0, 5, 1, 0))
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.BadParams            # AXIS_OUT_OF_RANGE
    w = W.build_template("gemm", {})
    w.view_a.a_shape = [0]
    w.view_b.a_shape = [0]
    with pytest.raises(Error) as e:
        Plan(w)
    assert e.value.code == ErrorCode.OutOfRange           # phase_range on an empty extent
    with pytest.raises(Error) as e:
        Plan(W.build_template("gemm", {}), FLAG_ARGMIN)
    assert e.value.code == ErrorCode.UnsupportedProgram   # argmin needs the SAD kernel


@pytest.mark.parametrize("make", [
    lambda: W.conv_nchw_view(0, 64, 14, 14, 64, 3, 1, 1),     # empty batch
    lambda: W.maxpool_nchw_view(0, 8, 16, 16),
    lambda: W.me_view(64, 128, 16, 16, pairs=0),               # no frame pairs
])
def test_empty_outputs_rejected_like_reference_tensor(make):
    # the reference builds the output Tensor from p_shape, and Tensor rejects
    # zero extents with BadParams (tensor.hpp:167-169): no empty run exists
    with pytest.raises(Error) as e:
        Plan(make())
    assert e.value.code == ErrorCode.BadParams


def test_reject_out_of_range_views_go_to_checking_interpreter():
    w = W.build_template("maxpool", {"h": 4, "w": 4, "k": 2})
    w.view_a.terms[1].offset = -1
    assert Plan(w).kernel == Kernel.GENERIC   # the interpreter raises OutOfRange at run time


def test_generators_match_reference_fill_random():
    from tests.golden_io import load
    g = load()
    for seed in (1, 2, 3, 4, 5, 2001, 2002):
        assert np.array_equal(W.gen_uniform([256], seed), g[f"fill_f32/{seed}"])
        assert np.array_equal(W.gen_range_i16([256], seed), g[f"fill_i16/{seed}"])


def test_bf16_conversion_rne():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.3e38, np.inf, -0.0], np.float32)
    b = W.to_bf16_bits(x)
    back = W.bf16_bits_to_f32(b)
    assert back[0] == 1.0 and back[1] == 1.0 and back[2] == 1.015625 and back[3] == -2.5
    assert np.isinf(back[5]) and np.signbit(back[6])


def test_device_entry_points_fail_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    w = W.config_workload("C1", scale=8)
    with pytest.raises(Error) as e:
        Plan(w).run_host(w.src_a, w.src_b)
    assert e.value.code == ErrorCode.Cuda


def test_gemm_lowers_to_tensor_core_kernel_real32_only():
    from paper_1911_03458_b200 import Kernel, Plan
    from paper_1911_03458_b200 import workloads as W
    w = W.build_template("gemm", {"m": 33, "n": 40, "k": 70})
    W.fill_random(w, 1, 2)
    p = Plan(w)
    assert p.kernel == Kernel.CONV_TC and "gemm M=33 N=40 K=70" in p.description
    wf = W.build_template("gemm", {"m": 5, "n": 6, "k": 7, "fix": 1, "frac": 6})
    W.fill_random(wf, 1, 2)
    assert Plan(wf).kernel == Kernel.GENERIC  # FIX16: exact interpreter


def test_maxpool_reject_view_b_goes_to_error_path():
    # run_full gathers port B at every step (engine.hpp:128-133) although the
    # max program never reads it: an out-of-range REJECT view_b must raise
    # OutOfRange like the reference, so K1 must not take such a workload
    w = W.maxpool_nchw_view(2, 3, 8, 8)
    assert Plan(w).kernel == Kernel.MAXPOOL
    w.view_b.boundary = W.Boundary.Reject
    assert Plan(w).kernel == Kernel.MAXPOOL          # in range: still K1
    w.view_b.terms = [ViewTerm(0, 0, 1, 0)]            # image index into a (1,) source
    assert Plan(w).kernel == Kernel.GENERIC


def _me_pair_views(h, wd, r, pairs=None):
    w16 = W.me_view(h, wd, 16, r, pairs=pairs)
    w8 = W.me_view(h, wd, 8, r, pairs=pairs)
    return w16, w8


def test_multi_plan_fuses_c5_block_sizes():
    from paper_1911_03458_b200 import PlanGroup
    w16, w8 = _me_pair_views(2160, 3840, 32, pairs=4)
    g = PlanGroup([w16, w8], FLAG_ARGMIN | FLAG_NO_MAP)
    assert g.kernel == Kernel.SAD and "fused" in g.description
    b16, b8 = 4 * 135 * 240, 4 * 270 * 480
    assert g.info.aux_elems == 3 * (b16 + b8) and g.info.out_elems == 0
    assert [m["aux_offset"] for m in g.members] == [0, 3 * b16]
    assert g.info.n_outputs == (b16 + b8) * 65 * 65
    assert g.info.algorithmic_ops == (b16 * 256 + b8 * 64) * 65 * 65
    assert g.info.executed_ops == b8 * 64 * 65 * 65    # the 16x16 SADs are sums of 8x8 ones
    assert g.info.launches_per_run == 1
    # member order does not matter
    g2 = PlanGroup([w8, w16], FLAG_ARGMIN | FLAG_NO_MAP)
    assert g2.kernel == Kernel.SAD and [m["aux_offset"] for m in g2.members] == [0, 3 * b8]
    # host pipelining slices by frame pairs; every record range lands once
    sl = g.host_slices()
    assert len(sl) >= 2
    fine = sorted((s["aux_lo"], s["aux_hi"]) for s in sl)
    coarse = sorted((s["aux2_lo"], s["aux2_hi"]) for s in sl)
    assert fine[0][0] == 4 * 3 * b16 and fine[-1][1] == 4 * 3 * (b16 + b8)
    assert coarse[0][0] == 0 and coarse[-1][1] == 4 * 3 * b16
    for lst in (fine, coarse):
        assert all(a[1] == b[0] for a, b in zip(lst, lst[1:]))


def test_multi_plan_unfusable_runs_members():
    from paper_1911_03458_b200 import PlanGroup
    # +/-16 window: no fused kernel; H = 72: 9 rows of 8x8 blocks are not 2 x 4
    for h, r in ((2160, 16), (72, 32)):
        w16, w8 = _me_pair_views(h, 256, r)
        g = PlanGroup([w16, w8], FLAG_ARGMIN | FLAG_NO_MAP)
        assert g.kernel == Kernel.MULTI and g.info.launches_per_run == 2
    # maps requested: separate launches too
    w16, w8 = _me_pair_views(2160, 3840, 32)
    assert PlanGroup([w16, w8], FLAG_ARGMIN).kernel == Kernel.MULTI
    # a conv and a max-pool over different sources: BadParams
    c = W.conv_nchw_view(1, 8, 10, 10, 4)
    m = W.maxpool_nchw_view(1, 8, 10, 10)
    with pytest.raises(Error) as ei:
        PlanGroup([c, m])
    assert ei.value.code == ErrorCode.BadParams


def test_u16_sad_map_lowering():
    # an exact uint16 SAD map (8-bit 16x16 blocks: every SAD <= 65,280) halves
    # the map's bytes; other kernels do not take it
    w = W.me_view(64, 96, 16, 16)
    w.dtype_out = W.Dtype.U16
    plan = Plan(w, FLAG_ARGMIN)
    assert plan.kernel == Kernel.SAD
    assert plan.info.out_bytes == 2 * plan.info.out_elems
    c = W.conv_nchw_view(1, 8, 10, 10, 4)
    c.dtype_out = W.Dtype.U16
    with pytest.raises(Error):
        Plan(c)


def test_plan_member_of_single_plan_is_itself():
    w = W.maxpool_nchw_view(1, 2, 8, 8)
    plan = Plan(w)
    info = _capi.PlanInfoC()
    oo, ao = C.c_int64(-1), C.c_int64(-1)
    assert plan.lib.merit_dev_plan_member(plan.handle, 0, C.byref(info), C.byref(oo), C.byref(ao)) == 0
    assert info.n_outputs == plan.info.n_outputs and oo.value == 0 and ao.value == 0
    assert plan.lib.merit_dev_plan_member(plan.handle, 1, C.byref(info), None, None) != 0
