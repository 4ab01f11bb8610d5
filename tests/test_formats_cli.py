"""Reference file formats and the device CLI.

MRT1 bytes are pinned to the reference's own Tensor::write / Tensor::read
(tensor.hpp:123-163, through the compiled reference shim); manifests follow
tools/merit.cpp:102-118 + serialize.hpp; `bin/merit-dev run` is checked on CPU
with --dry-run (lowering + TilingPlan traffic) and on the GPU end to end
against the reference engine.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import binding as O
from paper_1911_03458_b200 import Error, ErrorCode, formats as F
from paper_1911_03458_b200 import workloads as W

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_1911_03458_b200" / "bin" / "merit-dev"
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built")


def _cli(*args):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True)


# ---------------------------------------------------------------- MRT1 ----
@needs_ref
@pytest.mark.parametrize("arr,frac", [
    (np.arange(24, dtype=np.float32).reshape(2, 3, 4) - 7.5, 0),
    (np.array([-32768, -1, 0, 1, 32767], np.int16), 9),
    (np.float32([np.inf, -0.0, 1e-38]), 0),
])
def test_mrt1_bytes_match_reference_writer(tmp_path, arr, frac):
    p = tmp_path / "t.mrt"
    F.write_mrt1(p, arr, frac)
    assert p.read_bytes() == O.ref_mrt1_bytes(arr, frac)
    got, fb = F.read_mrt1(p)
    ref, rfb = O.ref_mrt1_parse(p.read_bytes())
    assert fb == rfb == (frac if arr.dtype == np.int16 else 0)
    assert got.tobytes() == ref.tobytes() == np.ascontiguousarray(arr).tobytes()


@needs_ref
@pytest.mark.parametrize("data,code", [
    (b"MRT2\x00\x00\x01\x00\x01\x00\x00\x00", ErrorCode.BadMagic),
    (b"MRT1\x02\x00\x01\x00\x01\x00\x00\x00", ErrorCode.UnknownDtype),
    (b"MRT1\x00\x00\x01\x00\x02\x00\x00\x00\x00\x00\x80\x3f", ErrorCode.TruncatedPayload),
    (b"MRT1\x00\x00\x00\x00", ErrorCode.TruncatedPayload),     # rank 0
    (b"MRT1\x00\x00\x01\x00\x00\x00\x00\x00", ErrorCode.BadParams),  # extent 0
])
def test_mrt1_read_errors_like_reference(tmp_path, data, code):
    p = tmp_path / "bad.mrt"
    p.write_bytes(data)
    with pytest.raises(Error) as e:
        F.read_mrt1(p)
    with pytest.raises(Error) as r:
        O.ref_mrt1_parse(data)
    assert e.value.code == r.value.code == code


# ------------------------------------------------------------ manifests ----
@pytest.mark.parametrize("name,prm", [
    ("conv2d", {"h": 9, "w": 8, "k": 3}), ("maxpool", {"h": 9, "w": 11, "k": 3}),
    ("bilateral", {"h": 9, "w": 8, "k": 5}), ("gemm", {"m": 4, "n": 5, "k": 6, "fix": 1, "frac": 6}),
])
def test_manifest_round_trip(tmp_path, name, prm):
    w = W.build_template(name, prm)
    W.fill_random(w, 3, 4)
    path = F.write_manifest(tmp_path, w, "2x2,3x3")
    w2, tiling = F.load_manifest(path)
    assert tiling == "2x2,3x3"
    assert F.view_to_json(w2.view_a) == F.view_to_json(w.view_a)
    assert F.view_to_json(w2.view_b) == F.view_to_json(w.view_b)
    assert F.program_to_json(w2.program) == F.program_to_json(w.program)
    assert np.asarray(w2.src_a).tobytes() == np.asarray(w.src_a).tobytes()


def test_manifest_errors(tmp_path):
    w = W.build_template("conv2d", {"h": 6, "w": 6, "k": 3})
    W.fill_random(w, 1, 2)
    path = F.write_manifest(tmp_path, w)
    m = json.loads(path.read_text())
    m["program"]["segments"][0][0]["op"] = "FMA"
    path.write_text(json.dumps(m))
    with pytest.raises(Error) as e:
        F.load_manifest(path)
    assert e.value.code == ErrorCode.BadParams and "unknown op" in str(e.value)
    with pytest.raises(Error) as e:
        F.load_manifest(tmp_path / "missing.json")
    assert e.value.code == ErrorCode.Usage


# ------------------------------------------------------------------ CLI ----
@needs_ref
def test_cli_dry_run_traffic_matches_reference(tmp_path):
    w = W.build_template("conv2d", {"h": 68, "w": 68, "k": 5, "pad": 0})
    W.fill_random(w, 3, 4)
    path = F.write_manifest(tmp_path, w, "16x8,5x5")
    r = _cli("run", "--manifest", path, "--dry-run")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    _, ref = O.ref_run_tiled(w, [16, 8], [5, 5])
    assert list(rep["traffic"].values()) == [int(v) for v in ref]
    assert rep["naive_unrolled_words"] == 64 * 64 * 25 and rep["output_shape"] == [64, 64]
    assert rep["traffic"]["scratchpad_peak_words_a"] == 240


def test_cli_exit_codes(tmp_path):
    assert _cli("run").returncode == 2                                        # usage: no manifest
    assert _cli("run", "--manifest", tmp_path / "none.json").returncode == 2  # cannot open (Usage)
    assert _cli("frobnicate").returncode == 2
    w = W.build_template("maxpool", {"h": 6, "w": 6, "k": 2})
    W.fill_random(w, 1, 2)
    path = F.write_manifest(tmp_path, w)
    r = _cli("run", "--manifest", path, "--tile", "3", "--dry-run")
    assert r.returncode == 2                                                  # malformed tile (Usage)
    (tmp_path / "workload_a.mrt").write_bytes(b"XXXX")
    r = _cli("run", "--manifest", path, "--dry-run")
    assert r.returncode == 1 and "bad magic" in r.stderr                      # BadMagic -> 1


@pytest.mark.gpu
@pytest.mark.parametrize("name,prm,tol", [
    ("maxpool", {"h": 17, "w": 23, "k": 3, "stride": 2}, 0.0),
    ("conv2d", {"h": 20, "w": 20, "cin": 16, "cout": 32}, 1e-4),
    ("motion_estimation", {"h": 32, "w": 48, "blk": 8, "r": 4}, 0.0),
    ("bilateral", {"h": 9, "w": 8, "k": 5}, 0.0),
])
def test_cli_run_matches_reference_engine(cuda, tmp_path, name, prm, tol):
    w = W.build_template(name, prm)
    W.fill_random(w, 5, 6)
    if W.template_shares_input(name):
        w.src_b = w.src_a
    path = F.write_manifest(tmp_path, w)
    out = tmp_path / "out.mrt"
    r = _cli("run", "--manifest", path, "--out", out)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    got, _ = F.read_mrt1(out)
    want = O.ref_run_full(w) if O.ref_available() else O.run_full(w)
    assert list(got.shape) == rep["output_shape"]
    if tol == 0.0:
        assert got.tobytes() == np.asarray(want).tobytes()
    else:
        assert np.max(np.abs(got - want) / (1 + np.abs(want))) <= tol
    assert rep["checksum"] == pytest.approx(float(np.sum(got, dtype=np.float64)), rel=1e-9, abs=1e-9)
