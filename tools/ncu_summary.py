"""Summarise ncu captures into files committed under profiles/.

usage: python tools/ncu_summary.py OUT_DIR TAG=CONFIG ...   (run in this container)

For every TAG it reads gpurun_out/prof_TAG.ncu-rep (one `ncu --set full`
capture of the dominant kernel) and gpurun_out/launches_TAG.csv (the
`--metrics gpu__time_duration.sum` launch list of the same bench command) and
writes OUT_DIR/TAG_full.json, OUT_DIR/TAG_launches.json, and merges the DRAM
bytes per launch into profiles/ncu_traffic.json (keyed by CONFIG), which
bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_active_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "smem_lsu_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "smem_tc_wavefronts_pct": ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "dyn_smem_bytes": ("launch__shared_mem_per_block_dynamic", None),
}


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def raw_metrics(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, vals = rows[0], rows[2] if len(rows) > 2 else rows[1]
    return dict(zip(hdr, vals))


def full_summary(rep: Path):
    d = raw_metrics(rep)
    s = {"kernel": d.get("Kernel Name", "")[:160]}
    for k, (m, _) in KEYS.items():
        v = _num(d.get(m, ""))
        if v is not None:
            s[k] = v
    if "duration_us" in s:  # base units: ns
        s["duration_us"] = s["duration_us"] / 1e3
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: _num(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and _num(v) is not None}
    tot = sum(stalls.values()) or 1.0
    s["stall_mix_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
    if "dram_read_bytes" in s and "dram_write_bytes" in s:
        s["dram_bytes_per_launch"] = s["dram_read_bytes"] + s["dram_write_bytes"]
    return s


def launch_summary(path: Path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = defaultdict(list)
    for r in rows[1:]:
        v = _num(r[vi])
        if v is not None:
            per[r[ki]].append(v)
    total = sum(sum(v) for v in per.values()) or 1.0
    return {"note": "ncu launch list (cold-cache, serialised replay): per-kernel share of the bench command",
            "kernels": [{"kernel": k[:120], "launches": len(v), "mean_us": round(sum(v) / len(v) / 1e3, 3),
                         "share_pct": round(100 * sum(v) / total, 1)}
                        for k, v in sorted(per.items(), key=lambda x: -sum(x[1]))]}


def main():
    out = Path(sys.argv[1]).resolve()
    out.mkdir(parents=True, exist_ok=True)
    traffic_path = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for arg in sys.argv[2:]:
        tag, cfg = arg.split("=")
        rep = ROOT / "gpurun_out" / f"prof_{tag}.ncu-rep"
        lst = ROOT / "gpurun_out" / f"launches_{tag}.csv"
        if rep.exists():
            s = full_summary(rep)
            (out / f"{tag}_full.json").write_text(json.dumps(s, indent=1) + "\n")
            if "dram_bytes_per_launch" in s:
                traffic[cfg] = {"dram_bytes_per_launch": s["dram_bytes_per_launch"], "kernel": s["kernel"],
                                "source": f"{out.relative_to(ROOT)}/{tag}_full.json (ncu --set full)"}
            print(tag, json.dumps({k: s[k] for k in ("duration_us", "dram_bytes_per_launch") if k in s}))
        if lst.exists():
            (out / f"{tag}_launches.json").write_text(json.dumps(launch_summary(lst), indent=1) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
