"""Write profiles/<round>/README.md from the committed bench lines and ncu summaries.

usage: python tools/profiles_readme.py r01 TAG [C2=TAG2 ...]   (per-config capture tags)
"""
import json
import sys
from pathlib import Path

rnd, tag = sys.argv[1], sys.argv[2]
tags = {c: tag for c in ["C1", "C2", "C3", "C4", "C5"]}
tags.update(a.split("=") for a in sys.argv[3:])
d = Path(__file__).resolve().parents[1] / "profiles" / rnd
out = [f"# profiles/{rnd} — measurements (B200, sm_100a)", "",
       "Files: `bench_C*.json` = the `python bench.py --config C*` line (default settings);",
       "`bench_reference_C*.json` = `bench.py --impl reference --config C*` (the reference on the host cores);",
       "`<tag>_c*_full.json` = summary of one `ncu --set full --clock-control none` capture of the dominant kernel",
       "(`tools/refresh_profiles.sh`, summarised by `tools/ncu_summary.py`);",
       "`<tag>_c*_launches.json` = the `--metrics gpu__time_duration.sum` launch list of the same short bench command.",
       "ncu times are cold-cache and serialised (and run at the ncu-observed clock), so only the kernel's share of the",
       "step is comparable with the bench, not the absolute time.", "",
       "| config | kernel | bench ms/step | value (Goutputs/s) | roofline frac | ncu µs | ncu SM clock | tensor pipe % | "
       "ALU pipe % | issue active % | DRAM B / launch | top stalls |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for c in ["C1", "C2", "C3", "C4", "C5"]:
    b = json.loads((d / f"bench_{c}.json").read_text().strip().splitlines()[-1])
    f = json.loads((d / f"{tags[c]}_{c.lower()}_full.json").read_text())
    st = ", ".join(f"{k} {v}" for k, v in list(f["stall_mix_pct"].items())[:3])
    out.append(f"| {c} | `{b['roofline']['kernel']}` | {b['ms_per_step']} | {b['value']:.1f} | "
               f"{b['roofline']['frac']:.3f} ({b['roofline']['bound']}) | {f['duration_us']:.1f} | "
               f"{f['sm_clock_hz'] / 1e9:.2f} GHz | {f['tensor_pipe_active_pct']} | {f['alu_pipe_active_pct']} | "
               f"{f['issue_active_pct']} | {f['dram_bytes_per_launch']:.3e} | {st} |")
for rc in ["C5", "C2"]:
    rp = d / f"bench_reference_{rc}.json"
    if not rp.exists():
        continue
    r = json.loads(rp.read_text().strip().splitlines()[-1])
    ol = r.get("cpu_baseline_oracle_loop", {})
    out += ["", f"Reference arm ({rc}): {r['value']:.3e} Goutputs/s on {r['cpu_baseline']['cores']} host cores "
            f"({r['cpu_baseline'].get('cpu', '')}; {r['cpu_baseline']['kind']}; sample: {r['cpu_baseline']['sample']})."
            + (f"  The reference's oracle loop on the same cores: {ol['value']:.3e} Goutputs/s ({ol['sample']})." if ol else "")]
out.append("")
(d / "README.md").write_text("\n".join(out) + "\n")
print("\n".join(out[-9:]))
