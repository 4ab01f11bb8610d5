#!/bin/bash
# Refresh the committed measurements on the GPU box (run under gpurun):
#   bench lines (default settings, CPU baseline included) -> gpurun_out/bench_<tag>_<C>.json
#   ncu launch list + one --set full capture of the dominant kernel per config,
#   each only after the same bench command exited 0 without ncu.
# Then, in the container: python tools/ncu_summary.py profiles/<round> <tag>_c1=C1 ...
# usage: tools/refresh_profiles.sh TAG [configs...]
set -u
TAG=$1; shift
CONFIGS=${*:-C1 C2 C3 C4 C5}
mkdir -p gpurun_out
declare -A KERN=([C1]=maxpool [C2]=sad_ [C3]=conv_s1 [C4]=conv_tma [C5]=sad_async)
for C in $CONFIGS; do
  c=$(echo "$C" | tr 'C' 'c')
  timeout 900 python bench.py --config "$C" > "gpurun_out/bench_${TAG}_${C}.json" 2> "gpurun_out/bench_${TAG}_${C}.err" || { echo "$C bench failed"; continue; }
  SHORT="python bench.py --config $C --steps 6 --warmup 3 --no-cpu-baseline --soak 0 --e2e-steps 1"
  $SHORT > "gpurun_out/plain_${TAG}_${c}.log" 2>&1 || { echo "$C short run failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "gpurun_out/launches_${TAG}_${c}.csv" $SHORT > "gpurun_out/ncu_launch_${TAG}_${c}.log" 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KERN[$C]}" -s 3 -c 1 \
    -o "gpurun_out/prof_${TAG}_${c}" -f $SHORT > "gpurun_out/ncu_full_${TAG}_${c}.log" 2>&1
  echo "$C done"
done
for C in $CONFIGS; do
  if [[ "$C" == "C5" || "$C" == "C2" ]]; then
    timeout 900 python bench.py --impl reference --config "$C" > "gpurun_out/bench_${TAG}_ref_${C}.json" 2>&1
  fi
done
