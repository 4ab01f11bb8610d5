#!/bin/bash
# Profile one config on the GPU box: plain run, launch list, full capture of the top kernel.
# usage: tools/profile.sh C2 sad_kernel [tag]
set -u
CFG=$1; KERN=$2; TAG=${3:-$1}
CMD="python bench.py --config $CFG --steps 6 --warmup 3 --no-cpu-baseline --soak 0 --e2e-steps 1"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KERN -s 3 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile $TAG rc=$?"
