#!/bin/bash
# Bench + ncu evidence for one config. Usage: scripts/gpu_profile.sh TAG [bench args...]
# Writes gpurun_out/bench_TAG.json, launches_TAG.csv, prof_TAG.ncu-rep
TAG=$1; shift
mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile $TAG rc=$?"
