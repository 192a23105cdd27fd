#!/bin/bash
# ncu of the default (lane-group) step kernel on the bench workload; full set, source-level.
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$CMD > gpurun_out/prof_lane_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 \
    -o gpurun_out/prof_lane -f $CMD > gpurun_out/prof_lane_ncu.log 2>&1
echo "prof rc=$?"
