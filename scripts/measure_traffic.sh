#!/bin/bash
# DRAM traffic of the step kernel over a window of consecutive iterations of the timed bench loop
# (ncu, --cache-control none so L2 state carries between launches exactly as in the timed run).
# Every kernel is captured: a step's outputs stay in L2 at its end and reach DRAM when the next
# L2 flush (a 512 MiB read) evicts them, so the step's traffic = its own reads + writes plus the
# write-back its dirty lines cause inside the following flush kernel.
# Usage: scripts/measure_traffic.sh TAG [bench args...]   -> gpurun_out/traffic_TAG.csv
TAG=$1; shift
CMD="python bench.py --steps 14 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$CMD > gpurun_out/traffic_plain_$TAG.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none -s 12 -c 26 --csv --log-file gpurun_out/traffic_$TAG.csv \
    $CMD > gpurun_out/traffic_ncu_$TAG.log 2>&1
echo "traffic $TAG rc=$?"
