#!/bin/bash
# ncu of the one-thread-per-env step kernel on the bench workload (nav N=4 fp64).
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
$CMD > gpurun_out/prof_env_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 \
    -o gpurun_out/prof_env -f $CMD > gpurun_out/prof_env_ncu.log 2>&1
echo "rc=$?"
