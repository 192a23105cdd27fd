#!/bin/bash
CMD="python bench.py --task material_transport --robots 10 --envs 131072 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --policy mlp"
$CMD > gpurun_out/prof_pol_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:policy_kernel -s 3 -c 1 -o gpurun_out/prof_policy -f $CMD > gpurun_out/prof_pol_ncu.log 2>&1
echo "prof rc=$?"
