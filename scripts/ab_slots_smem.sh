#!/bin/bash
# rware shelf centres read from shared memory (default build) vs indexed reads of the kernel-parameter copy (lib_prev).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])" 2>&1 | tail -1; }
S=paper_2505_06771_b200/libmrsim_cuda.so
for rep in 1 2; do
for tn in rware:4:65536:100 rware:6:65536:100 navigation:4:65536:70; do
  IFS=: read t n e h <<< "$tn"; A="--task $t --robots $n --envs $e --max-steps $h"
  echo "$t N=$n: param $(run build/ab/lib_prev.so $A) | smem $(run $S $A)"
done; done
