#!/bin/bash
# ptxas knobs on the whole library: -regUsageLevel 2 / 8 (default 5) and -allow-expensive-optimizations, vs the shipped build.
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])" 2>&1 | tail -1; }
S=paper_2505_06771_b200/libmrsim_cuda.so
for tn in navigation:4:65536:70 discovery:6:32768:100 material_transport:10:131072:70 arctic_transport:10:131072:100 rware:6:65536:100; do
  IFS=: read t n e h <<< "$tn"
  A="--task $t --robots $n --envs $e --max-steps $h"
  echo "$t N=$n: shipped $(run $S $A) | rul2 $(run build/ab/lib_rul2.so $A) | rul8 $(run build/ab/lib_rul8.so $A) | aeo $(run build/ab/lib_aeo.so $A) | shipped $(run $S $A)"
done
