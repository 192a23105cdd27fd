#!/bin/bash
# A/B of the default build vs build/ab/lib_prev.so (set per experiment; see the commit that uses it).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])" 2>&1 | tail -1; }
S=paper_2505_06771_b200/libmrsim_cuda.so
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 foraging:4:65536:100 material_transport:10:131072:70 arctic_transport:10:131072:100 rware:6:65536:100; do
  IFS=: read t n e h <<< "$tn"; A="--task $t --robots $n --envs $e --max-steps $h"
  echo "$t N=$n: prev $(run build/ab/lib_prev.so $A) | new $(run $S $A)"
done; done
