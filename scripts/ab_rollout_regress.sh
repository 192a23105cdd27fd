#!/bin/bash
# Single-step kernel before (build/ab/pre: the tree before mrsim_rollout) vs after (this tree).
run() { (cd $1 && timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1) | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 material_transport:10:131072:70 rware:4:65536:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: pre $(run build/ab/pre --task $t --robots $n --envs $e --max-steps $h) | templated $(run . --task $t --robots $n --envs $e --max-steps $h --rollout 0)"
done; done
