#!/bin/bash
# Split steps (two half-step warp tasks per env group; default when the batch is < 8 task rounds) vs whole steps
# (MRSIM_SPLIT=0), same library.
run() { MRSIM_SPLIT=$1 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 40 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 predator_prey:6:32768:100 foraging:4:65536:100 navigation:4:16384:70; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n B=$e: whole $(run 0 --task $t --robots $n --envs $e --max-steps $h) | split $(run 1 --task $t --robots $n --envs $e --max-steps $h)"
done; done
