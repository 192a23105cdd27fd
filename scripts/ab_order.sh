#!/bin/bash
# (The MRSIM_TASK_ORDER variant was measured here and reverted.)
# Cost-ordered warp-task dispatch on (default) vs off (MRSIM_TASK_ORDER=0), same library, interleaved.
run() { MRSIM_TASK_ORDER=$1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 navigation:4:262144:70 discovery:6:32768:100 material_transport:10:131072:70 arctic_transport:10:131072:100 rware:6:65536:100 foraging:4:65536:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n B=$e: off $(run 0 --task $t --robots $n --envs $e --max-steps $h) | on $(run 1 --task $t --robots $n --envs $e --max-steps $h)"
done; done
