#!/bin/bash
# QP warm start on every task (lib_warm2, -DMRSIM_QP_WARM=2) vs arctic only (default), after the counted GJ loops + L=16 at 4 blocks.
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for tn in material_transport:10:131072:70 discovery:6:32768:100 navigation:4:65536:70 rware:6:65536:100 predator_prey:6:32768:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: default $(run paper_2505_06771_b200/libmrsim_cuda.so --task $t --robots $n --envs $e --max-steps $h) | warm-all $(run build/ab/lib_warm2.so --task $t --robots $n --envs $e --max-steps $h)"
done
