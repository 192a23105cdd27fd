#!/bin/bash
# Caller actions read before the state loads (default build) vs after them (lib_prev): host-buffer e2e and device value.
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 60 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"; }
for rep in 1 2 3; do
  echo "nav: after $(run build/ab/lib_prev.so) | first $(run paper_2505_06771_b200/libmrsim_cuda.so)"
done
echo "disc6: after $(run build/ab/lib_prev.so --task discovery --robots 6 --envs 32768 --max-steps 100) | first $(run paper_2505_06771_b200/libmrsim_cuda.so --task discovery --robots 6 --envs 32768 --max-steps 100)"
