#!/bin/bash
# Warm-start Gauss-Jordan with one sync per pivot (deferred pivot-row scale; default build) vs two (lib_prev).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
  echo "arctic N=10: two-sync $(run build/ab/lib_prev.so --task arctic_transport --robots 10 --envs 131072 --max-steps 100) | one-sync $(run paper_2505_06771_b200/libmrsim_cuda.so --task arctic_transport --robots 10 --envs 131072 --max-steps 100)"
done
