#!/bin/bash
# Host-step error word written by the step kernel's last warp (default build) vs a copy after the kernel (lib_prev).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 60 --rollout 0 ${@:2} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))" 2>&1 | tail -1; }
for rep in 1 2 3; do
  echo "prev $(run build/ab/lib_prev.so) | epilogue $(run paper_2505_06771_b200/libmrsim_cuda.so)"
done
