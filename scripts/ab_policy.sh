#!/bin/bash
# Feedforward policy + step with the shipped hybrid (warp-per-env for N <= 4, tiled GEMM above).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 --policy mlp ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms' % (d['ms_per_step']))" 2>&1 | tail -1; }
for tn in navigation:4:65536:70 rware:4:65536:100 discovery:6:32768:100 material_transport:10:131072:70; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n policy+step: hybrid $(run build/ab/lib_hybrid.so --task $t --robots $n --envs $e --max-steps $h)"
done
