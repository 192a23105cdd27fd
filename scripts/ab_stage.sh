#!/bin/bash
# Warp-staged float4 obs stores on the device path (lib_stage1 = default) vs direct per-lane stores (lib_stage0).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms e2e %.4g' % (d['value'], d['ms_per_step'], d['e2e']['value']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 rware:4:65536:100 material_transport:10:131072:70 arctic_transport:10:131072:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: direct $(run build/ab/lib_stage0.so --task $t --robots $n --envs $e --max-steps $h) | staged-float4 $(run build/ab/lib_stage1.so --task $t --robots $n --envs $e --max-steps $h)"
done; done
