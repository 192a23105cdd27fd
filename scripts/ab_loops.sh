#!/bin/bash
# QP slot loops two slots per trip (lib_loops = default build) vs one (lib_base).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in arctic_transport:10:131072:100 material_transport:10:131072:70 discovery:6:32768:100 navigation:4:65536:70 rware:6:65536:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: base $(run build/ab/lib_base.so --task $t --robots $n --envs $e --max-steps $h) | loops2 $(run build/ab/lib_loops.so --task $t --robots $n --envs $e --max-steps $h)"
done; done
