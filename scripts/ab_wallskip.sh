#!/bin/bash
# Lane-group scan with the exact wall-row skip (lib_wallskip = default build) vs without (lib_warm1).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 rware:4:65536:100 material_transport:10:131072:70 arctic_transport:10:131072:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: before $(run build/ab/lib_warm1.so --task $t --robots $n --envs $e --max-steps $h) | wall-skip $(run build/ab/lib_wallskip.so --task $t --robots $n --envs $e --max-steps $h)"
done
done
