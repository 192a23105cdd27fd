#!/bin/bash
# Resident blocks per SM for the L = 4 / 8 step kernels: 3 (12 warps) vs 4 (16 warps, default).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for tn in navigation:4:65536:70 navigation:4:262144:70 discovery:6:32768:100 foraging:4:65536:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n B=$e: minb4 $(run build/ab/lib_minb4.so --task $t --robots $n --envs $e --max-steps $h) | minb5 $(run build/ab/lib_minb5.so --task $t --robots $n --envs $e --max-steps $h)"
done
