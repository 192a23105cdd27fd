#!/bin/bash
# QP warm start: Gauss-Jordan rebuild (w1 = default) vs bordered rebuild (round-2 first version) vs off.
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for tn in arctic_transport:10:131072:100 material_transport:10:131072:70 discovery:6:32768:100 navigation:4:65536:70; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: off $(run build/ab/lib_warm0.so --task $t --robots $n --envs $e --max-steps $h) | bordered $(run build/ab/lib_warm1_bordered.so --task $t --robots $n --envs $e --max-steps $h) | GJ-arctic $(run build/ab/lib_warm1.so --task $t --robots $n --envs $e --max-steps $h) | GJ-all $(run build/ab/lib_warm2.so --task $t --robots $n --envs $e --max-steps $h)"
done
