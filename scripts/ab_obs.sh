#!/bin/bash
# rware obstacle rows: rsqrt + slot-indexed centres (lib_obsrsqrt = default build) vs sqrt/divide + register copies (lib_warm1).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in rware:4:65536:100 rware:6:65536:100 navigation:4:65536:70; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: before $(run build/ab/lib_warm1.so --task $t --robots $n --envs $e --max-steps $h) | after $(run build/ab/lib_obsrsqrt.so --task $t --robots $n --envs $e --max-steps $h)"
done; done
