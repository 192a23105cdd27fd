#!/bin/bash
# A/B of the QP warm start: MRSIM_QP_WARM = 0 (off), 1 (arctic only, default), 2 (every task).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for tn in arctic_transport:10:131072 material_transport:10:131072 discovery:6:32768 predator_prey:6:32768 rware:6:65536 navigation:4:65536 foraging:6:65536; do
  IFS=: read t n e <<< "$tn"
  line="$t N=$n B=$e:"
  for w in 0 1 2; do line="$line | w$w $(run build/ab/lib_warm$w.so --task $t --robots $n --envs $e --max-steps $([ $t = navigation ] && echo 70 || ([ $t = material_transport ] && echo 70 || echo 100)))"; done
  echo "$line"
done
