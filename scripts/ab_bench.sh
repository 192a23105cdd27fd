#!/bin/bash
# A/B throughput of library builds: scripts/ab_bench.sh "lib1 lib2 ..." "task:N task:N ..."
for lib in $1; do
  for tn in $2; do
    t=${tn%%:*}; n=${tn##*:}
    v=$(MRSIM_LIB_PATH=$lib timeout 300 python bench.py --task $t --robots $n --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.4g robot/s %.3f ms' % (d['value'], d['robot_steps_per_s'], d['ms_per_step']))" 2>&1)
    echo "$lib $t N=$n: $v"
  done
done
