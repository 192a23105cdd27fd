#!/bin/bash
# A/B of the env kernel (default build) vs the lane-group kernel on N <= 4 workloads, fp64.
run() { timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for envs in 65536 262144; do
  echo "env-kernel envs=$envs: $(run --envs $envs) | lane-groups $(run --envs $envs --lane-groups)"
done
for t in warehouse:4 random_waypoints:4 foraging:4; do
  echo "$t: env $(run --task ${t%%:*} --robots 4) | lane-groups $(run --task ${t%%:*} --robots 4 --lane-groups)"
done
