#!/bin/bash
# Host-buffer obs: warp stage at the cost of a resident block (default rule) vs the QP-workspace stage (no smem cost;
# MRSIM_AB_WS=1 on build/ab/lib_abws.so).
run() { MRSIM_LIB_PATH=build/ab/lib_abws.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 30 --rollout 0 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e %.4g' % d['e2e']['value'])" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in discovery:6:32768:100 material_transport:10:131072:70 rware:6:65536:100 foraging:6:65536:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: warp-stage $(run --task $t --robots $n --envs $e --max-steps $h) | ws-stage $(MRSIM_AB_WS=1 run --task $t --robots $n --envs $e --max-steps $h)"
done; done
