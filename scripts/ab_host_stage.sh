#!/bin/bash
# Host-path (zero-copy) obs: warp-staged float4 blocks even when the stage costs a resident block
# (MRSIM_FORCE_OBS_STAGE=1 on build/ab/lib_stage.so) vs the default rule (stage only when free).
run() { MRSIM_LIB_PATH=build/ab/lib_stage.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 30 --rollout 0 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))" 2>&1 | tail -1; }
for tn in discovery:6:32768:100 material_transport:10:131072:70 predator_prey:6:32768:100 rware:6:65536:100 arctic_transport:10:131072:100; do
  IFS=: read t n e h <<< "$tn"
  echo "$t N=$n: default $(run --task $t --robots $n --envs $e --max-steps $h) | forced $(MRSIM_FORCE_OBS_STAGE=1 run --task $t --robots $n --envs $e --max-steps $h)"
done
