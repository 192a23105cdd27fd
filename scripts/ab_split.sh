#!/bin/bash
# Split steps (half-step warp tasks; build/ab/lib_split.so with MRSIM_SPLIT=1) vs the same build whole-step vs the
# shipped kernel, same box.
run() { timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])" 2>&1 | tail -1; }
for rep in 1 2; do
for tn in navigation:4:65536:70 discovery:6:32768:100 predator_prey:6:32768:100; do
  IFS=: read t n e h <<< "$tn"
  a=$(run --task $t --robots $n --envs $e --max-steps $h)
  b=$(MRSIM_LIB_PATH=build/ab/lib_split.so run --task $t --robots $n --envs $e --max-steps $h)
  c=$(MRSIM_SPLIT=1 MRSIM_LIB_PATH=build/ab/lib_split.so run --task $t --robots $n --envs $e --max-steps $h)
  echo "$t N=$n B=$e: shipped $a | split-build whole $b | split-build split $c"
done; done
