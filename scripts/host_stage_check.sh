#!/bin/bash
# Host-path tests and e2e per task after the host obs-stage rule (capi.cu: stage when it costs <= 1 block, not arctic).
python -m pytest tests -q -m gpu -p no:cacheprovider -k "host or dropin or invalid or earlier" 2>&1 | tail -2
run() { timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 30 --rollout 0 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))" 2>&1 | tail -1; }
for tn in navigation:4:65536:70 discovery:6:32768:100 material_transport:10:131072:70 rware:6:65536:100 rware:4:65536:100 foraging:6:65536:100 arctic_transport:10:131072:100; do
  IFS=: read t n e h <<< "$tn"; echo "$t N=$n: $(run --task $t --robots $n --envs $e --max-steps $h)"
done
