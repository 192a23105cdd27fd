#!/bin/bash
# rware obstacle-slot indices packed in 4-bit nibbles (fewer registers): 3 blocks (lib_opk3) and 4 blocks (lib_opk4)
# vs the shipped build (int per slot, 3 blocks).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g' % d['value'])"; }
for rep in 1 2; do for n in 4 6; do
  echo "rware N=$n: shipped $(run paper_2505_06771_b200/libmrsim_cuda.so --task rware --robots $n --envs 65536 --max-steps 100) | opk3 $(run build/ab/lib_opk3.so --task rware --robots $n --envs 65536 --max-steps 100) | opk4 $(run build/ab/lib_opk4.so --task rware --robots $n --envs 65536 --max-steps 100)"
done; done
