#!/bin/bash
# L = 16 step kernels (N = 9..16): 4 resident blocks per SM (<= 128 registers) vs 3 (default, <= 168).
run() { MRSIM_LIB_PATH=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --rollout 0 ${@:2} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g env/s %.3f ms' % (d['value'], d['ms_per_step']))" 2>&1 | tail -1; }
for rep in 1 2; do
  echo "arctic N=10: minb3 $(run paper_2505_06771_b200/libmrsim_cuda.so --task arctic_transport --robots 10 --envs 131072 --max-steps 100) | minb4 $(run build/ab/lib_l16minb4.so --task arctic_transport --robots 10 --envs 131072 --max-steps 100)"
  echo "MT N=10: minb3 $(run paper_2505_06771_b200/libmrsim_cuda.so --task material_transport --robots 10 --envs 131072) | minb4 $(run build/ab/lib_l16minb4.so --task material_transport --robots 10 --envs 131072)"
done
