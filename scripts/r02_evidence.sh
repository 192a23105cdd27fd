#!/bin/bash
# Round-2 evidence run: default bench (+ --verify), 2-rank bench, launch list, arctic N=10 ncu.
set -x
python bench.py --steps 50 --warmup 5 --verify > gpurun_out/e_bench_verify.json 2> gpurun_out/e_bench_verify.err
python bench.py --gpus 2 --steps 20 --warmup 5 --e2e-steps 5 --no-cpu-baseline > gpurun_out/e_bench_2rank.json 2> gpurun_out/e_bench_2rank.err
python bench.py --task arctic_transport --robots 10 --envs 131072 --max-steps 100 --steps 20 --warmup 3 --cpu-seconds 8 > gpurun_out/e_bench_arctic10.json 2> gpurun_out/e_bench_arctic10.err
python bench.py --task material_transport --robots 10 --envs 131072 --steps 20 --warmup 3 --cpu-seconds 8 > gpurun_out/e_bench_mt10.json 2> gpurun_out/e_bench_mt10.err
python bench.py --task discovery --robots 6 --envs 32768 --max-steps 100 --steps 50 --warmup 3 --cpu-seconds 8 > gpurun_out/e_bench_disc6.json 2> gpurun_out/e_bench_disc6.err
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/e_launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/e_launches_nav4.csv $CMD > gpurun_out/e_launch_ncu.log 2>&1
ACMD="python bench.py --task arctic_transport --robots 10 --envs 131072 --max-steps 100 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$ACMD > gpurun_out/e_arctic_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_arctic10 -f $ACMD > gpurun_out/e_arctic_ncu.log 2>&1
echo evidence done
