#!/bin/bash
# Round-2 final evidence on the shipped build.
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/f_gpu_tests.log 2>&1; tail -2 gpurun_out/f_gpu_tests.log
python bench.py --steps 50 --warmup 5 --verify > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
python scripts/sweep_batch.py rware > gpurun_out/f_sweep_rware.jsonl 2> gpurun_out/f_sweep_rware.err
bash scripts/prof_lane.sh > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/prof_lane.ncu-rep 30 > gpurun_out/f_ncu_nav4.txt 2>&1
echo final done
