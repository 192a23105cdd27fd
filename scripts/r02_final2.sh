#!/bin/bash
# Round-2 closing evidence on the shipped build: GPU suite (shipped + device-checks builds), smoke,
# bench lines (nav + verify, reference arm, 2 ranks, MT / arctic / discovery), nav launch list.
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g_gpu_tests.log 2>&1; echo "gpu suite: $(tail -1 gpurun_out/g_gpu_tests.log)"
bash scripts/device_checks.sh > gpurun_out/g_device_checks.log 2>&1; echo "checks suite: $(tail -1 gpurun_out/g_device_checks.log)"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1; tail -1 gpurun_out/g_smoke.log
python bench.py --steps 50 --warmup 5 --verify > gpurun_out/g_bench_verify.json 2> gpurun_out/g_bench_verify.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err
python bench.py --gpus 2 --steps 20 --warmup 5 --e2e-steps 5 --no-cpu-baseline > gpurun_out/g_bench_2rank.json 2> gpurun_out/g_bench_2rank.err
python bench.py --task arctic_transport --robots 10 --envs 131072 --max-steps 100 --steps 20 --warmup 3 --cpu-seconds 8 > gpurun_out/g_bench_arctic10.json 2> gpurun_out/g_bench_arctic10.err
python bench.py --task material_transport --robots 10 --envs 131072 --steps 20 --warmup 3 --cpu-seconds 8 > gpurun_out/g_bench_mt10.json 2> gpurun_out/g_bench_mt10.err
python bench.py --task discovery --robots 6 --envs 32768 --max-steps 100 --steps 50 --warmup 3 --cpu-seconds 8 > gpurun_out/g_bench_disc6.json 2> gpurun_out/g_bench_disc6.err
for f in gpurun_out/g_bench_*.json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d.get('value'), (d.get('e2e') or {}).get('value'), d.get('ms_per_step'), (d.get('verify') or {}).get('ok'))")"; done
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/g_launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/g_launches_nav4.csv $CMD > gpurun_out/g_launch_ncu.log 2>&1
echo final done
