# HB batched evaluation (config 3): tests, bench, per-kernel launch times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py -m gpu -q -x > gpurun_out/t_hb.log 2>&1; echo "hb tests rc=$?" > gpurun_out/hb.txt
tail -2 gpurun_out/t_hb.log >> gpurun_out/hb.txt
timeout 300 python bench.py --config c3 --steps 500 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_c3.log').read().strip().splitlines()[-1]); print('c3', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us', d['roofline'], d['e2e']['value'])" >> gpurun_out/hb.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv \
   python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/hb.txt
cat gpurun_out/hb.txt
