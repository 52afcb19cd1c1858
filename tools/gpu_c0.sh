# c0 with the clean-L2 scrub; c4 cold-L2 sweeps; ncu duration of the c0 kernel
mkdir -p gpurun_out
timeout 900 python bench.py --config c0 > gpurun_out/bench_c0.log 2>&1; echo "c0 rc=$?"; tail -1 gpurun_out/bench_c0.log | cut -c1-200
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c0.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['config']['l2'])
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:glm -c 30 --csv python bench.py --config c0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c0.csv 2> gpurun_out/ncu_c0.err; echo "ncu rc=$?"
