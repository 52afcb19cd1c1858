# correctness + bench + ncu evidence in one gpurun call
#   TESTS=1 BENCH=1 EXTRA=1 PROFILE=1 bash tools/gpu_check.sh
set -x
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
  for t in test_gpu_glm test_gpu_diff test_gpu_ising test_gpu_hb test_gpu_denoise test_gpu_rng test_gpu_hb_sweep test_gpu_dist test_cli; do
    timeout 900 python -m pytest tests/$t.py -m gpu -q > gpurun_out/$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/rc.txt
  done
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
fi
if [ "${EXTRA:-1}" = "1" ]; then
  for c in c1f32 c0 c2 c3 c3sweep c4 c4potts rng; do
    timeout 600 python bench.py --config $c ${EXTRA_ARGS:---no-cpu-baseline} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/rc.txt
  done
fi
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  echo "ncu-launch rc=$?" >> gpurun_out/rc.txt
  timeout 300 python tools/prof_glm.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 2 -c 1 \
      -o gpurun_out/glm_stream_full -f python tools/prof_glm.py > gpurun_out/ncu_full.log 2>&1
  echo "ncu-full rc=$?" >> gpurun_out/rc.txt
fi
cat gpurun_out/rc.txt
