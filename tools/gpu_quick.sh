# quick validation: selected tests + selected bench configs + ncu captures of small drivers
#   TESTS="test_gpu_ising" CONFIGS="c4 c4potts" NCU="tools/prof_ising.py:gibbs_packed tools/prof_hb.py:hb_kernel"
set -x
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
for t in ${TESTS:-}; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q > gpurun_out/$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/rc.txt
done
for c in ${CONFIGS:-}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/rc.txt
done
for spec in ${NCU:-}; do
  drv=${spec%%:*}; pat=${spec##*:}
  timeout 300 python $drv > gpurun_out/prof_plain_$pat.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 \
      -o gpurun_out/ncu_$pat -f python $drv > gpurun_out/ncu_$pat.log 2>&1
  echo "ncu $pat rc=$?" >> gpurun_out/rc.txt
done
cat gpurun_out/rc.txt
