# quick validation: selected tests + selected bench configs (+ optional ncu of one driver)
#   TESTS="test_gpu_ising" CONFIGS="c4 c4potts" NCU="tools/prof_ising.py:gibbs_packed" bash tools/gpu_quick.sh
set -x
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
for t in ${TESTS:-}; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q > gpurun_out/$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/rc.txt
done
for c in ${CONFIGS:-}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/rc.txt
done
if [ -n "${NCU:-}" ]; then
  drv=${NCU%%:*}; pat=${NCU##*:}
  timeout 300 python $drv ${NCU_ARGS:-} > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$pat -s 2 -c 1 \
      -o gpurun_out/ncu_$pat -f python $drv ${NCU_ARGS:-} > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/rc.txt
fi
cat gpurun_out/rc.txt
