O=gpurun_out/r02d
mkdir -p $O
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_PHASES.so timeout 300 python tools/c0_breakdown.py --tag PHASES > $O/phases.log 2>&1
timeout 300 python tools/diff_latency.py > $O/diff_latency.log 2>&1
timeout 300 python tools/diff_latency.py > /dev/null 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"diff_eval|glm_stream" -c 40 --csv \
    --log-file $O/diff_launches.csv python tools/diff_latency.py > /dev/null 2>&1
for t in 0 1; do timeout 600 python bench.py --config c4 --steps 1000 --warmup 10 --no-cpu-baseline --tune gibbs_smem=$t > $O/c4_smem$t.log 2>&1; done
for t in 0 1; do timeout 600 python bench.py --config c4potts --steps 1000 --warmup 10 --no-cpu-baseline --tune gibbs_smem=$t > $O/c4p_smem$t.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_ising.py tests/test_gpu_rng.py -q -p no:cacheprovider > $O/pytest.log 2>&1
tail -2 $O/pytest.log
