# r02 pass U: pm_glm_wait polling the completion word (tune glm_poll): GLM / ABI / dist tests + e2e A/B
O=gpurun_out/r02u
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_abi.py tests/test_gpu_dist.py tests/test_gpu_protocols.py tests/test_gpu_diff.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for t in 1 0 1 0; do timeout 600 python bench.py --config c0 --no-cpu-baseline --tune glm_poll=$t >> $O/c0_poll$t.log 2>&1; done
for t in 1 0; do timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 --tune glm_poll=$t >> $O/c1_poll$t.log 2>&1; done
cat $O/summary.txt
