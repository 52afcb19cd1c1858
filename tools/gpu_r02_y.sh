# r02 pass Y: default library after compiling the self-producing column path out: c0 breakdown + tests
O=gpurun_out/r02y
mkdir -p $O
timeout 300 python tools/c0_breakdown.py --tag default > $O/c0_breakdown.jsonl 2> $O/c0.err
timeout 300 python tools/e2e_breakdown.py > $O/e2e_c0.json 2>> $O/c0.err
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0_b.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py tests/test_gpu_hb.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
cat $O/c0_breakdown.jsonl $O/e2e_c0.json $O/summary.txt
