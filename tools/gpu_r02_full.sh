# full validation: smoke + every GPU test
O=gpurun_out/r02full
mkdir -p $O
timeout 600 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)" > $O/summary.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" >> $O/summary.txt
cat $O/summary.txt
