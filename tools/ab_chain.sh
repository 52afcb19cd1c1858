# A/B of the resident chain kernel knobs (unroll x CTAs per SM), 20 iterations at config-2 shape
mkdir -p gpurun_out
for u in 1 2 4; do for b in 1 2 3; do
  echo "U=$u B=$b $(PM_CHAIN_UNROLL=$u PM_CHAIN_BLOCKS_PER_SM=$b timeout 300 python tools/prof_chain.py 20 2>&1 | tail -1)" >> gpurun_out/ab_chain.txt
done; done
cat gpurun_out/ab_chain.txt
