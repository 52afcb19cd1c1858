# r02 pass I: pipeline floor (consumers' math compiled out) at the fp32-X and fp64 config-1 shapes
O=gpurun_out/r02i
mkdir -p $O
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_NO_COMPUTE.so timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_nocompute.log 2>&1
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_NO_COMPUTE.so timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=0 > $O/c1f32_nocompute_15w.log 2>&1
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_NO_COMPUTE.so timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 300 > $O/c1_nocompute.log 2>&1
tail -c 600 $O/*.log
