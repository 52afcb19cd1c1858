# A/B of the HB sweep kernel knobs (PM_HBS_SPEC speculation, PM_HBS_MINB CTAs/SM register budget)
mkdir -p gpurun_out
for cfg in "2 4" "2 7" "2 8" "1 8" "1 4"; do
  set -- $cfg
  PM_HBS_SPEC=$1 PM_HBS_MINB=$2 timeout 600 python bench.py --config c3sweep --steps 10 --warmup 2 --no-cpu-baseline \
    > gpurun_out/hbs_spec$1_minb$2.log 2>&1
done
