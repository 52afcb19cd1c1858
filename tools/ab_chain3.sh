for sp in 1 2 4 6; do for u in 1 2; do
  echo "SPEC=$sp U=$u $(PM_CHAIN_SPEC=$sp PM_CHAIN_UNROLL=$u PM_CHAIN_TIMING=1 python tools/c2_var.py 2>&1 | grep kernel | sed -n 3p)"
done; done
