# r02 pass F: fp32-X row-dot consumer A/B (tune f32_pairs=3, 7 and 15 consumer warps) + c4 e2e parts
O=gpurun_out/r02f
mkdir -p $O
cat > /tmp/rowdot_check.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import glm_oracle as gl
from paper_1310_1537_b200 import _lib, glm
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan
from paper_1310_1537_b200.sampler import GaussianPrior
from paper_1310_1537_b200.synthetic import baseline_design
for k, n in [(100, 40_001), (36, 9_999), (44, 70_000), (108, 5_000)]:
    for knobs in ({"f32_pairs": 3}, {"f32_pairs": 3, "stream_ncw": 15}):
        with _lib.tuned(**knobs):
            x, y, _, beta = baseline_design(n, k, seed=k)
            d = DesignMatrix(x, y); prior = GaussianPrior.isotropic(k, 0.0, 10.0)
            plan = ExecPlan(x_storage="f32")
            r = glm.log_posterior_grad(d, beta, prior, plan)
            xr = x.astype(np.float32).astype(np.float64)
            f, g = gl.log_posterior_grad(xr, y, beta, prior.mu, prior.sigma)
            ef = abs(r.f - f) / max(abs(f), 1.0); eg = float(np.max(np.abs(r.g - g) / np.maximum(np.abs(g), 1.0)))
            fl = glm.loglike(d, beta, plan); f0 = gl.loglike_grad(xr, y, beta)[0]
            print(k, n, knobs, d.on_device(0, "f32").geometry(), "rel f", ef, "rel g", eg, "loglike rel", abs(fl - f0) / abs(f0), flush=True)
            assert ef < 1e-10 and eg < 1e-10
            d.release_device()
PY
timeout 600 python /tmp/rowdot_check.py > $O/rowdot_check.log 2>&1; echo "rowdot check rc=$?" > $O/summary.txt
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_pairs1.log 2>&1
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 > $O/c1f32_rowdot7.log 2>&1
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 --tune stream_ncw=15 > $O/c1f32_rowdot15.log 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.log 2>&1
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1
cat $O/summary.txt
