# r02 pass J: row-dot consumer with self-producing consumer warps: parity + repeats + bench A/B
O=gpurun_out/r02l
mkdir -p $O
cat > /tmp/rowdot3_check.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import glm_oracle as gl
from paper_1310_1537_b200 import _lib, glm
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan
from paper_1310_1537_b200.sampler import GaussianPrior
from paper_1310_1537_b200.synthetic import baseline_design
for k, n in [(100, 40_001), (100, 1_000_003), (36, 9_999), (108, 5_000), (116, 33), (60, 200_000)]:
    for knobs in ({"f32_pairs": 3, "stream_ncw": 15}, {"f32_pairs": 3}, {"f32_pairs": 3, "stream_ncw": 15, "f32_selfprod": 1}, {"f32_pairs": 3, "stream_ncw": 15, "f32_selfprod": 0}):
        with _lib.tuned(**knobs):
            x, y, _, betas = baseline_design(n, k, seed=k, n_eval=2)
            d = DesignMatrix(x, y); prior = GaussianPrior.isotropic(k, 0.0, 10.0)
            plan = ExecPlan(x_storage="f32")
            r = glm.log_posterior_grad(d, betas[0], prior, plan)
            xr = x.astype(np.float32).astype(np.float64)
            f, g = gl.log_posterior_grad(xr, y, betas[0], prior.mu, prior.sigma)
            ef = abs(r.f - f) / max(abs(f), 1.0); eg = float(np.max(np.abs(r.g - g) / np.maximum(np.abs(g), 1.0)))
            fl = glm.loglike(d, betas[0], plan); f0 = gl.loglike_grad(xr, y, betas[0])[0]
            print(k, n, knobs, d.on_device(0, "f32").geometry(), "rel f", ef, "rel g", eg, flush=True)
            assert ef < 1e-10 and eg < 1e-10 and abs(fl - f0) / abs(f0) < 1e-10
            for i in range(30):
                o = glm.log_posterior_grad(d, betas[1], prior, plan)
                a = glm.log_posterior_grad(d, betas[0], prior, plan)
                assert a.f == r.f and np.array_equal(a.g, r.g), i
            d.release_device()
print("ok")
PY
timeout 900 python /tmp/rowdot3_check.py > $O/check.log 2>&1; echo "rowdot selfprod check rc=$?" > $O/summary.txt
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 --tune stream_ncw=15 > $O/c1f32_rowdot16_self3.log 2>&1
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 --tune stream_ncw=15 --tune f32_selfprod=0 > $O/c1f32_rowdot15_prod.log 2>&1
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 --tune stream_ncw=15 --tune f32_selfprod=1 > $O/c1f32_rowdot15_self1.log 2>&1
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_pairs1.log 2>&1
cat $O/summary.txt
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 --tune f32_pairs=3 > $O/c1f32_rowdot8_self3.log 2>&1
