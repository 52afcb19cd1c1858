import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import glm_oracle as gl
from paper_1310_1537_b200.hb import CsrGroups, hb_log_posterior_grad
for k, sizes in ((32, [100_000, 37, 250_001]), (32, [350_038]), (32, [64] * 5000), (30, [100_000, 37, 250_001])):
    gen = np.random.default_rng(k)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    x = gen.standard_normal((int(off[-1]), k)); y = (gen.random(int(off[-1])) < 0.45).astype(float)
    betas = gen.normal(0, 0.3, (len(sizes), k))
    fr, gr = gl.hb_log_posterior_grad(x, y, off, betas)
    for st in ("7", "14", "21"):
        os.environ["PM_HB_ROWS_STAGES"] = st
        errs = []
        for rep in range(3):
            res = hb_log_posterior_grad(CsrGroups(x, y, off), betas)
            f = np.array([r.f for r in res])
            errs.append(float(np.max(np.abs(f - fr) / np.abs(fr))))
        print(k, len(sizes), "stages", st, errs, flush=True)
