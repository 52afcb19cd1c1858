"""A/B: row-per-lane flat kernel with 7 vs 15 consumer warps at small K (N = 1e7)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402

n = 10_000_000
for k in (2, 4, 8, 12, 16):
    gen = np.random.default_rng(k)
    x = gen.standard_normal((n, k))
    y = (gen.random(n) < 0.5).astype(float)
    betas = gen.normal(0, 0.1, (50, k))
    res = {}
    for ncw in ("7", "15"):
        os.environ["PM_ROWS_NCW"] = ncw
        d = glm.DesignMatrix(x, y)
        dev = d.on_device(0)
        dev.time_launches(betas[:5], False, True)
        res[ncw] = dev.time_launches(betas, False, True) / len(betas)
        d.release_device()
    print(k, {kk: round(v * 1e3, 1) for kk, v in res.items()}, "us",
          {kk: round(n * (k * 8 + 8) / (v * 1e-3) / 1e9) for kk, v in res.items()}, "GB/s", flush=True)
