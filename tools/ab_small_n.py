"""Fixed per-launch cost of the flat GLM kernel: device time per launch vs N (K=32 fp64)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402

for n in (32, 4096, 100_000, 1_000_000):
    gen = np.random.default_rng(1)
    x = gen.standard_normal((n, 32))
    y = (gen.random(n) < 0.5).astype(float)
    betas = gen.normal(0, 0.1, (200, 32))
    d = glm.DesignMatrix(x, y)
    dev = d.on_device(0)
    dev.time_launches(betas[:10], False, True)
    ms = dev.time_launches(betas, False, True) / len(betas)
    print(os.environ.get("PM_LIB_PATH", "default").split("/")[-1], n, round(ms * 1e3, 2), "us", dev.geometry(), flush=True)
