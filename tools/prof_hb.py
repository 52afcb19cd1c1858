"""Small driver for ncu captures of the HB kernel (config 3 shape)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200.hb import CsrGroups  # noqa: E402
from paper_1310_1537_b200.synthetic import hb_design  # noqa: E402

x, y, off, betas, mu, tau = hb_design(1000, 20, seed=3)
dev = CsrGroups(x, y, off).on_device(0)
for _ in range(4):
    f, g = dev.eval(betas, mu, np.full(20, tau))
print("ok", float(f.sum()))
