"""Small driver for ncu captures of the HB sweep kernel (config-3 shape, 1 sweep)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200.glm import DesignMatrix  # noqa: E402
from paper_1310_1537_b200.hb import HbDataset, HbState  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior  # noqa: E402
from paper_1310_1537_b200.synthetic import hb_design  # noqa: E402

x, y, off, _, mu, tau = hb_design(1000, 20, seed=3)
ds = HbDataset([DesignMatrix(x[off[g]:off[g + 1]], y[off[g]:off[g + 1]]) for g in range(1000)])
prior = GaussianPrior(mu, np.full(20, tau))
st = HbState(ds, prior, seed=5)
for _ in range(2):
    st.sweeps(prior, 1)
print("ok", st.last_kernel_ms, st.total_evals)
