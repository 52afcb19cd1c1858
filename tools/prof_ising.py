"""Small driver for ncu captures of the packed Gibbs kernel (config 4 shape by default)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import ising  # noqa: E402
from paper_1310_1537_b200.rng import SitePhilox  # noqa: E402
from paper_1310_1537_b200.synthetic import ising_spins, potts_states  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--size", type=int, default=8192)
p.add_argument("--potts", action="store_true")
p.add_argument("--sweeps", type=int, default=3)
a = p.parse_args()
n = a.size
if a.potts:
    lat = ising.PottsLattice(potts_states(n, n, seed=0), 0.4407)
else:
    lat = ising.IsingLattice(ising_spins(n, n, seed=0), np.zeros((n, n)), 0.8814, boundary="periodic")
part = ising.color_lattice(lat)
ising.gibbs_sweeps(lat, part, SitePhilox(1), a.sweeps)
print("fast path", part.device.fast_path(), "mean", float(lat.s.mean()))
