"""Config-4 end-to-end breakdown: wall time of pack_from (H2D + validate + pack), n sweeps
(enqueue + device) and unpack_into (unpack + D2H) for the Ising and Potts lattices, pinned
and pageable spins.

python tools/c4_e2e_breakdown.py [--size 8192] [--sweeps 1000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import ising  # noqa: E402
from paper_1310_1537_b200.rng import SitePhilox  # noqa: E402
from paper_1310_1537_b200.synthetic import ising_spins, potts_states  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--size", type=int, default=8192)
p.add_argument("--sweeps", type=int, default=1000)
a = p.parse_args()
import torch  # noqa: E402

n = a.size
for model in ("ising", "potts"):
    for pinned in (True, False):
        if model == "ising":
            lat = ising.IsingLattice(ising_spins(n, n, seed=0), np.zeros((n, n)), 0.8814, boundary="periodic")
        else:
            lat = ising.PottsLattice(potts_states(n, n, seed=0), 0.4407, boundary="periodic")
        if pinned:
            ising.pin_lattice(lat)
        part = ising.color_lattice(lat)
        dev = part.device
        rng = SitePhilox(seed=2024)
        dev.sweeps(10, 2, rng.seed, 0, 0)
        torch.cuda.synchronize()
        res = {"model": model, "pinned": pinned}
        for rep in range(2):
            t0 = time.perf_counter()
            part.pack_from(lat)
            t1 = time.perf_counter()
            dev.sweeps(a.sweeps, 2, rng.seed, 0, 10)
            t2 = time.perf_counter()
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            part.unpack_into(lat)
            t4 = time.perf_counter()
            res[f"rep{rep}"] = {"pack_ms": round((t1 - t0) * 1e3, 2), "sweeps_call_ms": round((t2 - t1) * 1e3, 2),
                                "sync_ms": round((t3 - t2) * 1e3, 2), "unpack_ms": round((t4 - t3) * 1e3, 2),
                                "total_ms": round((t4 - t0) * 1e3, 2)}
        res["device_ms"] = round(dev.time_sweeps(a.sweeps, 2, rng.seed, 0, 10), 2)
        print(json.dumps(res), flush=True)
        dev.close()
