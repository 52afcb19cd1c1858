"""Small driver for ncu captures of the batch-RNG kernels (bench config `rng` shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import rng  # noqa: E402

u = rng.DeviateBuffer(rng.BufferKind.UNIFORM01, seed=9, owner=(0,))
z = rng.DeviateBuffer(rng.BufferKind.STD_NORMAL, seed=9, owner=(1,))
for _ in range(2):
    d = rng.gamma_batch(rng.GammaParams(2.0, 3.0), 10_000_000, u, z)
n = z.take_device(1 << 24)
print("ok", float(d.mean()), float(n.std()))
