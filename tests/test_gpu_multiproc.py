"""The cross-process exchange paths that bench.py takes at N > 1, run as 2 and 3 separate
PROCESSES on cuda:0 (tests/_mp_rank.py): real CUDA IPC handles exported with
pm_xchg_ipc_handle / pm_lat_strip_xchg_ipc_handle, all-gathered over gloo and opened with
pm_xchg_open_peer / pm_lat_strip_xchg_set_peers; the P2P deposits, system-scope release
flags and acquire waits inside the evaluation / half-sweep kernels.

Launch order is host-sequenced so that no kernel waits on a still-running kernel (ranks
sharing one GPU are time-sliced; see tests/_mp_rank.py).  Bar: 50 GLM evaluations and 20
strip sweeps (Ising and Potts) bit-identical to the single-process path -- the rank-ordered
fold of the shards' partials (pm_fold_rows, the NCCL path) and the C oracle's sweeps --
on every rank, and no exchange wait timed out.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import gibbs_oracle as go
from oracle import glm_oracle as gl

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import _mp_rank as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_exchange_across_processes(gpu, tmp_path, world):
    import ctypes

    import torch
    from paper_1310_1537_b200 import _lib
    from paper_1310_1537_b200.glm import DesignMatrix
    from paper_1310_1537_b200.parallel import partition
    from paper_1310_1537_b200.sampler import GaussianPrior
    from paper_1310_1537_b200.synthetic import baseline_design, ising_spins, potts_states

    port = _free_port()
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.dirname(HERE), os.environ.get("PYTHONPATH", "")]))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_mp_rank.py"), str(r), str(world), str(port),
                               str(tmp_path)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    try:
        for p in procs:
            out, _ = p.communicate(timeout=600)
            logs.append(out.decode(errors="replace")[-3000:])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert all(p.returncode == 0 for p in procs), "\n----\n".join(logs)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]

    # the single-process path: every shard's partial (rank 0 with the prior), ascending fold
    x, y, _, _ = baseline_design(mp.N_ROWS, mp.K, seed=5)
    prior = GaussianPrior.isotropic(mp.K, 0.0, 10.0)
    shards = [DesignMatrix(x[a:b], y[a:b]).on_device(0) for a, b in partition(mp.N_ROWS, world)]
    shards[0].set_prior(prior.mu, prior.sigma)
    part = torch.empty((world, mp.K + 1), dtype=torch.float64, device="cuda:0")
    fold = torch.empty(mp.K + 1, dtype=torch.float64, device="cuda:0")
    betas = mp.glm_betas()
    for i, beta in enumerate(betas):
        for r, d in enumerate(shards):
            d.eval_device(beta, True, part[r].data_ptr(), 0, with_prior=(r == 0))
        torch.cuda.synchronize()
        _lib.call("pm_fold_rows", ctypes.c_void_p(part.data_ptr()), world, mp.K + 1,
                  ctypes.c_void_p(fold.data_ptr()), None)
        torch.cuda.synchronize()
        ref = fold.cpu().numpy()
        for r in range(world):
            np.testing.assert_array_equal(ranks[r]["glm"][i], ref, err_msg=f"eval {i} rank {r}")
        if i % 17 == 0:
            f, g = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma)
            assert abs(ref[0] - f) / max(abs(f), 1) < 1e-10
            assert np.max(np.abs(ref[1:] - g) / np.maximum(np.abs(g), 1)) < 1e-10
    assert all(int(z["glm_timed_out"]) == 0 for z in ranks)

    for model in ("ising", "potts"):
        full = ising_spins(mp.H, mp.W, seed=8) if model == "ising" else potts_states(mp.H, mp.W, seed=8)
        got = np.concatenate([z[f"strip_{model}"] for z in ranks], axis=0)
        if model == "ising":
            ref = go.ising_sweeps(full, None, 0.8814, True, mp.SWEEPS, go.RNG_PHILOX4X32, mp.SEED, 0, 0)
        else:
            ref = go.potts_sweeps(full, 1.0986, True, mp.SWEEPS, go.RNG_PHILOX4X32, mp.SEED, 0, 0)
        np.testing.assert_array_equal(got, ref)
        assert all(int(z[f"strip_{model}_timed_out"]) == 0 for z in ranks)
