"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: the row split follows the
reference's partition rule and the rank-ordered fold of the (K+1) partials equals the
reference's ascending-worker merge bit for bit (glm.py:243-250).  The per-rank partial
is produced by the oracle here (no GPU); on the box it is the fused kernel's output."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import glm_oracle as gl
        from paper_1310_1537_b200.dist import gather_partials, shard_bounds
        z = golden("glm.npz")
        x, y, beta = z["c0_x"], z["c0_y"], z["c0_beta"]
        a, b = shard_bounds(x.shape[0], world, rank)
        f, g = gl.block_fg(x[a:b], y[a:b], beta)
        part = torch.from_numpy(np.concatenate([[f], g]))
        tot = gather_partials(part).numpy()
        q.put((rank, a, b, tot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_ordered_fold_equals_reference_merge(world):
    from oracle import glm_oracle as gl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z = golden("glm.npz")
    f_ref, g_ref = gl.loglike_grad(z["c0_x"], z["c0_y"], z["c0_beta"], workers=world)
    bounds = [(a, b) for _, a, b, _ in res]
    assert bounds == gl.partition(z["c0_x"].shape[0], world)
    for _, _, _, tot in res:
        assert tot[0] == f_ref and np.array_equal(tot[1:], g_ref)  # identical on every rank
    assert abs(res[0][3][0] - float(z["c0_f"])) / abs(float(z["c0_f"])) < 1e-13
