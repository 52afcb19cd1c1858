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


# ---------------------------------------------------------------------------
# lattice strips: the halo-exchange schedule of paper_1310_1537_b200.dist, driven by a CPU
# emulation of the strip half-sweep (same global row / colour / RNG-site indexing as the
# device kernel), must reproduce the full-lattice oracle bit for bit for any strip count.
# ---------------------------------------------------------------------------

class _CpuStrip:
    def __init__(self, full, w, row0, rows):
        import math
        self.H, self.W = full.shape
        self.W2 = self.W // 2
        self.row0, self.rows, self.w = row0, rows, w
        self.math = math
        self.pk = [torch.zeros((rows + 2, self.W2), dtype=torch.uint8) for _ in range(2)]
        for r in range(rows):
            i = row0 + r
            for j in range(self.W):
                self.pk[(i + j) & 1][r + 1, j // 2] = int(full[i, j]) & 0xFF

    def row(self, colour, array_row):
        return self.pk[colour][array_row]

    def half_sweep(self, c, seed, sweep):
        from oracle import gibbs_oracle as go
        lib = go.load()
        other = self.pk[1 - c].numpy().view(np.int8)
        mine = self.pk[c].numpy()
        n0 = self.H * self.W2
        for r in range(1, self.rows + 1):
            i = self.row0 + r - 1
            o = (i + c) & 1
            for q in range(self.W2):
                nsum = int(other[r - 1, q]) + int(other[r + 1, q]) + int(other[r, (q - 1 + o) % self.W2]) + \
                    int(other[r, (q + o) % self.W2])
                wn = self.w * float(nsum)
                p = 1.0 / (1.0 + self.math.exp(-(0.0 + wn)))
                u = lib.oracle_site_uniform(c * n0 + i * self.W2 + q, sweep, seed)
                mine[r, q] = 0x01 if u < p else 0xFF

    def own(self):
        out = np.empty((self.rows, self.W), dtype=np.int8)
        for r in range(self.rows):
            i = self.row0 + r
            for j in range(self.W):
                out[r, j] = np.int8(np.uint8(self.pk[(i + j) & 1][r + 1, j // 2]))
        return out


def _strip_worker(rank, world, port, q, shape, sweeps, seed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_1537_b200.dist import strip_bounds, strip_sweeps
        from paper_1310_1537_b200.synthetic import ising_spins
        full = ising_spins(*shape, seed=4)
        a, b = strip_bounds(shape[0], world, rank)
        strip = _CpuStrip(full, 0.8814, a, b - a)
        strip_sweeps(strip, sweeps, seed, 0, rank, world)
        q.put((rank, a, strip.own()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_strip_halo_exchange_matches_full_lattice(world):
    from oracle import gibbs_oracle as go
    from paper_1310_1537_b200.synthetic import ising_spins
    shape, sweeps, seed = (12, 8), 3, 77
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strip_worker, args=(r, world, port, q, shape, sweeps, seed)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([r[2] for r in res], axis=0)
    ref = go.ising_sweeps(ising_spins(*shape, seed=4), None, 0.8814, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
    np.testing.assert_array_equal(got, ref)


def _xchg_worker(rank, world, port, q, fail_rank):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_1537_b200 import dist as pdist

        class FakeLib:
            """Stands in for libpmb200's pm_xchg_* on CPU: handles are 64 bytes naming the
            rank; rank `fail_rank` fails to map its peers."""

            def __init__(self):
                self.opened, self.destroyed = [], 0

            def load(self):
                return self

            def check(self, rc, what=""):
                if rc:
                    raise RuntimeError(what)

            def pm_xchg_create(self, device, world_, rank_, width, out):
                out._obj.value = 1000 + rank_
                return 0

            def pm_xchg_destroy(self, h):
                self.destroyed += 1
                return 0

            def call(self, name, *args):
                if name == "pm_xchg_ipc_handle":
                    import ctypes
                    ctypes.memmove(args[1], f"rank{rank}".encode().ljust(64, b"\0"), 64)
                elif name == "pm_xchg_open_peer":
                    import ctypes
                    if rank == fail_rank:
                        raise RuntimeError("cudaIpcOpenMemHandle: peer access unsupported")
                    self.opened.append((args[1], ctypes.string_at(args[2], 5)))

        fake = FakeLib()
        pdist._lib_override = fake
        x = pdist.PeerExchange(0, 5)
        q.put((rank, x.ok, sorted(fake.opened), fake.destroyed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_peer_exchange_setup_agrees_across_ranks(fail_rank):
    """PeerExchange's collective setup (gloo, world 3, libpmb200 stood in for on CPU): every
    rank opens every other rank's handle; if any rank cannot map a peer, ALL ranks report
    ok = False and release their mailbox (so every rank falls back to the NCCL path)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, opened, destroyed in res:
        assert ok == (fail_rank < 0)
        if rank != fail_rank:
            assert opened == [(p, f"rank{p}".encode()) for p in range(world) if p != rank]
        assert destroyed == (0 if ok else 1)


def _halo_worker(rank, world, port, q, fail_rank):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_1537_b200.dist import start_peer_halos

        class FakeStrip:
            """The strip's pm_lat_strip_xchg_* calls stood in for on CPU."""

            def __init__(self):
                self.peers, self.started = None, False

            def xchg_ipc_handle(self):
                return f"mb{rank}".encode().ljust(64, b"\0")

            def xchg_mailbox(self):
                return 4096 + rank

            def xchg_set_peers(self, up=None, down=None, up_ipc=None, down_ipc=None):
                if rank == fail_rank:
                    raise RuntimeError("cudaIpcOpenMemHandle failed")
                self.peers = (up, down, up_ipc[:3] if up_ipc else None, down_ipc[:3] if down_ipc else None)

            def xchg_start(self):
                self.started = True

        s = FakeStrip()
        ok = start_peer_halos(s, rank, world)
        q.put((rank, ok, s.started, s.peers))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,fail_rank", [(3, -1), (3, 2), (1, -1)])
def test_peer_halo_setup_neighbours_and_agreement(world, fail_rank):
    """start_peer_halos (gloo, CPU stand-in strips): rank r maps rank r-1 as the strip above
    and r+1 below (periodic; world 1 maps itself by pointer); a failure on any rank leaves
    every rank on the NCCL path (nobody starts the peer exchange)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, started, peers in res:
        assert ok == (fail_rank < 0) and started == ok
        if ok and world == 1:
            assert peers == (4096, 4096, None, None)
        elif ok:
            assert peers == (None, None, f"mb{(rank - 1) % world}".encode(), f"mb{(rank + 1) % world}".encode())
