"""Row sharding across ranks (one process per GPU, torch.distributed over NCCL).

The reference splits rows across worker threads and per-shard private copies
(parallel.py:30-46, glm.py:143-158, 439-454) and merges the (f, g) partials in
ascending worker order (glm.py:243-250).  Here each rank holds the rows
`partition(N, world)[rank]` on its own GPU; one evaluation is

    rank-local fused kernel -> (K+1) doubles on the device
    -> NCCL all-gather of the partials (one exchange step)
    -> sum in ascending rank order (bitwise identical on every rank)
    -> + prior terms (sampler.py:55-58), once.

`ordered_sum` and `gather_partials` are the collective logic; they are exercised
with the gloo backend on CPU tensors in tests/test_dist_gloo.py.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .glm import DesignMatrix, GradResult, _check_beta
from .parallel import partition

__all__ = ["shard_bounds", "ordered_sum", "gather_partials", "PeerExchange", "DistributedDesign",
           "strip_bounds", "exchange_halos", "LatticeStrip", "start_peer_halos", "strip_sweeps"]


def shard_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Rows owned by `rank` (parallel.py:30-46: the first n % world ranks get one extra)."""
    return partition(n_rows, world)[rank]


def ordered_sum(gathered):
    """Sum the rows of a (world, K+1) tensor in ascending rank order (fixed association)."""
    acc = gathered[0].clone()
    for r in range(1, gathered.shape[0]):
        acc += gathered[r]
    return acc


def torch_stream_handle(device) -> int:
    """cudaStream_t of torch's current stream on `device` for the C ABI.  torch reports the
    legacy default stream as 0, which the ABI reads as "the handle's own stream"; pass
    cudaStreamLegacy (0x1) instead so the launch really lands on torch's stream."""
    import torch
    return torch.cuda.current_stream(device).cuda_stream or 1


def gather_partials(part, group=None):
    """All-gather every rank's (K+1) partial and fold them in rank order.

    NCCL: one all_gather_into_tensor + one fold launch (pm_fold_rows) on the current
    stream; gloo (CPU tensors, the tests): the same ascending-rank fold in torch.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(part.shape), dtype=part.dtype, device=part.device)
        dist.all_gather_into_tensor(out, part.contiguous(), group=group)
        from . import _lib
        tot = torch.empty_like(part)
        _lib.call("pm_fold_rows", ctypes.c_void_p(out.data_ptr()), world, part.numel(),
                  ctypes.c_void_p(tot.data_ptr()), ctypes.c_void_p(torch_stream_handle(part.device)))
        return tot
    parts = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(parts, part.contiguous(), group=group)
    return ordered_sum(torch.stack(parts))


class PeerExchange:
    """Mailboxes of the peer-memory exchange (pm_xchg_*): every rank's (K+1) partial goes
    straight into all ranks' device memory from the finishing CTA of its own evaluation
    kernel (P2P stores over NVLink/NVSwitch, CUDA IPC mappings), so one evaluation is ONE
    launch with no NCCL call and no fold launch.  Built collectively; `ok` is False on every
    rank if any rank could not map a peer (then the NCCL path is used)."""

    def __init__(self, device: int, width: int, group=None):
        import torch.distributed as dist

        from . import _lib
        _lib = _lib_override or _lib  # tests stand in for the library on CPU
        self._lib = _lib
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._h = None
        err = ""
        try:
            h = ctypes.c_void_p()
            _lib.check(_lib.load().pm_xchg_create(device, self.world, self.rank, width, ctypes.byref(h)),
                       "pm_xchg_create")
            self._h = h
            buf = ctypes.create_string_buffer(64)
            _lib.call("pm_xchg_ipc_handle", h, ctypes.cast(buf, ctypes.c_void_p))
            mine = bytes(buf.raw)
        except Exception as e:  # noqa: BLE001 - any failure means: use NCCL on every rank
            mine, err = b"", str(e)
        handles = [None] * self.world
        dist.all_gather_object(handles, (mine, _hostname()), group=group)
        ok = all(hd[0] for hd in handles) and len({hd[1] for hd in handles}) == 1
        if ok:
            try:
                for p, (hd, _) in enumerate(handles):
                    if p != self.rank:
                        _lib.call("pm_xchg_open_peer", self._h, p, ctypes.cast(ctypes.c_char_p(hd), ctypes.c_void_p))
            except Exception as e:  # noqa: BLE001
                ok, err = False, str(e)
        flags = [None] * self.world
        dist.all_gather_object(flags, ok, group=group)
        self.ok = all(flags)
        self.error = err
        if not self.ok:
            self.close()

    def eval(self, dev, beta, with_prior: bool, out_ptr: int, stream: int) -> None:
        self._lib.call("pm_glm_eval_xchg", dev.handle, self._lib.dptr(beta), int(with_prior), self._h,
                       ctypes.c_void_p(out_ptr), ctypes.c_void_p(stream))

    def eval_phase(self, dev, beta, with_prior: bool, phase: int, out_ptr: int, stream: int) -> None:
        """Split form (pm_glm_eval_xchg_phase): 1 = deposit + flags, 2 = wait + fold.  With a
        barrier between every rank's phase 1 and any rank's phase 2, no kernel waits on a
        running kernel, so ranks sharing one GPU can use the real IPC exchange."""
        self._lib.call("pm_glm_eval_xchg_phase", dev.handle, self._lib.dptr(beta), int(with_prior), self._h,
                       int(phase), ctypes.c_void_p(out_ptr or None), ctypes.c_void_p(stream))

    def timed_out(self) -> bool:
        v = ctypes.c_int32()
        self._lib.call("pm_xchg_status", self._h, ctypes.byref(v))
        return bool(v.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.load().pm_xchg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_lib_override = None


def _hostname() -> str:
    import socket
    return socket.gethostname()


class DistributedDesign:
    """This rank's row shard on its GPU.  One evaluation is one kernel launch whose finishing
    CTA exchanges the (K+1) partials with the other ranks through peer memory and folds them
    in ascending rank order (PeerExchange, NCCL backend, world > 1); otherwise (gloo, world 1,
    exchange="nccl", or a node without peer mappings) one kernel, one NCCL all-gather and one
    fold launch.  Rank 0's kernel adds the prior terms (the same device finaliser as the
    single-GPU path), so the rank-ordered fold holds them exactly once.

    exchange: "auto" (peer exchange for NCCL groups of > 1 rank), "peer" (also for a
    1-rank group: exercises the exchange kernel on one GPU) or "nccl"."""

    def __init__(self, local: DesignMatrix, device: int, x_storage: str = "f64", group=None,
                 exchange: str = "auto"):
        import torch
        import torch.distributed as dist
        self.local = local
        self.device = device
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.dev = local.on_device(device, x_storage)
        self.k = local.n_cols
        self._buf = torch.empty(self.k + 1, dtype=torch.float64, device=f"cuda:{device}")
        self._out = torch.empty(self.k + 1, dtype=torch.float64, device=f"cuda:{device}")
        self.xchg = None
        if exchange not in ("auto", "peer", "nccl"):
            raise ValueError(f"exchange must be auto, peer or nccl, got {exchange!r}")
        want = exchange
        if (want in ("auto", "peer") and dist.is_initialized() and dist.get_backend(group) == "nccl"
                and (dist.get_world_size(group) > 1 or want == "peer")):
            x = PeerExchange(device, self.k + 1, group)
            self.xchg = x if x.ok else None

    @property
    def exchange(self) -> str:
        return "peer" if self.xchg is not None else "nccl"

    def _partial(self, beta: np.ndarray, prior=None):
        stream = torch_stream_handle(self.device)
        with_prior = prior is not None and self.rank == 0
        if with_prior:
            self.dev.set_prior(prior.mu, prior.sigma)
        self.dev.eval_device(beta, True, self._buf.data_ptr(), stream, with_prior=with_prior)
        return self._buf

    def log_posterior_grad_device(self, beta, prior=None):
        """(f, g) as a device tensor of K+1 doubles, identical on every rank."""
        beta = _check_beta(beta, self.k)
        if self.xchg is not None:
            with_prior = prior is not None and self.rank == 0
            if with_prior:
                self.dev.set_prior(prior.mu, prior.sigma)
            self.xchg.eval(self.dev, beta, with_prior, self._out.data_ptr(), torch_stream_handle(self.device))
            return self._out
        return gather_partials(self._partial(beta, prior), self.group)

    def log_posterior_grad(self, beta, prior=None) -> GradResult:
        out = self.log_posterior_grad_device(beta, prior).cpu().numpy()
        # a timed-out exchange writes NaN (the status read is a device round trip: only then)
        if self.xchg is not None and np.isnan(out[0]) and self.xchg.timed_out():
            raise RuntimeError("peer exchange timed out: a rank did not take part in the evaluation")
        return GradResult(float(out[0]), out[1:].copy())


# ---------------------------------------------------------------------------
# lattice strips with halo-row exchange
# ---------------------------------------------------------------------------

def strip_bounds(height: int, world: int, rank: int) -> tuple[int, int]:
    """Global rows owned by `rank` (same partition rule as the rows of X)."""
    return partition(height, world)[rank]


def exchange_halos(first_row, last_row, top_halo, bottom_halo, rank: int, world: int, group=None) -> None:
    """Refresh the halo rows of one colour after that colour was updated.

    The row above a strip belongs to rank (rank-1) % world (its last own row), the row
    below to rank (rank+1) % world (its first own row); the lattice is periodic.  Every
    rank issues its operations in the same canonical order (send up, send down, receive
    from below, receive from above) so FIFO-matched transports (NCCL) and tag-matched
    ones (gloo) pair them identically, including world == 2 where up == down.
    """
    if world == 1:
        top_halo.copy_(last_row)
        bottom_halo.copy_(first_row)
        return
    import torch.distributed as dist
    up, down = (rank - 1) % world, (rank + 1) % world
    gu = dist.get_global_rank(group, up) if group is not None else up
    gd = dist.get_global_rank(group, down) if group is not None else down
    ops = [dist.P2POp(dist.isend, first_row, gu, group, tag=0),
           dist.P2POp(dist.isend, last_row, gd, group, tag=1),
           dist.P2POp(dist.irecv, bottom_halo, gd, group, tag=0),
           dist.P2POp(dist.irecv, top_halo, gu, group, tag=1)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class _DevBuf:
    """__cuda_array_interface__ view of raw device bytes (torch.as_tensor consumes it)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class LatticeStrip:
    """This rank's strip of a periodic H x W lattice on its GPU (pm_lat_create_strip)."""

    def __init__(self, height: int, width: int, row0: int, rows: int, device: int,
                 model: str = "ising", w: float = 0.0, coupling: float = 0.0):
        import ctypes

        from . import _lib
        self._lib = _lib
        _lib.require_device(device)
        h = ctypes.c_void_p()
        m = _lib.PM_MODEL_ISING if model == "ising" else _lib.PM_MODEL_POTTS4
        _lib.check(_lib.load().pm_lat_create_strip(device, height, width, row0, rows, m, ctypes.byref(h)),
                   "pm_lat_create_strip")
        self._h = h
        self.height, self.width, self.row0, self.rows, self.device = height, width, row0, rows, device
        if model == "ising":
            _lib.call("pm_lat_set_ising", h, float(w), None)
        else:
            _lib.call("pm_lat_set_potts", h, float(coupling))
        self._views = {}
        self.peer_exchange = False  # True after xchg_start: half-sweeps exchange halos themselves

    def set_spins(self, own_rows: np.ndarray) -> None:
        s = np.ascontiguousarray(own_rows, dtype=np.int8)
        assert s.shape == (self.rows, self.width)
        self._lib.call("pm_lat_set_spins", self._h, self._lib.i8ptr(s))

    def get_spins(self) -> np.ndarray:
        import torch
        torch.cuda.synchronize(self.device)  # half-sweeps and exchanges run on torch's stream
        out = np.empty((self.rows, self.width), dtype=np.int8)
        self._lib.call("pm_lat_get_spins", self._h, self._lib.i8ptr(out))
        return out

    def row(self, colour: int, array_row: int):
        """torch uint8 tensor aliasing packed row `array_row` of `colour` (0/rows+1 = halos)."""
        import ctypes

        import torch
        key = (colour, array_row)
        t = self._views.get(key)
        if t is None:
            p = ctypes.c_void_p()
            self._lib.call("pm_lat_strip_row", self._h, int(colour), int(array_row), ctypes.byref(p))
            t = torch.as_tensor(_DevBuf(p.value, self.width // 2), device=f"cuda:{self.device}")
            self._views[key] = t
        return t

    # ---- peer-memory halo exchange (pm_lat_strip_xchg_*) ----
    def xchg_mailbox(self) -> int:
        import ctypes
        p = ctypes.c_void_p()
        self._lib.call("pm_lat_strip_xchg_create", self._h, ctypes.byref(p))
        return p.value

    def xchg_ipc_handle(self) -> bytes:
        import ctypes
        self.xchg_mailbox()
        buf = ctypes.create_string_buffer(64)
        self._lib.call("pm_lat_strip_xchg_ipc_handle", self._h, ctypes.cast(buf, ctypes.c_void_p))
        return bytes(buf.raw)

    def xchg_set_peers(self, up=None, down=None, up_ipc: bytes = None, down_ipc: bytes = None) -> None:
        """Neighbour mailboxes: same-process device pointers (up/down) or IPC handles."""
        import ctypes

        def h(b):
            return None if b is None else ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p)
        self._lib.call("pm_lat_strip_xchg_set_peers", self._h, ctypes.c_void_p(up), h(up_ipc),
                       ctypes.c_void_p(down), h(down_ipc))

    def xchg_start(self) -> None:
        import ctypes
        self._lib.call("pm_lat_strip_xchg_start", self._h, ctypes.c_void_p(torch_stream_handle(self.device)))
        self.peer_exchange = True

    def xchg_timed_out(self) -> bool:
        import ctypes
        v = ctypes.c_int32()
        self._lib.call("pm_lat_strip_xchg_status", self._h, ctypes.byref(v))
        return bool(v.value)

    def half_sweep(self, colour: int, seed: int, sweep: int) -> None:
        import ctypes

        stream = torch_stream_handle(self.device)
        self._lib.call("pm_lat_strip_half_sweep", self._h, int(colour), ctypes.c_uint64(seed),
                       ctypes.c_uint64(sweep), ctypes.c_void_p(stream))

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._views.clear()
            self._lib.load().pm_lat_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def start_peer_halos(strip, rank: int, world: int, group=None) -> bool:
    """Set up the peer-memory halo exchange for a strip (collective over the group): mailbox
    IPC handles all-gathered, neighbours (rank-1, rank+1, periodic) mapped; every rank agrees
    on the outcome, so on failure all ranks keep the NCCL path.  Call after set_spins."""
    import torch.distributed as dist
    ok, err, mine = True, "", b""
    try:
        mine = strip.xchg_ipc_handle()
    except Exception as e:  # noqa: BLE001
        ok, err = False, str(e)
    handles = [None] * world
    dist.all_gather_object(handles, (mine, ok), group=group)
    ok = all(o for _, o in handles)
    if ok:
        up, down = (rank - 1) % world, (rank + 1) % world
        try:
            if world == 1:
                mb = strip.xchg_mailbox()
                strip.xchg_set_peers(up=mb, down=mb)
            else:
                strip.xchg_set_peers(up_ipc=handles[up][0], down_ipc=handles[down][0])
        except Exception as e:  # noqa: BLE001
            ok, err = False, str(e)
    flags = [None] * world
    dist.all_gather_object(flags, ok, group=group)
    if not all(flags):
        return False
    strip.xchg_start()
    return True


def strip_sweeps(strip, n_sweeps: int, seed: int, sweep0: int, rank: int, world: int, group=None) -> None:
    """n_sweeps full sweeps of a strip-decomposed lattice: per colour, the device half-sweep
    then one halo exchange of that colour (bit-identical to the single-GPU sweep).  After
    start_peer_halos the half-sweep kernels exchange the halo rows themselves (P2P stores +
    flags), so this is just the sequence of half-sweep launches."""
    if getattr(strip, "peer_exchange", False):
        for t in range(n_sweeps):
            for c in (0, 1):
                strip.half_sweep(c, seed, sweep0 + t)
        return
    r = strip.rows
    for c in (0, 1):  # halos of both colours must be current before the first half-sweep
        exchange_halos(strip.row(c, 1), strip.row(c, r), strip.row(c, 0), strip.row(c, r + 1), rank, world, group)
    for t in range(n_sweeps):
        for c in (0, 1):
            strip.half_sweep(c, seed, sweep0 + t)
            exchange_halos(strip.row(c, 1), strip.row(c, r), strip.row(c, 0), strip.row(c, r + 1), rank, world,
                           group)
