"""Reduced parity subset for compute-sanitizer (memcheck / racecheck / synccheck, one tool
per gpurun call): every kernel family with a hand-rolled protocol runs at a small size --
the TMA/mbarrier stream kernel in all consumer layouts (fp64 columns / pairs, fp32 columns /
pairs / whole tile), the row-per-lane kernel, the wide kernel, the HB rows kernel with the
separate and the fused (per-group ticket) fold, the packed and generic Gibbs half-sweeps,
lattice strips with the in-kernel halo exchange (flags, acquire waits), the peer-exchange
evaluation (split phases), the multi-delta diff / commit kernels and the cooperative chain
kernel.  Each result is checked against the oracle so a silent corruption also fails.

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_subset.py
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import gibbs_oracle as go  # noqa: E402
from oracle import glm_oracle as gl  # noqa: E402
from paper_1310_1537_b200 import _lib, glm, hb, ising  # noqa: E402
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan  # noqa: E402
from paper_1310_1537_b200.rng import SitePhilox  # noqa: E402
from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior, run_chain  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design, ising_spins, potts_states  # noqa: E402


def close(a, b, tol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) < tol


def glm_cases():
    gen = np.random.default_rng(1)
    for k, n, xs, knobs in [(100, 4099, "f64", {}), (100, 4099, "f64", {"f64_pairs": 0}),
                            (100, 4099, "f32", {}), (100, 4099, "f32", {"f32_pairs": 0}),
                            (100, 4099, "f32", {"f32_pairs": 1}), (100, 4099, "f32", {"f32_pairs": 4}),
                            (100, 4099, "f32", {"f32_selfprod": 0}),
                            (64, 2049, "f32", {"f32_pairs": 2}), (20, 70_001, "f64", {"glm_rows": 1}),
                            (300, 1500, "f64", {}), (32, 100_000, "f64", {})]:
        with _lib.tuned(**knobs):
            x, y, _, beta = baseline_design(n, k, seed=k + n)
            d = DesignMatrix(x, y)
            prior = GaussianPrior.isotropic(k, 0.0, 10.0)
            r = glm.log_posterior_grad(d, beta, prior, ExecPlan(x_storage=xs))
            xr = x.astype(np.float32).astype(np.float64) if xs == "f32" else x
            f, g = gl.log_posterior_grad(xr, y, beta, prior.mu, prior.sigma)
            assert close(r.f, f, 1e-10) and close(r.g, g, 1e-10), (k, n, xs, knobs)
            d.release_device()
    print("glm ok", flush=True)


def hb_cases():
    from paper_1310_1537_b200.synthetic import hb_design
    for knobs in ({}, {"hb_fused": 0}, {"hb_rows": 0}, {"hb_mapped_out": 0}, {"hb_selfprod": 0, "hb_rows_ncw": 7},
                  {"hb_rows_ncw": 15}, {"hb_mapped_in": 1}):
        with _lib.tuned(**knobs):
            x, y, off, betas, mu, tau = hb_design(40, 20, seed=3, mean_rows=300)
            dev = hb.CsrGroups(x, y, off).on_device(0)
            f, g = dev.eval(betas, mu, np.full(20, tau))
            fr, gr = gl.hb_log_posterior_grad(x, y, off, betas, mu, np.full(20, tau))
            assert close(f, fr, 1e-10) and close(g, gr, 1e-10), knobs
            dev.close()
    print("hb ok", flush=True)


def gibbs_cases():
    s0 = ising_spins(64, 128, seed=2)
    lat = ising.IsingLattice(s0, np.zeros(s0.shape), 0.8814, boundary="periodic")
    part = ising.color_lattice(lat)
    ising.gibbs_sweeps(lat, part, SitePhilox(5), 3)
    assert np.array_equal(lat.s, go.ising_sweeps(s0, None, 0.8814, True, 3, go.RNG_PHILOX4X32, 5, 0, 0))
    p0 = potts_states(64, 128, seed=2)
    plat = ising.PottsLattice(p0, 0.7)
    ising.potts_sweeps(plat, ising.color_lattice(plat), SitePhilox(5), 3)
    assert np.array_equal(plat.s, go.potts_sweeps(p0, 0.7, True, 3, go.RNG_PHILOX4X32, 5, 0, 0))
    f0 = ising_spins(13, 10, seed=4)
    b = np.random.default_rng(0).normal(0, 0.5, f0.shape)
    flat = ising.IsingLattice(f0, b, 0.6)
    ising.gibbs_sweeps(flat, ising.color_lattice(flat), SitePhilox(7), 2)
    assert np.array_equal(flat.s, go.ising_sweeps(f0, b, 0.6, False, 2, go.RNG_PHILOX4X32, 7, 0, 0))
    print("gibbs ok", flush=True)


def strip_cases():
    import torch
    from paper_1310_1537_b200.dist import LatticeStrip, strip_bounds
    H, W = 48, 64
    full = ising_spins(H, W, seed=8)
    strips = []
    for k in range(3):
        a, b = strip_bounds(H, 3, k)
        s = LatticeStrip(H, W, a, b - a, 0, model="ising", w=0.8814)
        s.set_spins(full[a:b])
        strips.append(s)
    boxes = [s.xchg_mailbox() for s in strips]
    for k, s in enumerate(strips):
        s.xchg_set_peers(up=boxes[(k - 1) % 3], down=boxes[(k + 1) % 3])
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for s in strips:
            s.xchg_start()
        for t in range(4):
            for c in (0, 1):
                for s in strips:
                    s.half_sweep(c, 11, t)
    torch.cuda.synchronize()
    got = np.concatenate([s.get_spins() for s in strips], axis=0)
    assert np.array_equal(got, go.ising_sweeps(full, None, 0.8814, True, 4, go.RNG_PHILOX4X32, 11, 0, 0))
    assert not any(s.xchg_timed_out() for s in strips)
    for s in strips:
        s.close()
    print("strips ok", flush=True)


def xchg_cases():
    import torch
    from paper_1310_1537_b200.parallel import partition
    x, y, _, beta = baseline_design(9001, 100, seed=9)
    devs = [DesignMatrix(x[a:b], y[a:b]).on_device(0) for a, b in partition(9001, 2)]
    hs = []
    for r in range(2):
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pm_xchg_create(0, 2, r, 101, ctypes.byref(h)))
        hs.append(h)
    boxes = []
    for h in hs:
        p = ctypes.c_void_p()
        _lib.call("pm_xchg_mailbox", h, ctypes.byref(p))
        boxes.append(p.value)
    for r in range(2):
        _lib.call("pm_xchg_set_peer_ptr", hs[r], 1 - r, ctypes.c_void_p(boxes[1 - r]))
    out = [torch.empty(101, dtype=torch.float64, device="cuda") for _ in range(2)]
    st = torch.cuda.Stream()
    for phase in (1, 2):
        for r in range(2):
            _lib.call("pm_glm_eval_xchg_phase", devs[r].handle, _lib.dptr(beta), 0, hs[r], phase,
                      ctypes.c_void_p(out[r].data_ptr() if phase == 2 else None), ctypes.c_void_p(st.cuda_stream))
    torch.cuda.synchronize()
    f, g = gl.loglike_grad(x, y, beta)
    got = out[0].cpu().numpy()
    assert close(got[0], f, 1e-10) and close(got[1:], g, 1e-10)
    for h in hs:
        _lib.load().pm_xchg_destroy(h)
    print("xchg ok", flush=True)


def chain_cases():
    from oracle import sampler_oracle as so
    x, y, _, _ = baseline_design(3000, 6, seed=3)
    d = DesignMatrix(x, y)
    prior = GaussianPrior.isotropic(6, 0.0, 10.0)
    out = run_chain(d, prior, ChainConfig(n_iter=4, n_burnin=0, seed=9))
    ref, evals = so.run_chain(x, y, prior.mu, prior.sigma, 4, 0, seed=9)
    assert np.max(np.abs(out.draws - ref)) <= 1e-6 and out.accept_evals == evals
    ws = glm.GlmWorkspace(d, np.zeros(6))
    v = glm.diff_loglike_multi(ws, d, 2, [0.1, -0.2, 0.3])
    glm.commit_update(ws, 2, 0.1)
    ws.validate(d)
    assert np.all(np.isfinite(v))
    print("chain/diff ok", flush=True)


if __name__ == "__main__":
    _lib.require_device(0)
    glm_cases()
    hb_cases()
    gibbs_cases()
    strip_cases()
    xchg_cases()
    chain_cases()
    print("sanitize subset done")
