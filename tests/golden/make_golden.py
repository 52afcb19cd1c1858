"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the development container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by calling the reference package `parmcmc`
(/root/reference/pkg/src/parmcmc) through its public API; the committed .npz
files pin both the CPU oracle (tests/test_oracle.py) and the device path
(tests/test_gpu_*.py).  The only non-API step is `periodic_ising`, which feeds
the reference's unmodified gibbs_sweep (ising.py:175-187) a ColorPartition whose
neighbour table is rebuilt with wrap-around indices, and the
site-Philox uniforms, which come from a duck-typed buffer (only `.take(n)` is
used by gibbs_sweep, ising.py:185).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import parmcmc  # noqa: E402  (reference)
from parmcmc import glm as rglm  # noqa: E402
from parmcmc import hb as rhb  # noqa: E402
from parmcmc import ising as ris  # noqa: E402
from parmcmc import rng as rrng  # noqa: E402
from parmcmc import sampler as rsmp  # noqa: E402

from oracle import gibbs_oracle  # noqa: E402  (site-Philox uniforms for the periodic case)

assert "reference" in os.path.abspath(parmcmc.__file__), parmcmc.__file__


def random_instance(n, k, seed):
    """test_glm.py:20-25."""
    gen = np.random.default_rng(seed)
    x = gen.standard_normal((n, k)) * gen.uniform(0.5, 2.0)
    y = (gen.random(n) < 0.5).astype(float)
    beta = gen.normal(0.0, 1.0, k)
    return x, y, beta


def baseline_design(n, k, seed, intercept=True):
    """SURVEY §8(d) generator (one gen, fixed draw order)."""
    gen = np.random.default_rng(seed)
    x = np.empty((n, k))
    if intercept:
        x[:, 0] = 1.0
        x[:, 1:] = gen.standard_normal((n, k - 1))
    else:
        x[:, :] = gen.standard_normal((n, k))
    beta_true = gen.normal(0.0, 0.5, k)
    from scipy.special import expit
    y = (gen.random(n) < expit(x @ beta_true)).astype(np.float64)
    beta_eval = gen.normal(0.0, 0.1, k)
    return x, y, beta_eval


def glm_fixture():
    cases = [(16, 3, 11), (23, 5, 7), (1, 1, 0), (37, 4, 1), (501, 7, 42), (1000, 6, 9),
             (1499, 23, 3000), (257, 32, 5), (300, 33, 6), (200, 64, 7), (150, 100, 8),
             (96, 129, 9), (64, 256, 10), (40, 300, 12), (33, 700, 13)]
    out = {}
    for i, (n, k, seed) in enumerate(cases):
        x, y, beta = random_instance(n, k, seed)
        data = rglm.DesignMatrix(x, y)
        res = rglm.loglike_grad(data, beta, rglm.ExecPlan(rglm.Strategy.PLF, workers=1))
        f_only = rglm.loglike(data, beta)
        prior = rsmp.GaussianPrior(np.linspace(-0.5, 0.5, k), np.linspace(0.5, 3.0, k))
        lp = res.f + sum(prior.logpdf_coord(j, beta[j]) for j in range(k))
        out[f"x{i}"], out[f"y{i}"], out[f"beta{i}"] = x, y, beta
        out[f"f{i}"], out[f"g{i}"], out[f"fl{i}"] = res.f, res.g, f_only
        out[f"mu{i}"], out[f"sigma{i}"], out[f"lp{i}"] = prior.mu, prior.sigma, lp
    # BASELINE config 0 shape (intercept column), scaled rows; prior N(0, 10^2)
    x, y, beta = baseline_design(1500, 32, 2024)
    data = rglm.DesignMatrix(x, y)
    res = rglm.loglike_grad(data, beta)
    prior = rsmp.GaussianPrior.isotropic(32, 0.0, 10.0)
    lp = res.f + sum(prior.logpdf_coord(j, beta[j]) for j in range(32))
    out.update(c0_x=x, c0_y=y, c0_beta=beta, c0_f=res.f, c0_g=res.g, c0_lp=lp)
    out["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "glm.npz"), **out)


def diff_fixture():
    x, y, beta = random_instance(300, 6, 4)
    data = rglm.DesignMatrix(x, y)
    ws = rglm.GlmWorkspace(data, beta)
    gen = np.random.default_rng(12)
    ops = []
    vals = []
    for _ in range(60):
        k = int(gen.integers(6))
        d = float(gen.normal(0, 0.5))
        if gen.random() < 0.5:
            vals.append(rglm.diff_loglike(ws, data, k, d))
            ops.append((0, k, d))
        else:
            rglm.commit_update(ws, k, d)
            vals.append(np.nan)
            ops.append((1, k, d))
    np.savez_compressed(os.path.join(HERE, "diff.npz"), x=x, y=y, beta=beta, ops=np.array(ops),
                        vals=np.array(vals), xbeta=ws.xbeta, beta_final=ws.beta_current)


def rng_fixture():
    out = {}
    for seed in (0, 5, 33):
        buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, capacity=64, seed=seed)
        out[f"u{seed}"] = buf.take(1000)
        bg = np.random.Philox(np.random.SeedSequence(seed))
        out[f"key{seed}"] = np.array(bg.state["state"]["key"], dtype=np.uint64)
    buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, capacity=16, seed=17, owner=(3,))
    out["u17_3"] = buf.take(100)
    out["key17_3"] = np.array(np.random.Philox(np.random.SeedSequence(17, spawn_key=(3,))).state["state"]["key"],
                              dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def random_lattice(h, w, coupling=0.8, seed=0):
    """test_ising.py:17-21."""
    gen = np.random.default_rng(seed)
    s = gen.choice([-1, 1], size=(h, w)).astype(np.int8)
    b = gen.normal(0.0, 0.7, size=(h, w))
    return ris.IsingLattice(s, b, coupling)


def ising_fixture():
    out = {}
    cases = [((4, 5), 0.9, 0, 100, 3), ((6, 6), 0.8, 8, 21, 25), ((5, 7), 0.8, 2, 4, 10), ((1, 5), 0.5, 3, 6, 7),
             ((3, 1), 0.7, 4, 9, 5), ((8, 9), 0.8, 3, 5, 10), ((1, 1), 0.5, 1, 0, 4), ((16, 12), 0.44, 7, 77, 30),
             ((33, 17), 1.1, 9, 90, 12)]
    for i, (shape, cpl, lseed, bseed, sweeps) in enumerate(cases):
        lat = random_lattice(*shape, coupling=cpl, seed=lseed)
        out[f"s0_{i}"], out[f"b_{i}"] = lat.s.copy(), lat.b.copy()
        part = ris.color_lattice(lat)
        buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, seed=bseed)
        for _ in range(sweeps):
            ris.gibbs_sweep(lat, part, buf)
        out[f"s1_{i}"] = lat.s.copy()
        out[f"meta_{i}"] = np.array([shape[0], shape[1], sweeps, bseed], dtype=np.int64)
        out[f"w_{i}"] = cpl
    # image-bias lattice (two bias classes), from_image path (ising.py:73-82)
    img = ris.flip_noise(ris.synthetic_binary_image(20, 24), 0.15, seed=2)
    lat = ris.IsingLattice.from_image(img, 1.0, 1.5)
    out["img_s0"], out["img_b"] = lat.s.copy(), lat.b.copy()
    part = ris.color_lattice(lat)
    buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, seed=9)
    for _ in range(60):
        ris.gibbs_sweep(lat, part, buf)
    out["img_s1"] = lat.s.copy()
    # partition accessors and the stationary log weight (ising.py:84-93, 134-150)
    out["img_nsum0"], out["img_nsum1"] = part.neighbor_spin_sum(0), part.neighbor_spin_sum(1)
    out["img_packed0"], out["img_packed1"] = part.packed_s[0].copy(), part.packed_s[1].copy()
    out["img_logw"] = np.float64(lat.log_weight())
    out["logw_cases"] = np.array([ris.IsingLattice(out[f"s1_{i}"], out[f"b_{i}"], float(out[f"w_{i}"])).log_weight()
                                  for i in range(len(cases))])
    out["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "ising.npz"), **out)


class _SiteUniforms:
    """Duck-typed rng_buffer: take(n_c) returns the sweep's site-Philox uniforms."""

    def __init__(self, seed, n0, n1, sweep0=0):
        self.seed, self.n0, self.n1, self.sweep, self.colour = seed, n0, n1, sweep0, 0
        self._cur = None

    def take(self, n):
        if self.colour == 0:
            self._cur = gibbs_oracle.site_uniforms(self.seed, self.sweep, self.n0 + self.n1)
            out = self._cur[: self.n0]
            assert n == self.n0
        else:
            out = self._cur[self.n0:]
            assert n == self.n1
            self.sweep += 1
        self.colour ^= 1
        return out


def periodic_partition(lat):
    """A reference ColorPartition whose neighbour table wraps around."""
    part = ris.color_lattice(lat)
    h, w = lat.height, lat.width
    ii, jj = np.indices((h, w))
    pos = np.empty(h * w, dtype=np.int64)
    for c in (0, 1):
        pos[part.colors[c]] = np.arange(part.colors[c].size)
    for c in (0, 1):
        cols = []
        for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            nf = (((ii + di) % h) * w + (jj + dj) % w).ravel()[part.colors[c]]
            cols.append(pos[nf])
        part.packed_nbr[c] = np.ascontiguousarray(np.stack(cols, axis=1))
    return part


def periodic_fixture():
    out = {}
    cases = [((4, 4), 0.8814, 0.0, 1, 3, 40), ((6, 8), 0.6, 0.3, 2, 99, 15), ((8, 32), 0.8814, 0.0, 3, 7, 10),
             ((16, 64), 0.5, -0.2, 4, 12345678901, 6)]
    for i, (shape, w, b, lseed, seed, sweeps) in enumerate(cases):
        gen = np.random.default_rng(lseed)
        s = gen.choice([-1, 1], size=shape).astype(np.int8)
        lat = ris.IsingLattice(s, np.full(shape, b), w)
        out[f"s0_{i}"] = s.copy()
        part = periodic_partition(lat)
        hw = shape[0] * shape[1]
        buf = _SiteUniforms(seed, (hw + 1) // 2, hw // 2)
        for _ in range(sweeps):
            ris.gibbs_sweep(lat, part, buf)
        out[f"s1_{i}"] = lat.s.copy()
        out[f"meta_{i}"] = np.array([shape[0], shape[1], sweeps, seed], dtype=np.uint64)
        out[f"wb_{i}"] = np.array([w, b])
    out["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "periodic.npz"), **out)


def sampler_fixture():
    data, _ = rglm.synthetic_logistic(120, 4, seed=0)
    prior = rsmp.GaussianPrior.isotropic(4, sigma=5.0)
    cfg = rsmp.ChainConfig(n_iter=30, n_burnin=5, seed=77)
    a = rsmp.run_chain(data, prior, cfg)
    data2, _ = rglm.synthetic_logistic(400, 5, seed=8)
    cfg2 = rsmp.ChainConfig(n_iter=40, n_burnin=0, seed=31)
    b = rsmp.run_chain(data2, prior if False else rsmp.GaussianPrior.isotropic(5, sigma=5.0), cfg2)
    np.savez_compressed(os.path.join(HERE, "sampler.npz"), x=data.x, y=data.y, draws=a.draws,
                        evals=a.accept_evals, x2=data2.x, y2=data2.y, draws2=b.draws, evals2=b.accept_evals)


def hb_fixture():
    ds, betas_true = rhb.synthetic_hb_dataset(5, 3, 60, seed=3)
    prior = rsmp.GaussianPrior(np.array([0.2, -0.1, 0.3]), np.array([0.3, 0.3, 0.3]))
    gen = np.random.default_rng(1)
    betas = prior.mu + prior.sigma * gen.standard_normal((5, 3))
    f = np.empty(5)
    g = np.empty((5, 3))
    for m, grp in enumerate(ds.groups):
        r = rglm.loglike_grad(grp, betas[m])
        f[m] = r.f + sum(prior.logpdf_coord(k, betas[m, k]) for k in range(3))
        g[m] = r.g - (betas[m] - prior.mu) / prior.sigma ** 2
    x = np.concatenate([grp.x for grp in ds.groups])
    y = np.concatenate([grp.y for grp in ds.groups])
    off = np.concatenate([[0], np.cumsum([grp.n_rows for grp in ds.groups])]).astype(np.int64)
    np.savez_compressed(os.path.join(HERE, "hb.npz"), x=x, y=y, offsets=off, betas=betas, mu=prior.mu,
                        sigma=prior.sigma, f=f, g=g)


def denoise_fixture():
    """Reference denoiser (ising.py:257-290), its per-sweep trace, the differential
    sweep's flip counter and cached sums (ising.py:190-254), and PBM bytes."""
    import tempfile
    out = {}
    cases = [((64, 64), "two_region", 0.1, 3, 1.0, 2.0, 30, 10, 4), ((32, 32), "two_region", 0.1, 5, 1.0, 2.0, 20, 5, 6),
             ((48, 48), "all_ones", 0.1, 7, 1.0, 2.0, 25, 8, 8), ((24, 24), "two_region", 0.0, 0, 1.0, 8.0, 12, 4, 1),
             ((16, 16), "two_region", 0.2, 9, 1.0, 2.0, 0, 0, 1), ((16, 16), "two_region", 0.2, 9, 1.0, 2.0, 5, 5, 2),
             ((37, 23), "two_region", 0.25, 11, 0.7, 1.5, 9, 3, 12345), ((1, 9), "two_region", 0.3, 1, 1.0, 1.0, 7, 2, 3)]
    for i, (shape, kind, rate, nseed, w, bscale, sweeps, burnin, seed) in enumerate(cases):
        noisy = ris.flip_noise(ris.synthetic_binary_image(*shape, kind=kind), rate, seed=nseed)
        trace = []
        restored = ris.denoise(noisy, w=w, bias_scale=bscale, sweeps=sweeps, burnin=burnin, seed=seed,
                               trace_out=trace)
        restored_diff = ris.denoise(noisy, w=w, bias_scale=bscale, sweeps=sweeps, burnin=burnin, seed=seed,
                                    use_diff=True)
        assert (restored == restored_diff).all()
        buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, seed=seed)
        out[f"noisy_{i}"], out[f"out_{i}"] = noisy, restored
        out[f"trace_{i}"] = np.array(trace, dtype=np.float64)
        out[f"par_{i}"] = np.array([w, bscale, sweeps, burnin, seed], dtype=np.float64)
        out[f"key_{i}"] = np.array(buf._gen.bit_generator.state["state"]["key"], dtype=np.uint64)
    # differential sweeps: flips_last_sweep and the cached sums after each sweep
    img = ris.flip_noise(ris.synthetic_binary_image(20, 24), 0.15, seed=2)
    lat = ris.IsingLattice.from_image(img, 1.0, 1.5)
    part = ris.color_lattice(lat)
    zc = ris.ZCache(lat, part)
    buf = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, seed=9)
    flips, nsums = [], []
    for _ in range(12):
        ris.gibbs_sweep_diff(lat, part, zc, buf)
        flips.append(zc.flips_last_sweep)
        nsums.append(np.concatenate([zc.nsum(0), zc.nsum(1)]))
    out["diff_img"], out["diff_s1"] = img, lat.s.copy()
    out["diff_flips"], out["diff_nsum"] = np.array(flips, dtype=np.int64), np.stack(nsums)
    out["diff_z"] = zc.z_grid(lat, part)
    # PBM bytes written by the reference (P1 and P4, with a ragged P4 row)
    with tempfile.TemporaryDirectory() as d:
        for fmt in ("P1", "P4"):
            pimg = ris.flip_noise(ris.synthetic_binary_image(7, 13), 0.4, seed=11)
            path = os.path.join(d, f"x.{fmt}")
            ris.write_pbm(path, pimg, fmt=fmt)
            with open(path, "rb") as fh:
                out[f"pbm_{fmt}"] = np.frombuffer(fh.read(), dtype=np.uint8)
            out["pbm_img"] = pimg
    out["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "denoise.npz"), **out)


GAMMA_CASES = [(2.0, 3.0, 9, 3000), (1.0, 1.0, 4, 2000), (0.3, 2.0, 5, 1500), (5.5, 0.7, 6, 1000),
               (1.0000001, 1.0, 7, 500), (50.0, 2.0, 1, 500), (0.999, 1.0, 2, 400)]
DIRICHLET_CASES = [([2.0, 3.0, 5.0], 11, 500), ([1.0] * 100, 12, 40), ([0.1, 0.5, 1.0, 2.0], 13, 300), ([1.0], 14, 20),
                   ([0.05] * 5, 15, 200), ([3.0] * 7, 16, 150), ([1.5] * 130, 17, 10)]


def rng_batch_fixture():
    """Reference normal streams, Gamma and Dirichlet draws with their stream consumption
    (rng.py:59-215), on owner streams (0,) uniform / (1,) normal as _bench_sources."""
    out = {}
    for tag, cap, seed, owner, n in (("n8", 4096, 8, (), 4099), ("n10", 3, 10, (1,), 1001)):
        out[f"normal_{tag}"] = rrng.DeviateBuffer(rrng.BufferKind.STD_NORMAL, cap, seed, owner=owner).take(n)
    for i, (alpha, rate, seed, n) in enumerate(GAMMA_CASES):
        u = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, 8192, seed, owner=(0,))
        z = rrng.DeviateBuffer(rrng.BufferKind.STD_NORMAL, 8192, seed, owner=(1,))
        out[f"gamma_{i}"] = np.array([rrng.gamma_sample(rrng.GammaParams(alpha, rate), u, z) for _ in range(n)])
        out[f"gamma_used_{i}"] = np.array([u.consumed, z.consumed], dtype=np.int64)
    for i, (alphas, seed, n) in enumerate(DIRICHLET_CASES):
        u = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, 8192, seed, owner=(0,))
        z = rrng.DeviateBuffer(rrng.BufferKind.STD_NORMAL, 8192, seed, owner=(1,))
        out[f"dir_{i}"] = np.array([rrng.dirichlet_sample(alphas, u, z) for _ in range(n)])
        out[f"dir_used_{i}"] = np.array([u.consumed, z.consumed], dtype=np.int64)
    # independent owner streams (2s,) uniform / (2s+1,) normal
    draws, used = [], []
    for s in range(8):
        u = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, 8192, 21, owner=(2 * s,))
        z = rrng.DeviateBuffer(rrng.BufferKind.STD_NORMAL, 8192, 21, owner=(2 * s + 1,))
        draws.append([rrng.gamma_sample(rrng.GammaParams(0.7, 1.5), u, z) for _ in range(50)])
        used.append([u.consumed, z.consumed])
    out["gstreams"], out["gstreams_used"] = np.array(draws), np.array(used, dtype=np.int64)
    draws, used = [], []
    for s in range(5):
        u = rrng.DeviateBuffer(rrng.BufferKind.UNIFORM01, 8192, 22, owner=(2 * s,))
        z = rrng.DeviateBuffer(rrng.BufferKind.STD_NORMAL, 8192, 22, owner=(2 * s + 1,))
        draws.append([rrng.dirichlet_sample([0.5, 1.0, 2.0], u, z) for _ in range(20)])
        used.append([u.consumed, z.consumed])
    out["dstreams"], out["dstreams_used"] = np.array(draws), np.array(used, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "rng_batch.npz"), **out)


def hb_sweep_fixture():
    """Reference hierarchical Gibbs sweeps (HbState + hb_sweep, hb.py:110-168)."""
    out = {}
    # case 0: the reference generator, isotropic prior, 3 sweeps
    ds, _ = rhb.synthetic_hb_dataset(6, 3, 80, seed=4)
    prior = rsmp.GaussianPrior.isotropic(3)
    # case 1: ragged groups (1..150 rows), non-zero prior mean, neval 3, small buffers
    groups = [rglm.synthetic_logistic(n, 3, seed=40 + i, beta=np.array([0.5, -1.0, 0.25]))[0]
              for i, n in enumerate([1, 7, 33, 64, 150])]
    ds1 = rhb.HbDataset(groups)
    prior1 = rsmp.GaussianPrior(np.array([0.2, -0.1, 0.3]), np.array([0.5, 0.5, 0.5]))
    for c, (d, pr, seed, cap, neval, sweeps) in enumerate([(ds, prior, 5, 8192, 1, 3), (ds1, prior1, 6, 7, 3, 4)]):
        st = rhb.HbState(d, pr, seed=seed, buffer_capacity=cap)
        pol = rhb.MappingPolicy(rhb.MappingMode.COARSE, workers=1, neval=neval)
        traj = []
        for _ in range(sweeps):
            traj.append(np.array(rhb.hb_sweep(d, st, pr, pol)))
        out[f"betas_{c}"] = np.stack(traj)
        out[f"evals_{c}"] = np.int64(st.total_evals)
        out[f"used_{c}"] = np.array([b.consumed for b in st.buffers], dtype=np.int64)
        out[f"x_{c}"] = np.concatenate([g.x for g in d.groups])
        out[f"y_{c}"] = np.concatenate([g.y for g in d.groups])
        out[f"off_{c}"] = np.concatenate([[0], np.cumsum([g.n_rows for g in d.groups])]).astype(np.int64)
        out[f"prior_{c}"] = np.stack([pr.mu, pr.sigma])
        out[f"meta_{c}"] = np.array([seed, cap, neval, sweeps], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "hb_sweep.npz"), **out)


if __name__ == "__main__":
    glm_fixture()
    diff_fixture()
    rng_fixture()
    ising_fixture()
    periodic_fixture()
    sampler_fixture()
    hb_fixture()
    denoise_fixture()
    rng_batch_fixture()
    hb_sweep_fixture()
    for fn in sorted(os.listdir(HERE)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(HERE, fn)))
