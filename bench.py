#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric: log-posterior+gradient evals/s
and achieved HBM GB/s, logistic GLM, fp64).

Default workload = BASELINE config 1 (N=1e7, K=100 fp64, fresh beta ~ N(0, 0.1^2) per
step, prior N(0, 10^2)), the largest configuration that fits one GPU (8.08 GB of X).
One step = one log-posterior + gradient evaluation over all N rows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c1|c1f32|c0|c2|c3|c3sweep|c4|c4potts|rng] [--force-dist]

N>1 runs one process per GPU under torch.distributed.run (NCCL): rows are split by
the reference's partition rule, each rank streams its shard and the (K+1)-double
partials are all-gathered and summed in rank order (--force-dist runs that rank path
as a 1-rank group on one GPU).  c4 at N>1 splits the lattice into row strips with halo
exchange; the other configs are replicas.

`--impl reference` times the UNMODIFIED reference on this host's cores: `parmcmc` 0.1.0
installed from the reference tree into baseline/_ref by __graft_entry__.build()
(pip --target, git-ignored, travels to the GPU box like libpmb200.so), called through its
own public API -- glm.loglike_grad(DesignMatrix, beta, ExecPlan(PLF, workers)) plus the
GaussianPrior terms -- on the FULL config (every step evaluates all N rows; no sample
scaling).  Both BASELINE.md §3 thread settings run, each in a fresh subprocess:
(i) PLF workers=1 with OPENBLAS_NUM_THREADS=C, (ii) PLF workers=C with OpenBLAS 1; the
faster is the line's value.  Without baseline/_ref the numpy restatement in
oracle/glm_oracle.py stands in (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))


def _early_args():
    p = argparse.ArgumentParser(add_help=False)
    p.add_argument("--impl", default="b200")
    p.add_argument("--cpu-worker", action="store_true")
    p.add_argument("--ref-worker", action="store_true")
    p.add_argument("--setting", default="ii")
    a, _ = p.parse_known_args()
    return a


def _affinity_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_EA = _early_args()
if _EA.cpu_worker or (_EA.ref_worker and _EA.setting == "ii"):
    # BASELINE.md §3 setting (ii): workers = cores, one BLAS thread each (set before numpy loads)
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
elif _EA.ref_worker:
    # setting (i): one PLF worker, OpenBLAS over all cores
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = str(_affinity_cores())

import numpy as np  # noqa: E402

sys.path.insert(0, ROOT)

CONFIGS = {
    "c0": dict(n=100_000, k=32, x_storage="f64", desc="config 0: N=1e5 K=32 fp64 log-posterior+gradient"),
    "c1": dict(n=10_000_000, k=100, x_storage="f64", desc="config 1: N=1e7 K=100 fp64 log-posterior+gradient"),
    "c1f32": dict(n=10_000_000, k=100, x_storage="f32",
                  desc="config 1 fp32-X/fp64-accumulate: N=1e7 K=100 log-posterior+gradient"),
    "c2": dict(chain_n=1_000_000, k=50, desc="config 2: slice-within-Gibbs chain, N=1e6 K=50 fp64 (iterations)"),
    "c3": dict(groups=1000, k=20, mean_rows=2000, desc="config 3: G=1000 n_g~Poisson(2000) K=20 HB batched"),
    "c4": dict(h=8192, w=8192, model="ising", desc="config 4: 8192^2 periodic Ising, Philox4x32 (seed,sweep,site)"),
    "c4potts": dict(h=8192, w=8192, model="potts", desc="config 4 Potts q=4 variant, 8192^2 periodic"),
    "c3sweep": dict(sweep_groups=1000, k=20, mean_rows=2000,
                    desc="config 3 shape, hierarchical Gibbs sweep: G=1000 groups x K=20 slice updates per sweep"),
    "rng": dict(draws=10_000_000, desc="batch RNG: 10M Gamma(2,3) draws per step on one stream pair (rng.py:246-300)"),
}

METRIC = "log-posterior+gradient evals/s and achieved HBM GB/s (logistic GLM, fp64)"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def load_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(key: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            v = json.load(fh).get(key)
        return None if v is None else float(v)
    except Exception:
        return None


class L2Scrub:
    """Evicts the inputs from L2 between timed launches: a 512 MiB write (larger than the
    126 MB L2), then a 256 MiB read of a second buffer so the timed launch does not pay
    for writing the scrub's dirty lines back to HBM (cold inputs, clean L2)."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.dirty = torch.empty(512 << 20, dtype=torch.uint8, device=device)
        self.clean = torch.ones(256 << 20, dtype=torch.uint8, device=device)

    def __call__(self):
        self.dirty.zero_()
        self.clean.max()
        self.torch.cuda.synchronize(self.dirty.device)


def issue_roofline(config: str, ms_per_sweep: float, clk: dict):
    """The Gibbs sweep's real bound: warp instructions issued per second (ncu count of one
    Ising / Potts half-sweep launch, profiles/traffic.json) against 148 SMs x 4 schedulers x the
    median SM clock sampled during the timed region."""
    n = load_traffic(f"{config}_warp_inst_per_half_sweep") if config in ("c4", "c4potts") else None
    if not n or not clk or not clk.get("sm_mhz"):
        return None
    achieved = 2 * n / (ms_per_sweep * 1e-3)
    peak = 148 * 4 * clk["sm_mhz"] * 1e6
    return {"achieved": achieved, "peak": peak, "unit": "warp instructions/s", "frac": achieved / peak,
            "source": "ncu smsp__inst_executed.sum per half-sweep (%s)"
            % ("profiles/r02_ncu_ising_raw.csv" if config == "c4" else "profiles/r01_ncu_gibbs_potts_raw.csv")}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        if os.environ.get("PM_BENCH_NO_CLOCKS"):
            return
        # In-process NVML polling (100 ms): a concurrent `nvidia-smi -lms` loop measurably
        # slows long cooperative kernels (config 2: 135 vs 180 iterations/s on B200).
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._stop = threading.Event()
            self._samples: list[tuple[float, int]] = []
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            time.sleep(0.12)
            return
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _poll(self):
        nv = self._nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self._samples.append((float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)),
                                      int(get_reasons(self._h))))
            except Exception:
                pass
            self._stop.wait(0.1)

    def stop(self) -> dict:
        if getattr(self, "_nvml", None) is not None:
            time.sleep(0.1)
            self._stop.set()
            self._t.join(timeout=2)
            bits = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                    "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
            reasons = sorted({n for _, r in self._samples for n, b in bits.items() if r & b})
            sms = [s for s, _ in self._samples]
            return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": self._max, "reasons": reasons,
                    "samples": len(sms), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------- distributed
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------- CPU baseline
def cpu_worker_other(args):
    """CPU oracle timings for configs 2-4 (bounded samples; see the `sample` strings)."""
    cores = host_cores()
    cfg = CONFIGS[args.config]
    if "chain_n" in cfg:
        from oracle import sampler_oracle as so
        from paper_1310_1537_b200.synthetic import baseline_design
        x, y, _, _ = baseline_design(cfg["chain_n"], cfg["k"], seed=2)
        t0 = time.perf_counter()
        _, evals = so.run_chain(x, y, np.zeros(cfg["k"]), np.full(cfg["k"], 10.0), 1, 0, seed=5, workers=cores)
        dt = time.perf_counter() - t0
        res = {"value": 1.0 / dt, "unit": "iterations/s", "cores": cores, "kind": "port",
               "sample": f"oracle/sampler_oracle.py run_chain, 1 iteration (K={cfg['k']} coordinate updates, "
                         f"{evals} evaluations) at N={cfg['chain_n']}, numpy diff_loglike over {cores} workers"}
    elif "groups" in cfg:
        from oracle import glm_oracle as gl
        from paper_1310_1537_b200.synthetic import hb_design
        x, y, off, betas, mu, tau = hb_design(cfg["groups"], cfg["k"], seed=3, mean_rows=cfg["mean_rows"])
        gl.hb_log_posterior_grad(x, y, off, betas, mu, np.full(cfg["k"], tau))
        t0 = time.perf_counter()
        for _ in range(3):
            gl.hb_log_posterior_grad(x, y, off, betas, mu, np.full(cfg["k"], tau))
        dt = (time.perf_counter() - t0) / 3
        res = {"value": 1.0 / dt, "unit": "launches/s", "cores": 1, "kind": "port",
               "sample": "oracle/glm_oracle.py hb_log_posterior_grad (per-group numpy loop, the reference's "
                         "hb.py:127-135 composition), full config-3 data, mean of 3 after 1 warm-up"}
    else:
        from oracle import gibbs_oracle as go
        from paper_1310_1537_b200.synthetic import ising_spins, potts_states
        h, w = cfg["h"], cfg["w"]
        t0 = time.perf_counter()
        if cfg["model"] == "ising":
            go.ising_sweeps(ising_spins(h, w, seed=0), None, 2 * 0.4407, True, 1, go.RNG_PHILOX4X32, 2024, 0, 0)
        else:
            go.potts_sweeps(potts_states(h, w, seed=0), 0.4407, True, 1, go.RNG_PHILOX4X32, 2024, 0, 0)
        dt = time.perf_counter() - t0
        res = {"value": 1.0 / dt, "unit": "sweeps/s", "cores": 1, "kind": "port",
               "sample": f"oracle/gibbs_oracle.c (scalar C restatement of ising.py:175-187 + Philox4x32), "
                         f"1 sweep at {h}x{w}, 1 core"}
    print(json.dumps(res))


def cpu_baseline_other(config: str) -> dict:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--cpu-worker", "--config", config]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, check=True).stdout
        return json.loads(out.strip().splitlines()[-1])
    except Exception as exc:
        return {"value": None, "unit": None, "cores": host_cores(), "kind": "port", "sample": f"failed: {exc}"}


def cpu_worker_main(args):
    """Subprocess body for the non-GLM configs' CPU baselines (cpu_worker_other)."""
    return cpu_worker_other(args)


# ---------------------------------------------------------------------------- reference (CPU)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_installed() -> bool:
    """The unmodified reference package, pip-installed by __graft_entry__.build()."""
    return os.path.isfile(os.path.join(REF_DIR, "parmcmc", "glm.py"))


def save_glm_inputs(x, y, betas) -> str:
    """Park the inputs as .npy files (memory-mapped by the timing subprocesses, so the
    8 GB design is generated once): /dev/shm when it has room, else the temp dir."""
    import tempfile
    need = x.nbytes + y.nbytes + betas.nbytes + (1 << 28)
    base = None
    try:
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize > 2 * need:
            base = "/dev/shm"
    except OSError:
        pass
    d = tempfile.mkdtemp(prefix="pm_ref_", dir=base)
    np.save(os.path.join(d, "x.npy"), x)
    np.save(os.path.join(d, "y.npy"), y)
    np.save(os.path.join(d, "betas.npy"), betas)
    return d


def ref_worker_main(args):
    """Subprocess: time the CPU log-posterior + gradient on the full inputs in args.data.
    Unmodified reference (baseline/_ref): f = loglike_grad(...).f + sum_k prior.logpdf_coord,
    g = loglike_grad(...).g - (beta - mu) / sigma^2 (glm.py:351-364, sampler.py:55-58)."""
    cores = _affinity_cores()
    workers = 1 if args.setting == "i" else cores
    x = np.load(os.path.join(args.data, "x.npy"), mmap_mode="r")
    y = np.load(os.path.join(args.data, "y.npy"))
    betas = np.load(os.path.join(args.data, "betas.npy"))
    k = x.shape[1]
    mu, sigma = np.zeros(k), np.full(k, 10.0)
    if args.ref_kind == "reference":
        sys.path.insert(0, REF_DIR)
        from parmcmc import glm as rglm
        from parmcmc.sampler import GaussianPrior
        data = rglm.DesignMatrix(x, y)
        plan = rglm.ExecPlan(rglm.Strategy.PLF, workers=workers)
        prior = GaussianPrior(mu, sigma)

        def evaluate(beta):
            r = rglm.loglike_grad(data, beta, plan)
            f = r.f + sum(prior.logpdf_coord(j, float(beta[j])) for j in range(k))
            return f, r.g - (beta - prior.mu) / prior.sigma ** 2
        what = (f"unmodified parmcmc (baseline/_ref) glm.loglike_grad + GaussianPrior.logpdf_coord, "
                f"ExecPlan(PLF, workers={workers})")
    else:
        from oracle import glm_oracle as gl
        xa = np.ascontiguousarray(x)

        def evaluate(beta):
            return gl.log_posterior_grad(xa, y, beta, mu, sigma, workers=workers)
        what = f"oracle/glm_oracle.py log_posterior_grad (numpy restatement of PLF), {workers} workers"
    for i in range(args.warmup):
        evaluate(betas[i % len(betas)])
    times = []
    f = None
    for i in range(args.steps):
        t0 = time.perf_counter()
        f, _ = evaluate(betas[(args.warmup + i) % len(betas)])
        times.append(time.perf_counter() - t0)
    print(json.dumps({"times": times, "total_s": sum(times), "median_s": statistics.median(times),
                      "cores": cores, "workers": workers, "blas": os.environ.get("OPENBLAS_NUM_THREADS"),
                      "setting": args.setting, "kind": args.ref_kind, "what": what, "last_f": f}))


def run_ref_settings(data_dir: str, steps: int, warmup: int, settings=("ii", "i")) -> dict:
    """each thread setting in a fresh subprocess (the BLAS env var must be
    set before numpy loads); returns {"settings": {...}, "best": name, "kind": ...}."""
    kind = "reference" if reference_installed() else "port"
    out = {}
    for st in settings:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--ref-worker", "--setting", st, "--data", data_dir,
               "--steps", str(steps), "--warmup", str(warmup), "--ref-kind", kind]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, check=True)
            out[st] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:  # reported, never fatal
            tail = getattr(exc, "stderr", "") or ""
            out[st] = {"error": f"{exc} {tail[-300:]}"}
    ok = {k: v for k, v in out.items() if "total_s" in v}
    best = min(ok, key=lambda k: ok[k]["total_s"] / len(ok[k]["times"])) if ok else None
    return {"settings": out, "best": best, "kind": kind}


def _settings_summary(res: dict) -> str:
    parts = []
    for st, v in res["settings"].items():
        if "total_s" in v:
            rate = len(v["times"]) / v["total_s"]
            parts.append(f"({st}) workers={v['workers']} OPENBLAS_NUM_THREADS={v['blas']}: {rate:.3f} evals/s "
                         f"(median {v['median_s']*1e3:.0f} ms){' <- faster' if st == res['best'] else ''}")
        else:
            parts.append(f"({st}) failed: {v.get('error', '?')[:200]}")
    return "; ".join(parts)


def glm_inputs(cfg: dict, n_betas: int, seed: int = 7):
    from paper_1310_1537_b200.synthetic import baseline_design
    x, y, _, betas = baseline_design(cfg["n"], cfg["k"], seed=seed, n_eval=max(n_betas, 2))
    if cfg.get("x_storage") == "f32":  # fp32-X: the reference runs on the fp32-rounded X (as f64)
        x = x.astype(np.float32).astype(np.float64)
    return x, y, np.ascontiguousarray(betas)


def cpu_baseline(cfg: dict, x, y, betas) -> dict:
    """The GPU arm's cpu_baseline: the unmodified reference on the same full inputs, both
    thread settings, 2 warm-up + 3 timed evaluations each (~10-20 s of CPU work at c1)."""
    import shutil
    d = save_glm_inputs(x, y, betas)
    try:
        res = run_ref_settings(d, steps=3, warmup=2)
    finally:
        shutil.rmtree(d, ignore_errors=True)
    best = res["settings"].get(res["best"]) if res["best"] else None
    if best is None:
        return {"value": None, "unit": "evals/s", "cores": host_cores(), "kind": res["kind"],
                "sample": _settings_summary(res)}
    return {"value": len(best["times"]) / best["total_s"], "unit": "evals/s", "cores": best["cores"],
            "kind": res["kind"],
            "sample": (f"{best['what']}: full N={cfg['n']} rows x K={cfg['k']} per evaluation (no scaling), "
                       f"same X/y as the GPU arm, 3 timed evaluations after 2 warm-up per setting; "
                       + _settings_summary(res))}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import shutil
    cores = host_cores()
    n_full, k = cfg["n"], cfg["k"]
    x, y, betas = glm_inputs(cfg, args.warmup + args.steps)
    d = save_glm_inputs(x, y, betas)
    del x, y
    try:
        res = run_ref_settings(d, steps=args.steps, warmup=args.warmup)
    finally:
        shutil.rmtree(d, ignore_errors=True)
    if res["best"] is None:
        print(json.dumps({"impl": "reference", "unavailable": _settings_summary(res)[:400]}), flush=True)
        return
    best = res["settings"][res["best"]]
    ms_per_step = best["total_s"] / len(best["times"]) * 1e3
    value = 1000.0 / ms_per_step
    sample = (f"{best['what']}: every step evaluates the full N={n_full} x K={k} design (no sample scaling); "
              f"{args.warmup} warm-up + {args.steps} timed steps per setting, each setting in a fresh "
              f"subprocess; " + _settings_summary(res))
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8d generator, seed 7)",
        "config": {"workload": cfg["desc"], "N": n_full, "K": k, "x_storage": cfg.get("x_storage", "f64"),
                   "rows_per_step": n_full, "thread_setting": res["best"]},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": res["kind"], "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "median_ms_per_step": best["median_s"] * 1e3,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- B200 arm: GLM
def run_glm(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_1310_1537_b200 import glm as pglm
    from paper_1310_1537_b200.parallel import partition
    from paper_1310_1537_b200.sampler import GaussianPrior
    from paper_1310_1537_b200.synthetic import baseline_design_rows

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    # the rank path (DistributedDesign: NCCL all-gather + ordered fold) runs for N > 1, and at
    # N = 1 with --force-dist (a 1-rank NCCL group) so the multi-GPU code is exercised on one GPU
    dist_mode = ws > 1 or args.force_dist
    if dist_mode:
        if ws == 1:
            import socket
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if "MASTER_PORT" not in os.environ:
                with socket.socket() as s:
                    s.bind(("127.0.0.1", 0))
                    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_full, k = cfg["n"], cfg["k"]
    a, b = partition(n_full, ws)[rank]
    n_local = b - a
    steps, warmup = args.steps, args.warmup
    # ONE global design (seed 7, the reference arm's inputs): every rank draws the whole
    # generator stream chunk by chunk and keeps its own rows (bit-identical to slicing the
    # single-process design); rank 0 of a multi-rank run keeps all rows for the check below
    n_betas = warmup + 2 * steps
    if ws == 1 or rank == 0:
        x_all, y_all, betas = glm_inputs(cfg, n_betas)
        x, y = x_all[a:b], y_all[a:b]
    else:
        x, y, _, betas = baseline_design_rows(n_full, k, 7, a, b, n_eval=n_betas)
        x_all = y_all = None
        if cfg.get("x_storage") == "f32":
            x = x.astype(np.float32).astype(np.float64)
    data = pglm.DesignMatrix(x, y)
    del x
    prior = GaussianPrior.isotropic(k, 0.0, 10.0)
    plan = pglm.ExecPlan(pglm.Strategy.B200, device=local, x_storage=cfg["x_storage"])
    dev = data.on_device(local, cfg["x_storage"])
    geo = dev.geometry()

    dev.set_prior(prior.mu, prior.sigma)  # every rank: the kernel-only timing below adds it
    if dist_mode:
        from paper_1310_1537_b200.dist import DistributedDesign
        dd = DistributedDesign(data, device=local, x_storage=cfg["x_storage"], exchange=args.exchange)

        def step_dev(beta):
            return dd.log_posterior_grad_device(beta, prior)

        def step_e2e(beta):
            return dd.log_posterior_grad(beta, prior)
    else:
        def step_dev(beta):
            dev.launch(beta, True, True)
            dev.wait(True)

        def step_e2e(beta):
            return pglm.log_posterior_grad(data, beta, prior, plan)

    def barrier():
        if dist_mode:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(local)

    # warm-up (untimed)
    for i in range(warmup):
        step_dev(betas[i])
        step_e2e(betas[i])
    barrier()

    # ---- device-timed region: K steps, inputs resident, events on the launching stream
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    block = np.ascontiguousarray(betas[warmup:warmup + steps])
    xs_bytes = 8 if cfg["x_storage"] == "f64" else 4
    flush_l2 = n_local * (k * xs_bytes + 8) < 256e6   # inputs not larger than the 126 MB L2
    flush = L2Scrub(f"cuda:{local}") if flush_l2 else None   # evicts X and y from L2

    if not dist_mode and flush_l2:
        # each launch preceded by an L2 scrub on the same stream, CUDA events around the launch
        # only (pm_glm_time_cold): cold inputs, device time without the host's launch latency
        dev_ms = dev.time_cold(block, with_prior=True, want_grad=True)
    elif not dist_mode:
        # K launches bracketed by CUDA events on the launching (handle) stream
        dev_ms = dev.time_launches(block, with_prior=True, want_grad=True)
    else:
        # rank steps (kernel + all-gather + fold) on torch's stream, events on that stream
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tstream = torch.cuda.current_stream(local)
        if flush_l2:
            dev_ms = 0.0
            for i in range(steps):
                flush()
                dist.barrier(device_ids=[local])
                ev0.record(tstream)
                step_dev(block[i])
                ev1.record(tstream)
                torch.cuda.synchronize(local)
                dev_ms += ev0.elapsed_time(ev1)
        else:
            ev0.record(tstream)
            for i in range(steps):
                step_dev(block[i])
            ev1.record(tstream)
            torch.cuda.synchronize(local)
            dev_ms = ev0.elapsed_time(ev1)
    barrier()
    clk = clocks.stop()

    # ---- kernel-only timing of the dominant kernel (handle stream, back-to-back launches)
    kern_ms = dev_ms / steps if flush_l2 else dev.time_launches(block, with_prior=True, want_grad=True) / steps

    # ---- end-to-end through the public API (host beta in, host (f, g) out, every step)
    barrier()
    if flush_l2:
        e2e_s = 0.0
        for i in range(steps):
            flush()
            t0 = time.perf_counter()
            res = step_e2e(betas[warmup + steps + i])
            e2e_s += time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        for i in range(steps):
            res = step_e2e(betas[warmup + steps + i])
        e2e_s = time.perf_counter() - t0
    barrier()
    assert np.isfinite(res.f) and np.all(np.isfinite(res.g))

    # rank path: rank 0 checks the folded (f, g) against a 1-GPU evaluation of ALL rows of
    # the same global design (different CTA partition, so within 1e-10, not bitwise)
    check = None
    if dist_mode:
        probe = betas[0]
        got = step_e2e(probe)
        if rank == 0:
            full = pglm.DesignMatrix(x_all, y_all)
            ref = pglm.log_posterior_grad(full, probe, prior, pglm.ExecPlan(pglm.Strategy.B200, device=local,
                                                                              x_storage=cfg["x_storage"]))
            rf = abs(got.f - ref.f) / max(abs(ref.f), 1.0)
            rg = float(np.max(np.abs(got.g - ref.g) / np.maximum(np.abs(ref.g), 1.0)))
            check = {"beta": "first warm-up beta", "rel_f": rf, "rel_g": rg, "tol": 1e-10,
                     "ok": bool(rf < 1e-10 and rg < 1e-10)}
            full.release_device()
            del full
            assert check["ok"], check
        barrier()

    # max over ranks
    t = torch.tensor([dev_ms, e2e_s, kern_ms], dtype=torch.float64, device=f"cuda:{local}")
    if dist_mode:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_s, kern_ms = (float(v) for v in t.cpu())

    xs = 8 if cfg["x_storage"] == "f64" else 4
    bytes_eval_local = n_local * (k * xs + 8)          # N (K b_x + b_y)
    bytes_eval_total = n_full * (k * xs + 8)
    ms_per_step = dev_ms / steps
    value = 1000.0 / ms_per_step
    peak, peak_src = load_peaks()
    achieved = bytes_eval_local / (kern_ms * 1e-3) / 1e9
    e2e_value = steps / e2e_s
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws, "steps": steps, "warmup": warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if cfg["x_storage"] == "f64" else "f64 (X stored f32)",
            "data": "synthetic (SURVEY §8d generator: X[:,0]=1, X[:,1:]~N(0,1), y~Bern(sigmoid(X beta_true)))",
            "config": {"workload": cfg["desc"], "N": n_full, "K": k, "rows_per_gpu": n_local,
                       "x_storage": cfg["x_storage"], "parallelism": f"row-shard x{ws}",
                       "l2": (f"L2 scrubbed on the launching stream (512 MiB write + 256 MiB read of a clean buffer) before every timed evaluation, events around the evaluation alone; inputs "
                              f"{bytes_eval_local/1e6:.1f} MB < L2" if flush_l2 else
                              f"inputs larger than L2 ({bytes_eval_local/1e9:.2f} GB per GPU per eval)"),
                       "prior": "N(0, 10^2) iid", "beta": "fresh N(0, 0.1^2) per step"},
            "achieved_gbs": bytes_eval_total / (ms_per_step * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_of_8tbs_spec": achieved / 8000.0,
                         "traffic": load_traffic(f"{args.config}"),
                         "algorithmic_bytes_per_launch": bytes_eval_local,
                         "kernel_ms": kern_ms, "peak_source": peak_src,
                         "kernel": f"glm_stream_kernel ({geo['kernel']}, grid {geo['grid']} x {geo['threads']} "
                                   f"threads, {geo['stages']} TMA stages, {geo['smem_bytes']} B smem)"},
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": 8 * k,
                    "d2h_bytes_per_step": 8 * (k + 1),
                    "path": (("paper_1310_1537_b200.dist.DistributedDesign.log_posterior_grad (per rank: ONE "
                              "launch -- kernel, peer-memory exchange of the (K+1) partials, ordered fold -- "
                              "(f,g) to host)" if dd.exchange == "peer" else
                              "paper_1310_1537_b200.dist.DistributedDesign.log_posterior_grad (per rank: kernel, "
                              "NCCL all-gather of the (K+1) partials, ordered fold, (f,g) to host)") if dist_mode else
                             "paper_1310_1537_b200.glm.log_posterior_grad (C-ABI pm_glm_launch/wait; beta in "
                             "kernel params, (f,g) written to mapped pinned host memory)")},
            # + the fold launch per step on the NCCL path (NCCL's own kernels not counted)
            "gpu_launches": steps * (2 if dist_mode and dd.exchange == "nccl" else 1),
            "clocks": clk,
        }
        if dist_mode and dd.exchange == "peer":
            line["config"]["collective"] = ("peer-memory exchange inside the evaluation kernel: the finishing CTA "
                                            "stores the K+1 partial into every rank's mailbox (CUDA IPC, "
                                            "NVLink/NVSwitch), flag + wait, rank-ordered fold (no NCCL call)")
        elif dist_mode:
            line["config"]["collective"] = "NCCL all_gather_into_tensor of K+1 doubles + pm_fold_rows per step"
        if dist_mode and check is not None:
            line["check_vs_1gpu"] = check
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, x_all, y_all, betas[:5])
        print(json.dumps(line), flush=True)
    if dist_mode:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- B200 arm: chain
def run_chain_bench(args, cfg):
    """Config 2: `steps` sampler iterations (each = K coordinate updates) of run_chain."""
    import torch
    from paper_1310_1537_b200 import glm as pglm
    from paper_1310_1537_b200.rng import BufferKind, DeviateBuffer
    from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior, run_chain
    from paper_1310_1537_b200.synthetic import baseline_design
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    n, k = cfg["chain_n"], cfg["k"]
    x, y, _, _ = baseline_design(n, k, seed=2)
    data = pglm.DesignMatrix(x, y)
    prior = GaussianPrior.isotropic(k, 0.0, 10.0)
    if args.warmup:
        run_chain(data, prior, ChainConfig(n_iter=args.warmup, n_burnin=0, seed=5))
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    out = run_chain(data, prior, ChainConfig(n_iter=args.steps, n_burnin=0, seed=5),
                    rng=DeviateBuffer(BufferKind.UNIFORM01, seed=5))
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    peak, src = load_peaks()
    evals = out.accept_evals
    dev_s = out.kernel_ms / 1e3
    if rank == 0:
        print(json.dumps({
            "metric": "slice-within-Gibbs iterations/s (config 2)", "value": args.steps / dev_s,
            "unit": "iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True, "scaling": "replicas only",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8d config 2 generator)",
            "config": {"workload": cfg["desc"], "N": n, "K": k, "seed": 5,
                       "timing": "value: CUDA events around the one cooperative chain kernel; e2e: host wall "
                                 "of run_chain (uniform stream position in, draws out)"},
            "log_posterior_evals_per_s": evals / dev_s, "evals_per_coordinate": evals / (args.steps * k),
            "roofline": {"bound": "dependent evaluations (one grid sync per pass) + fp64 softplus issue",
                         "achieved": evals * 24 * n / dev_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": evals * 24 * n / dev_s / 1e9 / peak, "traffic": None, "peak_source": src,
                         "note": "achieved = the reference's per-evaluation bytes (xbeta, xt[k], y) x evaluations"},
            "e2e": {"value": args.steps / wall, "unit": "iterations/s", "h2d_bytes_per_step": 8 * 3 * k / args.steps,
                    "d2h_bytes_per_step": 8 * k},
            "gpu_launches": 1, "clocks": clk,
            "cpu_baseline": None if args.no_cpu_baseline else cpu_baseline_other(args.config)}), flush=True)


# ---------------------------------------------------------------------------- B200 arm: HB
def run_hb(args, cfg):
    import torch
    from paper_1310_1537_b200.hb import CsrGroups
    from paper_1310_1537_b200.synthetic import hb_design
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    x, y, off, betas, mu, tau = hb_design(cfg["groups"], cfg["k"], seed=3, mean_rows=cfg["mean_rows"])
    csr = CsrGroups(x, y, off)
    dev = csr.on_device(local)
    sigma = np.full(cfg["k"], tau)
    for _ in range(args.warmup):
        dev.eval(betas, mu, sigma)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ms = dev.time_evals(betas, mu, sigma, n=args.steps) / args.steps  # device, CUDA events
    clk = clocks.stop()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dev.eval(betas, mu, sigma)
    e2e_ms = (time.perf_counter() - t0) / args.steps * 1e3
    n = int(off[-1])
    bytes_launch = n * (cfg["k"] * 8 + 8)
    peak, src = load_peaks()
    if rank == 0:
        print(json.dumps({
            "metric": "HB batched log-posterior+gradient launches/s (G groups per launch)", "value": 1000.0 / ms,
            "unit": "launches/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY §8d config 3 generator)",
            "config": {"workload": cfg["desc"], "rows": n, "K": cfg["k"], "groups": cfg["groups"]},
            "group_evals_per_s": cfg["groups"] * 1000.0 / ms,
            "roofline": {"bound": "hbm", "achieved": bytes_launch / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": bytes_launch / (ms * 1e-3) / 1e9 / peak, "traffic": load_traffic(args.config),
                         "peak_source": src},
            "e2e": {"value": 1000.0 / e2e_ms, "unit": "launches/s", "h2d_bytes_per_step": betas.nbytes,
                    "d2h_bytes_per_step": 8 * cfg["groups"] * (cfg["k"] + 1)},
            "gpu_launches": args.steps, "clocks": clk,
            "cpu_baseline": None if args.no_cpu_baseline else cpu_baseline_other(args.config)}), flush=True)


# ---------------------------------------------------------------------------- B200 arm: Gibbs
def run_gibbs_strips(args, cfg):
    """N>1: horizontal strips, one per rank; halo rows exchanged by the half-sweep kernels
    through peer memory (start_peer_halos), or over NCCL per half-sweep (--exchange nccl, or
    if a peer mapping fails on any rank)."""
    import torch
    import torch.distributed as dist
    from paper_1310_1537_b200.dist import LatticeStrip, start_peer_halos, strip_bounds, strip_sweeps
    from paper_1310_1537_b200.synthetic import ising_spins, potts_states
    ws, rank, local = dist_env()
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h, w = cfg["h"], cfg["w"]
    a, b = strip_bounds(h, ws, rank)
    full = ising_spins(h, w, seed=0) if cfg["model"] == "ising" else potts_states(h, w, seed=0)
    strip = LatticeStrip(h, w, a, b - a, local, model=cfg["model"], w=2 * 0.4407, coupling=0.4407)
    strip.set_spins(full[a:b])
    del full
    peer = args.exchange != "nccl" and start_peer_halos(strip, rank, ws)
    seed = 2024
    strip_sweeps(strip, args.warmup, seed, 0, rank, ws)
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    strip_sweeps(strip, args.steps, seed, args.warmup, rank, ws)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    peak, src = load_peaks()
    if rank == 0:
        print(json.dumps({
            "metric": "Gibbs sweeps/s (red-black checkerboard)", "value": 1000.0 / ms, "unit": "sweeps/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8 spins, u32 Philox",
            "data": "synthetic iid uniform initial state",
            "config": {"workload": cfg["desc"], "H": h, "W": w, "beta_J": 0.4407,
                       "parallelism": f"row strips x{ws}, " + (
                           "halo rows stored into the neighbours' mailboxes by the half-sweep kernels "
                           "(P2P, flags; no NCCL call)" if peer else "NCCL halo exchange per half-sweep")},
            "msite_per_s": h * w / (ms * 1e-3) / 1e6,
            "roofline": {"bound": "issue (Philox4x32) + halo latency", "achieved": 2 * h * w / (ms * 1e-3) / 1e9,
                         "peak": peak * ws, "unit": "GB/s", "frac": 2 * h * w / (ms * 1e-3) / 1e9 / (peak * ws),
                         "traffic": None, "peak_source": src},
            "e2e": {"value": 1000.0 / ms, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 2 * args.steps, "clocks": clk}), flush=True)
    strip.close()
    dist.destroy_process_group()


def run_gibbs(args, cfg):
    import torch
    from paper_1310_1537_b200 import ising
    from paper_1310_1537_b200.rng import SitePhilox
    from paper_1310_1537_b200.synthetic import ising_spins, potts_states
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    h, w = cfg["h"], cfg["w"]
    if ws > 1:
        return run_gibbs_strips(args, cfg)
    if cfg["model"] == "ising":
        lat = ising.IsingLattice(ising_spins(h, w, seed=0), np.zeros((h, w)), 2 * 0.4407, boundary="periodic")
    else:
        lat = ising.PottsLattice(potts_states(h, w, seed=0), 0.4407, boundary="periodic")
    ising.pin_lattice(lat)  # page-locked spins: the e2e spin I/O is one DMA each way
    part = ising.color_lattice(lat, device=local)
    dev = part.device
    assert dev.fast_path()
    rng = SitePhilox(seed=2024)
    dev.sweeps(args.warmup, 2, rng.seed, 0, rng.sweep)
    rng.advance(args.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ms = dev.time_sweeps(args.steps, 2, rng.seed, 0, rng.sweep) / args.steps  # CUDA events, handle stream
    clk = clocks.stop()
    # cold-L2 variant: the 2 x 32 MiB lattice state is L2-resident across sweeps by design;
    # also time single sweeps after evicting it (512 MiB write)
    flush = L2Scrub(f"cuda:{local}")
    cold_ms = 0.0
    n_cold = min(50, args.steps)
    for t in range(n_cold):
        flush()
        cold_ms += dev.time_sweeps(1, 2, rng.seed, 0, rng.sweep + args.steps + t)
    del flush
    # end to end: spins in from host, sweeps, spins out (one untimed spin round trip first, as
    # every other timed region here has its warm-up: the first one after the cold-L2 loop
    # intermittently took ~50 ms on the pack step, whatever the model)
    part.pack_from(lat)
    part.unpack_into(lat)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    part.pack_from(lat)
    t1 = time.perf_counter()
    dev.sweeps(args.steps, 2, rng.seed, 0, rng.sweep + args.steps)
    t2 = time.perf_counter()
    part.unpack_into(lat)
    e2e = time.perf_counter() - t0
    e2e_parts = {"pack_ms": (t1 - t0) * 1e3, "sweeps_ms": (t2 - t1) * 1e3, "unpack_ms": (t0 + e2e - t2) * 1e3}
    peak, src = load_peaks()
    bytes_sweep = 2 * h * w
    if rank == 0:
        print(json.dumps({
            "metric": "Gibbs sweeps/s (red-black checkerboard)", "value": 1000.0 / ms, "unit": "sweeps/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8 spins, u32 Philox",
            "data": "synthetic iid uniform initial state",
            "config": {"workload": cfg["desc"], "H": h, "W": w, "beta_J": 0.4407,
                       "l2": "lattice state (2 x 32 MiB packed int8) is L2-resident across the sweeps by design; "
                             "cold_l2_sweeps_per_s flushes L2 (512 MiB write + 256 MiB clean read) before each timed sweep"},
            "cold_l2_sweeps_per_s": 1000.0 * n_cold / cold_ms,
            "msite_per_s": h * w / (ms * 1e-3) / 1e6,
            "roofline": {"bound": "issue (Philox4x32) -- HBM fraction reported for context",
                         "achieved": bytes_sweep / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": bytes_sweep / (ms * 1e-3) / 1e9 / peak, "traffic": load_traffic(args.config),
                         "peak_source": src},
            "issue_roofline": issue_roofline(args.config, ms, clk),
            "e2e": {"value": args.steps / e2e, "unit": "sweeps/s", "h2d_bytes_per_step": h * w / args.steps,
                    "d2h_bytes_per_step": h * w / args.steps, "parts": e2e_parts},
            "gpu_launches": 2 * args.steps, "clocks": clk,
            "cpu_baseline": None if args.no_cpu_baseline else cpu_baseline_other(args.config)}), flush=True)


# ---------------------------------------------------------------------------- B200 arm: HB Gibbs sweep
def run_hb_sweep(args, cfg):
    """Device-resident hierarchical Gibbs sweeps (hb_sweep, hb.py:138-168) at the config-3 shape."""
    import torch
    from paper_1310_1537_b200.glm import DesignMatrix
    from paper_1310_1537_b200.hb import HbDataset, HbState
    from paper_1310_1537_b200.sampler import GaussianPrior
    from paper_1310_1537_b200.synthetic import hb_design
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    x, y, off, _, mu, tau = hb_design(cfg["groups"], cfg["k"], seed=3, mean_rows=cfg["mean_rows"])
    G, K = cfg["groups"], cfg["k"]
    ds = HbDataset([DesignMatrix(x[off[g]:off[g + 1]], y[off[g]:off[g + 1]]) for g in range(G)])
    prior = GaussianPrior(mu, np.full(K, tau))
    st = HbState(ds, prior, seed=5, device=local)
    st.sweeps(prior, args.warmup)
    ev0 = st.total_evals
    clocks = ClockSampler(local)
    clocks.start()
    kernel_ms, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        st.sweeps(prior, 1)
        walls.append(time.perf_counter() - t0)
        kernel_ms.append(st.last_kernel_ms)
    clk = clocks.stop()
    ms = statistics.mean(kernel_ms)
    evals = (st.total_evals - ev0) / args.steps
    n = int(off[-1])
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import sampler_oracle as so
        sample = 20
        t0 = time.perf_counter()
        for g in range(sample):
            so.run_chain(x[off[g]:off[g + 1]], y[off[g]:off[g + 1]], mu, np.full(K, tau), 1, 0,
                         rng=so.UniformStream(5, owner=(g,)))
        dt = (time.perf_counter() - t0) * G / sample
        cpu = {"value": 1.0 / dt, "unit": "sweeps/s", "cores": 1, "kind": "port",
               "sample": f"oracle/sampler_oracle.py run_chain (numpy restatement of the reference's per-group "
                         f"slice-within-Gibbs, hb.py:127-135) for {sample} of {G} groups, 1 sweep, scaled x{G/sample:g}"}
    peak, src = load_peaks()
    row_bytes = 24  # xbeta, xt[k], y per row per conditional evaluation (L2-resident group working set)
    if rank == 0:
        print(json.dumps({
            "metric": "hierarchical Gibbs sweeps/s (hb_sweep, every group's K coordinates once)",
            "value": 1000.0 / ms, "unit": "sweeps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY §8d config 3 generator, seed 3); streams seed 5, owner (g,)",
            "config": {"workload": cfg["desc"], "rows": n, "K": K, "groups": G},
            "coordinate_updates_per_s": G * K * 1000.0 / ms,
            "conditional_evals_per_s": evals * 1000.0 / ms,
            "roofline": {"bound": "latency (CTA-serial slice control flow) -- row-stream rate for context",
                         "achieved": evals / G * n * row_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": evals / G * n * row_bytes / (ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "peak_source": src},
            "e2e": {"value": 1.0 / statistics.mean(walls), "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 8 * G * (K + 2)},
            "gpu_launches": args.steps, "clocks": clk, "cpu_baseline": cpu}), flush=True)
    st.close()


# ---------------------------------------------------------------------------- B200 arm: batch RNG
def run_rng(args, cfg):
    """Device batch RNG: Gamma(2, 3) draws/s on one (uniform, normal) stream
    pair -- the reference's rng_bench GAMMA cell (rng.py:246-300) -- plus stream fill rates."""
    import ctypes

    import torch
    from paper_1310_1537_b200 import _lib
    from paper_1310_1537_b200 import rng as prng
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    n = cfg["draws"]
    params = prng.GammaParams(2.0, 3.0)
    u = prng.DeviateBuffer(prng.BufferKind.UNIFORM01, seed=9, owner=(0,))
    z = prng.DeviateBuffer(prng.BufferKind.STD_NORMAL, seed=9, owner=(1,))
    for _ in range(args.warmup):
        prng.gamma_batch(params, n, u, z, local)
    clocks = ClockSampler(local)
    clocks.start()
    dev_ms, walls = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        prng.gamma_batch(params, n, u, z, local, timing=dev_ms)
        walls.append(time.perf_counter() - t0)
    clk = clocks.stop()
    ms = statistics.mean(dev_ms)
    # stream fill rates into device memory (8 B written per deviate)
    n_fill = 1 << 28
    buf = torch.empty(n_fill, dtype=torch.float64, device=f"cuda:{local}")
    fill = {}
    k0, k1 = u.stream_key()
    for name, kind in (("uniform01", _lib.PM_RNG_KIND_UNIFORM01), ("std_normal", _lib.PM_RNG_KIND_STD_NORMAL)):
        t = ctypes.c_float()
        for _ in range(2):
            _lib.call("pm_rng_fill", local, kind, ctypes.c_uint64(k0), ctypes.c_uint64(k1), ctypes.c_uint64(0), n_fill,
                      buf.data_ptr(), 1, ctypes.byref(t))
        fill[name] = {"deviates_per_s": n_fill / (t.value * 1e-3), "write_gb_per_s": 8 * n_fill / (t.value * 1e-3) / 1e9}
    del buf
    dms = []
    prng.dirichlet_batch(np.ones(100), 100_000, u, z, local)
    prng.dirichlet_batch(np.ones(100), 100_000, u, z, local, timing=dms)
    peak, src = load_peaks()
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import rng_oracle as ro
        m = 30_000
        t0 = time.perf_counter()
        ro.gamma_draws(2.0, 3.0, m, u.stream_key(), 0, z.stream_key(), 0)
        dt = time.perf_counter() - t0
        cpu = {"value": m / dt, "unit": "draws/s", "cores": 1, "kind": "port",
               "sample": f"oracle/rng_oracle.py gamma_draws (restatement of rng.py:163-198, scalar Python, "
                         f"numpy streams), {m} Gamma(2,3) draws, 1 core -- the reference's per-call cost model"}
    if rank == 0:
        print(json.dumps({
            "metric": "Gamma(2,3) draws/s on one buffered stream pair (device two-scan sampler)",
            "value": n / (ms * 1e-3), "unit": "draws/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "numpy Philox4x64 streams, seed 9, owners (0,) uniform / (1,) normal",
            "config": {"workload": cfg["desc"], "draws_per_step": n},
            "cycles_per_sample_at_2.6GHz": ms * 1e-3 * 2.6e9 / n,
            "stream_fill": fill,
            "dirichlet_k100_vectors_per_s": 100_000 / (dms[0] * 1e-3),
            "roofline": {"bound": "issue (Philox4x64 + fp64 log/sincos) -- HBM fraction of the fill kernel for context",
                         "achieved": fill["uniform01"]["write_gb_per_s"], "peak": peak, "unit": "GB/s",
                         "frac": fill["uniform01"]["write_gb_per_s"] / peak, "traffic": None, "peak_source": src},
            "e2e": {"value": n / statistics.mean(walls), "unit": "draws/s", "h2d_bytes_per_step": 32,
                    "d2h_bytes_per_step": 8 * n},
            "gpu_launches": None, "clocks": clk, "cpu_baseline": cpu}), flush=True)


def main():
    p = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=None)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                   help="GLM rank path: peer-memory exchange in the kernel (auto: N>1) or NCCL all-gather")
    p.add_argument("--tune", action="append", default=[], metavar="KNOB=VALUE",
                   help="A/B: kernel-dispatch override through pm_tune_set (e.g. f32_pairs=0); repeatable")
    p.add_argument("--force-dist", action="store_true",
                   help="GLM configs: use the per-rank NCCL path even at N=1 (a 1-rank group)")
    # internal: CPU baseline subprocess
    p.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--sample-rows", type=int, default=0, help=argparse.SUPPRESS)
    p.add_argument("--k", type=int, default=0, help=argparse.SUPPRESS)
    p.add_argument("--reps", type=int, default=5, help=argparse.SUPPRESS)
    p.add_argument("--x-storage", default="f64", help=argparse.SUPPRESS)
    p.add_argument("--ref-worker", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--setting", default="ii", choices=["i", "ii"], help=argparse.SUPPRESS)
    p.add_argument("--data", default="", help=argparse.SUPPRESS)
    p.add_argument("--ref-kind", default="reference", choices=["reference", "port"], help=argparse.SUPPRESS)
    args = p.parse_args()
    if args.cpu_worker:
        cpu_worker_main(args)
        return
    if args.ref_worker:
        ref_worker_main(args)
        return
    cfg = CONFIGS[args.config]
    if args.tune and args.impl == "b200":
        from paper_1310_1537_b200 import _lib
        for kv in args.tune:
            knob, val = kv.split("=", 1)
            _lib.set_tune(knob.strip(), int(val))
    if args.impl == "reference":
        args.steps = args.steps or 5
        args.warmup = args.warmup if args.warmup is not None else 3
        if "n" not in cfg:
            ws, rank, _ = dist_env()
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for GLM configs"}))
            return
        run_reference(args, cfg)
        return
    if "n" in cfg:
        args.steps = args.steps or 1000
        args.warmup = args.warmup if args.warmup is not None else 10
        run_glm(args, cfg)
    elif "chain_n" in cfg:
        args.steps = args.steps or 20
        args.warmup = args.warmup if args.warmup is not None else 3
        run_chain_bench(args, cfg)
    elif "sweep_groups" in cfg:
        args.steps = args.steps or 20
        args.warmup = args.warmup if args.warmup is not None else 3
        cfg = dict(cfg, groups=cfg["sweep_groups"])
        run_hb_sweep(args, cfg)
    elif "groups" in cfg:
        args.steps = args.steps or 200
        args.warmup = args.warmup if args.warmup is not None else 5
        run_hb(args, cfg)
    elif "draws" in cfg:
        args.steps = args.steps or 10
        args.warmup = args.warmup if args.warmup is not None else 3
        run_rng(args, cfg)
    else:
        args.steps = args.steps or 1000
        args.warmup = args.warmup if args.warmup is not None else 10
        run_gibbs(args, cfg)


if __name__ == "__main__":
    main()
