"""CLI front end (reference cli.py; its tests test_cli.py restated).

The usage / input-error paths need no device and run on CPU; the end-to-end
commands are gpu-marked.
"""

import numpy as np
import pytest

from paper_1310_1537_b200 import cli, perf
from paper_1310_1537_b200.images import flip_noise, read_pbm, synthetic_binary_image, write_pbm


def read_csv_rows(path):
    lines = [ln for ln in path.read_text().splitlines() if ln and not ln.startswith("#")]
    return lines[0], lines[1:]


# ----------------------------------------------------------------- CPU: usage and input errors
def test_bench_missing_k_is_usage_error(tmp_path):
    assert cli.main(["bench", "--N", "100", "--out", str(tmp_path / "x.csv")]) == 2


def test_bench_bad_config_is_input_error(tmp_path):
    cfgfile = tmp_path / "bad.cfg"
    cfgfile.write_text("nonsense = 1\n")
    assert cli.main(["bench", "--config", str(cfgfile)]) == 2


def test_bench_internal_error_returns_one(tmp_path, monkeypatch):
    def boom(cfg):
        raise RuntimeError("kaput")
    monkeypatch.setattr(perf, "run_grid", boom)
    assert cli.main(["bench", "--N", "10", "--K", "2", "--out", str(tmp_path / "x.csv")]) == 1


def test_glm_sample_input_errors(tmp_path, capsys):
    bad = tmp_path / "bad.csv"
    bad.write_text("1.0,oops,1\n")
    assert cli.main(["glm-sample", "--data", str(bad), "--out", str(tmp_path / "o.csv")]) == 2
    assert "column 2" in capsys.readouterr().err
    assert cli.main(["glm-sample", "--data", str(tmp_path / "missing.csv"), "--out", str(tmp_path / "o.csv")]) == 2
    nb = tmp_path / "nb.csv"
    nb.write_text("0.5,2\n0.1,0\n")
    assert cli.main(["glm-sample", "--data", str(nb), "--out", str(tmp_path / "o.csv")]) == 2
    assert cli.main(["glm-sample", "--out", str(tmp_path / "o.csv")]) == 2


def test_ising_denoise_unreadable_image(tmp_path):
    assert cli.main(["ising-denoise", "--in", str(tmp_path / "nope.pbm"), "--out", str(tmp_path / "o.pbm")]) == 2
    garbage = tmp_path / "garbage.pbm"
    garbage.write_bytes(b"GIF89a....")
    assert cli.main(["ising-denoise", "--in", str(garbage), "--out", str(tmp_path / "o.pbm")]) == 2


def test_ising_denoise_zero_sweeps_is_identity_without_device(tmp_path):
    noisy = flip_noise(synthetic_binary_image(32, 32), 0.1, seed=3)
    path = tmp_path / "noisy.pbm"
    write_pbm(path, noisy)
    out = tmp_path / "same.pbm"
    assert cli.main(["ising-denoise", "--in", str(path), "--out", str(out), "--sweeps", "0", "--burnin", "0"]) == 0
    np.testing.assert_array_equal(read_pbm(out), noisy)


def test_rng_bench_unknown_mode_or_dist_is_input_error(tmp_path):
    assert cli.main(["rng-bench", "--modes", "bogus", "--out", str(tmp_path / "r.csv")]) == 2
    assert cli.main(["rng-bench", "--dists", "cauchy", "--out", str(tmp_path / "r.csv")]) == 2


def test_grid_config_parsing_and_sidecar(tmp_path):
    cfgfile = tmp_path / "g.cfg"
    cfgfile.write_text("N = 200, 400\nK = 3\nstrategies = plf, b200\nworkers = 1\nevals = 2\nreps = 2\n"
                       "cpu_clock_ghz = 3.0\nhbm_gbs = 7000.0\ndevice = 0\n")
    cfg = perf.parse_grid_config(cfgfile)
    assert cfg.n_rows == [200, 400] and cfg.hw.cpu_clock_ghz == 3.0 and cfg.dev.hbm_gbs == 7000.0
    rec = perf.BenchRecord.from_wall("grad/b200", 1000, 3, 1, 1, 0.001, 10, 2.6)
    out = tmp_path / "s.csv"
    perf.write_bench_csv([rec], out, failures=[("cell", "boom")])
    text = out.read_text()
    assert "# roofline n_cols=3 compute_min_cpr=" in text and "device_memory_min_cpr=" in text
    assert "[failed: boom]" in text
    # the reference machine's bound formulas (perf.py:64-82)
    assert perf.compute_min_cpr(perf.REFERENCE_MACHINE, 10) == pytest.approx(20 / 128)
    assert perf.memory_min_cpr(perf.REFERENCE_MACHINE, 10) == pytest.approx(2.6 * 88 / 102.4)


# ----------------------------------------------------------------- GPU: end to end
@pytest.mark.gpu
def test_bench_inline_grid_and_determinism(gpu, tmp_path):
    outs = []
    for name in ("a.csv", "b.csv"):
        out = tmp_path / name
        rc = cli.main(["bench", "--N", "500", "--K", "6", "--strategies", "som,b200", "--workers", "1,4",
                       "--evals", "2", "--reps", "2", "--seed", "3", "--out", str(out)])
        assert rc == 0
        header, rows = read_csv_rows(out)
        assert header.startswith("label,") and len(rows) == 4
        outs.append([",".join(np.array(r.split(","))[[0, 1, 2, 3, 4, 7]]) for r in rows])
    assert outs[0] == outs[1]


@pytest.mark.gpu
def test_bench_config_file_wins_and_failures_flagged(gpu, tmp_path):
    cfgfile = tmp_path / "grid.cfg"
    cfgfile.write_text("N = 200\nK = 3\nstrategies = plf\nworkers = 1\nevals = 2\nreps = 2\n")
    out = tmp_path / "c.csv"
    assert cli.main(["bench", "--config", str(cfgfile), "--N", "999999", "--K", "77", "--out", str(out)]) == 0
    _, rows = read_csv_rows(out)
    assert len(rows) == 1 and rows[0].split(",")[1] == "200"
    # an absurdly slow device model makes every cell violate the compute bound
    cfgfile.write_text("N = 200\nK = 4\nstrategies = b200\nworkers = 1\nevals = 2\nreps = 2\nwarmup = 0\n"
                       "fp64_tflops = 1e-9\n")
    out = tmp_path / "f.csv"
    assert cli.main(["bench", "--config", str(cfgfile), "--out", str(out)]) == 0
    assert "[failed:" in out.read_text()


@pytest.mark.gpu
def test_glm_sample_commands(gpu, tmp_path, capsys):
    out = tmp_path / "draws.csv"
    assert cli.main(["glm-sample", "--synthetic", "200,3", "--iters", "40", "--burnin", "10", "--seed", "5",
                     "--out", str(out)]) == 0
    assert "posterior_mean:" in capsys.readouterr().out
    assert np.loadtxt(out, delimiter=",", skiprows=1).shape == (30, 3)
    args = ["glm-sample", "--synthetic", "150,3", "--iters", "30", "--burnin", "5", "--seed", "9"]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(args + ["--diff-update", "--out", str(a)]) == 0
    assert cli.main(args + ["--no-diff-update", "--out", str(b)]) == 0
    da, db = (np.loadtxt(p, delimiter=",", skiprows=1) for p in (a, b))
    assert np.max(np.abs(da - db)) <= 1e-6
    data_file = tmp_path / "d.csv"
    gen = np.random.default_rng(0)
    x = gen.standard_normal((50, 2))
    y = (gen.random(50) < 0.5).astype(int)
    np.savetxt(data_file, np.column_stack([x, y]), delimiter=",", fmt="%.8g")
    assert cli.main(["glm-sample", "--data", str(data_file), "--iters", "20", "--burnin", "5",
                     "--out", str(tmp_path / "o.csv")]) == 0


@pytest.mark.gpu
def test_ising_denoise_commands(gpu, tmp_path):
    img = synthetic_binary_image(32, 32)
    noisy = flip_noise(img, 0.1, seed=3)
    path = tmp_path / "noisy.pbm"
    write_pbm(path, noisy, fmt="P4")
    out, trace = tmp_path / "restored.pbm", tmp_path / "trace.csv"
    assert cli.main(["ising-denoise", "--in", str(path), "--out", str(out), "--w", "1.0", "--bias", "2.0",
                     "--sweeps", "25", "--burnin", "8", "--seed", "7", "--trace", str(trace)]) == 0
    assert (read_pbm(out) != img).mean() < (noisy != img).mean()
    assert trace.read_text().startswith("sweep,flip_fraction")
    outs = []
    for name in ("r1.pbm", "r2.pbm"):
        o = tmp_path / name
        assert cli.main(["ising-denoise", "--in", str(path), "--out", str(o), "--sweeps", "15", "--burnin", "5",
                         "--seed", "21", "--diff-update", "--fmt", "P1"]) == 0
        outs.append(o.read_bytes())
    assert outs[0] == outs[1]


@pytest.mark.gpu
def test_hb_and_rng_bench_commands(gpu, tmp_path):
    out = tmp_path / "hb.csv"
    assert cli.main(["hb-bench", "--groups", "3", "--K", "3", "--navg", "60,120", "--neval", "1,2",
                     "--modes", "coarse,fine", "--sweeps", "2", "--reps", "1", "--out", str(out)]) == 0
    _, rows = read_csv_rows(out)
    assert len(rows) == 8
    out = tmp_path / "rng.csv"
    assert cli.main(["rng-bench", "--dists", "uniform,normal,gamma,dirichlet", "--n", "20000",
                     "--out", str(out)]) == 0
    header, rows = read_csv_rows(out)
    assert header == "dist,mode,n,cycles_per_sample,waste_fraction" and len(rows) == 4
