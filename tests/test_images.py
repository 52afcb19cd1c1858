"""Host-side image helpers of the denoising pipeline against reference fixtures (CPU only).

Mirrors the reference's own image tests (test_ising.py:311-332) and pins the
bytes written and the noise draws against tests/golden/denoise.npz, which
make_golden.py produced with the unmodified reference (ising.py:297-406).
"""

import numpy as np
import pytest

from conftest import golden
from paper_1310_1537_b200 import ising
from paper_1310_1537_b200.images import flip_noise, read_pbm, synthetic_binary_image, write_pbm


@pytest.mark.parametrize("fmt", ["P1", "P4"])
def test_pbm_bytes_match_reference(tmp_path, fmt):
    z = golden("denoise.npz")
    path = tmp_path / f"x.{fmt}"
    write_pbm(path, z["pbm_img"], fmt=fmt)
    assert path.read_bytes() == z[f"pbm_{fmt}"].tobytes()
    ref = tmp_path / f"ref.{fmt}"
    ref.write_bytes(z[f"pbm_{fmt}"].tobytes())
    np.testing.assert_array_equal(read_pbm(ref), z["pbm_img"])


@pytest.mark.parametrize("fmt", ["P1", "P4"])
@pytest.mark.parametrize("shape", [(5, 5), (7, 13), (3, 8), (1, 1), (2, 17)])
def test_pbm_round_trip(tmp_path, fmt, shape):
    img = flip_noise(synthetic_binary_image(*shape), 0.4, seed=11)
    path = tmp_path / f"img_{fmt}_{shape[0]}x{shape[1]}.pbm"
    write_pbm(path, img, fmt=fmt)
    np.testing.assert_array_equal(read_pbm(path), img)


def test_pbm_reads_comments_and_rejects_garbage(tmp_path):
    path = tmp_path / "c.pbm"
    path.write_text("P1\n# a comment\n3 2\n0 1 0\n1 1 0\n")
    np.testing.assert_array_equal(read_pbm(path), [[0, 1, 0], [1, 1, 0]])
    path.write_text("P1 # inline\n3 # w\n2\n010110\n")
    np.testing.assert_array_equal(read_pbm(path), [[0, 1, 0], [1, 1, 0]])
    for body in ("P5\n2 2\n", "P1\n4 4\n0 1\n", "P1\n0 3\n", "P4\n8 2\n\x01", "P1\n3\n"):
        bad = tmp_path / "bad.pbm"
        bad.write_text(body)
        with pytest.raises(ValueError):
            read_pbm(bad)


def test_write_pbm_rejects_bad_images(tmp_path):
    with pytest.raises(ValueError):
        write_pbm(tmp_path / "a.pbm", np.zeros((0, 3)))
    with pytest.raises(ValueError):
        write_pbm(tmp_path / "a.pbm", np.array([[0, 2]]))
    with pytest.raises(ValueError):
        write_pbm(tmp_path / "a.pbm", np.zeros((2, 2)), fmt="P2")


def test_noisy_images_match_reference_draws():
    z = golden("denoise.npz")
    kinds = ["two_region", "two_region", "all_ones", "two_region", "two_region", "two_region", "two_region",
             "two_region"]
    rates = [0.1, 0.1, 0.1, 0.0, 0.2, 0.2, 0.25, 0.3]
    nseeds = [3, 5, 7, 0, 9, 9, 11, 1]
    for i in range(int(z["n_cases"])):
        shape = z[f"noisy_{i}"].shape
        img = flip_noise(synthetic_binary_image(*shape, kind=kinds[i]), rates[i], seed=nseeds[i])
        np.testing.assert_array_equal(img, z[f"noisy_{i}"], err_msg=f"case {i}")


def test_flip_noise_counts_and_validation():
    img = synthetic_binary_image(20, 30)
    for rate in (0.0, 0.05, 0.5, 1.0):
        assert int((flip_noise(img, rate, seed=4) != img).sum()) == int(round(rate * img.size))
    with pytest.raises(ValueError):
        flip_noise(img, 1.5)
    with pytest.raises(ValueError):
        synthetic_binary_image(0, 3)
    with pytest.raises(ValueError):
        synthetic_binary_image(3, 3, kind="stripes")
    assert synthetic_binary_image(2, 2, kind="all_zeros").sum() == 0


def test_denoise_host_validation_needs_no_device():
    # reference order (ising.py:268-271): image validation, then the sweep counts
    with pytest.raises(ValueError):
        ising.denoise(np.empty((0, 0)))
    with pytest.raises(ValueError):
        ising.denoise(np.array([[0, 2]]))
    with pytest.raises(ValueError):
        ising.denoise(np.zeros((3, 3), dtype=np.uint8), sweeps=-1)
    noisy = flip_noise(synthetic_binary_image(16, 16), 0.2, seed=9)
    np.testing.assert_array_equal(ising.denoise(noisy, sweeps=0, burnin=0, seed=1), noisy)
    np.testing.assert_array_equal(ising.denoise(noisy, sweeps=4, burnin=4, seed=1), noisy)
