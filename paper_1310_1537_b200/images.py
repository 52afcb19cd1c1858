"""Binary-image I/O and synthesis for the denoising pipeline (host side).

Mirror of the reference's PBM helpers and test-image generators
(ising.py:297-406).  These are file/format utilities around the device sweep,
not part of the hot path:

  * read_pbm(path)            P1 (ASCII) or P4 (raw) -> (H, W) uint8 in {0, 1},
                              1 = black passed through unchanged (ising.py:297-324);
                              '#' comments allowed anywhere in the header;
                              ValueError on bad magic, bad size or short raster.
  * write_pbm(path, img, fmt) raw P4 (default) or ASCII P1 (ising.py:352-370).
  * synthetic_binary_image    "two_region" | "all_ones" | "all_zeros" (ising.py:373-392).
  * flip_noise(img, rate, seed)  flips exactly round(rate*size) distinct pixels
                              drawn by numpy default_rng(seed).choice without
                              replacement (ising.py:395-406) -- the same draw, so
                              the noisy images are identical to the reference's.
"""

from __future__ import annotations

import numpy as np

__all__ = ["read_pbm", "write_pbm", "synthetic_binary_image", "flip_noise"]


def _header(raw: bytes) -> tuple[list[bytes], int]:
    """Magic, width, height tokens and the offset of the first raster byte.

    Comments run from '#' to end of line.  After the third token exactly one
    whitespace byte separates header from raster (that matters for P4).
    """
    toks: list[bytes] = []
    pos, n = 0, len(raw)
    while pos < n and len(toks) < 3:
        ch = raw[pos:pos + 1]
        if ch in (b" ", b"\t", b"\r", b"\n"):
            pos += 1
            continue
        if ch == b"#":
            eol = pos
            while eol < n and raw[eol:eol + 1] not in (b"\r", b"\n"):
                eol += 1
            pos = eol
            continue
        end = pos
        while end < n and raw[end:end + 1] not in (b" ", b"\t", b"\r", b"\n"):
            end += 1
        toks.append(raw[pos:end])
        pos = end
        if len(toks) == 3 and pos < n:
            pos += 1
    return toks, pos


def read_pbm(path) -> np.ndarray:
    """Read a P1/P4 PBM into a (H, W) uint8 {0,1} array."""
    with open(path, "rb") as fh:
        raw = fh.read()
    toks, off = _header(raw)
    if len(toks) < 3:
        raise ValueError(f"{path}: truncated PBM header")
    magic = toks[0]
    try:
        width, height = int(toks[1]), int(toks[2])
    except ValueError as exc:
        raise ValueError(f"{path}: non-numeric PBM dimensions") from exc
    if width < 1 or height < 1:
        raise ValueError(f"{path}: bad dimensions {width}x{height}")
    npix = width * height
    if magic == b"P1":
        text = raw[off:].decode("ascii", "ignore")
        digits = []
        for line in text.splitlines():
            digits.extend(ch for ch in line.partition("#")[0] if ch in "01")
        if len(digits) < npix:
            raise ValueError(f"{path}: expected {npix} pixels, found {len(digits)}")
        return (np.frombuffer("".join(digits[:npix]).encode("ascii"), dtype=np.uint8) - ord("0")
                ).reshape(height, width).copy()
    if magic == b"P4":
        stride = (width + 7) >> 3
        need = height * stride
        body = raw[off:off + need]
        if len(body) < need:
            raise ValueError(f"{path}: expected {need} data bytes, found {len(body)}")
        packed = np.frombuffer(body, dtype=np.uint8).reshape(height, stride)
        return np.ascontiguousarray(np.unpackbits(packed, axis=1)[:, :width])
    raise ValueError(f"{path}: unsupported magic {magic!r} (want P1 or P4)")


def _check_image(img: np.ndarray) -> None:
    if img.ndim != 2 or img.size == 0:
        raise ValueError("image must be non-empty 2-D")
    if not np.isin(img, (0, 1)).all():
        raise ValueError("image entries must be 0 or 1")


def write_pbm(path, image01, fmt: str = "P4") -> None:
    """Write a {0,1} image as raw P4 (default) or ASCII P1."""
    img = np.asarray(image01)
    _check_image(img)
    if fmt not in ("P1", "P4"):
        raise ValueError(f"fmt must be 'P1' or 'P4', got {fmt!r}")
    height, width = img.shape
    if fmt == "P4":
        payload = np.packbits(img.astype(np.uint8), axis=1).tobytes()
        with open(path, "wb") as fh:
            fh.write(b"P4\n%d %d\n" % (width, height))
            fh.write(payload)
        return
    rows = "\n".join(" ".join("1" if v else "0" for v in row) for row in img.tolist())
    with open(path, "w") as fh:
        fh.write(f"P1\n{width} {height}\n{rows}\n")


def synthetic_binary_image(height: int, width: int, kind: str = "two_region", seed: int = 0) -> np.ndarray:
    """Deterministic {0,1} test images ("two_region": right half set, plus one
    set rectangle on the left and one cleared rectangle on the right)."""
    if height < 1 or width < 1:
        raise ValueError("image dimensions must be >= 1")
    if kind == "all_ones":
        return np.ones((height, width), dtype=np.uint8)
    if kind == "all_zeros":
        return np.zeros((height, width), dtype=np.uint8)
    if kind != "two_region":
        raise ValueError(f"unknown image kind {kind!r}")
    img = np.zeros((height, width), dtype=np.uint8)
    img[:, width // 2:] = 1
    r0, r1, r2 = height // 4, height // 2, 3 * height // 4
    img[r0:r1, width // 8:width // 3] = 1
    img[r1:r2, 2 * width // 3:7 * width // 8] = 0
    return img


def flip_noise(image01, rate: float, seed: int = 0) -> np.ndarray:
    """Flip exactly round(rate * size) distinct, uniformly chosen pixels."""
    out = np.asarray(image01).copy()  # C order, so the flat view below aliases it
    if not (0.0 <= rate <= 1.0):
        raise ValueError("rate must be in [0, 1]")
    count = int(round(rate * out.size))
    if count:
        picks = np.random.default_rng(seed).choice(out.size, size=count, replace=False)
        view = out.reshape(-1)
        view[picks] = 1 - view[picks]
    return out
