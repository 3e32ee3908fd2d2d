"""Caller-side input formats on the host: circumscribed-square side, PNM files
(tt_prep_side, tt_pnm_read, tt_pgm_write) and the oracle's restatement of the
device preparation kernel."""
import os

import numpy as np
import pytest

import oracle as O
import paper_1604_03410_b200 as tt


@pytest.mark.parametrize("h,w", [(1, 1), (3, 4), (256, 256), (480, 640), (17, 1000), (999, 2)])
def test_prep_side_is_the_smallest_square_whose_disk_holds_the_picture(h, w):
    n = tt.prep_side(h, w)
    assert (n - 1) ** 2 >= h * h + w * w > (n - 2) ** 2
    assert n >= max(h, w)


def test_pgm_round_trip(tmp_path):
    img = np.linspace(0.0, 1.0, 7 * 5, dtype=np.float32).reshape(7, 5)
    p = str(tmp_path / "a.pgm")
    tt.write_pgm(p, img, 0.0, 1.0)
    back = tt.read_pnm(p)
    assert back.shape == (7, 5) and back.dtype == np.uint8
    assert np.array_equal(back, np.floor(img.astype(np.float64) * 255.0 + 0.5).astype(np.uint8))  # lround


def test_ppm_reader_with_comments(tmp_path):
    rgb = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    p = tmp_path / "b.ppm"
    p.write_bytes(b"P6\n# made by a test\n3 2\n255\n" + rgb.tobytes())
    assert np.array_equal(tt.read_pnm(str(p)), rgb)


@pytest.mark.parametrize("content", [b"P3\n1 1\n255\n0 0 0", b"P5\n2 2\n65535\n" + bytes(8), b"P5\n4 4\n255\n" + bytes(3)])
def test_pnm_reader_rejects_unsupported_or_truncated_files(tmp_path, content):
    p = tmp_path / "bad.pnm"
    p.write_bytes(content)
    with pytest.raises(Exception):
        tt.read_pnm(str(p))


def test_oracle_prep_places_and_converts():
    rgb = np.zeros((2, 4, 3), np.uint8)
    rgb[..., 0] = 255
    out = O.prep(rgb, 6)
    assert out.shape == (6, 6)
    assert np.all(out[2:4, 1:5] == np.float32(np.float32(0.299) * np.float32(255.0)) / np.float32(255.0))
    assert out.sum() == out[2:4, 1:5].sum()
