"""Device preparation of 8-bit pictures (tt_prep_device) against the oracle's
restatement, and a picture through the whole path: file -> prep -> fused
kernel, with the mass check that motivates the circumscribed square."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("h,w,ch", [(1, 1, 1), (5, 7, 3), (240, 320, 3), (100, 37, 1), (256, 256, 3)])
def test_prep_matches_oracle_bitwise(gpu, h, w, ch):
    rng = np.random.default_rng(h * 1000 + w + ch)
    pix = rng.integers(0, 256, size=(h, w, ch) if ch == 3 else (h, w), dtype=np.uint8)
    n = tt.prep_side(h, w)
    d_pix = torch.from_numpy(pix.copy()).cuda()
    d_img = torch.full((n, n), float("nan"), device="cuda")
    tt.prep_device(d_pix.data_ptr(), h, w, ch, n, d_img.data_ptr())
    torch.cuda.synchronize()
    ref = O.prep(pix, n)
    assert np.array_equal(d_img.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_picture_file_through_the_path_keeps_its_mass(gpu, tmp_path):
    h, w = 60, 90
    yy, xx = np.mgrid[0:h, 0:w]
    rgb = np.stack([(xx * 2) % 256, (yy * 4) % 256, (xx + yy) % 256], -1).astype(np.uint8)
    p = tmp_path / "pic.ppm"
    p.write_bytes(b"P6\n%d %d\n255\n" % (w, h) + rgb.tobytes())
    pix = tt.read_pnm(str(p))
    n = tt.prep_side(h, w)
    d_pix = torch.from_numpy(pix.copy()).cuda()
    d_img = torch.empty((n, n), device="cuda")
    tt.prep_device(d_pix.data_ptr(), h, w, 3, n, d_img.data_ptr())
    img = d_img.cpu().numpy()
    ctx = tt.create_context(gpu)
    out, med, rep = tt.TraceTransform(ctx, n, 36)(img)
    assert rep.ok()
    # T0 of every angle integrates the whole picture: bilinear resampling on the pixel grid
    # conserves mass up to interpolation at the (zero) border of the inscribed disk
    mass = img.astype(np.float64).sum()
    t0 = out[:, 0, :].astype(np.float64).sum(axis=1)
    assert np.all(np.abs(t0 - mass) <= 2e-3 * mass)
    ctx.destroy()
