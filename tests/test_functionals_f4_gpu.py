"""Row f4 on the GPU: the orthonormal (square) sinogram input frame and the
Hermite P-functionals, against the oracle -- the frame
bit-exact (tto_orthonormal), the Hermite centre equal to the circus median
index of the replayed schedule, the Hermite values within an f64 tolerance of
the f64 restatement evaluated at that centre."""
import numpy as np
import pytest

import oracle as O
import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    c.destroy()


@pytest.mark.parametrize("h,w,A", [(256, 256, 360), (100, 180, 90), (300, 200, 128), (64, 64, 361), (512, 384, 720),
                                   (7, 5, 4)])
def test_orthonormal_frame_bit_exact(ctx, h, w, A):
    img = O.synth(O.PHANTOM, max(h, w))[:h, :w].copy()
    got = tt.orthonormal_image(ctx, img, A)
    ref = O.orthonormal(img, A)
    assert got.shape == (A, A) and tt.orthonormal_side(A) == O.orthonormal_side(A)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _check_hermite(sino, hp, center, orders):
    n = sino.shape[-1]
    _, _, rmed = O.circus(sino)
    assert np.array_equal(center, rmed), "centre differs from the circus (P2) median index"
    H, M = O.hermite(sino, center, orders)
    err = np.abs(hp - H) / (1e-9 * M + 1e-300)
    assert np.all(err <= 1.0), float(err.max())


@pytest.mark.parametrize("orders", [1, 4, 8])
@pytest.mark.parametrize("kind", [tt.DISK, tt.PHANTOM, tt.SPARSE])
def test_hermite_on_sinogram_rows(ctx, kind, orders):
    n, A = 128, 24
    img = tt.synth_image(kind, n)
    sino, _, rep = tt.TraceTransform(ctx, n, A)(img)
    assert rep.ok()
    hp, center = tt.hermite(ctx, sino, orders)
    assert hp.shape == (A, 6, orders) and center.shape == (A, 6)
    _check_hermite(sino, hp, center, orders)


@pytest.mark.parametrize("n", [1, 2, 33, 1000, 4096])
def test_hermite_edge_lengths_and_centres(ctx, n):
    rng = np.random.default_rng(n)
    rows = rng.random((7, n)).astype(np.float32)
    rows[1] = 0.0                      # S = 0: centre 0, only the upper side
    rows[2, :] = 0.0
    rows[2, -1] = 1.0                  # centre n-1: only the lower side
    rows[3, :] = 0.0
    rows[3, 0] = 1.0                   # centre 0
    hp, center = tt.hermite(ctx, rows, 5)
    _check_hermite(rows, hp, center, 5)


def test_orthonormal_sinogram_pipeline(ctx):
    """Picture -> orthonormal frame -> trace transform (A lines per angle, A angles) -> circus +
    Hermite features: every stage on the device, each checked against the oracle."""
    import torch
    h, w, A = 200, 150, 96
    img = O.synth(O.DISK, 200)[:h, :w].copy()
    d_img = torch.from_numpy(img).cuda()
    frame = torch.empty((A, A), device="cuda")
    tt.orthonormal_device(d_img.data_ptr(), h, w, A, frame.data_ptr())
    torch.cuda.synchronize()
    f = frame.cpu().numpy()
    assert np.array_equal(f.view(np.uint32), O.orthonormal(img, A).view(np.uint32))
    sino, med, rep = tt.TraceTransform(ctx, A, A)(f)
    c, s, wt = tt.make_tables(A, A)
    ref, rmed, _, _ = O.transform(f, A, c, s, wt, mode=O.REPLAY)
    assert np.array_equal(sino.view(np.uint32), ref.view(np.uint32)) and np.array_equal(med, rmed)
    d_sino = torch.from_numpy(sino).cuda()
    hp = torch.empty((A, 6, 3), dtype=torch.float64, device="cuda")
    cen = torch.empty((A, 6), dtype=torch.int32, device="cuda")
    tt.hermite_device(d_sino.data_ptr(), A, A * 6, 3, hp.data_ptr(), cen.data_ptr())
    torch.cuda.synchronize()
    _check_hermite(sino, hp.cpu().numpy(), cen.cpu().numpy(), 3)
