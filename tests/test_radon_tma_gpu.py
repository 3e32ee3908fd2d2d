"""T0 (Radon) through TMA-staged shared-memory tiles (sampler 2).

The tile kernel keeps the texture kernel's per-tap arithmetic, slot order and
butterfly, so its sinogram must equal the texture path's bit for bit, and the
oracle's replay of the NS = 32 schedule (TTO_REPLAY); launches it does not
serve (T0-T5, n <= 704, n % 4 != 0) fall back to the texture gather.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu


def _bitwise_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


def _raw(img, n, a0, a_count, A_total, sampler, pair_stride=0, partner_row=0, full=False):
    c, s, w = tt.make_tables(n, A_total)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    d_img, ct, st, wt = dev(img), dev(c), dev(s), dev(w)
    F = 6 if full else 1
    out = torch.full((a_count, F, n), float("nan"), device="cuda")
    med = torch.empty((a_count, 2, n), dtype=torch.int32, device="cuda") if full else None
    tt.trace_device(d_img.data_ptr(), n, a0, a_count, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                    med.data_ptr() if full else 0, full=full, sampler=sampler, pair_stride=pair_stride,
                    partner_row=partner_row)
    torch.cuda.synchronize()
    return out.cpu().numpy(), c, s, w


@pytest.mark.parametrize("n,A,kind", [(516, 6, tt.PHANTOM), (1000, 8, tt.DISK), (1024, 12, tt.SPARSE),
                                      (1028, 6, tt.DISK), (2048, 8, tt.PHANTOM), (3000, 4, tt.SPARSE),
                                      (4096, 6, tt.DISK), (4100, 3, tt.PHANTOM), (8192, 2, tt.DISK), (20000, 2, tt.DISK)])
def test_tma_radon_equals_texture_and_replay(gpu, n, A, kind):
    img = tt.synth_image(kind, n)
    got, c, s, w = _raw(img, n, 0, A, A, sampler=2)
    tex, _, _, _ = _raw(img, n, 0, A, A, sampler=1)
    assert _bitwise_equal(got, tex), "TMA tiles differ from the texture gather"
    rout, _, _, _ = O.transform(img, n, c, s, w, mode=O.REPLAY, full=False)
    assert _bitwise_equal(got, rout)
    fails, st = O.check(img, n, c, s, w, got, None, full=False)
    assert fails == 0, st


@pytest.mark.parametrize("A", [72, 360, 1440])
def test_tma_radon_every_angle_class(gpu, A):
    """Full angle grids (every pitch choice and tile shape), n = 2048: bit-identical to the texture path."""
    n = 2048
    img = tt.synth_image(tt.PHANTOM, n)
    got, _, _, _ = _raw(img, n, 0, A, A, sampler=2)
    tex, _, _, _ = _raw(img, n, 0, A, A, sampler=1)
    assert _bitwise_equal(got, tex)


def test_tma_radon_orientation_shard_and_unpaired(gpu):
    """An orientation shard with its mirror half (pair_stride = A/2, partner_row) and an unpaired odd
    launch (no mirror sharing) -- both bit-identical to the texture path."""
    n, A = 2048, 48
    img = tt.synth_image(tt.DISK, n)
    got, _, _, _ = _raw(img, n, 5, 8, A, sampler=2, pair_stride=A // 2)
    tex, _, _, _ = _raw(img, n, 5, 8, A, sampler=1, pair_stride=A // 2)
    assert _bitwise_equal(got, tex)
    got, _, _, _ = _raw(img, n, 3, 7, A, sampler=2)
    tex, _, _, _ = _raw(img, n, 3, 7, A, sampler=1)
    assert _bitwise_equal(got, tex)


def test_tma_radon_unmirrored_partner(gpu):
    """Tables whose partner angle is not the exact negation: the tile kernel samples the partner in a
    second pass (as the texture kernel does)."""
    n, A = 1536, 8
    img = tt.synth_image(tt.SPARSE, n)
    c, s, w = tt.make_tables(n, A)
    c2, s2 = c.copy(), s.copy()
    c2[A // 2:] = np.nextafter(c2[A // 2:], np.float32(2))  # break the bitwise mirror
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    d_img, ct, st, wt = dev(img), dev(c2), dev(s2), dev(w)
    outs = []
    for smp in (2, 1):
        out = torch.full((A, 1, n), float("nan"), device="cuda")
        tt.trace_device(d_img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(), 0,
                        full=False, sampler=smp)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert _bitwise_equal(outs[0], outs[1])
    rout, _, _, _ = O.transform(img, n, c2, s2, w, mode=O.REPLAY, full=False)
    assert _bitwise_equal(outs[0], rout)


@pytest.mark.parametrize("n,full", [(512, False), (704, False), (1030, False), (2048, True)])
def test_tma_sampler_falls_back_to_texture(gpu, n, full):
    """Launches the tile kernel does not serve run the texture gather (same bits as sampler 1)."""
    A = 4
    img = tt.synth_image(tt.PHANTOM, n)
    got, _, _, _ = _raw(img, n, 0, A, A, sampler=2, full=full)
    tex, _, _, _ = _raw(img, n, 0, A, A, sampler=1, full=full)
    assert _bitwise_equal(got, tex)


def test_tma_context_sampler(gpu):
    """The drop-in flow (cuda_launch of radon on a DeviceContext) with sampler 2."""
    n, A = 2048, 6
    img = tt.synth_image(tt.DISK, n)
    ctx = tt.create_context(gpu)
    try:
        ctx.set_sampler(2)
        tr = tt.TraceTransform(ctx, n, A, full=False)
        out, _, rep = tr(img)
        assert rep.ok()
        rout, _, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY, full=False)
        assert _bitwise_equal(out, rout)
    finally:
        ctx.destroy()
