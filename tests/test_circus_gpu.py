"""P-functionals / circus stage: bit-exact vs the oracle's
replay of the one-warp schedule; P1/P3 within tolerance of the f64 truth and
P2 taken at an eps-median of the f64 prefix."""
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


def _check_against_truth(sino, circ):
    rc, r64, rm = O.circus(sino)
    assert np.array_equal(circ.view(np.uint32), rc.view(np.uint32)), "differs bitwise from the replay"
    n = sino.shape[-1]
    chain = (n + 31) // 32 + 10
    eps = 2 * chain * 2.0 ** -24
    p1_err = np.abs(circ[..., 0] - r64[..., 0]) / (1e-4 * np.abs(r64[..., 0]) + 1e-30 + eps * r64[..., 0])
    assert np.all(p1_err <= 1.0)
    assert np.array_equal(circ[..., 2], r64[..., 2].astype(np.float32))
    # P2 = s[m] at the replayed (== GPU) median index m, which must be an eps-median of the f64 prefix
    rows = sino.reshape(-1, n).astype(np.float64)
    m = rm.reshape(-1).astype(np.int64)
    P = np.cumsum(rows, axis=1)
    S = P[:, -1]
    Pm = np.take_along_axis(P, m[:, None], 1)[:, 0]
    Pprev = np.where(m > 0, np.take_along_axis(P, np.maximum(m - 1, 0)[:, None], 1)[:, 0], 0.0)
    ok = np.where(S > 0, (2 * Pm >= S * (1 - eps)) & ((m == 0) | (2 * Pprev < S * (1 + eps))), m == 0)
    assert ok.all()
    assert np.array_equal(circ.reshape(-1, 3)[:, 1], sino.reshape(-1, n)[np.arange(m.size), m])


@pytest.mark.parametrize("n,A,kind", [(64, 10, tt.DISK), (256, 360, tt.PHANTOM), (1000, 8, tt.SPARSE),
                                      (1024, 24, tt.DISK)])
def test_circus_of_trace_output(ctx, n, A, kind):
    img = tt.synth_image(kind, n)
    tr = tt.TraceTransform(ctx, n, A)
    sino, _, _ = tr(img)
    circ = tt.circus(ctx, sino)
    assert circ.shape == (A, 6, 3)
    _check_against_truth(sino, circ)


def test_circus_edge_rows(ctx):
    rng = np.random.default_rng(3)
    sino = np.stack([np.zeros(77), np.ones(77), rng.random(77) ** 8, np.eye(1, 77, 76)[0], np.eye(1, 77, 0)[0]])
    circ = tt.circus(ctx, sino.astype(np.float32))
    _check_against_truth(sino.astype(np.float32), circ)


def test_resident_flow_with_features(ctx):
    n, A = 512, 40
    img = tt.synth_image(tt.PHANTOM, n)
    tr = tt.TraceTransform(ctx, n, A, features=True)
    out = np.empty(tr.out_shape(), np.float32)
    med = np.empty((A, 2, n), np.int32)
    circ = np.empty((A, 6, 3), np.float32)
    tr.run_resident(img, out, med, circ)
    ref, _, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
    rc, _, _ = O.circus(out)
    assert np.array_equal(circ.view(np.uint32), rc.view(np.uint32))


@pytest.mark.parametrize("fused", [0, 1], ids=["separate", "fused"])
@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("n,A,batch,pair", [(64, 10, 1, 0), (128, 9, 1, 0), (256, 12, 3, 0), (1024, 8, 1, 0),
                                            (1000, 6, 1, 0), (2048, 4, 1, 0), (4096, 2, 1, 0), (256, 16, 1, 8),
                                            (256, 16, 1, 4)])
def test_trace_circus_output_equals_separate_stage(gpu, n, A, batch, pair, sampler, fused):
    """tt_trace_desc.circ: the P stage of a raw trace launch -- a separate circus launch on the same
    stream, or with TT_TRACE_FUSED_P (texture sampler) P-CTAs appended to the trace launch (warp per row,
    waiting on per-unit line counters) -- bit-identical to tt_circus_device over the same rows, and to the
    oracle's replay; covers sub-warp segments, W > 1 warps per line, batches, unpaired units and
    explicit mirror-half shards."""
    import torch
    c, s, w = tt.make_tables(n, A)
    imgs = np.stack([tt.synth_image(tt.PHANTOM, n, 7 + b) for b in range(batch)])
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    img, ct, st, wt = dev(imgs), dev(c), dev(s), dev(w)
    a_count = A if pair == 0 else 2 * (A // 4)
    out = torch.empty((batch, a_count, 6, n), device="cuda")
    med = torch.empty((batch, a_count, 2, n), dtype=torch.int32, device="cuda")
    circ = torch.full((batch, a_count, 6, 3), float("nan"), device="cuda")
    tex = None
    if sampler == 1:
        tex = tt.trace.image_atlas(img.data_ptr(), n, batch) if batch > 1 else tt.trace.image_texture(img.data_ptr(), n)
    for _ in range(2):  # the per-unit counters reset themselves: a second launch must work the same
        tt.trace_device(img.data_ptr(), n, 0, a_count, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                        med.data_ptr(), sampler=sampler, tex=tex, batch=batch, pair_stride=pair,
                        circ_ptr=circ.data_ptr(), fused_p=bool(fused))
    ref = torch.empty_like(circ)
    tt.circus_device(out.data_ptr(), n, batch * a_count * 6, ref.data_ptr())
    torch.cuda.synchronize()
    if tex is not None:
        tt.trace.image_texture_destroy(tex)
    got = circ.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.cpu().numpy().view(np.uint32))
    _check_against_truth(out.cpu().numpy(), got)
