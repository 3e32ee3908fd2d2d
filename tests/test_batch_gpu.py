"""Batched feature extraction (config C4 shape): trace_t05_batch over a stack
of images — every image bit-identical to its own single-image replay, through
the drop-in facade (texture atlas) and the raw device entry (strided LDG)."""
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


def _imgs(B, n):
    kinds = (tt.DISK, tt.PHANTOM, tt.SPARSE)
    return np.stack([tt.synth_image(kinds[b % 3], n, tt.SEEDS[kinds[b % 3]] + b) for b in range(B)])


@pytest.mark.parametrize("sampler", [1, 0], ids=["tex-atlas", "ldg"])
@pytest.mark.parametrize("B,n,A", [(6, 128, 24), (3, 100, 9), (40, 256, 36)])
def test_batch_facade_bit_exact_per_image(ctx, sampler, B, n, A):
    ctx.set_sampler(sampler)
    imgs = _imgs(B, n)
    tr = tt.TraceTransform(ctx, n, A, batch=B)
    out, med, rep = tr(imgs)
    assert rep.ok() and out.shape == (B, A, 6, n)
    for b in range(B):
        ref, rmed, _, _ = O.transform(imgs[b], n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
        assert np.array_equal(out[b].view(np.uint32), ref.view(np.uint32)), b
        assert np.array_equal(med[b], rmed), b
    ctx.set_sampler(1)


def test_batch_raw_strided_and_atlas(ctx):
    B, n, A = 5, 64, 10
    imgs = _imgs(B, n)
    stride = n * n + 37  # padded image stride (LDG path)
    flat = np.zeros(B * stride, np.float32)
    for b in range(B):
        flat[b * stride:b * stride + n * n] = imgs[b].reshape(-1)
    c, s, w = tt.make_tables(n, A)
    d = {k: ctx.mem_alloc(x.nbytes) for k, x in (("img", flat), ("c", c), ("s", s), ("w", w))}
    for k, x in (("img", flat), ("c", c), ("s", s), ("w", w)):
        ctx.memcpy_htod(d[k], x)
    out_d = ctx.mem_alloc(B * A * 6 * n * 4)
    med_d = ctx.mem_alloc(B * A * 2 * n * 4)
    P = {k: ctx.device_pointer(v) for k, v in d.items()}
    for sampler in (0, 1):
        tt.trace_device(P["img"], n, 0, A, P["c"], P["s"], P["w"], ctx.device_pointer(out_d),
                        ctx.device_pointer(med_d), sampler=sampler, stream=ctx.stream, batch=B, img_stride=stride)
        ctx.synchronize()
        out = np.empty((B, A, 6, n), np.float32)
        med = np.empty((B, A, 2, n), np.int32)
        ctx.memcpy_dtoh(out, out_d)
        ctx.memcpy_dtoh(med, med_d)
        for b in range(B):
            ref, rmed, _, _ = O.transform(imgs[b], n, c, s, w, mode=O.REPLAY)
            assert np.array_equal(out[b].view(np.uint32), ref.view(np.uint32)), (sampler, b)
            assert np.array_equal(med[b], rmed)


def test_batch_features_resident(ctx):
    B, n, A = 8, 128, 16
    imgs = _imgs(B, n)
    tr = tt.TraceTransform(ctx, n, A, batch=B, features=True)
    out = np.empty(tr.out_shape(), np.float32)
    circ = np.empty((B, A, 6, 3), np.float32)
    tr.run_resident(imgs, out, None, circ)
    rc, _, _ = O.circus(out)
    assert np.array_equal(circ.view(np.uint32), rc.view(np.uint32))
    for b in (0, B - 1):
        ref, _, _, _ = O.transform(imgs[b], n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
        assert np.array_equal(out[b].view(np.uint32), ref.view(np.uint32))
