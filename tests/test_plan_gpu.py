"""Pipelined host-to-host plans (tt_plan_*): chunked launches with overlapped
downloads must reproduce the single-launch drop-in path bit-for-bit."""
import numpy as np
import pytest

import paper_1604_03410_b200 as tt
from paper_1604_03410_b200.trace import NF

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    c.destroy()


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("n,A,full,chunks", [(256, 360, True, 0), (256, 360, True, 7), (1000, 12, True, 5),
                                             (128, 9, True, 3), (64, 10, False, 4), (1024, 16, True, 8)])
def test_plan_equals_one_launch(ctx, n, A, full, chunks, sampler):
    ctx.set_sampler(sampler)
    img = tt.synth_image(tt.PHANTOM, n)
    ref_out, ref_med, rep = tt.TraceTransform(ctx, n, A, full=full)(img)
    assert rep.ok()
    plan = tt.Plan(ctx, n, A, full=full, features=full, chunks=chunks)
    F = NF if full else 1
    out = np.full((A, F, n), np.nan, np.float32)
    med = np.full((A, 2, n), -7, np.int32) if full else None
    circ = np.zeros((A, NF, 3), np.float32) if full else None
    for _ in range(2):  # reusable
        plan.run(img, out, med, circ)
    assert np.array_equal(_bits(out), _bits(ref_out))
    if full:
        assert np.array_equal(med, ref_med)
        assert np.array_equal(_bits(circ), _bits(tt.circus(ctx, ref_out)))
    plan.destroy()


def test_plan_angle_range_and_partial_outputs(ctx):
    n, A, a0, cnt = 256, 40, 6, 20
    img = tt.synth_image(tt.DISK, n)
    ref_out, ref_med, _ = tt.TraceTransform(ctx, n, A, a0=a0, a_count=cnt)(img)
    plan = tt.Plan(ctx, n, A, a0=a0, a_count=cnt, chunks=3)
    out = np.empty((cnt, NF, n), np.float32)
    plan.run(img, out)  # medians and features not requested
    assert np.array_equal(_bits(out), _bits(ref_out))
    plan.destroy()


@pytest.mark.parametrize("world,rank", [(2, 0), (2, 1), (4, 3), (3, 1)])
def test_plan_mirror_half_shard_equals_rows_of_the_whole(ctx, world, rank):
    """An orientation shard with its mirror half (pair_stride = A/2): rows [cnt] + [cnt] equal the
    corresponding rows (a0.., A/2+a0..) of the whole transform, bit for bit."""
    from paper_1604_03410_b200 import shard
    ctx.set_sampler(1)
    n, A = 256, 40
    img = tt.synth_image(tt.PHANTOM, n)
    whole, wmed, _ = tt.TraceTransform(ctx, n, A)(img)
    a0, cnt, h = shard.orientation_shard(A, world, rank)
    plan = tt.Plan(ctx, n, A, a0=a0, a_count=2 * cnt, pair_stride=h, chunks=3)
    out = np.full((2 * cnt, NF, n), np.nan, np.float32)
    med = np.full((2 * cnt, 2, n), -1, np.int32)
    plan.run(img, out, med)
    rows = shard.shard_rows(A, world, rank)
    assert np.array_equal(_bits(out), _bits(whole[rows])) and np.array_equal(med, wmed[rows])
    plan.destroy()
    with pytest.raises(tt.Error):  # odd a_count / partner angles outside the grid
        tt.Plan(ctx, n, A, a0=a0, a_count=3, pair_stride=h)
    with pytest.raises(tt.Error):
        tt.Plan(ctx, n, A, a0=h, a_count=2 * cnt, pair_stride=h)


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("chunks", [0, 2, 3])
def test_plan_batched_features(ctx, chunks, sampler):
    ctx.set_sampler(sampler)
    n, A, B = 128, 12, 3
    imgs = np.stack([tt.synth_image(tt.DISK, n, tt.SEEDS[tt.DISK] + b) for b in range(B)])
    plan = tt.Plan(ctx, n, A, features=True, batch=B, chunks=chunks)
    out = np.empty((B, A, NF, n), np.float32)
    med = np.empty((B, A, 2, n), np.int32)
    circ = np.empty((B, A, NF, 3), np.float32)
    plan.run(imgs, out, med, circ)
    for b in range(B):
        ro, rm, _ = tt.TraceTransform(ctx, n, A)(imgs[b])
        assert np.array_equal(_bits(out[b]), _bits(ro)) and np.array_equal(med[b], rm)
        assert np.array_equal(_bits(circ[b]), _bits(tt.circus(ctx, ro)))
    plan.destroy()


def test_plan_counts_bytes_and_launches(ctx):
    n, A = 256, 24
    plan = tt.Plan(ctx, n, A, chunks=4)
    c0 = ctx.counters()
    out = np.empty((A, NF, n), np.float32)
    plan.run(tt.synth_image(tt.DISK, n), out)
    c1 = ctx.counters()
    assert c1["bytes_h2d"] - c0["bytes_h2d"] == n * n * 4
    assert c1["bytes_d2h"] - c0["bytes_d2h"] == out.nbytes
    assert c1["gpu_kernel_launches"] - c0["gpu_kernel_launches"] == plan.chunks == 4
    plan.destroy()


def test_plan_rejects_bad_descriptors(ctx):
    with pytest.raises(Exception):
        tt.Plan(ctx, 0, 10)
    with pytest.raises(Exception):
        tt.Plan(ctx, 64, 10, a0=5, a_count=10)
    with pytest.raises(Exception):
        tt.Plan(ctx, 64, 0)


def test_plan_validates_host_arrays_and_closes(ctx):
    n, A = 64, 8
    img = tt.synth_image(tt.DISK, n)
    with tt.Plan(ctx, n, A) as plan:
        with pytest.raises(ValueError):
            plan.run(img, np.empty((A, NF, n - 1), np.float32))       # wrong size
        with pytest.raises(ValueError):
            plan.run(img, np.empty((A, NF, n), np.float64))           # wrong dtype
        with pytest.raises(ValueError):
            plan.run(img[:, :-1].copy())                              # wrong image size
        out = np.empty((A, NF, n), np.float32)
        plan.run(img, out)
    assert not plan._p
    with pytest.raises(ValueError):
        plan.run(img, out)                                            # destroyed


@pytest.mark.parametrize("slots", [1, 2, 3])
def test_overlapping_submissions_equal_separate_runs(ctx, slots):
    n, A = 256, 48
    imgs = [tt.synth_image(k, n) for k in (tt.DISK, tt.PHANTOM, tt.SPARSE, tt.DISK)]
    plan = tt.Plan(ctx, n, A, features=True, chunks=3, slots=slots)
    refs = []
    for img in imgs:
        o, m, c = np.empty((A, NF, n), np.float32), np.empty((A, 2, n), np.int32), np.empty((A, NF, 3), np.float32)
        plan.run(img, o, m, c)
        refs.append((o, m, c))
    outs = [(np.full((A, NF, n), np.nan, np.float32), np.zeros((A, 2, n), np.int32), np.zeros((A, NF, 3), np.float32))
            for _ in imgs]
    for img, (o, m, c) in zip(imgs, outs):
        plan.submit(img, o, m, c)
    plan.wait()
    for (o, m, c), (ro, rm, rc) in zip(outs, refs):
        assert np.array_equal(_bits(o), _bits(ro)) and np.array_equal(m, rm) and np.array_equal(_bits(c), _bits(rc))
    plan.destroy()


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("n,A,batch,chunks", [(256, 360, 1, 0), (256, 40, 1, 3), (128, 12, 3, 2)])
def test_graph_plan_replays_the_captured_submission(ctx, sampler, n, A, batch, chunks):
    """tt_plan_desc.graph: the first submission per slot and host-buffer set is captured into a CUDA
    graph and later ones replay it (the steady state: one input buffer refilled per image, the
    output buffers alternating with the two slots); outputs (sinograms, medians, fused circus)
    equal the enqueued plan's bit for bit, new host buffers re-capture, counters advance per
    submission."""
    ctx.set_sampler(sampler)
    imgs = [np.stack([tt.synth_image(kind, n, 3 + k + b) for b in range(batch)]) for k, kind in
            enumerate((tt.PHANTOM, tt.DISK, tt.SPARSE, tt.PHANTOM))]
    if batch == 1:
        imgs = [im[0] for im in imgs]
    ref_plan = tt.Plan(ctx, n, A, features=True, batch=batch, chunks=chunks)
    gplan = tt.Plan(ctx, n, A, features=True, batch=batch, chunks=chunks, graph=True, slots=2)
    shape = ((batch,) if batch > 1 else ()) + (A,)
    bufs = [(np.zeros(shape + (NF, n), np.float32), np.zeros(shape + (2, n), np.int32),
             np.zeros(shape + (NF, 3), np.float32)) for _ in range(2)]
    h_img = np.empty_like(imgs[0])
    for j in range(8):
        h_img[...] = imgs[j % len(imgs)]
        o, m, c = bufs[j % 2]
        c0 = ctx.counters()
        gplan.run(h_img, o, m, c)
        c1 = ctx.counters()
        ro, rm, rc = (np.empty_like(x) for x in (o, m, c))
        ref_plan.run(h_img, ro, rm, rc)
        assert np.array_equal(_bits(o), _bits(ro)) and np.array_equal(m, rm) and np.array_equal(_bits(c), _bits(rc))
        assert c1["bytes_h2d"] - c0["bytes_h2d"] == h_img.nbytes
        assert c1["bytes_d2h"] - c0["bytes_d2h"] == o.nbytes + m.nbytes + c.nbytes
    assert gplan.captures == 2  # one per slot; the other six submissions replayed
    other = np.empty_like(bufs[0][0])
    gplan.run(h_img, other)  # a different buffer set re-captures
    assert gplan.captures == 3 and np.array_equal(_bits(other), _bits(bufs[1][0]))
    gplan.destroy()
    ref_plan.destroy()
