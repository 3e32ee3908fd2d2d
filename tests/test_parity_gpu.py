"""Parity of the sm_100a trace kernels with the CPU oracle (spec DESIGN.md §2.5).

Every case is launched through the drop-in path (cuda_launch of the
trace_t05 / radon signatures on a DeviceContext) and checked two ways:
  1. bit-exact (sinograms and median indices) against the oracle's replay of
     the kernel's reduction schedule (TTO_REPLAY);
  2. against the f64 truth within rtol 1e-4 plus the condition-aware floor,
     medians exact except eps-ties (north_star's tolerance).
"""
import numpy as np
import pytest

import oracle as O
import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu

SMALL = [  # (n, A, kind)
    (1, 3, tt.DISK), (2, 4, tt.DISK), (16, 8, tt.DISK), (31, 7, tt.PHANTOM), (33, 5, tt.SPARSE),
    (100, 13, tt.SPARSE), (128, 24, tt.DISK), (255, 9, tt.PHANTOM), (256, 360, tt.DISK),  # C1
    (300, 20, tt.PHANTOM), (512, 16, tt.SPARSE), (1000, 8, tt.DISK), (1001, 6, tt.PHANTOM), (1024, 16, tt.PHANTOM),
    (2047, 3, tt.SPARSE), (3000, 2, tt.DISK),
    (1536, 5, tt.DISK), (2048, 6, tt.SPARSE), (4096, 3, tt.DISK), (8192, 2, tt.PHANTOM), (16384, 1, tt.DISK),
]


@pytest.fixture(scope="module")
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    c.destroy()


def _bitwise_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


def _run(ctx, img, n, A, full=True, sampler=0, a0=0, a_count=None):
    ctx.set_sampler(sampler)
    tr = tt.TraceTransform(ctx, n, A, full=full, a0=a0, a_count=a_count)
    out, med, rep = tr(img)
    assert rep.ok()
    return tr, out, med


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("n,A,kind", SMALL)
def test_fused_t05_bit_exact_vs_replay_and_within_tolerance_of_f64(ctx, n, A, kind, sampler):
    img = tt.synth_image(kind, n)
    tr, out, med = _run(ctx, img, n, A, sampler=sampler)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, rout), "GPU differs bitwise from the replay of its schedule"
    assert np.array_equal(med, rmed)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med)
    assert fails == 0, st


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
@pytest.mark.parametrize("n,A,kind", [(64, 12, tt.DISK), (256, 360, tt.PHANTOM), (777, 5, tt.SPARSE),
                                      (1025, 4, tt.PHANTOM), (2048, 6, tt.PHANTOM), (4096, 2, tt.DISK),
                                      (8192, 2, tt.SPARSE), (20000, 1, tt.DISK)])
def test_radon_t0_bit_exact(ctx, n, A, kind, sampler):
    img = tt.synth_image(kind, n)
    tr, out, _ = _run(ctx, img, n, A, full=False, sampler=sampler)
    rout, _, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY, full=False)
    assert _bitwise_equal(out, rout)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, None, full=False)
    assert fails == 0, st


@pytest.mark.parametrize("sampler", [0, 1, 2], ids=["ldg", "tex", "tma"])
@pytest.mark.parametrize("n,A,full", [(64, 16, True), (300, 12, True), (1028, 8, False)])
def test_non_finite_pixels_stay_local(ctx, n, A, full, sampler):
    """Inf / NaN pixels (one at the corner (0,0), which every out-of-range LDG tap addresses) reach
    only the lines whose in-range taps touch them: every other line is bit-exact against the replay,
    and a line is non-finite exactly where the replay's is (out-of-range taps select +0,
    they never multiply a fetched pixel by 0)."""
    img = tt.synth_image(tt.PHANTOM, n)
    img[0, 0] = np.nan
    img[n // 2, 1] = np.inf
    img[1, n - 2] = -np.inf
    tr, out, med = _run(ctx, img, n, A, full=full, sampler=sampler)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY, full=full)
    F = 6 if full else 1
    out, rout = out.reshape(A, F, n), rout.reshape(A, F, n)
    bad = ~np.isfinite(rout).all(axis=1)  # [A][n] lines with a non-finite functional in the replay
    assert bad.sum() < bad.size // 4, "most lines non-finite: out-of-range taps leak the bad pixels"
    assert np.array_equal(~np.isfinite(out).all(axis=1), bad)
    good = np.broadcast_to(~bad[:, None, :], out.shape)
    assert _bitwise_equal(out[good], rout[good])
    if full:
        mg = np.broadcast_to(~bad[:, None, :], med.shape)
        assert np.array_equal(med[mg], rmed[mg])


def test_radon_equals_t0_of_full_kernel(ctx):
    n, A = 300, 17
    img = tt.synth_image(tt.PHANTOM, n)
    _, full, _ = _run(ctx, img, n, A)
    _, t0, _ = _run(ctx, img, n, A, full=False)
    assert _bitwise_equal(full[:, 0, :], t0[:, 0, :])


def test_dropin_angle_subrange_bit_exact(ctx):
    """A drop-in launch of an angle sub-range (a0, a_count) replays exactly."""
    n, A = 200, 24
    img = tt.synth_image(tt.DISK, n)
    for a0, cnt in [(0, 6), (6, 6), (12, 11), (23, 1)]:
        tr, part, pmed = _run(ctx, img, n, A, a0=a0, a_count=cnt)
        rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, a0=a0, a_count=cnt, mode=O.REPLAY)
        assert _bitwise_equal(part, rout) and np.array_equal(pmed, rmed)


def _raw(ctx, img, n, c, s, w, a0, a_count, pair_stride, full=True, sampler=0):
    """tt_trace_device on context-owned buffers (the multi-GPU driver's entry)."""
    F = 6 if full else 1
    bufs = {k: ctx.mem_alloc(x.nbytes) for k, x in (("img", img), ("c", c), ("s", s), ("w", w))}
    for k, x in (("img", img), ("c", c), ("s", s), ("w", w)):
        ctx.memcpy_htod(bufs[k], np.ascontiguousarray(x))
    out_d = ctx.mem_alloc(a_count * F * n * 4)
    med_d = ctx.mem_alloc(a_count * 2 * n * 4)
    ptr = {k: ctx.device_pointer(v) for k, v in bufs.items()}
    tt.trace_device(ptr["img"], n, a0, a_count, ptr["c"], ptr["s"], ptr["w"], ctx.device_pointer(out_d),
                    ctx.device_pointer(med_d), full=full, sampler=sampler, stream=ctx.stream,
                    pair_stride=pair_stride)
    ctx.synchronize()
    out = np.empty((a_count, F, n), np.float32)
    med = np.empty((a_count, 2, n), np.int32)
    ctx.memcpy_dtoh(out, out_d)
    ctx.memcpy_dtoh(med, med_d)
    for b in list(bufs.values()) + [out_d, med_d]:
        ctx.mem_free(b)
    return out, med


@pytest.mark.parametrize("sampler", [0, 1], ids=["ldg", "tex"])
def test_orientation_shards_with_mirror_halves_are_exact_slices(ctx, sampler):
    """Multi-GPU sharding (row e): rank r of G takes angles [r*A/2G, (r+1)*A/2G)
    plus their mirrors (pair_stride = A/2); the shards are bit-identical to the
    corresponding rows of the single-launch transform."""
    n, A, G = 160, 48, 4
    img = tt.synth_image(tt.PHANTOM, n)
    c, s, w = tt.make_tables(n, A)
    whole, wmed = _raw(ctx, img, n, c, s, w, 0, A, 0, sampler=sampler)
    rout, rmed, _, _ = O.transform(img, n, c, s, w, mode=O.REPLAY)
    assert _bitwise_equal(whole, rout) and np.array_equal(wmed, rmed)
    h = A // 2
    for r in range(G):
        a0, cnt = r * h // G, (r + 1) * h // G - r * h // G
        part, pmed = _raw(ctx, img, n, c, s, w, a0, 2 * cnt, h, sampler=sampler)
        assert _bitwise_equal(part[:cnt], whole[a0:a0 + cnt])
        assert _bitwise_equal(part[cnt:], whole[h + a0:h + a0 + cnt])
        assert np.array_equal(pmed[:cnt], wmed[a0:a0 + cnt]) and np.array_equal(pmed[cnt:], wmed[h + a0:h + a0 + cnt])
        ro, rm = O.replay_launch(img, n, c, s, w, a0=a0, units=cnt, pair_stride=h)
        assert _bitwise_equal(part, ro) and np.array_equal(pmed, rm)


def test_unpaired_raw_launch_matches_unpaired_replay(ctx):
    n, A = 96, 10
    img = tt.synth_image(tt.SPARSE, n)
    c, s, w = tt.make_tables(n, A)
    out, med = _raw(ctx, img, n, c, s, w, 0, A, -1)
    ro, rm = O.replay_launch(img, n, c, s, w, a0=0, units=A, pair_stride=0)
    assert _bitwise_equal(out, ro) and np.array_equal(med, rm)
    fails, st = O.check(img, n, c, s, w, out, med)
    assert fails == 0, st


@pytest.mark.parametrize("n", [64, 255, 512, 700])
def test_clipped_t0_off_grid_and_near_axis_angles(ctx, n):
    """Texture T0 launches sample only the tap range that can lie inside the image
    (clip_range, a superset solved with a 2-pixel margin): off-grid angles, angles a
    few ulps from the axes (direction cosines below the 2^-20 cut-off, and just
    above it) and exact axes must give the replay's bits, which walks every tap."""
    rng = np.random.default_rng(n)
    th = np.concatenate([rng.uniform(0, 2 * np.pi, 10),
                         [0.0, np.pi / 2, np.pi, 1e-7, np.pi / 2 + 3e-7, 2.0 ** -19, 2.0 ** -21, np.pi / 4,
                          -2.0 ** -20 + np.pi]])
    c = np.cos(th).astype(np.float32)
    s = np.sin(th).astype(np.float32)
    _, _, w = tt.make_tables(n, 2)
    img = tt.synth_image(tt.PHANTOM, n) + np.float32(0.25)  # non-zero up to the image border
    out, _ = _raw(ctx, img, n, c, s, w, 0, len(th), -1, full=False, sampler=1)
    ro, _ = O.replay_launch(img, n, c, s, w, a0=0, units=len(th), pair_stride=0, full=False)
    assert _bitwise_equal(out, ro)


@pytest.mark.parametrize("n", [64, 256, 512])
def test_texture_handle_follows_images(ctx, n):
    """A texture handle refreshed from alternating device images (pitch-linear views for n <= 256,
    array copies above) samples whichever image it was last pointed at, and the in-place rewrite of an
    image is seen by the next launch."""
    import torch

    c, s, w = tt.make_tables(n, 8)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    imgs = [d(tt.synth_image(k, n)) for k in (tt.PHANTOM, tt.DISK)]
    ct, st, wt = d(c), d(s), d(w)
    tex = tt.trace.image_texture(imgs[0].data_ptr(), n)
    try:
        for step, k in enumerate([0, 1, 0, 1]):
            if step == 2:
                imgs[0].mul_(0.5)  # rewritten in place between launches
            tt.trace.image_texture_update(tex, imgs[k].data_ptr())
            out = torch.empty((8, 6, n), device="cuda")
            med = torch.empty((8, 2, n), dtype=torch.int32, device="cuda")
            tt.trace_device(imgs[k].data_ptr(), n, 0, 8, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                            med.data_ptr(), sampler=1, tex=tex, pair_stride=-1)
            torch.cuda.synchronize()
            host = imgs[k].cpu().numpy()
            ro, rm = O.replay_launch(host, n, c, s, w, a0=0, units=8, pair_stride=0)
            assert _bitwise_equal(out.cpu().numpy(), ro) and np.array_equal(med.cpu().numpy(), rm), (step, k)
        # an image that is not texture-aligned (4 bytes into a buffer): the handle falls back to an array copy
        buf = torch.zeros(n * n + 1, device="cuda")
        buf[1:].copy_(imgs[1].reshape(-1))
        odd = buf[1:].view(n, n)
        tt.trace.image_texture_update(tex, odd.data_ptr())
        out = torch.empty((8, 6, n), device="cuda")
        med = torch.empty((8, 2, n), dtype=torch.int32, device="cuda")
        tt.trace_device(odd.data_ptr(), n, 0, 8, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                        med.data_ptr(), sampler=1, tex=tex, pair_stride=-1)
        torch.cuda.synchronize()
        ro, rm = O.replay_launch(odd.cpu().numpy(), n, c, s, w, a0=0, units=8, pair_stride=0)
        assert _bitwise_equal(out.cpu().numpy(), ro) and np.array_equal(med.cpu().numpy(), rm), "unaligned"
    finally:
        tt.trace.image_texture_destroy(tex)


def test_zero_image_gives_zero_functionals_and_zero_medians(ctx):
    n, A = 64, 6
    img = np.zeros((n, n), np.float32)
    _, out, med = _run(ctx, img, n, A)
    assert not out.any() and not med.any()


def test_constant_image_ties_are_accepted(ctx):
    n, A = 128, 16
    img = np.ones((n, n), np.float32)
    tr, out, med = _run(ctx, img, n, A)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med)
    assert fails == 0, st


def test_random_dense_image_large_dynamic_range(ctx):
    n, A = 257, 11
    rng = np.random.default_rng(5)
    img = (rng.random((n, n), dtype=np.float32) ** 4 * 1e3).astype(np.float32)
    tr, out, med = _run(ctx, img, n, A)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med)
    assert fails == 0, st


def test_deterministic_across_launches(ctx):
    n, A = 512, 30
    img = tt.synth_image(tt.PHANTOM, n)
    _, a, ma = _run(ctx, img, n, A)
    _, b, mb = _run(ctx, img, n, A)
    assert _bitwise_equal(a, b) and np.array_equal(ma, mb)


@pytest.mark.slow
def test_config2_full_size_1024_720(ctx):
    """C2 (1024^2, 720 angles, T0-T5) at full size: bit-exact vs replay, tolerance vs f64."""
    n, A = 1024, 720
    img = tt.synth_image(tt.DISK, n)
    tr, out, med = _run(ctx, img, n, A)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med)
    assert fails == 0, st


@pytest.mark.slow
def test_config3_4096_1440_angle_subsample(ctx):
    """C3 (4096^2, 1440 angles): full-size lines on a strided subset of angles."""
    n, A = 4096, 1440
    img = tt.synth_image(tt.DISK, n)
    for a0 in (0, 181, 719, 1100):
        tr, out, med = _run(ctx, img, n, A, a0=a0, a_count=2)
        rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, a0=a0, a_count=2, mode=O.REPLAY)
        assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)
        fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med, a0=a0)
        assert fails == 0, st


def test_size_independent_properties_at_8192(ctx):
    """Beyond oracle-friendly sizes: T0 of the angle pair (theta, theta+pi)
    sums the same lines in opposite order, so T0(a, p) ~= T0(a+A/2, n-1-p);
    the medians satisfy m + m(reversed) ~ n-1."""
    n, A = 8192, 4
    img = tt.synth_image(tt.DISK, n)
    _, out, med = _run(ctx, img, n, A)
    t0, t0r = out[0, 0].astype(np.float64), out[2, 0, ::-1].astype(np.float64)
    mask = t0 > 1.0
    assert mask.sum() > n // 2
    assert np.max(np.abs(t0[mask] - t0r[mask]) / t0[mask]) < 1e-3
    assert np.all(out[:, 1:] >= 0)


def test_texture_cache_follows_image_rewrites(ctx):
    """The texture sampler caches a block-linear copy per image allocation; every
    write to the allocation (H2D copy, a kernel storing into it) must refresh it."""
    n, A = 128, 8
    ctx.set_sampler(1)
    tr = tt.TraceTransform(ctx, n, A)
    out = np.empty(tr.out_shape(), np.float32)
    med = np.empty((A, 2, n), np.int32)
    imgs = [tt.synth_image(k, n) for k in (tt.DISK, tt.PHANTOM, tt.SPARSE)]
    for img in imgs + imgs[:1]:
        tr.run_resident(img, out, med)
        ref, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
        assert _bitwise_equal(out, ref) and np.array_equal(med, rmed)
    # a native kernel writing into the image buffer (scale by 2) also invalidates the copy
    img = imgs[1]
    tr.run_resident(img, out, med)
    mod = ctx.module_load(tt.render_module(tt.KernelAst("scale", ["a", "k"]), [(True, "f32"), (False, "f32")], "s"))
    fn = ctx.get_function(mod, "scale")
    r = tr._resident()
    flat = tt.GridConfig((1, 1, 1), (1, 1, 1))
    ctx.memcpy_htod(r["img"], (img * np.float32(2.0)).astype(np.float32))
    tr.launch_resident()
    ctx.memcpy_dtoh(out, r["out"])
    ref, _, _, _ = O.transform((img * np.float32(2.0)).astype(np.float32), n, tr.ctab, tr.stab, tr.wtab,
                               mode=O.REPLAY)
    assert _bitwise_equal(out, ref)
    assert ctx.launch(fn, flat, [r["img"], np.float32(0.5)]).ok()  # kernel write -> generation bump
    tr.launch_resident()
    ctx.memcpy_dtoh(out, r["out"])
    img2 = (img * np.float32(2.0)).astype(np.float32)
    img2.reshape(-1)[0] = img2.reshape(-1)[0] * np.float32(0.5)
    ref, _, _, _ = O.transform(img2, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, ref)
    ctx.set_sampler(0)


def test_tiny_and_denormal_values_exact(ctx):
    """sqrt of zero / denormal / tiny samples (the kernel's exact fast sqrt path)."""
    n, A = 64, 6
    img = (tt.synth_image(tt.DISK, n) * np.float32(1e-38)).astype(np.float32)
    for sampler in (0, 1):
        tr, out, med = _run(ctx, img, n, A, sampler=sampler)
        rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
        assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)


@pytest.mark.parametrize("n,A", [(256, 6), (1024, 4), (2048, 2)])
def test_mixed_magnitude_values_exact(ctx, n, A):
    """Pixels spanning denormals to 1e25 in one image: tap pairs whose square roots take
    different (scaled / unscaled) paths inside one packed sqrt2_rn, on each schedule."""
    rng = np.random.default_rng(n)
    expo = rng.uniform(-44.0, 25.0, size=(n, n))
    img = (tt.synth_image(tt.DISK, n).astype(np.float64) * 10.0 ** expo).astype(np.float32)
    img[rng.random((n, n)) < 0.05] = 0.0
    tr, out, med = _run(ctx, img, n, A, sampler=1)
    ctx.set_sampler(0)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
    assert _bitwise_equal(out, rout) and np.array_equal(med, rmed)


@pytest.mark.parametrize("n,A", [(256, 12), (1000, 6), (1024, 8)])
def test_prepared_weight_layout_equals_per_call_conversion(ctx, n, A):
    """tt_weights_soa + tt_trace_desc.wsoa gives the same bits as the per-call conversion."""
    img = tt.synth_image(tt.PHANTOM, n)
    c, s, w = tt.make_tables(n, A)
    ref, rmed = _raw(ctx, img, n, c, s, w, 0, A, 0)
    bufs = {k: ctx.mem_alloc(x.nbytes) for k, x in (("img", img), ("c", c), ("s", s), ("w", w))}
    for k, x in (("img", img), ("c", c), ("s", s), ("w", w)):
        ctx.memcpy_htod(bufs[k], np.ascontiguousarray(x))
    ws = ctx.mem_alloc(24 * n)
    out_d, med_d = ctx.mem_alloc(A * 6 * n * 4), ctx.mem_alloc(A * 2 * n * 4)
    ptr = {k: ctx.device_pointer(v) for k, v in bufs.items()}
    tt.weights_soa(ptr["w"], n, ctx.device_pointer(ws), ctx.stream)
    for _ in range(2):  # reused across launches
        tt.trace_device(ptr["img"], n, 0, A, ptr["c"], ptr["s"], ptr["w"], ctx.device_pointer(out_d),
                        ctx.device_pointer(med_d), stream=ctx.stream, wsoa_ptr=ctx.device_pointer(ws))
    ctx.synchronize()
    out = np.empty((A, 6, n), np.float32)
    med = np.empty((A, 2, n), np.int32)
    ctx.memcpy_dtoh(out, out_d)
    ctx.memcpy_dtoh(med, med_d)
    for b in list(bufs.values()) + [ws, out_d, med_d]:
        ctx.mem_free(b)
    assert _bitwise_equal(out, ref) and np.array_equal(med, rmed)


def _random_configs(count=24, seed=20260417):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.choice([int(rng.integers(2, 700)), int(2 ** rng.integers(3, 11))]))
        A = int(rng.integers(1, 40))
        a0 = int(rng.integers(0, A))
        cnt = int(rng.integers(1, A - a0 + 1))
        out.append((n, A, a0, cnt, int(rng.integers(0, 3)), int(rng.integers(0, 2)), bool(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("n,A,a0,cnt,kind,sampler,full", _random_configs())
def test_random_configurations_bit_exact_vs_replay(ctx, n, A, a0, cnt, kind, sampler, full):
    """Seeded random sizes / angle ranges / images / samplers / functional sets."""
    img = tt.synth_image([tt.DISK, tt.PHANTOM, tt.SPARSE][kind], n)
    tr, out, med = _run(ctx, img, n, A, full=full, sampler=sampler, a0=a0, a_count=cnt)
    rout, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, a0=a0, a_count=cnt, mode=O.REPLAY, full=full)
    assert _bitwise_equal(out, rout)
    if full:
        assert np.array_equal(med, rmed)
    fails, st = O.check(img, n, tr.ctab, tr.stab, tr.wtab, out, med if full else None, a0=a0, full=full)
    assert fails == 0, st
