"""The DeviceContext contract of /root/reference/proj/tests/test_driver.cpp,
re-run against the CUDA-backed context (native sm_100a kernels, pooled HBM).
Test names follow the reference's TEST_CASEs."""
import json

import numpy as np
import pytest

import paper_1604_03410_b200 as tt
from paper_1604_03410_b200 import GridConfig

pytestmark = pytest.mark.gpu

VADD_F32 = tt.render_module(tt.KernelAst("vadd", ["a", "b", "c"]), [(True, "f32")] * 3, "vadd$9e81eb78751b412a")


@pytest.fixture
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    if not c.destroyed():
        c.destroy()


def test_fresh_context_has_zeroed_counters(ctx):  # test_driver.cpp:35-46
    c = ctx.counters()
    for k in ("modules_loaded", "functions_resolved", "launches", "allocs", "frees", "bytes_h2d", "bytes_d2h"):
        assert c[k] == 0
    assert c["launch_log"] == []


def test_context_destruction_poisons_the_handle(ctx):  # :48-56
    p = ctx.mem_alloc(16)
    ctx.destroy()
    with pytest.raises(tt.ContextDestroyed):
        ctx.destroy()
    with pytest.raises(tt.ContextDestroyed):
        ctx.mem_free(p)
    with pytest.raises(tt.ContextDestroyed):
        ctx.mem_alloc(4)
    with pytest.raises(tt.ContextDestroyed):
        ctx.module_load(".module m\n")


def test_module_loading(ctx):  # :58-83
    h1 = ctx.module_load(VADD_F32)
    h2 = ctx.module_load(VADD_F32)
    assert h1 != h2
    assert ctx.counters()["modules_loaded"] == 2
    with pytest.raises(tt.VptxSyntaxError):
        ctx.module_load("not a module")
    assert ctx.counters()["modules_loaded"] == 2
    with pytest.raises(tt.ValidationFailed):
        ctx.module_load(".module m\n.kernel k() {\n}\n.kernel k() {\n}\n")
    assert ctx.counters()["modules_loaded"] == 2


def test_function_resolution(ctx):  # :85-117
    md = ctx.module_load(VADD_F32)
    f1 = ctx.get_function(md, "vadd")
    f2 = ctx.get_function(md, "vadd")
    assert f1 != f2
    assert ctx.counters()["functions_resolved"] == 2
    with pytest.raises(tt.FunctionNotFound):
        ctx.get_function(md, "nosuch")
    cfg = GridConfig((4, 1, 1))
    ga, gb, gc1, gc2 = (ctx.mem_alloc(16) for _ in range(4))
    ctx.memcpy_htod(ga, np.array([1, 2, 3, 4], np.float32))
    ctx.memcpy_htod(gb, np.array([5, 6, 7, 8], np.float32))
    assert ctx.launch(f1, cfg, [ga, gb, gc1]).ok()
    assert ctx.launch(f2, cfg, [ga, gb, gc2]).ok()
    c1, c2 = np.zeros(4, np.float32), np.zeros(4, np.float32)
    ctx.memcpy_dtoh(c1, gc1)
    ctx.memcpy_dtoh(c2, gc2)
    assert np.array_equal(c1, c2) and list(c1) == [6, 8, 10, 12]
    ctx.module_unload(md)
    with pytest.raises(tt.FunctionNotFound):
        ctx.launch(f1, GridConfig(), [])


def test_memory_transfer_accounting_is_exact(ctx):  # :119-157
    p = ctx.mem_alloc(48)
    assert ctx.counters()["allocs"] == 1
    host = np.full(12, 1.5, np.float32)
    ctx.memcpy_htod(p, host, 48)
    assert ctx.counters()["bytes_h2d"] == 48
    back = np.zeros(12, np.float32)
    ctx.memcpy_dtoh(back, p, 48)
    assert ctx.counters()["bytes_d2h"] == 48 and np.array_equal(back, host)
    big = np.zeros(13, np.float32)
    with pytest.raises(tt.OutOfBounds):
        ctx.memcpy_htod(p, big, 49)
    assert ctx.counters()["bytes_h2d"] == 48
    with pytest.raises(tt.OutOfBounds):
        ctx.memcpy_dtoh(big, p, 52)
    assert ctx.counters()["bytes_d2h"] == 48
    z1, z2 = ctx.mem_alloc(0), ctx.mem_alloc(0)
    assert z1.base != 0 and z2.base != 0 and z1.base != z2.base and z1.length == 0
    other = tt.create_context()
    foreign = other.mem_alloc(16)
    with pytest.raises(tt.ArgumentMismatch):
        ctx.memcpy_htod(foreign, host, 4)
    other.destroy()
    ctx.mem_free(p)
    assert ctx.counters()["frees"] == 1
    with pytest.raises(tt.DoubleFree):
        ctx.mem_free(p)
    with pytest.raises(tt.UseAfterFree):
        ctx.memcpy_htod(p, host, 4)
    with pytest.raises(tt.UseAfterFree):
        ctx.memcpy_dtoh(back, p, 4)


def test_allocations_are_zero_filled_even_when_pool_memory_is_recycled(ctx):
    for _ in range(3):
        p = ctx.mem_alloc(1 << 20)
        h = np.full(1 << 18, 7.0, np.float32)
        ctx.memcpy_htod(p, h)
        ctx.mem_free(p)
    q = ctx.mem_alloc(1 << 20)
    got = np.ones(1 << 18, np.float32)
    ctx.memcpy_dtoh(got, q)
    assert not got.any()


def test_addresses_are_never_reused(ctx):
    bases = set()
    for _ in range(50):
        p = ctx.mem_alloc(100)
        assert p.base not in bases and p.base % 256 == 0 and p.base >= 4096
        bases.add(p.base)
        ctx.mem_free(p)


def test_multi_kernel_modules_resolve_each_kernel_independently(ctx):  # :159-184
    text = (".module pair\n"
            ".kernel vadd(.param ptr.global.i32 a, .param ptr.global.i32 b, .param ptr.global.i32 c) {\n  ret\n}\n"
            ".kernel scale(.param ptr.global.f32 a, .param f32 k) {\n  ret\n}\n"
            ".kernel first(.param ptr.global.i32 out) {\n  ret\n}\n")
    md = ctx.module_load(text)
    fv = ctx.get_function(md, "vadd")
    fs = ctx.get_function(md, "scale")
    with pytest.raises(tt.FunctionNotFound):  # no native implementation: never a CPU fallback
        ctx.get_function(md, "first")
    a = ctx.mem_alloc(8)
    ctx.memcpy_htod(a, np.array([11, 20], np.int32))
    assert ctx.launch(fv, GridConfig((2, 1, 1)), [a, a, a]).ok()
    v = np.zeros(2, np.int32)
    ctx.memcpy_dtoh(v, a)
    assert list(v) == [22, 40]
    f = ctx.mem_alloc(8)
    ctx.memcpy_htod(f, np.array([1.5, -2.0], np.float32))
    assert ctx.launch(fs, GridConfig((1, 1, 1), (2, 1, 1)), [f, np.float32(3.0)]).ok()
    w = np.zeros(2, np.float32)
    ctx.memcpy_dtoh(w, f)
    assert list(w) == [4.5, -6.0]


def test_stale_and_foreign_handles_are_rejected(ctx):  # :186-206
    md = ctx.module_load(VADD_F32)
    fn = ctx.get_function(md, "vadd")
    other = tt.create_context()
    with pytest.raises(tt.ArgumentMismatch):
        other.get_function(md, "vadd")
    other.destroy()
    p = ctx.mem_alloc(4)
    ctx.mem_free(p)
    with pytest.raises(tt.UseAfterFree):
        ctx.launch(fn, GridConfig(), [p, p, p])
    ctx.module_unload(md)
    with pytest.raises(tt.ArgumentMismatch):
        ctx.get_function(md, "vadd")


def test_launch_argument_checking(ctx):  # :208-227
    md = ctx.module_load(VADD_F32)
    fn = ctx.get_function(md, "vadd")
    p = ctx.mem_alloc(4)
    with pytest.raises(tt.ArgumentMismatch):
        ctx.launch(fn, GridConfig(), [p, p])
    with pytest.raises(tt.ArgumentMismatch):
        ctx.launch(fn, GridConfig(), [p, p, np.float32(1.5)])
    with pytest.raises(tt.LaunchConfigError):
        ctx.launch(fn, GridConfig((0, 1, 1)), [p, p, p])
    with pytest.raises(tt.LaunchConfigError):
        ctx.launch(fn, GridConfig((1, 1, 1), (2048, 1, 1)), [p, p, p])
    assert ctx.counters()["launches"] == 0
    r = ctx.launch(fn, GridConfig((2, 1, 1)), [p, p, p])  # index 2 in a one-element array
    assert not r.ok()
    assert r.trap.kind == tt.api.TrapKind.GlobalOutOfBounds
    c = ctx.counters()
    assert c["launches"] == 1 and len(c["launch_log"]) == 1 and c["launch_log"][0]["kernel"] == "vadd"


def test_the_manual_host_flow(ctx):  # :229-280 (paper Listing 2)
    md = ctx.module_load(VADD_F32)
    vadd_fun = ctx.get_function(md, "vadd")
    a = np.array([(i * 37) % 100 for i in range(12)], np.float32)
    b = np.array([(i * 91) % 100 for i in range(12)], np.float32)
    ga, gb, gc = ctx.mem_alloc(48), ctx.mem_alloc(48), ctx.mem_alloc(48)
    ctx.memcpy_htod(ga, a, 48)
    ctx.memcpy_htod(gb, b, 48)
    assert ctx.launch(vadd_fun, GridConfig((12, 1, 1), (1, 1, 1)), [ga, gb, gc]).ok()
    c = np.zeros(12, np.float32)
    ctx.memcpy_dtoh(c, gc, 48)
    assert np.array_equal(c, a + b)
    for g in (ga, gb, gc):
        ctx.mem_free(g)
    ctx.module_unload(md)
    k = ctx.counters()
    assert (k["modules_loaded"], k["functions_resolved"], k["launches"], k["allocs"], k["frees"]) == (1, 1, 1, 3, 3)
    assert (k["bytes_h2d"], k["bytes_d2h"]) == (96, 48)
    assert len(k["launch_log"]) == 1
    rec = k["launch_log"][0]
    assert (rec["h2d_bytes"], rec["d2h_bytes"], rec["grid"]) == (96, 48, [12, 1, 1])


def test_counter_snapshot_exports_stable_json_field_names(ctx):  # :282-306
    md = ctx.module_load(VADD_F32)
    fn = ctx.get_function(md, "vadd")
    p = ctx.mem_alloc(16)
    h = np.ones(4, np.float32)
    ctx.memcpy_htod(p, h, 16)
    ctx.launch(fn, GridConfig((4, 1, 1)), [p, p, p])
    ctx.memcpy_dtoh(h, p, 16)
    j = ctx.counters_json()
    json.dumps(j)
    for key in ("modules_loaded", "functions_resolved", "launches", "allocs", "frees", "bytes_h2d", "bytes_d2h",
                "launch_log"):
        assert key in j
    assert j["modules_loaded"] == 1 and j["launches"] == 1
    log = j["launch_log"][0]
    assert (log["kernel"], log["h2d_bytes"], log["d2h_bytes"], log["grid"][0]) == ("vadd", 16, 16, 4)
    assert list(h) == [2, 2, 2, 2]


def test_distinct_contexts_are_fully_independent(gpu):  # :308-316
    c1, c2 = tt.create_context(gpu), tt.create_context(gpu)
    c1.mem_alloc(64)
    assert c1.counters()["allocs"] == 1 and c2.counters()["allocs"] == 0
    c2.module_load(VADD_F32)
    assert c1.counters()["modules_loaded"] == 0
    assert c1.id != c2.id
    c1.destroy()
    c2.destroy()


def test_trace_launch_contract(ctx):
    """The native trace kernels' own launch rules: coverage, bounds -> trap, no side effects."""
    n, A = 64, 4
    mod = tt.render_module(tt.TRACE_T05, [(True, "f32"), (False, "i32"), (True, "f32"), (True, "f32"),
                                          (True, "f32"), (True, "f32"), (True, "i32"), (False, "i32")], "t")
    fn = ctx.get_function(ctx.module_load(mod), "trace_t05")
    c, s, w = tt.make_tables(n, A)
    bufs = [ctx.mem_alloc(x) for x in (n * n * 4, A * 4, A * 4, 8 * n * 4, A * 6 * n * 4, A * 2 * n * 4)]
    for b, h in zip(bufs[1:4], (c, s, w)):
        ctx.memcpy_htod(b, h)
    img, ct, st, wt, out, med = bufs
    args = [img, np.int32(n), ct, st, wt, out, med, np.int32(0)]
    assert ctx.launch(fn, GridConfig((A, 1, 1), (n, 1, 1)), args).ok()
    with pytest.raises(tt.LaunchConfigError):  # lines p >= 32 not covered
        ctx.launch(fn, GridConfig((A, 1, 1), (32, 1, 1)), args)
    r = ctx.launch(fn, GridConfig((A + 1, 1, 1), (n, 1, 1)), args)  # one angle too many for ctab/out
    assert not r.ok() and r.trap.kind == tt.api.TrapKind.GlobalOutOfBounds
    with pytest.raises(tt.ArgumentMismatch):
        ctx.launch(fn, GridConfig((A, 1, 1), (n, 1, 1)), args[:7] + [np.int64(0)])


def test_sampler_selection_contract(gpu):
    """tt_ctx_set_sampler: 0 (L1 loads), 1 (texture), 2 (TMA tiles for the T0 launches they serve), 3
    (the default: tiles where they pay); anything else is TT_ERR_INVALID and leaves the sampler unchanged.
    Every sampler gives the same bits."""
    n, A = 1024, 4
    img = tt.synth_image(tt.PHANTOM, n)
    ctx = tt.create_context(gpu)
    try:
        outs = []
        for smp in (3, 2, 1, 0):
            if smp != 3:
                ctx.set_sampler(smp)
            out, _, rep = tt.TraceTransform(ctx, n, A, full=False)(img)
            assert rep.ok()
            outs.append(out.reshape(-1).view(np.uint32))
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
        for bad in (-1, 4, 7):
            with pytest.raises(tt.api.AbiError):
                ctx.set_sampler(bad)
    finally:
        ctx.destroy()
