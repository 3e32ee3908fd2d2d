"""The one-call facade contract of /root/reference/proj/tests/test_autolaunch.cpp
re-run against the CUDA-backed context: direction-exact transfers, the
per-signature method cache, Out buffers never uploaded, traps free buffers,
facade == manual flow, steady-state event stream."""
import numpy as np
import pytest

import paper_1604_03410_b200 as tt
from paper_1604_03410_b200 import GridConfig, cu_in, cu_inout, cu_out, cuda_launch

pytestmark = pytest.mark.gpu

VADD = tt.parse_kernel("kernel vadd(a, b, c) {\n  i = block_id_x() + (thread_id_x() - 1) * num_blocks_x();\n"
                       "  c[i] = a[i] + b[i];\n}\n")
COPY = tt.parse_kernel("kernel copy(a, b){ b[thread_id_x()] = a[thread_id_x()]; }")


def grid1d(blocks, threads):
    return GridConfig((blocks, 1, 1), (threads, 1, 1))


@pytest.fixture
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    c.destroy()


def test_one_call_flow_reproduces_manual_result_with_exact_transfer_counts(ctx):  # :38-62
    a = np.array([(i * 13) % 50 for i in range(12)], np.float32)
    b = np.array([(i * 29) % 50 for i in range(12)], np.float32)
    c = np.full(12, -1.0, np.float32)
    rep = cuda_launch(ctx, VADD, grid1d(12, 1), [cu_in(a), cu_in(b), cu_out(c)])
    assert rep.ok() and not rep.cache_hit
    assert (rep.bytes_h2d, rep.bytes_d2h) == (96, 48)
    assert np.array_equal(c.view(np.uint32), (a + b).view(np.uint32))
    k = ctx.counters()
    assert (k["allocs"], k["frees"], k["bytes_h2d"], k["bytes_d2h"]) == (3, 3, 96, 48)


def test_second_identical_call_is_a_pure_cache_hit(ctx):  # :64-85
    a, b, c = np.ones(12, np.float32), np.full(12, 2.0, np.float32), np.zeros(12, np.float32)
    first = cuda_launch(ctx, VADD, grid1d(12, 1), [cu_in(a), cu_in(b), cu_out(c)])
    loaded = ctx.counters()["modules_loaded"]
    second = cuda_launch(ctx, VADD, grid1d(12, 1), [cu_in(a), cu_in(b), cu_out(c)])
    assert not first.cache_hit and second.cache_hit
    assert ctx.counters()["modules_loaded"] == loaded
    assert np.all(c == 3.0)
    st = tt.cache_stats(ctx)
    assert (st.entries, st.hits, st.misses, st.compiles) == (1, 1, 1, 1)


def test_new_argument_types_trigger_a_new_compilation(ctx):  # :87-109
    af, bf, cf = np.ones(4, np.float32), np.full(4, 2, np.float32), np.zeros(4, np.float32)
    ad, bd, cd = np.ones(4), np.full(4, 2.0), np.zeros(4)
    cuda_launch(ctx, VADD, grid1d(4, 1), [cu_in(af), cu_in(bf), cu_out(cf)])
    cuda_launch(ctx, VADD, grid1d(4, 1), [cu_in(ad), cu_in(bd), cu_out(cd)])
    st = tt.cache_stats(ctx)
    assert (st.entries, st.compiles) == (2, 2)
    assert ctx.counters()["modules_loaded"] == 2
    assert np.array_equal(cd, np.full(4, 3.0))
    scale = tt.parse_kernel("kernel scale(a, k){ a[thread_id_x()] = a[thread_id_x()] * k; }")
    data = np.full(4, 2.0, np.float32)
    cuda_launch(ctx, scale, grid1d(1, 4), [cu_inout(data), np.float32(3.0)])
    assert tt.cache_stats(ctx).entries == 3
    assert np.array_equal(data, np.full(4, 6.0, np.float32))


@pytest.mark.parametrize("mode", ["in_out", "inout", "unwrapped"])
def test_directions_control_the_transfers_exactly(ctx, mode):  # :111-139
    n = 1024
    nbytes = n * 4
    src, dst = np.full(n, 5.0, np.float32), np.zeros(n, np.float32)
    h0, d0 = ctx.counters()["bytes_h2d"], ctx.counters()["bytes_d2h"]
    if mode == "in_out":
        cuda_launch(ctx, COPY, grid1d(1, n), [cu_in(src), cu_out(dst)])
        assert ctx.counters()["bytes_h2d"] - h0 == nbytes and ctx.counters()["bytes_d2h"] - d0 == nbytes
        assert np.array_equal(dst, src)
    else:
        args = [cu_inout(src), cu_inout(dst)] if mode == "inout" else [src, dst]
        rep = cuda_launch(ctx, COPY, grid1d(1, n), args)
        assert (rep.bytes_h2d, rep.bytes_d2h) == (2 * nbytes, 2 * nbytes)


def test_out_arrays_never_upload(ctx):  # :141-155
    k = tt.parse_kernel("kernel add_to(inp, out){ t = thread_id_x(); out[t] = inp[t] + out[t]; }")
    inp = np.full(8, 3.0, np.float32)
    poisoned = np.full(8, 777.0, np.float32)
    rep = cuda_launch(ctx, k, grid1d(1, 8), [cu_in(inp), cu_out(poisoned)])
    assert rep.ok() and rep.bytes_h2d == 32
    assert np.array_equal(poisoned, np.full(8, 3.0, np.float32))


def test_unregistered_signature_fails_before_any_allocation(ctx):  # :157-169 analogue
    a, out = np.ones(4, np.float64), np.zeros(4, np.float64)
    with pytest.raises(tt.FunctionNotFound):
        cuda_launch(ctx, COPY, grid1d(1, 4), [cu_in(a), cu_out(out)])  # copy(f64[],f64[]) has no native kernel
    assert ctx.counters()["allocs"] == 0


def test_a_trap_still_frees_the_buffers_and_skips_downloads(ctx):  # :171-184
    out = np.full(4, 9, np.int32)
    a = np.ones(1, np.int32)
    rep = cuda_launch(ctx, VADD, grid1d(4, 1), [cu_in(a), cu_in(a), cu_out(out[:1].copy())])
    assert not rep.ok()
    assert rep.trap.kind == tt.api.TrapKind.GlobalOutOfBounds
    assert rep.bytes_d2h == 0
    k = ctx.counters()
    assert k["allocs"] == k["frees"]
    assert rep.to_json()["trap"]["kind"] == "GlobalOutOfBounds"


def test_arity_errors_are_reported_against_the_kernel(ctx):  # :186-190
    with pytest.raises(tt.ArityError):
        cuda_launch(ctx, VADD, grid1d(1, 1), [cu_in(np.ones(4, np.float32))])


def test_equivalence_facade_equals_manual_driver_sequence(gpu):  # :192-219
    a = (np.arange(12, dtype=np.float32) * np.float32(0.37)).astype(np.float32)
    b = ((11 - np.arange(12, dtype=np.float32)) * np.float32(1.91)).astype(np.float32)
    c_facade = np.zeros(12, np.float32)
    ctx1 = tt.create_context(gpu)
    cuda_launch(ctx1, VADD, grid1d(12, 1), [cu_in(a), cu_in(b), cu_out(c_facade)])
    ctx2 = tt.create_context(gpu)
    md = ctx2.module_load(tt.render_module(VADD, [(True, "f32")] * 3, "vadd$manual"))
    fn = ctx2.get_function(md, "vadd")
    ga, gb, gc = ctx2.mem_alloc(48), ctx2.mem_alloc(48), ctx2.mem_alloc(48)
    ctx2.memcpy_htod(ga, a, 48)
    ctx2.memcpy_htod(gb, b, 48)
    assert ctx2.launch(fn, grid1d(12, 1), [ga, gb, gc]).ok()
    c_manual = np.zeros(12, np.float32)
    ctx2.memcpy_dtoh(c_manual, gc, 48)
    assert c_facade.tobytes() == c_manual.tobytes()
    ctx1.destroy()
    ctx2.destroy()


def test_steady_state_performs_only_alloc_copy_launch_copy_free_events(ctx):  # :221-233
    a, b, c = np.ones(8, np.float32), np.full(8, 2.0, np.float32), np.zeros(8, np.float32)
    cuda_launch(ctx, VADD, grid1d(8, 1), [cu_in(a), cu_in(b), cu_out(c)])
    mark = len(ctx.events())
    for _ in range(5):
        cuda_launch(ctx, VADD, grid1d(8, 1), [cu_in(a), cu_in(b), cu_out(c)])
    ev = ctx.events()[mark:]
    assert ev and set(ev) <= {"Alloc", "H2D", "Launch", "D2H", "Free"}


def test_trace_transform_one_call_flow_counts(ctx):
    """The path itself through the facade: exact bytes, one compile per signature."""
    n, A = 128, 10
    tr = tt.TraceTransform(ctx, n, A)
    img = tt.synth_image(tt.DISK, n)
    out, med, rep = tr(img)
    assert rep.ok() and not rep.cache_hit
    assert rep.bytes_h2d == n * n * 4 + 2 * A * 4 + 8 * n * 4
    assert rep.bytes_d2h == A * 6 * n * 4 + A * 2 * n * 4
    out2, med2, rep2 = tr(img)
    assert rep2.cache_hit and np.array_equal(out, out2) and np.array_equal(med, med2)
    # per call: the pass-2 weight layout of the freshly uploaded wtab + the fused kernel
    assert ctx.counters()["gpu_kernel_launches"] == 4
