"""VPTX kernels without a native implementation run through the JIT
(tt_jit.h: VPTX -> CUDA C++ -> NVRTC -> sm_100a) behind module_load /
get_function / launch, against golden vectors from the reference's own front
end and emulator (tests/golden/jit_golden.json, oracle/ref_jit_golden.cpp):
bit-exact outputs, and the same first trap (kind, thread, block, instruction)."""
import json
import os

import numpy as np
import pytest

import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "jit_golden.json")))
DT = {"f32": (np.float32, np.uint32), "i32": (np.int32, np.uint32), "f64": (np.float64, np.uint64),
      "i64": (np.int64, np.uint64)}


@pytest.fixture(scope="module")
def ctx(gpu):
    c = tt.create_context(gpu)
    yield c
    c.destroy()


def _unbits(vals, t):
    dt, ut = DT[t]
    return np.asarray(vals, dtype=ut).view(dt)


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_jit_matches_reference_emulator(ctx, case):
    mh = ctx.module_load(case["vptx"])
    fn = ctx.get_function(mh, case["kernel"])
    args, bufs = [], {}
    for a in case["args"]:
        t = a["type"]
        if t.endswith("[]"):
            host = _unbits(a["data"], t[:-2])
            p = ctx.mem_alloc(host.nbytes)
            ctx.memcpy_htod(p, host)  # Out buffers start zero-filled on both sides
            bufs[a["index"]] = (p, host, t[:-2])
            args.append(p)
        else:
            args.append(DT[t][0](a["value"]))
    cfg = tt.GridConfig(tuple(case["grid"]), tuple(case["block"]), case["shared_extra"])
    res = ctx.launch(fn, cfg, args)
    if case["trap"] is None:
        assert res.ok(), res.trap
        for idx, want in case["outputs"].items():
            p, host, t = bufs[int(idx)]
            got = np.empty_like(host)
            ctx.memcpy_dtoh(got, p)
            w = np.asarray(want, dtype=DT[t][1])
            g = got.view(DT[t][1])
            if t in ("f32", "f64"):  # NaN payloads are not part of the contract (x86 vs GPU default NaN)
                nan = np.isnan(got) & np.isnan(w.view(DT[t][0]))
                g, w = g[~nan], w[~nan]
            assert np.array_equal(g, w), (case["name"], idx)
    else:
        tr = case["trap"]
        assert not res.ok()
        assert int(res.trap.kind) == tr["kind"]
        assert tuple(res.trap.thread) == tuple(tr["thread"]) and tuple(res.trap.block) == tuple(tr["block"])
        assert res.trap.instr_index == tr["instr_index"]
    for p, _, _ in bufs.values():
        ctx.mem_free(p)


def test_jit_function_is_reusable_and_unloads(ctx):
    case = GOLDEN[0]  # vadd
    mh = ctx.module_load(case["vptx"])
    fn = ctx.get_function(mh, case["kernel"])
    n = 12
    a = np.arange(n, dtype=np.float32)
    b = np.full(n, 0.5, np.float32)
    pa, pb, pc = ctx.mem_alloc(a.nbytes), ctx.mem_alloc(b.nbytes), ctx.mem_alloc(a.nbytes)
    ctx.memcpy_htod(pa, a)
    ctx.memcpy_htod(pb, b)
    for _ in range(3):
        assert ctx.launch(fn, tt.GridConfig((n, 1, 1), (1, 1, 1)), [pa, pb, pc]).ok()
    c = np.empty(n, np.float32)
    ctx.memcpy_dtoh(c, pc)
    assert np.array_equal(c, a + b)
    ctx.mem_free(pa)
    # a freed argument buffer is rejected before launch (UseAfterFree), as for native kernels
    with pytest.raises(Exception):
        ctx.launch(fn, tt.GridConfig((n, 1, 1), (1, 1, 1)), [pa, pb, pc])
    ctx.module_unload(mh)
    with pytest.raises(Exception):
        ctx.launch(fn, tt.GridConfig((n, 1, 1), (1, 1, 1)), [pb, pb, pc])
    ctx.mem_free(pb)
    ctx.mem_free(pc)


def test_jit_rejects_invalid_bodies_with_validation_failed(ctx):
    bad = ".module m\n.kernel k(.param ptr.global.f32 a) {\n  .reg f32 %f\n  add.f32 %f, %f, %nope\n  ret\n}\n"
    mh = ctx.module_load(bad)
    with pytest.raises(tt.ValidationFailed):
        ctx.get_function(mh, "k")


TRACE_VPTX = open(os.path.join(os.path.dirname(__file__), "golden", "trace_t05.vptx")).read()


def _run_dsl_trace(ctx, img, n, A, c, s, w, block=64):
    """oracle/trace_t05.krn as the reference front end compiles it, run through the JIT
    (renamed so the native fused kernel does not replace it)."""
    mh = ctx.module_load(TRACE_VPTX.replace(".kernel trace_t05(", ".kernel trace_t05_dsl(", 1))
    fn = ctx.get_function(mh, "trace_t05_dsl")
    bufs = [ctx.mem_alloc(x.nbytes) for x in (img, c, s, w)]
    for b, x in zip(bufs, (img, c, s, w)):
        ctx.memcpy_htod(b, np.ascontiguousarray(x))
    out_d, med_d = ctx.mem_alloc(A * 6 * n * 4), ctx.mem_alloc(A * 2 * n * 4)
    res = ctx.launch(fn, tt.GridConfig((A, (n + block - 1) // block, 1), (block, 1, 1)),
                     [bufs[0], np.int32(n), bufs[1], bufs[2], bufs[3], out_d, med_d, np.int32(0)])
    out = np.empty((A, 6, n), np.float32)
    med = np.empty((A, 2, n), np.int32)
    ctx.memcpy_dtoh(out, out_d)
    ctx.memcpy_dtoh(med, med_d)
    for b in bufs + [out_d, med_d]:
        ctx.mem_free(b)
    return res, out, med


@pytest.mark.parametrize("n,A,kind", [(32, 6, tt.DISK), (64, 10, tt.PHANTOM), (100, 7, tt.SPARSE)])
def test_jit_of_the_reference_dsl_trace_kernel_equals_seq32_oracle(ctx, n, A, kind):
    """The trace transform written in the reference DSL, compiled by the reference front end and
    run through the JIT, equals the oracle's SEQ32 mode (= the reference emulator, tier 2)
    bit-for-bit: the JIT, the oracle and the emulator agree on every bit of the path."""
    import oracle as O

    img = tt.synth_image(kind, n)
    c, s, w = tt.make_tables(n, A)
    res, out, med = _run_dsl_trace(ctx, img, n, A, c, s, w)
    assert res.ok(), res.trap
    rout, rmed, _, _ = O.transform(img, n, c, s, w, mode=O.SEQ32)
    assert np.array_equal(out.view(np.uint32), rout.view(np.uint32))
    assert np.array_equal(med, rmed)


def test_foreign_body_with_a_native_name_runs_as_written(ctx):
    """A user kernel that only shares the name and signature of a native kernel is compiled from
    its own body (no silent substitution): here a `trace_t05` whose body writes 7.0 to out[0]."""
    header = TRACE_VPTX.split("{", 1)[0]  # .module + .kernel with the native signature
    vptx = (header + "{\n  .reg f32 %v\n  .reg i64 %a\n  mov.f32 %v, 0f40E00000\n  mov.i64 %a, out\n"
            "  st.global.f32 [%a], %v\n  ret\n}\n")
    mh = ctx.module_load(vptx)
    fn = ctx.get_function(mh, "trace_t05")
    n = 8
    bufs = [ctx.mem_alloc(64 * 4) for _ in range(6)]
    res = ctx.launch(fn, tt.GridConfig((1, 1, 1), (1, 1, 1)),
                     [bufs[0], np.int32(n), bufs[1], bufs[2], bufs[3], bufs[4], bufs[5], np.int32(0)])
    assert res.ok(), res.trap
    out = np.empty(64, np.float32)
    ctx.memcpy_dtoh(out, bufs[4])
    assert out[0] == 7.0 and not out[1:].any()
    for b in bufs:
        ctx.mem_free(b)
