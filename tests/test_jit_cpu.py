"""VPTX -> CUDA C++ translation of the JIT (tt_jit_source), host only: every
golden kernel (the reference front end's own VPTX) translates, with the
emulator's semantics visible in the generated code (explicit _rn float
intrinsics, wrapping integer arithmetic, checked global/shared accesses)."""
import ctypes as C
import json
import os

import pytest

from paper_1604_03410_b200._lib import lib

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "jit_golden.json")))


def _source(vptx: str, kernel: str):
    t = vptx.encode()
    n = C.c_size_t()
    st = lib.tt_jit_source(t, len(t), kernel.encode(), None, 0, C.byref(n))
    if st != 0:
        return st, None
    buf = C.create_string_buffer(n.value)
    assert lib.tt_jit_source(t, len(t), kernel.encode(), buf, n.value, C.byref(n)) == 0
    return 0, buf.value.decode()


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_golden_kernels_translate(case):
    st, src = _source(case["vptx"], case["kernel"])
    assert st == 0 and "tt_jit_kernel" in src
    assert "tt_gcheck" in src or "tt_sh" in src
    if "add.f32" in case["vptx"]:
        assert "__fadd_rn" in src


def test_integer_division_traps_and_wraps():
    st, src = _source(next(c for c in GOLDEN if c["name"] == "mixed_ops")["vptx"], "mixed")
    assert st == 0
    assert "TT_TRAP(3," in src          # DivisionByZero
    assert "== -1 ?" in src             # INT_MIN / -1 wraps, INT_MIN % -1 == 0


def test_invalid_body_is_a_validation_error():
    bad = ".module m\n.kernel k(.param ptr.global.f32 a) {\n  .reg f32 %f\n  add.f32 %f, %f, %nope\n  ret\n}\n"
    st, _ = _source(bad, "k")
    assert st == 3  # TT_ERR_VALIDATION_FAILED


TRACE_VPTX = open(os.path.join(os.path.dirname(__file__), "golden", "trace_t05.vptx")).read()


def _fingerprint(vptx: str, kernel: str) -> int:
    t = vptx.encode()
    out = C.c_uint64()
    assert lib.tt_vptx_body_fingerprint(t, len(t), kernel.encode(), C.byref(out)) == 0
    return out.value


def test_trace_t05_body_fingerprint_is_the_registered_one():
    """The native fused kernel stands in for a `trace_t05` module only when its body is the
    reference front end's compilation of the documented DSL kernel (tests/golden/trace_t05.vptx);
    the constant registered in tt_context.cpp must be this file's fingerprint."""
    assert _fingerprint(TRACE_VPTX, "trace_t05") == 0x64a3da5074adf4b3


def test_fingerprint_ignores_layout_but_not_instructions():
    fp = _fingerprint(TRACE_VPTX, "trace_t05")
    spaced = TRACE_VPTX.replace("\n  ", "\n      ")
    assert _fingerprint(spaced, "trace_t05") == fp
    lines = TRACE_VPTX.splitlines()
    i = next(k for k, l in enumerate(lines) if "add.f32" in l)
    edited = "\n".join(lines[:i] + [lines[i].replace("add.f32", "sub.f32", 1)] + lines[i + 1:]) + "\n"
    assert _fingerprint(edited, "trace_t05") != fp
