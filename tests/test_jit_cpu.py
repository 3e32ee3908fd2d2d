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
