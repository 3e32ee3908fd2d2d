"""CPU-side checks of the product library: it loads, exports every symbol
include/tt_b200.h declares, and its host-side inputs (tables, synthetic
images) are bit-identical to the oracle's independent restatement.  No
compute calls are made (no GPU here)."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1604_03410_b200 as tt
from paper_1604_03410_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "tt_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    decl = _declared()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(_lib.lib, name), name
    assert set(decl) == set(_lib.EXPORTED)


def test_abi_version_and_registry():
    assert _lib.lib.tt_abi_version() == 1
    ks = tt.native_kernels()
    assert "trace_t05(f32[],i32,f32[],f32[],f32[],f32[],i32[],i32)" in ks
    assert "radon(f32[],i32,f32[],f32[],f32[],i32)" in ks
    assert "vadd(f32[],f32[],f32[])" in ks


@pytest.mark.parametrize("n,A", [(1, 1), (16, 8), (257, 360), (1024, 720)])
def test_tables_bit_identical_to_oracle(n, A):
    a = tt.make_tables(n, A)
    b = O.tables(n, A)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


@pytest.mark.parametrize("kind", [tt.DISK, tt.PHANTOM, tt.SPARSE])
@pytest.mark.parametrize("n", [1, 2, 31, 256])
def test_synthetic_images_bit_identical_to_oracle(kind, n):
    assert np.array_equal(tt.synth_image(kind, n).view(np.uint32), O.synth(kind, n).view(np.uint32))


def test_schedule_matches_oracle_replay_schedule():
    for n in (1, 2, 16, 64, 100, 101, 255, 256, 300, 512, 777, 1000, 1024, 1500, 2048, 4095, 4096, 8192, 16384):
        for full in (True, False):
            assert tt.schedule_slots(n, full) == O.schedule_slots(n, full)


def test_no_gpu_fails_loudly():
    if tt.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(tt.CudaError):
        tt.create_context()


def test_module_rendering_matches_reference_header_shape():
    k = tt.parse_kernel("kernel vadd(a, b, c) {\n  c[i] = a[i] + b[i];\n}\n")
    assert k.name == "vadd" and k.params == ["a", "b", "c"]
    text = tt.render_module(k, [(True, "f32")] * 3, "vadd$x")
    assert text.splitlines()[1] == ".kernel vadd(.param ptr.global.f32 a, .param ptr.global.f32 b, " \
                                   ".param ptr.global.f32 c) {"
