"""Spectral P-functional (tt_circus_fft_device: sum_k |F(s)_k|^4) against the
f64 numpy FFT of the same rows (oracle.pfft).  Tolerance: rtol 1e-4 (fp32 FFT, f64 powers
and result)."""
import numpy as np
import pytest

import oracle as O
import paper_1604_03410_b200 as tt

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _gpu_pfft(ctx, rows_host):
    rows_host = np.ascontiguousarray(rows_host, dtype=np.float32)
    r, n = rows_host.shape
    d_s = ctx.mem_alloc(max(rows_host.nbytes, 4))
    d_p = ctx.mem_alloc(max(r * 8, 8))
    ctx.memcpy_htod(d_s, rows_host)
    tt.circus_fft_device(ctx.device_pointer(d_s), n, r, ctx.device_pointer(d_p), ctx.stream)
    ctx.synchronize()
    out = np.empty(r, np.float64)
    ctx.memcpy_dtoh(out, d_p)
    return out


@pytest.fixture(scope="module")
def ctx(gpu):
    c = tt.create_context(0)
    yield c
    c.destroy()


@pytest.mark.parametrize("n,A,kind", [(256, 12, tt.DISK), (1024, 4, tt.PHANTOM), (1000, 4, tt.SPARSE),
                                      (777, 2, tt.DISK), (4096, 1, tt.DISK)])
def test_pfft_of_trace_sinograms_within_rtol_of_f64_fft(ctx, n, A, kind):
    tr = tt.TraceTransform(ctx, n, A, full=True)
    out, _, rep = tr(tt.synth_image(kind, n))
    assert rep.ok()
    rows = out.reshape(-1, n)
    got = _gpu_pfft(ctx, rows)
    ref = O.pfft(rows)
    assert np.all(np.abs(got - ref) <= RTOL * np.abs(ref) + 1e-30), np.max(np.abs(got - ref) / (ref + 1e-30))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 1000, 4095, 4097, 8192, 16384])
def test_pfft_edge_lengths(ctx, n):
    rng = np.random.default_rng(n)
    rows = rng.random((3, n)).astype(np.float32)
    rows[1] = 0.0
    rows[2, : n // 2] = 0.0
    got = _gpu_pfft(ctx, rows)
    ref = O.pfft(rows)
    assert got[1] == 0.0
    assert np.all(np.abs(got - ref) <= RTOL * np.abs(ref)), (got, ref)


def test_pfft_rejects_bad_arguments(ctx):
    d = ctx.mem_alloc(64)
    p = ctx.device_pointer(d)
    with pytest.raises(Exception):
        tt.circus_fft_device(p, 0, 1, p, ctx.stream)
    with pytest.raises(Exception):
        tt.circus_fft_device(p, 16385, 1, p, ctx.stream)
    tt.circus_fft_device(p, 16, 0, p, ctx.stream)  # no rows: no work


def test_pfft_through_cuda_launch_equals_device_entry(ctx):
    """The module path (cuda_launch of a `circus_fft(f32[],i32,i32,f64[])` kernel, bound natively)
    gives the same bits as tt_circus_fft_device."""
    rows = np.random.default_rng(5).random((2, 6, 512)).astype(np.float32)
    via_launch = tt.circus_fft(ctx, rows)
    assert via_launch.shape == (2, 6)
    assert np.array_equal(via_launch.reshape(-1), _gpu_pfft(ctx, rows.reshape(-1, 512)))
