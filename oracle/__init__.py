"""ctypes wrapper for the CPU oracle (TEST INFRASTRUCTURE — see tt_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtt_oracle.so")
TIER2_PATH = os.path.join(HERE, "_ref", "tt_tier2")
TIER2_KRN = os.path.join(HERE, "_ref", "trace_t05.krn")

F64, SEQ32, REPLAY = 0, 1, 2
DISK, PHANTOM, SPARSE = 0, 1, 2
SEEDS = {DISK: 20160412, PHANTOM: 7, SPARSE: 11}
NF = 6

_lib = None


def build(force: bool = False) -> None:
    subprocess.check_call(["make", "-C", HERE, "-s", "libtt_oracle.so"] + (["-B"] if force else []))


def build_ref() -> bool:
    """Compile oracle/_ref/tt_tier2 from the reference sources (container only)."""
    if not os.path.isdir("/root/reference/proj/include"):
        return os.path.exists(TIER2_PATH)
    subprocess.check_call(["make", "-C", HERE, "-s", "ref"])
    return True


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        fp = ctypes.POINTER(ctypes.c_float)
        ip = ctypes.POINTER(ctypes.c_int32)
        dp = ctypes.POINTER(ctypes.c_double)
        L.tto_tables.argtypes = [ctypes.c_int, ctypes.c_int, fp, fp, fp]
        L.tto_synth.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, fp]
        L.tto_line_samples.argtypes = [fp, ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_int, fp]
        L.tto_schedule_slots.argtypes = [ctypes.c_int, ctypes.c_int]
        L.tto_schedule_slots.restype = ctypes.c_int
        L.tto_transform.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, fp,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, ip, dp, dp, ctypes.c_int]
        L.tto_replay_launch.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, fp,
                                        ctypes.c_int, ctypes.c_int, fp, ip, ctypes.c_int]
        L.tto_circus.argtypes = [fp, ctypes.c_int, ctypes.c_int, fp, dp, ip, ctypes.c_int]
        L.tto_is_eps_median.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.tto_is_eps_median.restype = ctypes.c_int
        L.tto_line_f64.argtypes = [fp, ctypes.c_int, fp, ctypes.c_int, ctypes.c_int, dp, dp, ip]
        L.tto_check.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, fp,
                                ctypes.c_int, fp, ip, ctypes.c_double, ctypes.c_int, ctypes.c_double, dp, ctypes.c_int]
        L.tto_check.restype = ctypes.c_long
        L.tto_replay_units.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp, fp, fp, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, ip, ip, fp, ip, ctypes.c_int]
        L.tto_check_lines.argtypes = [fp, ctypes.c_int, fp, fp, fp, ctypes.c_int, ctypes.c_int, ip, ip, fp, ip,
                                      ctypes.c_double, ctypes.c_int, ctypes.c_double, dp, ctypes.c_int]
        L.tto_check_lines.restype = ctypes.c_long
        L.tto_orthonormal_side.argtypes = [ctypes.c_int]
        L.tto_orthonormal_side.restype = ctypes.c_int
        L.tto_orthonormal.argtypes = [fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, fp]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def _f(a):
    return _p(a, ctypes.c_float)


def tables(n: int, a_total: int):
    c = np.empty(a_total, np.float32)
    s = np.empty(a_total, np.float32)
    w = np.empty(8 * n, np.float32)
    lib().tto_tables(n, a_total, _f(c), _f(s), _f(w))
    return c, s, w


def synth(kind: int, n: int, seed: int | None = None) -> np.ndarray:
    img = np.empty((n, n), np.float32)
    lib().tto_synth(kind, SEEDS[kind] if seed is None else seed, n, _f(img))
    return img


def schedule_slots(n: int, full: bool = True) -> int:
    """Slots (lanes) per line of the B200 kernel for side n (8/16/32 or 32W; T0 only, n > 1024: 32)."""
    return lib().tto_schedule_slots(n, int(full))


def line_samples(img, n, c, s, p):
    v = np.empty(n, np.float32)
    lib().tto_line_samples(_f(np.ascontiguousarray(img, np.float32)), n, c, s, p, _f(v))
    return v


def transform(img, n, ctab, stab, wtab, *, a0=0, a_count=None, full=True, mode=F64, W=0, nthreads=0,
              want64=False):
    """Returns (out f32 [a][F][n], med i32 [a][2][n] or None, out64, absm)."""
    a_total = len(ctab)
    a_count = a_total - a0 if a_count is None else a_count
    F = NF if full else 1
    out = np.empty((a_count, F, n), np.float32)
    med = np.zeros((a_count, 2, n), np.int32) if full else None
    out64 = np.empty((a_count, F, n), np.float64) if (want64 and mode == F64) else None
    absm = np.empty((a_count, F, n), np.float64) if (want64 and mode == F64) else None
    lib().tto_transform(_f(np.ascontiguousarray(img, np.float32)), n, a0, a_count, a_total, _f(ctab), _f(stab),
                        _f(wtab), int(full), mode, W, _f(out), _p(med, ctypes.c_int32),
                        _p(out64, ctypes.c_double), _p(absm, ctypes.c_double), nthreads)
    return out, med, out64, absm


def replay_launch(img, n, ctab, stab, wtab, *, a0, units, pair_stride, full=True, W=0, nthreads=0):
    """Replay of one raw B200 launch (tt_trace_device with explicit structure).
    Returns (out [rows][F][n], med [rows][2][n]) with rows = units * (2 if pair_stride else 1)."""
    rows = units * (2 if pair_stride > 0 else 1)
    F = NF if full else 1
    out = np.zeros((rows, F, n), np.float32)
    med = np.zeros((rows, 2, n), np.int32)
    lib().tto_replay_launch(_f(np.ascontiguousarray(img, np.float32)), n, a0, units, pair_stride, _f(ctab),
                            _f(stab), _f(wtab), int(full), W, _f(out), _p(med, ctypes.c_int32), nthreads)
    return out, (med if full else None)


def replay_units(img, n, ctab, stab, wtab, *, a0, pair_stride, units_idx, lines, full=True, W=0, nthreads=0):
    """Replay of selected units (a0 + units_idx[k], lines[k]) of one launch.  Returns
    (out f32 [k][2][F], med i32 [k][2][2], partner_col [k]): the unit's line and its partner
    line (a0+ui+pair_stride, partner_col) -- n-1-p when the tables are exactly mirrored, else p;
    bit-identical to tto_replay_launch's rows."""
    ui = np.ascontiguousarray(units_idx, np.int32)
    pl = np.ascontiguousarray(lines, np.int32)
    F = NF if full else 1
    out = np.zeros((len(ui), 2, F), np.float32)
    med = np.zeros((len(ui), 2, 2), np.int32)
    lib().tto_replay_units(_f(np.ascontiguousarray(img, np.float32)), n, a0, pair_stride, _f(ctab), _f(stab),
                           _f(wtab), int(full), W, len(ui), _p(ui, ctypes.c_int32), _p(pl, ctypes.c_int32),
                           _f(out), _p(med, ctypes.c_int32), nthreads)
    pcol = pl.copy()
    if pair_stride > 0:
        a = a0 + ui
        cb, sb = np.asarray(ctab, np.float32).view(np.uint32), np.asarray(stab, np.float32).view(np.uint32)
        mir = (cb[a + pair_stride] == (cb[a] ^ 0x80000000)) & (sb[a + pair_stride] == (sb[a] ^ 0x80000000))
        pcol = np.where(mir, n - 1 - pl, pl).astype(np.int32)
    return out, (med if full else None), pcol


def check_lines(img, n, ctab, stab, wtab, a_list, p_list, gpu_out, gpu_med=None, *, full=True, rtol=1e-4, W=0,
                chain=0.0, nthreads=0):
    """Spec §2.5 checker on an explicit list of lines: gpu_out [k][F], gpu_med [k][2]."""
    a = np.ascontiguousarray(a_list, np.int32)
    p = np.ascontiguousarray(p_list, np.int32)
    st = np.zeros(4, np.float64)
    gm = None if gpu_med is None else np.ascontiguousarray(gpu_med, np.int32)
    fails = lib().tto_check_lines(_f(np.ascontiguousarray(img, np.float32)), n, _f(ctab), _f(stab), _f(wtab),
                                  int(full), len(a), _p(a, ctypes.c_int32), _p(p, ctypes.c_int32),
                                  _f(np.ascontiguousarray(gpu_out, np.float32)), _p(gm, ctypes.c_int32), rtol, W,
                                  chain, _p(st, ctypes.c_double), nthreads)
    return int(fails), {"worst": float(st[0]), "ties": int(st[1]), "median_bad": int(st[2]), "lines": int(st[3])}


def circus(sino, nthreads=0):
    """P-functionals of sinogram rows: returns (replay f32 [..., 3], f64 truth [..., 3], median idx)."""
    sino = np.ascontiguousarray(sino, np.float32)
    n = sino.shape[-1]
    rows = sino.size // n
    c = np.empty(sino.shape[:-1] + (3,), np.float32)
    c64 = np.empty(sino.shape[:-1] + (3,), np.float64)
    med = np.empty(sino.shape[:-1], np.int32)
    lib().tto_circus(_f(sino), n, rows, _f(c), _p(c64, ctypes.c_double), _p(med, ctypes.c_int32), nthreads)
    return c, c64, med


def pfft(sino):
    """Spectral P-functional of sinogram rows (P = sum_k |F(s)_k|^4, F the
    length-n DFT of the row), in f64 with numpy's FFT: the truth tt_circus_fft_device is
    checked against (rtol 1e-4).  Returns f64 [...]."""
    s = np.asarray(sino, dtype=np.float64)
    f = np.fft.fft(s, axis=-1)
    p2 = f.real * f.real + f.imag * f.imag
    return np.sum(p2 * p2, axis=-1)


def is_eps_median(v, m, eps):
    v = np.ascontiguousarray(v, np.float32)
    return bool(lib().tto_is_eps_median(_f(v), v.size, int(m), float(eps)))


def check(img, n, ctab, stab, wtab, gpu_out, gpu_med=None, *, a0=0, full=True, rtol=1e-4, W=0, chain=0.0,
          nthreads=0):
    """Spec §2.5 checker. Returns (fails, stats dict)."""
    gpu_out = np.ascontiguousarray(gpu_out, np.float32)
    a_count = gpu_out.shape[0]
    st = np.zeros(4, np.float64)
    gm = None if gpu_med is None else np.ascontiguousarray(gpu_med, np.int32)
    fails = lib().tto_check(_f(np.ascontiguousarray(img, np.float32)), n, a0, a_count, len(ctab), _f(ctab),
                            _f(stab), _f(wtab), int(full), _f(gpu_out), _p(gm, ctypes.c_int32), rtol, W, chain,
                            _p(st, ctypes.c_double), nthreads)
    return int(fails), {"worst": float(st[0]), "ties": int(st[1]), "median_bad": int(st[2]),
                        "lines": int(st[3])}


def tier2_sample(img, n, ctab, stab, wtab, *, angles, lines, threads):
    """Bounded sample for the reference benchmark arm: angles [0, angles),
    lines p < lines of each, one angle per host thread."""
    return tier2(img, n, ctab, stab, wtab, a0=0, a_count=angles, threads=threads, lines=lines)


def tier2(img, n, ctab, stab, wtab, *, a0=0, a_count=None, threads=1, lines=0):
    """Run the DSL trace kernel on the reference's emulator (oracle/_ref).

    Returns (out f32 [a][6][n], med i32 [a][2][n], report dict)."""
    if not os.path.exists(TIER2_PATH):
        raise FileNotFoundError(TIER2_PATH + " (build with `make -C oracle ref`)")
    a_count = len(ctab) - a0 if a_count is None else a_count
    with tempfile.TemporaryDirectory() as d:
        fin, fout = os.path.join(d, "in.bin"), os.path.join(d, "out.bin")
        with open(fin, "wb") as f:
            f.write(np.array([n, len(ctab)], np.int32).tobytes())
            for arr in (img, ctab, stab, wtab):
                f.write(np.ascontiguousarray(arr, np.float32).tobytes())
        r = subprocess.run([TIER2_PATH, fin, fout, str(a0), str(a_count), str(threads), TIER2_KRN, str(lines)],
                           check=True, capture_output=True, text=True)
        rep = json.loads(r.stdout.strip().splitlines()[-1])
        raw = np.fromfile(fout, dtype=np.uint8)
    nout = a_count * 6 * n * 4
    out = raw[:nout].view(np.float32).reshape(a_count, 6, n)
    med = raw[nout:].view(np.int32).reshape(a_count, 2, n)
    return out, med, rep


def prep(pix, n: int):
    """CPU restatement of tt_prep_device (tt_b200.h; caller-side input format):
    8-bit gray [h][w] or RGB [h][w][3] -> n x n f32 gray placed at
    ((n-w)//2, (n-h)//2), zeros elsewhere; gray = ((0.299 r + 0.587 g) + 0.114 b) / 255
    in IEEE f32 (numpy float32 arithmetic never contracts)."""
    pix = np.asarray(pix, np.uint8)
    h, w = pix.shape[:2]
    f = pix.astype(np.float32)
    if pix.ndim == 3:
        r, g, b = f[..., 0], f[..., 1], f[..., 2]
        v = (np.float32(0.299) * r + np.float32(0.587) * g) + np.float32(0.114) * b
    else:
        v = f
    v = (v / np.float32(255.0)).astype(np.float32)
    out = np.zeros((n, n), np.float32)
    y0, x0 = (n - h) // 2, (n - w) // 2
    out[y0:y0 + h, x0:x0 + w] = v
    return out


def orthonormal(img, angles: int):
    """CPU restatement of tt_orthonormal_device: bit-exact f32 frame [A][A]."""
    img = np.ascontiguousarray(img, np.float32)
    h, w = img.shape
    out = np.empty((angles, angles), np.float32)
    lib().tto_orthonormal(_f(img), h, w, angles, _f(out))
    return out


def orthonormal_side(angles: int) -> int:
    return lib().tto_orthonormal_side(angles)


def hermite(sino, center, orders: int):
    """Hermite P-functionals in f64 around the given per-row centres:
    returns (H f64 [..., orders], M f64 [..., orders] = sum_p |s_p psi_k(z_p)|, the scale of the
    rounding error).  psi_k(z) = h_k(z) exp(-z^2/2) / sqrt(2^k k! sqrt(pi)), h_k the physicists'
    Hermite polynomials; z_p = (p - c) * 10 / c below the centre, (p - c) * 10 / (n - 1 - c) above."""
    s = np.asarray(sino, np.float64)
    n = s.shape[-1]
    rows = s.reshape(-1, n)
    c = np.asarray(center, np.int64).reshape(-1)
    p = np.arange(n)[None, :]
    lo = np.where(c > 0, 10.0 / np.maximum(c, 1), 0.0)[:, None]
    hi = np.where(c < n - 1, 10.0 / np.maximum(n - 1 - c, 1), 0.0)[:, None]
    z = (p - c[:, None]) * np.where(p < c[:, None], lo, hi)
    e = np.exp(-0.5 * z * z)
    H = np.empty((rows.shape[0], orders))
    M = np.empty((rows.shape[0], orders))
    h0, h1 = np.ones_like(z), 2.0 * z
    for k in range(orders):
        norm = 1.0 / np.sqrt(2.0 ** k * math.factorial(k) * np.sqrt(np.pi))
        t = rows * e * norm * h0
        H[:, k] = t.sum(axis=1)
        M[:, k] = np.abs(t).sum(axis=1)
        h0, h1 = h1, 2.0 * z * h1 - 2.0 * (k + 1) * h0
    shp = s.shape[:-1] + (orders,)
    return H.reshape(shp), M.reshape(shp)
