"""Trace-transform entry points on top of the drop-in API.

``TraceTransform`` is the call a user of the reference makes for this path:
the DSL kernel ``trace_t05(img, n, ctab, stab, wtab, out, med, a0)``
(oracle/trace_t05.krn; grid = (angles, ceil(n/B)), block = (B)) launched
through ``cuda_launch`` — here bound to the fused sm_100a kernel.
``trace_device`` is the raw device-pointer entry used by the multi-GPU
driver and the device-resident benchmark leg.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import lib
from .api import (DeviceContext, GridConfig, KernelAst, _check, cu_in, cu_out, cuda_launch)

DISK, PHANTOM, SPARSE = 0, 1, 2
SEEDS = {DISK: 20160412, PHANTOM: 7, SPARSE: 11}
NF = 6

TRACE_T05 = KernelAst("trace_t05", ["img", "n", "ctab", "stab", "wtab", "out", "med", "a0"])
CIRCUS = KernelAst("circus", ["sino", "n", "rows", "circ"])
CIRCUS_FFT = KernelAst("circus_fft", ["sino", "n", "rows", "pf"])
TRACE_T05_BATCH = KernelAst("trace_t05_batch", ["img", "n", "ctab", "stab", "wtab", "out", "med", "a0", "batch"])
RADON = KernelAst("radon", ["img", "n", "ctab", "stab", "out", "a0"])
HERMITE = KernelAst("hermite", ["sino", "n", "rows", "orders", "hp", "center"])
ORTHONORMAL = KernelAst("orthonormal", ["img", "h", "w", "angles", "out"])


def make_tables(n: int, a_total: int):
    """ctab, stab [a_total] and wtab [n][8]."""
    c = np.empty(a_total, np.float32)
    s = np.empty(a_total, np.float32)
    w = np.empty(8 * n, np.float32)
    _check(lib.tt_make_tables(n, a_total, c.ctypes.data, s.ctypes.data, w.ctypes.data))
    return c, s, w


def synth_image(kind: int, n: int, seed: int | None = None) -> np.ndarray:
    img = np.empty((n, n), np.float32)
    _check(lib.tt_synth_image(kind, SEEDS[kind] if seed is None else seed, n, img.ctypes.data))
    return img


def schedule_slots(n: int, full: bool = True) -> int:
    """Slots (lanes) per line of the fused kernel: 8/16/32 (warp segment) or 32W (T0 only, n > 1024: 32)."""
    return lib.tt_schedule_slots(n, int(full))


def max_full_n() -> int:
    return lib.tt_max_full_n()


def launch_config(n: int, angles: int, block: int = 256, batch: int = 1) -> GridConfig:
    b = min(block, max(n, 1))
    return GridConfig((angles, (n + b - 1) // b, batch), (b, 1, 1))


class TraceTransform:
    """Sinograms T0..T5 (or T0 only) of n x n images over `angles` orientations.

    ``__call__(img)`` is the reference-style one-call flow (cuda_launch:
    alloc, upload, launch, download, free).  ``run_resident(img)`` keeps the
    tables and output buffers on the device between calls and moves only the
    image in and the sinograms out (the e2e benchmark path)."""

    def __init__(self, ctx: DeviceContext, n: int, angles: int, full: bool = True, a0: int = 0,
                 a_count: int | None = None, features: bool = False, batch: int = 1):
        self.ctx, self.n, self.angles, self.full = ctx, n, angles, full
        self.features = features and full  # P-functional (circus) stage after the trace kernel
        self.a0 = a0
        self.a_count = angles - a0 if a_count is None else a_count
        self.batch = batch  # > 1: trace_t05_batch over [batch][n][n] images (T0-T5 only)
        if batch > 1 and not full:
            raise ValueError("batched launches compute T0-T5")
        self.ctab, self.stab, self.wtab = make_tables(n, angles)
        self.F = NF if full else 1
        self.cfg = launch_config(n, self.a_count, batch=batch)
        self._res = None

    def out_shape(self):
        lead = (self.batch,) if self.batch > 1 else ()
        return lead + (self.a_count, self.F, self.n)

    def _med_elems(self):
        return self.batch * self.a_count * 2 * self.n

    def _circ_elems(self):
        return self.batch * self.a_count * NF * 3

    def __call__(self, img: np.ndarray):
        img = np.ascontiguousarray(img, np.float32)
        out = np.empty(self.out_shape(), np.float32)
        if self.batch > 1:
            med = np.empty(self.out_shape()[:-2] + (2, self.n), np.int32)
            rep = cuda_launch(self.ctx, TRACE_T05_BATCH, self.cfg,
                              [cu_in(img), np.int32(self.n), cu_in(self.ctab), cu_in(self.stab), cu_in(self.wtab),
                               cu_out(out), cu_out(med), np.int32(self.a0), np.int32(self.batch)])
        elif self.full:
            med = np.empty((self.a_count, 2, self.n), np.int32)
            rep = cuda_launch(self.ctx, TRACE_T05, self.cfg,
                              [cu_in(img), np.int32(self.n), cu_in(self.ctab), cu_in(self.stab), cu_in(self.wtab),
                               cu_out(out), cu_out(med), np.int32(self.a0)])
        else:
            med = None
            rep = cuda_launch(self.ctx, RADON, self.cfg,
                              [cu_in(img), np.int32(self.n), cu_in(self.ctab), cu_in(self.stab), cu_out(out),
                               np.int32(self.a0)])
        if not rep.ok():
            raise RuntimeError(f"trace launch trapped: {rep.trap}")
        return out, med, rep

    # ---- device-resident flow --------------------------------------------------
    def _resident(self):
        if self._res is None:
            ctx = self.ctx
            r = {"img": ctx.mem_alloc(self.batch * self.n * self.n * 4), "ctab": ctx.mem_alloc(self.ctab.nbytes),
                 "stab": ctx.mem_alloc(self.stab.nbytes), "wtab": ctx.mem_alloc(self.wtab.nbytes),
                 "out": ctx.mem_alloc(int(np.prod(self.out_shape())) * 4),
                 "med": ctx.mem_alloc(self._med_elems() * 4),
                 "circ": ctx.mem_alloc(self._circ_elems() * 4)}
            ctx.memcpy_htod(r["ctab"], self.ctab)
            ctx.memcpy_htod(r["stab"], self.stab)
            ctx.memcpy_htod(r["wtab"], self.wtab)
            kern = TRACE_T05_BATCH if self.batch > 1 else (TRACE_T05 if self.full else RADON)
            types = ([(True, "f32"), (False, "i32"), (True, "f32"), (True, "f32"), (True, "f32"), (True, "f32"),
                      (True, "i32"), (False, "i32")] if self.full else
                     [(True, "f32"), (False, "i32"), (True, "f32"), (True, "f32"), (True, "f32"), (False, "i32")])
            if self.batch > 1:
                types = types + [(False, "i32")]
            from .api import render_module
            mh = ctx.module_load(render_module(kern, types, kern.name + "$resident"))
            r["fn"] = ctx.get_function(mh, kern.name)
            mc = ctx.module_load(render_module(CIRCUS, [(True, "f32"), (False, "i32"), (False, "i32"), (True, "f32")],
                                               "circus$resident"))
            r["circus"] = ctx.get_function(mc, "circus")
            self._res = r
        return self._res

    def launch_resident(self):
        """Launch on the resident buffers (image already uploaded)."""
        r = self._resident()
        if self.batch > 1:
            args = [r["img"], np.int32(self.n), r["ctab"], r["stab"], r["wtab"], r["out"], r["med"],
                    np.int32(self.a0), np.int32(self.batch)]
        elif self.full:
            args = [r["img"], np.int32(self.n), r["ctab"], r["stab"], r["wtab"], r["out"], r["med"],
                    np.int32(self.a0)]
        else:
            args = [r["img"], np.int32(self.n), r["ctab"], r["stab"], r["out"], np.int32(self.a0)]
        res = self.ctx.launch(r["fn"], self.cfg, args)
        if not res.ok():
            raise RuntimeError(f"trace launch trapped: {res.trap}")
        if self.features:
            rows = self.batch * self.a_count * NF
            res = self.ctx.launch(r["circus"], GridConfig(((rows + 7) // 8, 1, 1), (256, 1, 1)),
                                  [r["out"], np.int32(self.n), np.int32(rows), r["circ"]])
            if not res.ok():
                raise RuntimeError(f"circus launch trapped: {res.trap}")

    def run_resident(self, img_host, out_host, med_host=None, circ_host=None):
        """H2D image -> fused kernel (-> circus) -> D2H sinograms (+ medians, + features)."""
        r = self._resident()
        self.ctx.memcpy_htod(r["img"], img_host, self.batch * self.n * self.n * 4)
        self.launch_resident()
        if out_host is not None:
            self.ctx.memcpy_dtoh(out_host, r["out"], int(np.prod(self.out_shape())) * 4)
        if med_host is not None and self.full:
            self.ctx.memcpy_dtoh(med_host, r["med"], self._med_elems() * 4)
        if circ_host is not None and self.features:
            self.ctx.memcpy_dtoh(circ_host, r["circ"], self._circ_elems() * 4)

    def resident_ptr(self, name: str) -> int:
        return self.ctx.device_pointer(self._resident()[name])

    def free_resident(self):
        if self._res is not None:
            for k in ("img", "ctab", "stab", "wtab", "out", "med", "circ"):
                self.ctx.mem_free(self._res[k])
            self._res = None


class Plan:
    """Host-to-host pipelined form of the path (tt_plan_*): tables, texture and
    outputs stay on the device; ``run`` uploads the image(s), runs the fused
    kernel in angle chunks while finished chunks download (overlapped D2H), runs
    the P-functional stage, and fills the given host arrays (pinned for overlap).
    Outputs equal one whole launch bit-for-bit."""

    def __init__(self, ctx: DeviceContext, n: int, angles: int, full: bool = True, a0: int = 0,
                 a_count: int | None = None, features: bool = False, batch: int = 1, chunks: int = 0,
                 slots: int = 0, pair_stride: int = 0, graph: bool = False):
        self.ctx, self.n, self.full, self.batch = ctx, n, full, batch
        self.a_count = angles - a0 if a_count is None else a_count
        self.features = features and full
        d = _lib.PlanDesc(n, angles, a0, self.a_count, int(full), int(self.features), batch, chunks, slots,
                          pair_stride, int(graph))
        self._p = C.c_void_p()
        _check(lib.tt_plan_create(ctx._p, C.byref(d), C.byref(self._p)), ctx._p)
        c = C.c_int()
        _check(lib.tt_plan_chunks(self._p, C.byref(c)))
        self.chunks = c.value

    @property
    def captures(self) -> int:
        """Graph mode: submissions captured into CUDA graphs so far (tt_plan_captures)."""
        c = C.c_int()
        _check(lib.tt_plan_captures(self._p, C.byref(c)))
        return c.value

    def run(self, img, out=None, med=None, circ=None) -> None:
        """Synchronous: returns with the host outputs filled."""
        self.submit(img, out, med, circ)
        self.wait()

    def wait(self) -> None:
        """Drain every submission (tt_plan_wait)."""
        _check(lib.tt_plan_wait(self._p), self.ctx._p)

    def submit(self, img, out=None, med=None, circ=None) -> None:
        """Asynchronous (tt_plan_submit): the arrays must stay alive and untouched until wait()."""
        def ptr(a, dt):
            if a is None:
                return None
            if a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
                raise ValueError(f"plan arrays must be C-contiguous {np.dtype(dt).name}")
            return C.c_void_p(a.ctypes.data)
        if not self._p:
            raise ValueError("plan destroyed")
        F = NF if self.full else 1
        lead = self.batch * self.a_count
        for a, size in ((out, lead * F * self.n), (med, lead * 2 * self.n), (circ, lead * NF * 3)):
            if a is not None and a.size != size:
                raise ValueError(f"output array has {a.size} elements, the plan writes {size}")
        if img.size != self.batch * self.n * self.n:
            raise ValueError(f"image array has {img.size} elements, the plan reads {self.batch * self.n * self.n}")
        _check(lib.tt_plan_submit(self._p, ptr(img, np.float32), ptr(out, np.float32),
                               ptr(med if self.full else None, np.int32), ptr(circ if self.features else None,
                                                                                np.float32)), self.ctx._p)

    def destroy(self) -> None:
        if self._p:
            lib.tt_plan_destroy(self._p)
            self._p = C.c_void_p()

    def __enter__(self) -> "Plan":
        return self

    def __exit__(self, *exc) -> None:
        self.destroy()


def trace_device(img_ptr: int, n: int, a0: int, a_count: int, ctab_ptr: int, stab_ptr: int, wtab_ptr: int,
                 out_ptr: int, med_ptr: int = 0, full: bool = True, sampler: int = 0, stream: int = 0,
                 tex=None, pair_stride: int = 0, batch: int = 1, img_stride: int = 0, wsoa_ptr: int = 0,
                 partner_row: int = 0, peer_out: bool = False, circ_ptr: int = 0, fused_p: bool = False) -> None:
    """Raw device-pointer launch (tt_trace_device / tt_trace_device_tex); pair_stride, batch, wsoa as in
    tt_b200.h (wsoa_ptr: a prepared weights_soa() buffer; 0 converts wtab per call; circ_ptr: the
    [rows][6][3] circus output, 0 = none; fused_p: compute it inside the trace launch, TT_TRACE_FUSED_P)."""
    d = _lib.TraceDesc(img_ptr, n, a0, a_count, int(full), ctab_ptr, stab_ptr, wtab_ptr or None, out_ptr,
                       med_ptr or None, sampler, pair_stride, batch, 0, img_stride, wsoa_ptr or None, partner_row,
                       (1 if peer_out else 0) | (2 if fused_p else 0), circ_ptr or None)
    if tex is not None:
        _check(lib.tt_trace_device_tex(C.byref(d), tex, C.c_void_p(stream)))
    else:
        _check(lib.tt_trace_device(C.byref(d), C.c_void_p(stream)))


def prep_side(h: int, w: int) -> int:
    """Side n of the square whose inscribed disk holds an h x w picture (tt_prep_side)."""
    return lib.tt_prep_side(h, w)


def read_pnm(path: str) -> np.ndarray:
    """Binary P5/P6 8-bit image -> uint8 [h][w] or [h][w][3] (tt_pnm_read)."""
    h, w, c = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib.tt_pnm_read(path.encode(), C.byref(h), C.byref(w), C.byref(c), None, 0))
    pix = np.empty((h.value, w.value, c.value), np.uint8)
    _check(lib.tt_pnm_read(path.encode(), C.byref(h), C.byref(w), C.byref(c), C.c_void_p(pix.ctypes.data),
                           pix.nbytes))
    return pix[..., 0] if c.value == 1 else pix


def write_pgm(path: str, img: np.ndarray, lo: float | None = None, hi: float | None = None) -> None:
    """f32 image -> 8-bit P5 file, linearly mapping [lo, hi] (default: min..max) to 0..255."""
    img = np.ascontiguousarray(img, np.float32)
    lo = float(img.min()) if lo is None else lo
    hi = float(img.max()) if hi is None else hi
    if hi <= lo:
        hi = lo + 1.0
    _check(lib.tt_pgm_write(path.encode(), C.c_void_p(img.ctypes.data), img.shape[0], img.shape[1], lo, hi))


def prep_device(pix_ptr: int, h: int, w: int, channels: int, n: int, img_ptr: int, stream: int = 0) -> None:
    """8-bit picture on device -> n x n f32 gray, centred, zero padded (tt_prep_device)."""
    _check(lib.tt_prep_device(C.c_void_p(pix_ptr), h, w, channels, n, C.c_void_p(img_ptr), C.c_void_p(stream)))


def ipc_export(ptr: int) -> bytes:
    """Inter-process handle (72 bytes) of a device pointer inside a cudaMalloc allocation."""
    h = _lib.IpcHandle()
    _check(lib.tt_ipc_export(C.c_void_p(ptr), C.byref(h)))
    return bytes(h)


def ipc_import(handle: bytes, device: int) -> int:
    """Map another process's exported device pointer into this one (peer access over NVLink)."""
    h = _lib.IpcHandle.from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib.tt_ipc_import(C.byref(h), device, C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    _check(lib.tt_ipc_close(C.c_void_p(ptr)))


class IpcBuffer:
    """A dedicated device allocation made for export (tt_ipc_alloc: one cudaMalloc, zero-filled), so its
    IPC handle is independent of the caching allocator's block layout.  Exposes
    ``__cuda_array_interface__`` (``torch.as_tensor(buf, device=...)`` views it without a copy); freed
    when the object is released (after every importer has closed its mapping)."""

    def __init__(self, device: int, shape, dtype):
        import numpy as np
        self.shape = tuple(int(x) for x in shape)
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        _check(lib.tt_ipc_alloc(int(device), max(nbytes, 1), C.byref(p)))
        self.ptr = p.value
        self.device = device

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self.dtype.str, "data": (self.ptr, False), "version": 3,
                "strides": None}

    def free(self) -> None:
        if getattr(self, "ptr", None):
            lib.tt_ipc_free(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # interpreter shutdown: the library may already be unloaded
            pass


def weights_soa(wtab_ptr: int, n: int, wsoa_ptr: int, stream: int = 0) -> None:
    """Regroup a device [n][8] weight table into the pass-2 layout (tt_weights_soa; 24n bytes)."""
    _check(lib.tt_weights_soa(C.c_void_p(wtab_ptr), n, C.c_void_p(wsoa_ptr), C.c_void_p(stream)))


def circus_device(sino_ptr: int, n: int, rows: int, circ_ptr: int, stream: int = 0) -> None:
    """P-functionals of `rows` device sinogram rows (tt_circus_device)."""
    _check(lib.tt_circus_device(C.c_void_p(sino_ptr), n, rows, C.c_void_p(circ_ptr), C.c_void_p(stream)))


def circus_fft_device(sino_ptr: int, n: int, rows: int, p_ptr: int, stream: int = 0) -> None:
    """Spectral P-functional sum_k |F(s)_k|^4 of `rows` device sinogram rows (tt_circus_fft_device)."""
    _check(lib.tt_circus_fft_device(C.c_void_p(sino_ptr), n, rows, C.c_void_p(p_ptr), C.c_void_p(stream)))


def circus(ctx: DeviceContext, sino: np.ndarray):
    """P-functionals of host sinogram rows through cuda_launch (circus kernel)."""
    sino = np.ascontiguousarray(sino, np.float32)
    n = sino.shape[-1]
    rows = sino.size // n
    circ = np.empty(sino.shape[:-1] + (3,), np.float32)
    rep = cuda_launch(ctx, CIRCUS, GridConfig(((rows + 7) // 8, 1, 1), (256, 1, 1)),
                      [cu_in(sino), np.int32(n), np.int32(rows), cu_out(circ)])
    if not rep.ok():
        raise RuntimeError(f"circus launch trapped: {rep.trap}")
    return circ


def circus_fft(ctx: DeviceContext, sino: np.ndarray):
    """Spectral P-functional sum_k |F(s)_k|^4 of host sinogram rows through cuda_launch (f64 per row)."""
    sino = np.ascontiguousarray(sino, np.float32)
    n = sino.shape[-1]
    rows = sino.size // n
    pf = np.empty(sino.shape[:-1], np.float64)
    rep = cuda_launch(ctx, CIRCUS_FFT, GridConfig((rows, 1, 1), (256, 1, 1)),
                      [cu_in(sino), np.int32(n), np.int32(rows), cu_out(pf)])
    if not rep.ok():
        raise RuntimeError(f"circus_fft launch trapped: {rep.trap}")
    return pf


def hermite(ctx: DeviceContext, sino: np.ndarray, orders: int = 4):
    """Hermite P-functionals H_0..H_{orders-1} of host sinogram rows around each row's weighted median
     through cuda_launch: returns (hp f64 [..., orders], center i32 [...])."""
    sino = np.ascontiguousarray(sino, np.float32)
    n = sino.shape[-1]
    rows = sino.size // n
    hp = np.empty(sino.shape[:-1] + (orders,), np.float64)
    center = np.empty(sino.shape[:-1], np.int32)
    rep = cuda_launch(ctx, HERMITE, GridConfig(((rows + 7) // 8, 1, 1), (256, 1, 1)),
                      [cu_in(sino), np.int32(n), np.int32(rows), np.int32(orders), cu_out(hp), cu_out(center)])
    if not rep.ok():
        raise RuntimeError(f"hermite launch trapped: {rep.trap}")
    return hp, center


def hermite_device(sino_ptr: int, n: int, rows: int, orders: int, hp_ptr: int, center_ptr: int = 0,
                   stream: int = 0) -> None:
    """Hermite P-functionals of `rows` device sinogram rows (tt_hermite_device)."""
    _check(lib.tt_hermite_device(C.c_void_p(sino_ptr), n, rows, orders, C.c_void_p(hp_ptr),
                                 C.c_void_p(center_ptr or None), C.c_void_p(stream)))


def orthonormal_side(angles: int) -> int:
    """Side s = ceil(angles / sqrt 2) the image is resampled to for a square sinogram."""
    return lib.tt_orthonormal_side(angles)


def orthonormal_image(ctx: DeviceContext, img: np.ndarray, angles: int) -> np.ndarray:
    """The orthonormal (square) sinogram input frame of a host image through
    cuda_launch: img (h x w) resampled to s x s and centred in angles x angles."""
    img = np.ascontiguousarray(img, np.float32)
    h, w = img.shape
    out = np.empty((angles, angles), np.float32)
    rep = cuda_launch(ctx, ORTHONORMAL, GridConfig((1, 1, 1), (256, 1, 1)),
                      [cu_in(img), np.int32(h), np.int32(w), np.int32(angles), cu_out(out)])
    if not rep.ok():
        raise RuntimeError(f"orthonormal launch trapped: {rep.trap}")
    return out


def orthonormal_device(img_ptr: int, h: int, w: int, angles: int, out_ptr: int, stream: int = 0) -> None:
    """tt_orthonormal_device: device image -> device angles x angles frame."""
    _check(lib.tt_orthonormal_device(C.c_void_p(img_ptr), h, w, angles, C.c_void_p(out_ptr), C.c_void_p(stream)))


def image_texture(img_ptr: int, n: int, stream: int = 0):
    t = C.c_void_p()
    _check(lib.tt_image_tex_create(C.c_void_p(img_ptr), n, C.c_void_p(stream), C.byref(t)))
    return t


def image_atlas(imgs_ptr: int, n: int, batch: int, img_stride: int = 0, stream: int = 0):
    """Texture atlas of a device batch of images (tt_image_atlas_create)."""
    t = C.c_void_p()
    _check(lib.tt_image_atlas_create(C.c_void_p(imgs_ptr), n, batch, img_stride, C.c_void_p(stream), C.byref(t)))
    return t


def image_texture_update(t, imgs_ptr: int, img_stride: int = 0, stream: int = 0) -> None:
    """Refresh a texture/atlas from device images (stream-ordered copy).  Small images (n <= 256) are
    gathered through a pitch-linear view of the image itself: nothing is copied, and a different image
    pointer switches the handle to that image's view."""
    _check(lib.tt_image_tex_update(t, C.c_void_p(imgs_ptr), img_stride, C.c_void_p(stream)))


def image_texture_destroy(t) -> None:
    lib.tt_image_tex_destroy(t)
