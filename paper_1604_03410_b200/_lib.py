"""ctypes binding of include/tt_b200.h.  Raises at import if libtt_b200.so
is missing (build it with ``python paper_1604_03410_b200/build.py`` or
``__graft_entry__.build()``) — there is deliberately no fallback."""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("TT_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtt_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python paper_1604_03410_b200/build.py` "
                      "(the trace transform has no CPU fallback)")


class Caps(C.Structure):
    _fields_ = [("max_block_threads", C.c_uint32), ("max_shared_bytes", C.c_uint64)]


class DevPtr(C.Structure):
    _fields_ = [("base", C.c_uint64), ("length", C.c_uint64), ("ctx_id", C.c_uint64)]


class Handle(C.Structure):
    _fields_ = [("ctx_id", C.c_uint64), ("id", C.c_uint64)]


class Grid(C.Structure):
    _fields_ = [("grid", C.c_uint32 * 3), ("block", C.c_uint32 * 3), ("shared_bytes_extra", C.c_uint64)]


class ArgValue(C.Union):
    _fields_ = [("i32", C.c_int32), ("i64", C.c_int64), ("f32", C.c_float), ("f64", C.c_double), ("ptr", DevPtr)]


class Arg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("v", ArgValue)]


class Trap(C.Structure):
    _fields_ = [("trapped", C.c_int32), ("kind", C.c_int32), ("thread", C.c_uint32 * 3), ("block", C.c_uint32 * 3),
                ("instr_index", C.c_uint64), ("code", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("modules_loaded", "functions_resolved", "launches", "allocs", "frees",
                                          "bytes_h2d", "bytes_d2h", "launch_log_size", "events_size",
                                          "gpu_kernel_launches")]


class PlanDesc(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("n", "a_total", "a0", "a_count", "full", "features", "batch", "chunks",
                                         "slots", "pair_stride", "graph")]


class TraceDesc(C.Structure):
    _fields_ = [("img", C.c_void_p), ("n", C.c_int32), ("a0", C.c_int32), ("a_count", C.c_int32),
                ("full", C.c_int32), ("ctab", C.c_void_p), ("stab", C.c_void_p), ("wtab", C.c_void_p),
                ("out", C.c_void_p), ("med", C.c_void_p), ("sampler", C.c_int32), ("pair_stride", C.c_int32),
                ("batch", C.c_int32), ("_pad2", C.c_int32), ("img_stride", C.c_int64), ("wsoa", C.c_void_p),
                ("partner_row", C.c_int32), ("flags", C.c_int32), ("circ", C.c_void_p)]


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 64), ("offset", C.c_uint64)]


ARG_I32, ARG_I64, ARG_F32, ARG_F64, ARG_PTR = range(5)

lib = C.CDLL(LIB_PATH)

_S = C.c_int  # tt_status
_sigs = {
    "tt_abi_version": (C.c_int, []),
    "tt_device_count": (_S, [C.POINTER(C.c_int)]),
    "tt_last_error": (C.c_char_p, [C.c_void_p]),
    "tt_native_kernels": (_S, [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tt_ctx_create": (_S, [C.c_int, C.POINTER(Caps), C.POINTER(C.c_void_p)]),
    "tt_ctx_destroy": (_S, [C.c_void_p]),
    "tt_ctx_release": (None, [C.c_void_p]),
    "tt_ctx_id": (_S, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "tt_ctx_synchronize": (_S, [C.c_void_p]),
    "tt_ctx_stream": (_S, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "tt_ctx_device": (_S, [C.c_void_p, C.POINTER(C.c_int)]),
    "tt_ctx_set_sampler": (_S, [C.c_void_p, C.c_int]),
    "tt_module_load": (_S, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(Handle)]),
    "tt_module_unload": (_S, [C.c_void_p, Handle]),
    "tt_get_function": (_S, [C.c_void_p, Handle, C.c_char_p, C.POINTER(Handle)]),
    "tt_mem_alloc": (_S, [C.c_void_p, C.c_uint64, C.POINTER(DevPtr)]),
    "tt_mem_free": (_S, [C.c_void_p, DevPtr]),
    "tt_memcpy_htod": (_S, [C.c_void_p, DevPtr, C.c_void_p, C.c_uint64]),
    "tt_memcpy_dtoh": (_S, [C.c_void_p, C.c_void_p, DevPtr, C.c_uint64]),
    "tt_mem_device_pointer": (_S, [C.c_void_p, DevPtr, C.POINTER(C.c_void_p)]),
    "tt_host_alloc": (_S, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "tt_host_free": (_S, [C.c_void_p]),
    "tt_launch": (_S, [C.c_void_p, Handle, C.POINTER(Grid), C.POINTER(Arg), C.c_int, C.POINTER(Trap)]),
    "tt_counters_get": (_S, [C.c_void_p, C.POINTER(Counters)]),
    "tt_counters_json": (_S, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tt_events": (_S, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tt_make_tables": (_S, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tt_synth_image": (_S, [C.c_int, C.c_uint64, C.c_int, C.c_void_p]),
    "tt_schedule_slots": (C.c_int, [C.c_int, C.c_int]),
    "tt_max_full_n": (C.c_int, []),
    "tt_count_inbounds_taps": (C.c_uint64, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_prep_side": (C.c_int, [C.c_int, C.c_int]),
    "tt_prep_device": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_pnm_read": (_S, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p,
                         C.c_size_t]),
    "tt_pgm_write": (_S, [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_float]),
    "tt_ffma_probe": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "tt_tld4_probe": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "tt_trace_device": (_S, [C.POINTER(TraceDesc), C.c_void_p]),
    "tt_weights_soa": (_S, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_ipc_export": (_S, [C.c_void_p, C.POINTER(IpcHandle)]),
    "tt_ipc_import": (_S, [C.POINTER(IpcHandle), C.c_int, C.POINTER(C.c_void_p)]),
    "tt_ipc_close": (_S, [C.c_void_p]),
    "tt_ipc_alloc": (_S, [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]),
    "tt_ipc_free": (_S, [C.c_void_p]),
    "tt_circus_device": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_circus_fft_device": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_image_tex_create": (_S, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tt_image_atlas_create": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tt_image_tex_update": (_S, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "tt_image_tex_destroy": (_S, [C.c_void_p]),
    "tt_trace_device_tex": (_S, [C.POINTER(TraceDesc), C.c_void_p, C.c_void_p]),
    "tt_jit_source": (_S, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tt_vptx_body_fingerprint": (_S, [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(C.c_uint64)]),
    "tt_hermite_device": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tt_orthonormal_side": (C.c_int, [C.c_int]),
    "tt_orthonormal_device": (_S, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "tt_plan_create": (_S, [C.c_void_p, C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]),
    "tt_plan_run": (_S, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tt_plan_submit": (_S, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tt_plan_wait": (_S, [C.c_void_p]),
    "tt_plan_chunks": (_S, [C.c_void_p, C.POINTER(C.c_int)]),
    "tt_plan_captures": (_S, [C.c_void_p, C.POINTER(C.c_int)]),
    "tt_plan_destroy": (_S, [C.c_void_p]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)
