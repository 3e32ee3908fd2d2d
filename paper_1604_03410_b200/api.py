"""Python mirror of the reference host API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/gridjit/{driver,autolaunch,errors,emulator}.hpp
so the tests read like the reference's test_driver.cpp / test_autolaunch.cpp.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import re
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib


# --------------------------------------------------------------- errors.hpp

class Error(RuntimeError):
    """gridjit::Error (errors.hpp:14)."""


class VptxSyntaxError(Error): pass        # errors.hpp:97
class ContextDestroyed(Error): pass       # errors.hpp:106
class ValidationFailed(Error): pass       # errors.hpp:111
class FunctionNotFound(Error): pass       # errors.hpp:125
class OutOfBounds(Error): pass            # errors.hpp:130
class DoubleFree(Error): pass             # errors.hpp:135
class UseAfterFree(Error): pass           # errors.hpp:140
class ArgumentMismatch(Error): pass       # errors.hpp:145
class LaunchConfigError(Error): pass      # errors.hpp:150
class ArityError(Error): pass             # errors.hpp:46
class CudaError(Error): pass              # CUDA runtime failure (no emulator analogue)
class AbiError(Error): pass               # misuse of the C ABI


_STATUS = {1: ContextDestroyed, 2: VptxSyntaxError, 3: ValidationFailed, 4: FunctionNotFound, 5: OutOfBounds,
           6: DoubleFree, 7: UseAfterFree, 8: ArgumentMismatch, 9: LaunchConfigError, 10: ArityError,
           11: CudaError, 12: AbiError}


def _check(status: int, ctx_ptr=None) -> None:
    if status == 0:
        return
    msg = lib.tt_last_error(ctx_ptr)
    raise _STATUS.get(status, Error)(msg.decode() if msg else f"status {status}")


# ----------------------------------------------------------- handle types

@dataclass(frozen=True)
class ModuleHandle:  # driver.hpp:31
    ctx_id: int
    id: int


@dataclass(frozen=True)
class FunctionHandle:  # driver.hpp:38
    ctx_id: int
    id: int


@dataclass(frozen=True)
class DevicePtr:  # driver.hpp:45
    base: int
    length: int
    ctx_id: int

    def _c(self):
        return _lib.DevPtr(self.base, self.length, self.ctx_id)


@dataclass
class GridConfig:  # emulator.hpp:42
    grid: tuple = (1, 1, 1)
    block: tuple = (1, 1, 1)
    shared_bytes_extra: int = 0

    def _c(self):
        g = _lib.Grid()
        for i in range(3):
            g.grid[i] = int(self.grid[i])
            g.block[i] = int(self.block[i])
        g.shared_bytes_extra = int(self.shared_bytes_extra)
        return g


class TrapKind(enum.IntEnum):  # emulator.hpp:61-68
    GlobalOutOfBounds = 0
    SharedOutOfBounds = 1
    UseOfFreedMemory = 2
    DivisionByZero = 3
    BarrierDivergence = 4
    ExplicitTrap = 5


@dataclass
class TrapInfo:  # emulator.hpp:60
    kind: TrapKind
    thread: tuple
    block: tuple
    instr_index: int = 0
    code: int = 0


@dataclass
class LaunchResult:  # emulator.hpp:99
    trap: TrapInfo | None = None

    def ok(self) -> bool:
        return self.trap is None


# Scalar launch arguments carry their type (LaunchArg variant, driver.hpp:52).
_SCALARS = {np.int32: _lib.ARG_I32, np.int64: _lib.ARG_I64, np.float32: _lib.ARG_F32, np.float64: _lib.ARG_F64}
_SIG_NAME = {np.int32: "i32", np.int64: "i64", np.float32: "f32", np.float64: "f64"}


def _to_c_arg(a) -> _lib.Arg:
    r = _lib.Arg()
    if isinstance(a, DevicePtr):
        r.kind = _lib.ARG_PTR
        r.v.ptr = a._c()
        return r
    if isinstance(a, (np.integer, np.floating)):
        t = type(a)
        if t not in _SCALARS:
            raise ArgumentMismatch(f"ArgumentMismatch: unsupported scalar type {t.__name__}")
        r.kind = _SCALARS[t]
        setattr(r.v, {0: "i32", 1: "i64", 2: "f32", 3: "f64"}[r.kind], a.item())
        return r
    if isinstance(a, bool) or not isinstance(a, (int, float)):
        raise ArgumentMismatch(f"ArgumentMismatch: unsupported launch argument {a!r}")
    # bare Python numbers: int -> i32 (i64 if it does not fit), float -> f64
    if isinstance(a, int):
        return _to_c_arg(np.int32(a) if -2**31 <= a < 2**31 else np.int64(a))
    return _to_c_arg(np.float64(a))


class _HostView:
    """(pointer, nbytes) of a host buffer; numpy arrays are used in place."""

    def __init__(self, buf, writable: bool):
        if isinstance(buf, np.ndarray):
            if not buf.flags.c_contiguous:
                raise AbiError("host buffers must be C-contiguous")
            if writable and not buf.flags.writeable:
                raise AbiError("destination buffer is read-only")
            self.ptr, self.nbytes, self.keep = buf.ctypes.data, buf.nbytes, buf
        elif isinstance(buf, (bytes, bytearray)):
            arr = np.frombuffer(buf, np.uint8) if isinstance(buf, bytes) else np.frombuffer(buf, np.uint8)
            self.ptr, self.nbytes, self.keep = arr.ctypes.data if arr.size else None, arr.size, arr
        elif isinstance(buf, int):
            self.ptr, self.nbytes, self.keep = buf, None, None
        else:
            raise AbiError(f"unsupported host buffer {type(buf).__name__}")


# ----------------------------------------------------------- driver.hpp

class MethodCache:  # driver.hpp:101-110
    def __init__(self):
        self.entries: dict[str, tuple[ModuleHandle, FunctionHandle]] = {}
        self.hits = 0
        self.misses = 0
        self.compiles = 0


class DeviceContext:
    """CUDA-backed DeviceContext (driver.hpp:112-330): one GPU, one stream."""

    def __init__(self, device: int = 0, caps: tuple | None = None):
        p = C.c_void_p()
        c = _lib.Caps(*caps) if caps is not None else None
        _check(lib.tt_ctx_create(device, C.byref(c) if c is not None else None, C.byref(p)))
        self._p = p
        self._destroyed = False
        self._cache = MethodCache()
        cid = C.c_uint64()
        _check(lib.tt_ctx_id(self._p, C.byref(cid)), self._p)
        self._id = cid.value
        self.device = device

    # lifecycle ---------------------------------------------------------
    @property
    def id(self) -> int:
        return self._id

    def destroy(self) -> None:
        _check(lib.tt_ctx_destroy(self._p), self._p)
        self._destroyed = True

    def destroyed(self) -> bool:
        return self._destroyed

    def __del__(self):
        p = getattr(self, "_p", None)
        if p:
            lib.tt_ctx_release(p)
            self._p = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if not self._destroyed:
            self.destroy()

    # modules -------------------------------------------------------------
    def module_load(self, text: str) -> ModuleHandle:
        b = text.encode()
        h = _lib.Handle()
        _check(lib.tt_module_load(self._p, b, len(b), C.byref(h)), self._p)
        return ModuleHandle(h.ctx_id, h.id)

    def module_unload(self, m: ModuleHandle) -> None:
        _check(lib.tt_module_unload(self._p, _lib.Handle(m.ctx_id, m.id)), self._p)

    def get_function(self, m: ModuleHandle, name: str) -> FunctionHandle:
        h = _lib.Handle()
        _check(lib.tt_get_function(self._p, _lib.Handle(m.ctx_id, m.id), name.encode(), C.byref(h)), self._p)
        return FunctionHandle(h.ctx_id, h.id)

    # memory ----------------------------------------------------------------
    def mem_alloc(self, nbytes: int) -> DevicePtr:
        d = _lib.DevPtr()
        _check(lib.tt_mem_alloc(self._p, int(nbytes), C.byref(d)), self._p)
        return DevicePtr(d.base, d.length, d.ctx_id)

    def mem_free(self, p: DevicePtr) -> None:
        _check(lib.tt_mem_free(self._p, p._c()), self._p)

    def memcpy_htod(self, dst: DevicePtr, src, nbytes: int | None = None) -> None:
        hv = _HostView(src, writable=False)
        n = hv.nbytes if nbytes is None else int(nbytes)
        if hv.nbytes is not None and n > hv.nbytes:
            raise AbiError("copy larger than the host buffer")
        _check(lib.tt_memcpy_htod(self._p, dst._c(), hv.ptr, n), self._p)

    def memcpy_dtoh(self, dst, src: DevicePtr, nbytes: int | None = None) -> None:
        hv = _HostView(dst, writable=True)
        n = (hv.nbytes if hv.nbytes is not None else src.length) if nbytes is None else int(nbytes)
        if hv.nbytes is not None and n > hv.nbytes:
            raise AbiError("copy larger than the host buffer")
        _check(lib.tt_memcpy_dtoh(self._p, hv.ptr, src._c(), n), self._p)

    def device_pointer(self, p: DevicePtr) -> int:
        out = C.c_void_p()
        _check(lib.tt_mem_device_pointer(self._p, p._c(), C.byref(out)), self._p)
        return out.value or 0

    @property
    def stream(self) -> int:
        out = C.c_void_p()
        _check(lib.tt_ctx_stream(self._p, C.byref(out)), self._p)
        return out.value or 0

    def set_sampler(self, sampler: int) -> None:
        """0 = global/L1 loads, 1 = texture gather, 2 = TMA tiles for the T0 launches they serve, 3 (default)
        = TMA tiles for T0 launches of >= 1.5e8 taps, the texture gather otherwise (trace kernels only)."""
        _check(lib.tt_ctx_set_sampler(self._p, int(sampler)), self._p)

    def synchronize(self) -> None:
        _check(lib.tt_ctx_synchronize(self._p), self._p)

    # launch ------------------------------------------------------------------
    def launch(self, fn: FunctionHandle, cfg: GridConfig, args: list) -> LaunchResult:
        n = len(args)
        arr = (_lib.Arg * max(n, 1))(*[_to_c_arg(a) for a in args])
        g = cfg._c()
        t = _lib.Trap()
        _check(lib.tt_launch(self._p, _lib.Handle(fn.ctx_id, fn.id), C.byref(g), arr, n, C.byref(t)), self._p)
        if not t.trapped:
            return LaunchResult(None)
        return LaunchResult(TrapInfo(TrapKind(t.kind), tuple(t.thread), tuple(t.block), t.instr_index, t.code))

    # introspection -------------------------------------------------------------
    def counters(self) -> dict:
        c = _lib.Counters()
        _check(lib.tt_counters_get(self._p, C.byref(c)), self._p)
        d = {k: getattr(c, k) for k, _ in _lib.Counters._fields_}
        d["launch_log"] = self.counters_json()["launch_log"]
        d["events"] = self.events()
        return d

    def counters_json(self) -> dict:
        need = C.c_size_t()
        _check(lib.tt_counters_json(self._p, None, 0, C.byref(need)), self._p)
        buf = C.create_string_buffer(need.value)
        _check(lib.tt_counters_json(self._p, buf, need.value, C.byref(need)), self._p)
        return json.loads(buf.value.decode())

    EVENTS = ("ModuleLoad", "FunctionResolve", "Alloc", "Free", "H2D", "D2H", "Launch")

    def events(self) -> list[str]:
        need = C.c_size_t()
        _check(lib.tt_events(self._p, None, 0, C.byref(need)), self._p)
        buf = (C.c_uint8 * max(need.value, 1))()
        _check(lib.tt_events(self._p, buf, need.value, C.byref(need)), self._p)
        return [self.EVENTS[buf[i]] for i in range(need.value)]

    def method_cache(self) -> MethodCache:
        if self._destroyed:
            raise ContextDestroyed("ContextDestroyed: operation on a destroyed context")
        return self._cache


def create_context(device: int = 0, caps: tuple | None = None) -> DeviceContext:  # driver.hpp:332
    return DeviceContext(device, caps)


def device_count() -> int:
    n = C.c_int()
    st = lib.tt_device_count(C.byref(n))
    return n.value if st == 0 else 0


def native_kernels() -> list[str]:
    need = C.c_size_t()
    _check(lib.tt_native_kernels(None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(lib.tt_native_kernels(buf, need.value, C.byref(need)))
    return [s for s in buf.value.decode().splitlines() if s]


# -------------------------------------------------------- autolaunch.hpp

class Direction(enum.Enum):  # autolaunch.hpp:33
    In = "in"
    Out = "out"
    InOut = "inout"


@dataclass
class KernelArg:  # autolaunch.hpp:46-107
    value: object
    direction: Direction = Direction.InOut

    @property
    def is_array(self) -> bool:
        return isinstance(self.value, np.ndarray)


def cu_in(a: np.ndarray) -> KernelArg:
    return KernelArg(a, Direction.In)


def cu_out(a: np.ndarray) -> KernelArg:
    return KernelArg(a, Direction.Out)


def cu_inout(a: np.ndarray) -> KernelArg:
    return KernelArg(a, Direction.InOut)


@dataclass
class KernelAst:
    """The launchable identity of a kernel: name + ordered parameter names.

    The reference's KernelAst (ast.hpp) carries a DSL body that its JIT
    compiles; here the body is bound to a native sm_100a kernel registered for
    the specialized signature, so only the header matters."""
    name: str
    params: list = field(default_factory=list)


_KHDR = re.compile(r"kernel\s+([A-Za-z_]\w*)\s*\(([^)]*)\)")


def parse_kernel(source: str) -> KernelAst:
    """Header of a gridjit DSL kernel (grammar.md: `kernel name(a, b) {...}`)."""
    src = "\n".join(line.split("#", 1)[0] for line in source.splitlines())
    m = _KHDR.search(src)
    if not m:
        raise Error("SyntaxError: no kernel definition found")
    params = [p.strip() for p in m.group(2).split(",") if p.strip()]
    return KernelAst(m.group(1), params)


def _arg_type(a: KernelArg) -> tuple[bool, str]:
    v = a.value
    if isinstance(v, np.ndarray):
        t = v.dtype.type
        if t not in _SIG_NAME:
            raise ArgumentMismatch(f"ArgumentMismatch: arrays must be i32/i64/f32/f64, got {v.dtype}")
        return True, _SIG_NAME[t]
    if isinstance(v, (np.integer, np.floating)) and type(v) in _SIG_NAME:
        return False, _SIG_NAME[type(v)]
    if isinstance(v, int) and not isinstance(v, bool):
        return False, "i32" if -2**31 <= v < 2**31 else "i64"
    if isinstance(v, float):
        return False, "f64"
    raise ArgumentMismatch(f"ArgumentMismatch: kernel arguments must be i32/i64/f32/f64, got {v!r}")


def render_module(kernel: KernelAst, types: list[tuple[bool, str]], module_name: str) -> str:
    """The VPTX module header a compile of this signature produces (vptx.hpp:327-340)."""
    ps = ", ".join(f".param {'ptr.global.' + t if is_ptr else t} {name}"
                   for (is_ptr, t), name in zip(types, kernel.params))
    return f".module {module_name}\n.kernel {kernel.name}({ps}) {{\n  ret\n}}\n"


def _fnv1a(s: str) -> str:  # Signature::hash, types.hpp:115-122
    h = 14695981039346656037
    for ch in s.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@dataclass
class LaunchReport:  # autolaunch.hpp:123-150
    kernel: str
    signature: str
    cache_hit: bool = False
    bytes_h2d: int = 0
    bytes_d2h: int = 0
    trap: TrapInfo | None = None

    def ok(self) -> bool:
        return self.trap is None

    def to_json(self) -> dict:
        j = {"kernel": self.kernel, "signature": self.signature, "cache_hit": self.cache_hit,
             "bytes_h2d": self.bytes_h2d, "bytes_d2h": self.bytes_d2h, "trap": None}
        if self.trap is not None:
            j["trap"] = {"kind": self.trap.kind.name, "block": list(self.trap.block),
                         "thread": list(self.trap.thread), "instr": self.trap.instr_index, "code": self.trap.code}
        return j


@dataclass
class CacheStats:  # autolaunch.hpp:152-157
    entries: int
    hits: int
    misses: int
    compiles: int


def cache_stats(ctx: DeviceContext) -> CacheStats:
    c = ctx.method_cache()
    return CacheStats(len(c.entries), c.hits, c.misses, c.compiles)


def cuda_launch(ctx: DeviceContext, kernel: KernelAst, cfg: GridConfig, args: list) -> LaunchReport:
    """One-call launch (autolaunch.hpp:167-245): signature -> method cache
    (compile = bind once per signature) -> alloc, upload In/InOut, launch,
    download Out/InOut (skipped on a trap), free."""
    if len(args) != len(kernel.params):
        raise ArityError(f"ArityError: kernel '{kernel.name}' expects {len(kernel.params)} argument(s), "
                         f"got {len(args)}")
    kargs = [a if isinstance(a, KernelArg) else KernelArg(a, Direction.InOut) for a in args]
    types = [_arg_type(a) for a in kargs]
    key = kernel.name + "(" + ",".join(t + ("[]" if p else "") for p, t in types) + ")"
    rep = LaunchReport(kernel.name, key)
    cache = ctx.method_cache()
    hit = cache.entries.get(key)
    if hit is not None:
        cache.hits += 1
        rep.cache_hit = True
        fn = hit[1]
    else:
        cache.misses += 1
        cache.compiles += 1
        mh = ctx.module_load(render_module(kernel, types, f"{kernel.name}${_fnv1a(key)}"))
        fn = ctx.get_function(mh, kernel.name)
        cache.entries[key] = (mh, fn)

    buffers, raw = [], []
    try:
        for a, (is_ptr, t) in zip(kargs, types):
            if not is_ptr:
                v = a.value
                raw.append(v if isinstance(v, (np.integer, np.floating)) else
                           {"i32": np.int32, "i64": np.int64, "f64": np.float64}[t](v))
                continue
            arr = a.value
            p = ctx.mem_alloc(arr.nbytes)
            buffers.append((p, a))
            if a.direction != Direction.Out:
                ctx.memcpy_htod(p, np.ascontiguousarray(arr), arr.nbytes)
                rep.bytes_h2d += arr.nbytes
            raw.append(p)
        res = ctx.launch(fn, cfg, raw)
        rep.trap = res.trap
        if res.ok():
            for p, a in buffers:
                if a.direction != Direction.In:
                    ctx.memcpy_dtoh(a.value, p, a.value.nbytes)
                    rep.bytes_d2h += a.value.nbytes
    finally:
        for p, _ in buffers:
            ctx.mem_free(p)
    return rep
