"""B200-native trace transform (arXiv 1604.03410 §7) behind the gridjit
driver/launch API.

The compute path is the sm_100a CUDA library ``libtt_b200.so`` (C ABI:
include/tt_b200.h).  This module is the Python mirror of the reference's host
API — ``DeviceContext`` / ``create_context`` (driver.hpp:112,332),
``cuda_launch`` / ``cu_in`` / ``cu_out`` / ``cu_inout`` (autolaunch.hpp:109-245)
and the exception taxonomy (errors.hpp) — used by the tests and the
benchmark.  C++ callers use include/tt/gridjit_b200.hpp instead.

There is no CPU fallback: importing works without a GPU (so the library can
be introspected), but every device operation raises ``CudaError`` when no
CUDA device is present, and a missing library raises at import.
"""
from ._lib import LIB_PATH, lib  # noqa: F401  (raises if the .so is missing)
from .api import (  # noqa: F401
    ArgumentMismatch, ArityError, CacheStats, ContextDestroyed, CudaError, DevicePtr, DeviceContext, Direction,
    DoubleFree, Error, FunctionHandle, FunctionNotFound, GridConfig, KernelAst, KernelArg, LaunchConfigError,
    LaunchReport, LaunchResult, ModuleHandle, OutOfBounds, TrapInfo, UseAfterFree, ValidationFailed,
    VptxSyntaxError, cache_stats, create_context, cu_in, cu_inout, cu_out, cuda_launch, device_count,
    native_kernels, parse_kernel, render_module,
)
from .trace import (  # noqa: F401
    CIRCUS, CIRCUS_FFT, DISK, PHANTOM, SEEDS, SPARSE, Plan, TRACE_T05, TRACE_T05_BATCH, RADON, TraceTransform, circus, circus_device, circus_fft, circus_fft_device, make_tables,
    ipc_close, ipc_export, ipc_import, max_full_n, prep_device, prep_side, read_pnm, write_pgm, schedule_slots, synth_image, trace_device, weights_soa,
    HERMITE, ORTHONORMAL, hermite, hermite_device, orthonormal_device, orthonormal_image, orthonormal_side,
)
