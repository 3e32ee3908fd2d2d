"""Time tt.Plan.run (host-to-host, pinned buffers) on C2 for several chunk counts."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402
from paper_1604_03410_b200._lib import lib  # noqa: E402

n, A = int(os.environ.get("TT_N", "1024")), int(os.environ.get("TT_A", "720"))
ctx = tt.create_context(0)


def pinned(shape, dt):
    p = C.c_void_p()
    assert lib.tt_host_alloc(int(np.prod(shape)) * np.dtype(dt).itemsize, C.byref(p)) == 0
    ct = C.c_float if dt == np.float32 else C.c_int32
    return np.ctypeslib.as_array((ct * int(np.prod(shape))).from_address(p.value)).reshape(shape)


img = pinned((n, n), np.float32)
img[:] = tt.synth_image(tt.DISK, n)
out, med, circ = pinned((A, 6, n), np.float32), pinned((A, 2, n), np.int32), pinned((A, 6, 3), np.float32)
for ch in [1, 2, 3, 5, 8, 12, 16, 24, 32]:
    plan = tt.Plan(ctx, n, A, features=True, chunks=ch)
    for _ in range(3):
        plan.run(img, out, med, circ)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        plan.run(img, out, med, circ)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(json.dumps({"n": n, "A": A, "chunks": plan.chunks, "median_ms": ts[10] * 1e3, "min_ms": ts[0] * 1e3}))
    plan.destroy()
