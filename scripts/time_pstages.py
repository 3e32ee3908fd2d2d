"""Device time of the sinogram consumers on C2-shaped rows (CUDA events, median of 20): the circus
(P1..P3), the spectral P-functional, the Hermite P-functionals (4 and 8 orders) and the orthonormal
frame.  One JSON line per stage."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402

n, A = int(os.environ.get("TT_N", "1024")), int(os.environ.get("TT_A", "720"))
rows = A * 6
sino = torch.rand((rows, n), device="cuda")
circ = torch.empty((rows, 3), device="cuda")
pf = torch.empty(rows, dtype=torch.float64, device="cuda")
hp = torch.empty((rows, 8), dtype=torch.float64, device="cuda")
cen = torch.empty(rows, dtype=torch.int32, device="cuda")
pic = torch.rand((600, 800), device="cuda")
frame = torch.empty((A, A), device="cuda")
stages = {
    "circus P1-P3": lambda: tt.circus_device(sino.data_ptr(), n, rows, circ.data_ptr()),
    "spectral P |F|^4": lambda: tt.circus_fft_device(sino.data_ptr(), n, rows, pf.data_ptr()),
    "Hermite 4 orders": lambda: tt.hermite_device(sino.data_ptr(), n, rows, 4, hp.data_ptr(), cen.data_ptr()),
    "Hermite 8 orders": lambda: tt.hermite_device(sino.data_ptr(), n, rows, 8, hp.data_ptr(), cen.data_ptr()),
    "orthonormal frame 600x800 -> AxA": lambda: tt.orthonormal_device(pic.data_ptr(), 600, 800, A, frame.data_ptr()),
}
for name, fn in stages.items():
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"stage": name, "n": n, "rows": rows, "median_ms": ts[len(ts) // 2]}), flush=True)
