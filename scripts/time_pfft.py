"""Time tt_circus_fft_device on the C2 sinogram rows (720 angles x 6 functionals x 1024) and on
4096-length rows; CUDA events on the launching stream.  One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402

for n, rows in ((1024, 720 * 6), (4096, 1440 * 6), (1000, 720 * 6)):
    s = torch.rand(rows, n, device="cuda")
    p = torch.empty(rows, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        tt.circus_fft_device(s.data_ptr(), n, rows, p.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tt.circus_fft_device(s.data_ptr(), n, rows, p.data_ptr(), st)
    e1.record()
    e1.synchronize()
    print(json.dumps({"n": n, "rows": rows, "ms": e0.elapsed_time(e1) / 10}))
