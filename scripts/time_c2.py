"""Time the fused kernel on C2 (or TT_N/TT_A) with CUDA events; prints one JSON line.
Use TT_LIB_PATH to time an experimental library variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402
from paper_1604_03410_b200.trace import image_texture  # noqa: E402

n = int(os.environ.get("TT_N", "1024"))
A = int(os.environ.get("TT_A", "720"))
c, s, w = tt.make_tables(n, A)
img = torch.from_numpy(tt.synth_image(tt.DISK, n)).cuda()
ct, st, wt = (torch.from_numpy(x).cuda() for x in (c, s, w))
out = torch.empty((A, 6, n), device="cuda")
med = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
wsoa = torch.empty(6 * n, device="cuda")
tt.weights_soa(wt.data_ptr(), n, wsoa.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
flush = torch.empty(64 << 20, device="cuda")
stream = torch.cuda.Stream()
sp = stream.cuda_stream
tex = image_texture(img.data_ptr(), n, sp)
ts = []
for i in range(25):
    with torch.cuda.stream(stream):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                    med.data_ptr(), stream=sp, tex=tex, wsoa_ptr=wsoa.data_ptr())
    e1.record(stream)
    e1.synchronize()
    if i >= 5:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"lib": os.environ.get("TT_LIB_PATH", "default"), "n": n, "A": A, "median_ms": ts[len(ts) // 2],
                  "min_ms": ts[0], "checksum": float(out.double().sum())}))
