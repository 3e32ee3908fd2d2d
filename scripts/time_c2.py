"""Time the fused kernel on C2 (or TT_N/TT_A; TT_FULL=0 for T0 only) with CUDA events; one JSON line.
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
full = os.environ.get("TT_FULL", "1") == "1"
reps = int(os.environ.get("TT_REPS", "20"))
F = 6 if full else 1
c, s, w = tt.make_tables(n, A)
img = torch.from_numpy(tt.synth_image(tt.DISK, n)).cuda()
ct, st, wt = (torch.from_numpy(x).cuda() for x in (c, s, w))
out = torch.empty((A, F, n), device="cuda")
med = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
wsoa = torch.empty(6 * n, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
stream = torch.cuda.Stream()
sp = stream.cuda_stream
tt.weights_soa(wt.data_ptr(), n, wsoa.data_ptr(), sp)
sampler = int(os.environ.get("TT_SAMPLER_ID", "1"))  # 1 texture gather, 0 LDG
tex = image_texture(img.data_ptr(), n, sp) if sampler == 1 else None
# TT_CIRC=1: circus output with the P stage fused into the trace launch; 2: separate circus launch
circ_mode = os.environ.get("TT_CIRC", "0")
circ = torch.empty((A, F, 3), device="cuda") if circ_mode in ("1", "2") and full else None
ts = []
for i in range(reps + 3):
    with torch.cuda.stream(stream):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                    med.data_ptr() if full else 0, full=full, sampler=sampler, stream=sp, tex=tex,
                    wsoa_ptr=wsoa.data_ptr(), circ_ptr=circ.data_ptr() if circ is not None else 0,
                    fused_p=circ_mode == "1")
    e1.record(stream)
    e1.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"lib": os.environ.get("TT_LIB_PATH", "default"), "n": n, "A": A, "full": full, "sampler": sampler,
                  "median_ms": ts[len(ts) // 2], "min_ms": ts[0], "checksum": float(out.double().sum())}))
