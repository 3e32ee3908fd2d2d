"""Minimal driver for ncu: launches the fused C2 kernel a few times (device-resident)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402
from paper_1604_03410_b200.trace import image_texture  # noqa: E402

n = int(os.environ.get("TT_N", "1024"))
A = int(os.environ.get("TT_A", "720"))
sampler = int(os.environ.get("TT_SAMPLER_PROF", "0"))
reps = int(os.environ.get("TT_REPS", "3"))
full = os.environ.get("TT_FULL", "1") == "1"
c, s, w = tt.make_tables(n, A)
img = torch.from_numpy(tt.synth_image(tt.DISK, n)).cuda()
ct, st, wt = (torch.from_numpy(x).cuda() for x in (c, s, w))
out = torch.empty((A, 6 if full else 1, n), device="cuda")
med = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
wsoa = torch.empty(6 * n, device="cuda")
tt.weights_soa(wt.data_ptr(), n, wsoa.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
stream = torch.cuda.current_stream().cuda_stream
tex = image_texture(img.data_ptr(), n, stream) if sampler == 1 else None
for _ in range(reps):
    tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                    med.data_ptr(), full=full, sampler=sampler, stream=stream, tex=tex, wsoa_ptr=wsoa.data_ptr())
torch.cuda.synchronize()
print("ok", float(out[:, 0].sum()))
