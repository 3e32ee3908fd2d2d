"""One small TMA-tile Radon launch vs the texture path (debugging aid for sampler 2)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_03410_b200 as tt  # noqa: E402

n, A = int(os.environ.get("TT_N", "2048")), int(os.environ.get("TT_A", "4"))
img = torch.from_numpy(tt.synth_image(tt.PHANTOM, n)).cuda()
c, s, w = (torch.from_numpy(x).cuda() for x in tt.make_tables(n, A))
outs = []
for smp in (2, 1):
    out = torch.full((A, n), float("nan"), device="cuda")
    tt.trace_device(img.data_ptr(), n, 0, A, c.data_ptr(), s.data_ptr(), w.data_ptr(), out.data_ptr(), 0, full=False,
                    sampler=smp)
    torch.cuda.synchronize()
    outs.append(out.cpu().numpy())
same = np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
print("tma == tex:", same, "nan rows:", int(np.isnan(outs[0]).any(axis=1).sum()),
      "max |diff|:", float(np.nanmax(np.abs(outs[0] - outs[1]))))
