"""Small launches of every kernel configuration for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402

ctx = tt.create_context(0)
for sampler in (0, 1):
    ctx.set_sampler(sampler)
    for n, A in [(64, 8), (100, 4), (300, 4), (512, 2), (1024, 2), (2048, 2), (4096, 2), (16384, 2)]:
        img = tt.synth_image(tt.PHANTOM, n)
        tr = tt.TraceTransform(ctx, n, A, features=True)
        out, med, rep = tr(img)
        assert rep.ok()
        tt.circus(ctx, out)
        tt.circus_fft(ctx, out)
        r = tt.TraceTransform(ctx, n, A, full=False)(img)
    B = 3
    imgs = np.stack([tt.synth_image(tt.DISK, 128, 20160412 + b) for b in range(B)])
    tt.TraceTransform(ctx, 128, 6, batch=B)(imgs)
ctx.destroy()
print("sanitize cases done")
