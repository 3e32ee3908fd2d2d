"""Small launches of every kernel configuration for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402

ctx = tt.create_context(0)
for sampler in (0, 1, 2):  # 2: TMA-staged tiles for the T0 launches with n > 1024
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

# raw entries: the fused P stage (appended P-CTAs), TMA Radon with a ragged n and an explicit shard,
# Hermite P-functionals and the orthonormal frame
import torch  # noqa: E402

for n, A, pair in [(256, 12, 0), (2048, 4, 0), (256, 16, 8)]:
    c, s, w = tt.make_tables(n, A)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    img, ct, st, wt = d(tt.synth_image(tt.PHANTOM, n)), d(c), d(s), d(w)
    out = torch.empty((A, 6, n), device="cuda")
    med = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
    circ = torch.empty((A, 6, 3), device="cuda")
    tex = tt.trace.image_texture(img.data_ptr(), n)
    tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                    med.data_ptr(), sampler=1, tex=tex, pair_stride=pair, circ_ptr=circ.data_ptr(), fused_p=True)
    torch.cuda.synchronize()
    tt.trace.image_texture_destroy(tex)
    hp = torch.empty((A * 6, 4), dtype=torch.float64, device="cuda")
    cen = torch.empty(A * 6, dtype=torch.int32, device="cuda")
    tt.hermite_device(out.data_ptr(), n, A * 6, 4, hp.data_ptr(), cen.data_ptr())
for n, A, a0, pair in [(1028, 6, 0, 0), (2052, 5, 0, 0), (2048, 8, 2, 8), (2048, 12, 0, 0), (4096, 8, 0, 0)]:
    c, s, w = tt.make_tables(n, 16 if pair else A)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    img, ct, st, wt = d(tt.synth_image(tt.SPARSE, n)), d(c), d(s), d(w)
    out = torch.empty((A if not pair else 8, n), device="cuda")
    tt.trace_device(img.data_ptr(), n, a0, A if not pair else 8, ct.data_ptr(), st.data_ptr(), wt.data_ptr(),
                    out.data_ptr(), 0, full=False, sampler=2, pair_stride=pair)
# texture T0 launches over the clipped tap range (NS >= 16), off-axis angles
for n, A in [(512, 12), (640, 8)]:
    c, s, w = tt.make_tables(n, A)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    img, ct, st, wt = d(tt.synth_image(tt.PHANTOM, n)), d(c), d(s), d(w)
    out = torch.empty((A, n), device="cuda")
    tex = tt.trace.image_texture(img.data_ptr(), n)
    tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(), 0,
                    full=False, sampler=1, tex=tex)
    torch.cuda.synchronize()
    tt.trace.image_texture_destroy(tex)
frame = torch.empty((90, 90), device="cuda")
pic = torch.rand((40, 50), device="cuda")
tt.orthonormal_device(pic.data_ptr(), 40, 50, 90, frame.data_ptr())
torch.cuda.synchronize()
print("sanitize cases done")
