"""Bit-exact parity against the replay oracle at large and ragged n (4097..16384, 2 angles, both samplers)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
import paper_1604_03410_b200 as tt
ctx = tt.create_context(0)
res = []
for n in (4097, 5000, 6000, 8192, 10000, 12345, 16384):
    for sampler in (0, 1):
        ctx.set_sampler(sampler)
        img = tt.synth_image(tt.PHANTOM, n, 99 + n)
        tr = tt.TraceTransform(ctx, n, 2, full=True)
        out, med, rep = tr(img)
        ref, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY)
        res.append((n, sampler, bool(rep.ok() and np.array_equal(out.view(np.uint32), ref.view(np.uint32)) and np.array_equal(med, rmed))))
print(json.dumps({"configs": len(res), "all_exact": all(r[2] for r in res), "bad": [r for r in res if not r[2]]}))
