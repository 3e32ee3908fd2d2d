"""Randomised parity stress: many (n, A, image kind, sampler, T0-only/T0-T5) configurations, each
checked bit-exactly against the schedule-replay oracle (and the medians exactly).  Prints one JSON
summary line; exit code 1 on any mismatch.  Usage: python scripts/parity_stress.py [count] [seed]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_1604_03410_b200 as tt  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1604)
ctx = tt.create_context(0)
bad, done = [], 0
for i in range(count):
    n = int(rng.choice([int(rng.integers(1, 160)), int(rng.integers(160, 1100)), int(rng.integers(1100, 3200))],
                       p=[0.3, 0.5, 0.2]))
    A = int(rng.integers(1, 9)) * (2 if rng.random() < 0.8 else 1)
    kind = int(rng.choice([tt.DISK, tt.PHANTOM, tt.SPARSE]))
    full = bool(rng.random() < 0.8)
    # samplers 0 (LDG), 1 (texture), 2 (TMA tiles for the T0 launches they serve, texture otherwise)
    sampler = int(rng.integers(0, 3))
    if not full and sampler == 2 and rng.random() < 0.5:  # bias T0 sizes towards the TMA kernel's range
        n = int(rng.integers(769, 5000)) // 4 * 4
    ctx.set_sampler(sampler)
    # angle sub-ranges (a0, a_count) and image batches (trace_t05_batch) as well
    a0 = int(rng.integers(0, A)) if rng.random() < 0.2 else 0
    a_count = int(rng.integers(1, A - a0 + 1)) if a0 else A
    batch = int(rng.integers(2, 4)) if (full and n <= 1100 and rng.random() < 0.15) else 1
    imgs = [tt.synth_image(kind, n, int(rng.integers(0, 1 << 30))) for _ in range(batch)]
    tr = tt.TraceTransform(ctx, n, A, full=full, a0=a0, a_count=a_count, batch=batch)
    out, med, rep = tr(np.stack(imgs) if batch > 1 else imgs[0])
    ok = rep.ok()
    for b, img in enumerate(imgs):
        ref, rmed, _, _ = O.transform(img, n, tr.ctab, tr.stab, tr.wtab, mode=O.REPLAY, full=full, a0=a0,
                                      a_count=a_count)
        ob = out[b] if batch > 1 else out
        ok = ok and np.array_equal(ob.view(np.uint32), ref.view(np.uint32))
        if full:
            ok = ok and np.array_equal(med[b] if batch > 1 else med, rmed)
    done += 1
    if not ok:
        bad.append({"n": n, "A": A, "a0": a0, "a_count": a_count, "batch": batch, "kind": kind,
                    "sampler": sampler, "full": full})
ctx.destroy()
print(json.dumps({"configs": done, "mismatches": len(bad), "first_bad": bad[:5]}))
sys.exit(1 if bad else 0)
