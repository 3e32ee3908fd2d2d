"""C3 e2e through tt.Plan at several chunk counts (graph and enqueued): per-step ms of pipelined submits."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_03410_b200 as tt  # noqa: E402

n, A, steps = int(os.environ.get("TT_N", "4096")), int(os.environ.get("TT_A", "1440")), 6
ctx = tt.create_context(0)
img = torch.from_numpy(tt.synth_image(tt.DISK, n)).pin_memory()
out = [torch.empty((A, 6, n)).pin_memory() for _ in range(2)]
med = [torch.empty((A, 2, n), dtype=torch.int32).pin_memory() for _ in range(2)]
for chunks in [int(x) for x in os.environ.get("TT_CHUNKS", "4,8,16,32").split(",")]:
    for graph in (False, True):
        plan = tt.Plan(ctx, n, A, chunks=chunks, graph=graph)
        for i in range(2):
            plan.submit(img.numpy(), out[i % 2].numpy(), med[i % 2].numpy())
        plan.wait()
        t0 = time.perf_counter()
        for i in range(steps):
            plan.submit(img.numpy(), out[i % 2].numpy(), med[i % 2].numpy())
        plan.wait()
        dt = (time.perf_counter() - t0) / steps
        print(json.dumps({"n": n, "A": A, "chunks": plan.chunks, "graph": graph, "ms_per_step": dt * 1e3}), flush=True)
        plan.destroy()
ctx.destroy()
