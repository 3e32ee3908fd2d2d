"""The multi-GPU public call (paper_1604_03410_b200.sharded.ShardedTrace) with
2 and 4 ranks on one GPU (gloo for the collectives, CUDA IPC for the P2P row
stores -- the same mechanism as peer access over NVLink between GPUs): the
host-to-host path (rank 0 upload + broadcast, chunked shard kernels writing
into rank 0's sinogram, per-chunk signals, chunked downloads) and the
device-resident path must both equal one single-GPU launch bit for bit, over
several consecutive overlapped submissions.  The same with assembly="gather"
(local shard blocks + one all-gather per step, the north_star's NCCL-gather
form and the fallback when the IPC mapping fails)."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, A, chunks, result, full=True, assembly="p2p"):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1604_03410_b200 as tt
    from paper_1604_03410_b200.sharded import ShardedTrace

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    F = 6 if full else 1
    # T0 at n > 704: the TMA tile kernel (explicitly: the default keeps launches this short on TLD4)
    st = ShardedTrace(n, A, dist, 0, chunks=chunks, full=full, assembly=assembly, sampler=None if full else 2)
    ok = st.assembly == assembly
    imgs = [tt.synth_image(kind, n) for kind in (tt.PHANTOM, tt.DISK, tt.SPARSE)]
    root = rank == 0
    hi = [torch.from_numpy(im).pin_memory() for im in imgs] if root else [None] * 3
    ho = [torch.full((A, F, n), float("nan")).pin_memory() for _ in imgs] if root else [None] * 3
    hm = [torch.full((A, 2, n), -1, dtype=torch.int32).pin_memory() for _ in imgs] if root else [None] * 3
    for i in range(3):  # consecutive submissions overlap (two image / output slots)
        st.submit(hi[i], ho[i], hm[i])
    st.wait()
    if root:
        ctx = tt.create_context(0)
        for i, im in enumerate(imgs):
            ref, rmed, rep = tt.TraceTransform(ctx, n, A, full=full)(im)
            ok &= rep.ok() and np.array_equal(ho[i].numpy().reshape(-1).view(np.uint32), ref.reshape(-1).view(np.uint32))
            if full:
                ok &= np.array_equal(hm[i].numpy(), rmed)
        ctx.destroy()
    # device-resident leg: image already in slot 0 on every rank
    st.img[0].copy_(torch.from_numpy(imgs[1]))
    torch.cuda.synchronize()
    st.run_device()
    st.wait()
    dist.barrier()
    if root:
        ctx = tt.create_context(0)
        ref, rmed, _ = tt.TraceTransform(ctx, n, A, full=full)(imgs[1])
        ok &= np.array_equal(st.out.cpu().numpy().reshape(-1).view(np.uint32), ref.reshape(-1).view(np.uint32))
        if full:
            ok &= np.array_equal(st.med.cpu().numpy(), rmed)
        ctx.destroy()
        result.put(bool(ok))
    st.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,A,chunks,full,assembly", [
    (2, 256, 40, 3, True, "p2p"), (4, 512, 24, 2, True, "p2p"), (3, 128, 18, 4, True, "p2p"),
    (2, 1024, 16, 2, False, "p2p"),
    (2, 256, 40, 3, True, "gather"), (4, 512, 24, 2, True, "gather"), (2, 1024, 16, 2, False, "gather")])
def test_sharded_trace_equals_one_launch(gpu, world, n, A, chunks, full, assembly):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, A, chunks, q, full, assembly)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=10) is True
