"""Direct-write orientation shards: two processes on one GPU (CUDA IPC, the
same mechanism as peer access over NVLink between GPUs) each run the fused
kernel on their shard with the output pointing into rank 0's sinogram buffer
(DESIGN.md §3.4).  The assembled sinogram must equal one whole launch bit-for-bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, A, result):
    import torch
    import torch.distributed as dist

    import paper_1604_03410_b200 as tt
    from paper_1604_03410_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    F = 6
    c, s, w = tt.make_tables(n, A)
    img = torch.from_numpy(tt.synth_image(tt.PHANTOM, n)).cuda()
    ct, st, wt = (torch.from_numpy(x).cuda() for x in (c, s, w))
    out = torch.full((A, F, n), float("nan"), device="cuda") if rank == 0 else None
    med = torch.full((A, 2, n), -1, dtype=torch.int32, device="cuda") if rank == 0 else None
    ptrs, close = shard.share_device_buffers([out.data_ptr(), med.data_ptr()] if rank == 0 else [], dist, 0)
    a0, cnt, pair, row0, prow = shard.direct_shard_rows(A, world, rank, F, n)
    tt.trace_device(img.data_ptr(), n, a0, cnt, ct.data_ptr(), st.data_ptr(), wt.data_ptr(),
                    ptrs[0] + row0 * F * n * 4, ptrs[1] + row0 * 2 * n * 4, pair_stride=pair, partner_row=prow,
                    peer_out=rank != 0)
    torch.cuda.synchronize()
    dist.barrier()  # every shard's rows are in rank 0's buffers
    if rank == 0:
        ref = torch.empty((A, F, n), device="cuda")
        rmed = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
        tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), ref.data_ptr(),
                        rmed.data_ptr())
        torch.cuda.synchronize()
        result.put(bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)) and torch.equal(med, rmed)))
    close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,A", [(2, 256, 40), (4, 512, 16)])
def test_direct_write_shards_assemble_the_full_sinogram(gpu, world, n, A):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, A, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=10) is True


def test_ipc_buffer_is_a_dedicated_exportable_allocation(gpu):
    """tt_ipc_alloc buffers (what ShardedTrace exports): zero-filled, viewed by torch without a copy, and
    exported at offset 0 of their own allocation (independent of the caching allocator's blocks)."""
    import torch

    from paper_1604_03410_b200.trace import IpcBuffer, ipc_export

    buf = IpcBuffer(gpu, (3, 5, 7), "float32")
    t = torch.as_tensor(buf, device=f"cuda:{gpu}")
    assert t.shape == (3, 5, 7) and t.data_ptr() == buf.ptr and float(t.abs().sum()) == 0.0
    t.fill_(2.5)
    assert float(torch.as_tensor(buf, device=f"cuda:{gpu}").sum()) == 2.5 * 105
    h = ipc_export(buf.ptr + 4 * 35)  # a pointer inside it: the handle carries the offset
    assert int.from_bytes(h[64:72], "little") == 4 * 35
    del t
    del buf
    torch.cuda.synchronize()
