"""Row (e) host logic on CPU: orientation shards with mirror halves, the
all-gather + reassembly, and image-batch shards, exercised by a world_size-2
gloo process group.  The per-rank compute is the oracle's replay of the
kernel's shard launch (bit-exact stand-in for the GPU on a CPU-only box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1604_03410_b200 import shard


def test_orientation_shards_partition_the_angle_set():
    for A in (2, 8, 360, 720, 1440, 2880):
        for G in (1, 2, 3, 4, 8):
            rows = [a for r in range(G) for a in shard.shard_rows(A, G, r)]
            assert sorted(rows) == list(range(A))
    with pytest.raises(ValueError):
        shard.orientation_shard(7, 2, 0)


def test_assemble_reorders_rank_blocks_into_angle_order():
    A, G = 16, 4
    blocks = [torch.tensor(shard.shard_rows(A, G, r), dtype=torch.float32)[:, None] for r in range(G)]
    full = shard.assemble(torch.cat(blocks), A, G)
    assert full[:, 0].tolist() == list(range(A))


def test_image_shards_cover_the_batch():
    for B, G in ((4096, 8), (10, 3), (1, 2)):
        got = []
        for r in range(G):
            lo, cnt = shard.image_shard(B, G, r)
            got += list(range(lo, lo + cnt))
        assert got == list(range(B))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, A = 48, 16
        img = O.synth(O.PHANTOM, n)
        c, s, w = O.tables(n, A)
        a0, cnt, h = shard.orientation_shard(A, world, rank)
        out, med = O.replay_launch(img, n, c, s, w, a0=a0, units=cnt, pair_stride=h)
        sino = shard.gather_sinograms(torch.from_numpy(out), A, dist)
        meds = shard.gather_sinograms(torch.from_numpy(med), A, dist)
        if rank == 0:
            whole, wmed = O.replay_launch(img, n, c, s, w, a0=0, units=h, pair_stride=h)
            ok = np.array_equal(sino.numpy().view(np.uint32), whole.view(np.uint32)) and \
                np.array_equal(meds.numpy(), wmed)
            q.put(ok)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_orientation_gather_is_bit_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def _init_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    os.environ.pop("TORCH_NCCL_ASYNC_ERROR_HANDLING", None)
    from paper_1604_03410_b200.sharded import chunk_bounds, init_process_group
    d = init_process_group("gloo", timeout_s=60)
    t = torch.ones(1)
    w = d.all_reduce(t, async_op=True)
    w.wait()
    ok = t.item() == world and os.environ["TORCH_NCCL_ASYNC_ERROR_HANDLING"] == "1"
    # chunk bounds partition every shard
    for cnt in (0, 1, 5, 90):
        for ch in (1, 3, 4):
            got = [u for c in range(ch) for u in range(*chunk_bounds(cnt, ch, c))]
            ok &= got == list(range(cnt))
    q.put(ok)
    d.destroy_process_group()


def test_sharded_init_sets_async_error_handling_and_timeout():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_init_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True and q.get(timeout=5) is True
