"""Orientation-sharded trace transform of one image across the GPUs of one node
(DESIGN.md §3.4): the multi-GPU public call.

One process per GPU (torchrun).  Rank r of G owns the orientation shard
``shard.orientation_shard(A, G, r)``: angles [a0, a0+cnt) and their mirrors
[A/2+a0, ...), launched as mirrored pairs (one sampling pass serves both
lines).  The data path of one ``submit``:

1. rank 0 uploads the image from pinned host memory (upload stream, two
   image slots so the next upload overlaps the current step);
2. one broadcast puts it on every GPU (NCCL over NVLink / NVSwitch) and each
   rank refreshes its texture from it (device-to-device copy);
3. each rank runs its shard in ``chunks`` angle chunks; the fused kernel of
   every chunk writes its sinogram and median rows straight into rank 0's
   full [A][F][n] / [A][2][n] buffers (CUDA IPC mapping = NVLink P2P stores,
   fenced at system scope) -- the sinogram assembly is the kernels' own
   stores, no gather collective;
4. after each chunk a 4-byte all_reduce on a signal stream tells rank 0 that
   chunk c of every shard has landed, and rank 0's copy stream downloads
   those rows to the host while later chunks compute.

Rank 0 holds two output slots; the broadcast that opens step i+2 waits for
step i's downloads on rank 0, and every rank's kernels are stream-ordered
after that broadcast, so no rank overwrites rows that are still being read.
``run_device`` is the same path without the host copies (image already on
every GPU): the device-resident leg of bench.py.  Results equal one
single-GPU launch bit-for-bit (tests/test_sharded_gpu.py).

``assembly="gather"`` is the north_star's literal form of step 3-4: every
rank's kernels write its shard into a local [2cnt] block (forward rows, then
mirror rows), ONE all-gather (NCCL over NVLink) of the flat out+median block
per step brings every shard to rank 0, which reorders them into angle order on
the device and downloads the whole sinogram.  It needs equal shards
((A/2) % G == 0).  It is also the fallback when the CUDA IPC mapping of rank
0's buffers fails (no peer access between two of the GPUs).

Failure detection: every collective is issued asynchronously and its Work
kept; ``check()`` (called by ``wait``) raises the first communicator error
(NCCL async errors surface through torch's watchdog when
TORCH_NCCL_ASYNC_ERROR_HANDLING is on -- ``init_process_group`` below sets it
and a bounded timeout).  Each step is bracketed by NVTX ranges.

The reference has no multi-device code; the
per-rank launch is tt_trace_device_tex (include/tt_b200.h), the drop-in
kernel entry.
"""
from __future__ import annotations

from . import shard
from .trace import (NF, IpcBuffer, image_texture, image_texture_destroy, image_texture_update, make_tables,
                    trace_device, weights_soa)


def init_process_group(backend: str = "nccl", device: int | None = None, timeout_s: float = 300.0):
    """torch.distributed.init_process_group for the sharded path: NCCL async-error handling on (a
    failed or hung peer tears the job down instead of hanging it), a bounded collective timeout, and
    the rank's device bound for NCCL."""
    import datetime
    import os

    import torch
    import torch.distributed as dist

    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    kw = {"timeout": datetime.timedelta(seconds=timeout_s)}
    if backend == "nccl" and device is not None:
        kw["device_id"] = torch.device("cuda", device)
    dist.init_process_group(backend, **kw)
    return dist


def chunk_bounds(cnt: int, chunks: int, c: int):
    """Units [u0, u1) of chunk c of a shard of `cnt` mirrored units."""
    return cnt * c // chunks, cnt * (c + 1) // chunks


class ShardedTrace:
    """Orientation-sharded T0..T5 (or T0) of one n x n image over a process group.

    Every rank constructs it (collectively); ``submit``/``wait`` run the
    host-to-host path (rank 0 passes the pinned host image and outputs, the
    other ranks pass nothing); ``run_device`` the device-resident one.
    Outputs on rank 0: ``out`` [A][F][n] f32 and ``med`` [A][2][n] i32."""

    def __init__(self, n: int, angles: int, dist, device: int, full: bool = True, chunks: int = 4,
                 sampler: int | None = None, group=None, root: int = 0, slots: int = 2, assembly: str = "p2p"):
        import torch

        self.torch, self.dist, self.group, self.root = torch, dist, group, root
        self.n, self.A, self.full, self.F = n, angles, full, (NF if full else 1)
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.a0, self.cnt, self.h = shard.orientation_shard(angles, self.world, self.rank)
        self.chunks = max(1, min(chunks, max(1, min(shard.orientation_shard(angles, self.world, r)[1]
                                                        for r in range(self.world)))))
        self.device = torch.device("cuda", device)
        if sampler is None:  # the measured-faster sampler: TMA tiles for the T0 launches they serve, else texture
            from .trace import schedule_slots
            units = min(shard.orientation_shard(angles, self.world, r)[1] for r in range(self.world))
            tma = (not full and n > 704 and n % 4 == 0 and schedule_slots(n, False) == 32
                   and (units // self.chunks) * n * n >= 1.5e8)  # tiles pay from ~1.5e8 taps per launch
            sampler = 2 if tma else 1
        self.sampler = sampler
        dev = self.device
        self.stream = torch.cuda.Stream(dev)       # texture refresh + shard kernels
        self.sig_stream = torch.cuda.Stream(dev)   # per-chunk completion signals
        self.up_stream = torch.cuda.Stream(dev)    # rank 0: image uploads
        self.copy_stream = torch.cuda.Stream(dev)  # rank 0: row downloads
        c, s, w = make_tables(n, angles)  # host f64 -> f32, bit-identical on every rank
        with torch.cuda.stream(self.stream):
            self.ctab, self.stab, self.wtab = (torch.from_numpy(x).to(dev) for x in (c, s, w))
            self.wsoa = torch.empty(6 * n, device=dev) if full else None
            self.img = [torch.zeros((n, n), device=dev) for _ in range(2)]  # broadcast targets (2 slots)
            self.signal = [torch.zeros(1, device=dev) for _ in range(self.chunks)]
            is_root = self.rank == root
            self.slots = slots if is_root else 0
            if assembly not in ("p2p", "gather"):
                raise ValueError(f"assembly must be 'p2p' or 'gather', not {assembly!r}")
            self._ipc_bufs = ([], [])
            if assembly == "p2p":
                # exported buffers are dedicated allocations (IpcBuffer), not caching-allocator blocks
                self._ipc_bufs = ([IpcBuffer(device, (angles, self.F, n), "float32") for _ in range(self.slots)],
                                  [IpcBuffer(device, (angles, 2, n), "int32") for _ in range(self.slots)])
                self.outs = [torch.as_tensor(b, device=dev) for b in self._ipc_bufs[0]]
                self.meds = [torch.as_tensor(b, device=dev) for b in self._ipc_bufs[1]]
        if full:
            weights_soa(self.wtab.data_ptr(), n, self.wsoa.data_ptr(), self.stream.cuda_stream)
        self.tex = image_texture(self.img[0].data_ptr(), n, self.stream.cuda_stream) if sampler == 1 else None
        self.stream.synchronize()
        nslots = [slots]
        dist.broadcast_object_list(nslots, src=root, group=group)
        self.nslots = nslots[0]
        self.peer, self._close = [], (lambda: None)
        if assembly == "p2p":
            # rank 0's output slots, mapped into every rank (CUDA IPC; NVLink peer access across GPUs)
            ptrs = [p for o, m in zip(self.outs, self.meds) for p in (o.data_ptr(), m.data_ptr())]
            try:
                self.peer, self._close = shard.share_device_buffers(ptrs if is_root else [], dist, device, src=root,
                                                                    group=group)
                ok = 1
            except Exception:  # e.g. no peer access between two of the GPUs
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=dev if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()) == 0:  # every rank agrees: fall back to the gather assembly
                self._close()
                self.peer, self._close = [], (lambda: None)
                self.outs = self.meds = []
                for bufs in self._ipc_bufs:
                    for b in bufs:
                        b.free()
                self._ipc_bufs = ([], [])
                assembly = "gather"
        self.assembly = assembly
        if assembly == "gather":
            h, G = angles // 2, self.world
            if h % G:
                raise ValueError("the gather assembly needs equal shards: (angles/2) % world == 0")
            rows = 2 * self.cnt
            self._nout = rows * self.F * n                 # f32 words of the local sinogram block
            self._nblk = self._nout + (rows * 2 * n if full else 0)  # + the i32 median block (same buffer)
            with torch.cuda.stream(self.stream):
                self.loc = torch.empty(self._nblk, device=dev)          # this rank's [2cnt] rows, flat
                self.raw = torch.empty((G, self._nblk), device=dev)    # every rank's block (all-gather target)
                self.outs = [torch.empty((angles, self.F, n), device=dev) for _ in range(self.slots)]
                self.meds = [torch.empty((angles, 2, n), dtype=torch.int32, device=dev) for _ in range(self.slots)]
            self.stream.synchronize()
        self.step = 0
        self._works = []
        self.copy_done = [None] * self.nslots
        self.up_done = [None, None]

    # ---- one step's pieces ----------------------------------------------------------
    def _launch(self, slot: int, k: int, c: int) -> None:
        u0, u1 = chunk_bounds(self.cnt, self.chunks, c)
        if u1 <= u0:
            return
        F, n = self.F, self.n
        if self.assembly == "p2p":
            row = self.a0 + u0  # forward rows; mirror rows at partner_row = A/2 further on
            out_ptr = self.peer[2 * slot] + row * F * n * 4
            med_ptr = self.peer[2 * slot + 1] + row * 2 * n * 4 if self.full else 0
            partner, peer = self.h, self.rank != self.root
        else:  # local [2cnt] block: forward rows u0.., mirror rows cnt + u0..
            out_ptr = self.loc.data_ptr() + u0 * F * n * 4
            med_ptr = self.loc.data_ptr() + (self._nout + u0 * 2 * n) * 4 if self.full else 0
            partner, peer = self.cnt, False
        trace_device(self.img[k].data_ptr(), n, self.a0 + u0, 2 * (u1 - u0), self.ctab.data_ptr(),
                     self.stab.data_ptr(), self.wtab.data_ptr(), out_ptr, med_ptr, full=self.full,
                     sampler=self.sampler, stream=self.stream.cuda_stream, tex=self.tex, pair_stride=self.h,
                     wsoa_ptr=self.wsoa.data_ptr() if self.full else 0, partner_row=partner,
                     peer_out=peer)

    def _gather(self, slot: int, host_out=None, host_med=None) -> None:
        """Gather assembly: one all-gather of every rank's flat block, rank 0 reorders the rows into
        angle order (``shard.assemble``) and downloads the whole sinogram."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            if self.dist.get_backend(self.group) == "nccl":
                w = self.dist.all_gather_into_tensor(self.raw, self.loc, group=self.group, async_op=True)
            else:  # gloo: the list form
                w = self.dist.all_gather(list(self.raw.unbind(0)), self.loc, group=self.group, async_op=True)
            w.wait()
            self._works.append(w)
            if self.rank != self.root:
                return
            G, cnt, F, n = self.world, self.cnt, self.F, self.n
            self.outs[slot].copy_(self.raw[:, :self._nout].reshape(G, 2, cnt, F, n).transpose(0, 1)
                                  .reshape(self.A, F, n))
            if self.full:
                self.meds[slot].copy_(self.raw[:, self._nout:].view(torch.int32).reshape(G, 2, cnt, 2, n)
                                      .transpose(0, 1).reshape(self.A, 2, n))
        if host_out is not None or host_med is not None:
            self.copy_stream.wait_stream(self.stream)
            with torch.cuda.stream(self.copy_stream):
                if host_out is not None:
                    host_out.copy_(self.outs[slot], non_blocking=True)
                if host_med is not None and self.full:
                    host_med.copy_(self.meds[slot], non_blocking=True)

    def _signal(self, c: int) -> None:
        """Chunk c of every shard has landed in rank 0's buffers once this all_reduce completes
        (each rank's contribution is stream-ordered after its chunk kernel)."""
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.sig_stream.wait_event(ev)
        with torch.cuda.stream(self.sig_stream):
            w = self.dist.all_reduce(self.signal[c], group=self.group, async_op=True)
            w.wait()  # the signal stream (not the host) waits for the collective
            self._works.append(w)

    def _rows(self, c: int):
        """Row ranges [r0, r1) of chunk c over every shard (forward and mirror halves)."""
        for r in range(self.world):
            a0, cnt, h = shard.orientation_shard(self.A, self.world, r)
            u0, u1 = chunk_bounds(cnt, self.chunks, c)
            if u1 > u0:
                yield a0 + u0, a0 + u1
                yield h + a0 + u0, h + a0 + u1

    def _body(self, slot: int, k: int, host_out=None, host_med=None) -> None:
        torch = self.torch
        if self.tex is not None:
            image_texture_update(self.tex, self.img[k].data_ptr(), 0, self.stream.cuda_stream)
        if self.assembly == "gather":
            for c in range(self.chunks):
                self._launch(slot, k, c)
            self._gather(slot, host_out, host_med)
            if self.rank == self.root:
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
                self.copy_done[slot] = ev
            return
        for c in range(self.chunks):
            self._launch(slot, k, c)
            self._signal(c)
            if self.rank == self.root and (host_out is not None or host_med is not None):
                ev = torch.cuda.Event()
                ev.record(self.sig_stream)
                self.copy_stream.wait_event(ev)
                with torch.cuda.stream(self.copy_stream):
                    for r0, r1 in self._rows(c):
                        if host_out is not None:
                            host_out[r0:r1].copy_(self.outs[slot][r0:r1], non_blocking=True)
                        if host_med is not None and self.full:
                            host_med[r0:r1].copy_(self.meds[slot][r0:r1], non_blocking=True)
        self.stream.wait_stream(self.sig_stream)  # the step ends when every chunk has been signalled
        if self.rank == self.root:
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
            self.copy_done[slot] = ev

    # ---- public calls -----------------------------------------------------------------
    def run_device(self) -> None:
        """Device-resident step: the shard kernels (image already in every rank's slot 0) with
        their chunk signals, on self.stream (enqueue only)."""
        slot = self.step % self.nslots
        with self.torch.cuda.nvtx.range("ShardedTrace.run_device"):
            self._body(slot, 0)
        self.step += 1

    def upload(self, host_img) -> None:
        """Rank 0: stage the next step's image (pinned host -> its image slot) on the upload stream."""
        torch = self.torch
        k = self.step % 2
        with torch.cuda.stream(self.up_stream):
            self.up_stream.wait_stream(self.stream)  # the slot's previous broadcast / texture refresh is done
            self.img[k].copy_(host_img, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.up_stream)
            self.up_done[k] = ev

    def submit(self, host_img=None, host_out=None, host_med=None) -> None:
        """Host-to-host step (enqueue only; ``wait`` drains).  Rank 0 passes the pinned host image
        [n][n] f32 and outputs [A][F][n] f32 / [A][2][n] i32 (torch CPU tensors); others pass None."""
        torch = self.torch
        k = self.step % 2
        slot = self.step % self.nslots
        if self.rank == self.root:
            if host_img is not None:
                self.upload(host_img)
            if self.up_done[k] is not None:
                self.stream.wait_event(self.up_done[k])
            if self.copy_done[slot] is not None:  # the slot's previous downloads are finished
                self.stream.wait_event(self.copy_done[slot])
        with torch.cuda.nvtx.range("ShardedTrace.submit"):
            with torch.cuda.stream(self.stream):
                w = self.dist.broadcast(self.img[k], src=self.root, group=self.group, async_op=True)
                w.wait()
                self._works.append(w)
            self._body(slot, k, host_out, host_med)
        self.step += 1

    def wait(self) -> None:
        for s in (self.up_stream, self.stream, self.sig_stream, self.copy_stream):
            s.synchronize()
        self.check()

    def check(self) -> None:
        """Raise the first error any finished collective of this object reported (communicator
        aborted, timeout); forget the finished ones."""
        live = []
        for w in self._works:
            if w.is_completed():
                try:
                    exc = w.exception()
                except Exception:  # backends without per-work exceptions (errors then surface from wait())
                    exc = None
                if exc is not None:
                    raise RuntimeError(f"ShardedTrace collective failed: {exc}")
            else:
                live.append(w)
        self._works = live

    @property
    def out(self):
        return self.outs[(self.step - 1) % self.nslots] if self.rank == self.root else None

    @property
    def med(self):
        return self.meds[(self.step - 1) % self.nslots] if self.rank == self.root else None

    def close(self) -> None:
        """Finish outstanding steps, unmap the peers' mappings and free rank 0's exported buffers (the
        tensors returned by ``out`` / ``med`` are invalid afterwards)."""
        self.wait()
        self.dist.barrier(group=self.group)  # no rank still writes into rank 0's buffers
        self._close()
        self.dist.barrier(group=self.group)  # every mapping closed before rank 0 frees the exported buffers
        self.outs = self.meds = []
        for bufs in self._ipc_bufs:
            for b in bufs:
                b.free()
        self._ipc_bufs = ([], [])
        if self.tex is not None:
            image_texture_destroy(self.tex)
            self.tex = None
