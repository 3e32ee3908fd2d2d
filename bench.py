#!/usr/bin/env python
"""Trace-transform benchmark (contract: one JSON line from rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c1|c4]
                  [--impl ours|reference] [--sampler 0|1]

Metric: sinogram samples/s = F*A*n per image per second (F = 6 for T0..T5),
whole job over all ranks.  A "step" is one pass of the hot path over one
image of the workload:
  c3 (default; BASELINE.json configs[2], the north_star's target workload):
     4096^2 image, 1440 angles, T0..T5; N>1: orientations sharded across ranks
     (strong scaling; paper_1604_03410_b200.sharded.ShardedTrace: the shard
     kernels write into rank 0's sinogram over NVLink P2P).
  c2 (configs[1]): 1024^2 image, 720 angles, T0..T5 + P-functionals (circus);
     N>1: one image per rank (weak scaling), features gathered over NCCL.
  c1: 256^2, 360 angles (the reference's CPU-runnable case).
  c4: 4096 x 256^2 images, 360 angles, T0..T5 + circus, images sharded.
A plain `python bench.py --gpus N` (no WORLD_SIZE) spawns the N ranks itself
through torch.distributed.run.
`value` times the fused kernel on device-resident inputs (CUDA events on the
launching stream, L2 flushed between steps, max over ranks); `e2e` times the
public API (tt.Plan.run / tt_plan_run: pinned H2D of the image, the chunked launches,
D2H of sinograms + medians).  `--impl reference` runs the reference's own
execution engine (oracle/_ref: the gridjit emulator running
oracle/trace_t05.krn) on a bounded sample, on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c1": dict(n=256, angles=360, full=True, features=False, desc="256^2 fp32, 360 angles x 256 lines, T0-T5"),
    "c2": dict(n=1024, angles=720, full=True, features=True,
               desc="1024^2 fp32, 720 angles x 1024 lines, T0-T5 + P-functionals (circus)"),
    "c3": dict(n=4096, angles=1440, full=True, features=False, orient=True,
               desc="4096^2 fp32, 1440 angles x 4096 lines, T0-T5"),
    "c4": dict(n=256, angles=360, full=True, features=True, batch=4096,
               desc="batched feature extraction: 4096 x 256^2 fp32, 360 angles, T0-T5 + circus"),
}
FLOPS_PER_TAP = {True: 34, False: 16}  # FMA = 2, in-bounds taps only
FLOPS_PER_TAP_EXEC = {True: 26, False: 9}  # the same, the sampling flops counted once per mirrored pair
METRIC = "trace-transform sinogram samples/s"
UNIT = "samples/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------- our arm

def fp32_peak_tflops(torch, tt, stream) -> float:
    """Measured FFMA throughput of this GPU at the current clocks (roofline denominator)."""
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    blocks, iters = props.multi_processor_count * 8, 4096
    buf = torch.empty(blocks, device="cuda")
    from paper_1604_03410_b200._lib import lib
    for _ in range(2):
        lib.tt_ffma_probe(buf.data_ptr(), blocks, 64, stream.cuda_stream)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.tt_ffma_probe(buf.data_ptr(), blocks, iters, stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    flops = blocks * 256.0 * iters * 128 * 2
    return flops / best / 1e12


def tex_peak_gathers(torch, stream) -> float:
    """Measured texture-gather throughput (TLD4 lane-gathers/s, L1-resident texture) of this GPU:
    the roofline of the sampling stage (one gather per sampled tap)."""
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    blocks, iters = props.multi_processor_count * 8, 1024
    buf = torch.empty(blocks, dtype=torch.int32, device="cuda")
    from paper_1604_03410_b200._lib import lib
    lib.tt_tld4_probe(buf.data_ptr(), blocks, 16, stream.cuda_stream)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.tt_tld4_probe(buf.data_ptr(), blocks, iters, stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return blocks * 256.0 * iters * 8 / best


def load_traffic(workload: str):
    """dram bytes per launch of the fused kernel (and its pipe utilisations) from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", f"ncu_{workload}_summary.json")
    try:
        with open(p) as f:
            j = json.load(f)
    except Exception:
        return None, None, None
    pipes = None
    if "issue_slots_busy_pct" in j:
        # north_star: "SM FP32 and shared-memory pipe utilisation" for L2-resident images
        pipes = {"issue_slots_busy": j["issue_slots_busy_pct"] / 100.0,
                 "l1tex_shared_throughput": j.get("l1tex_throughput_pct", 0.0) / 100.0,
                 "fma_pipe_cycles_active": j.get("fma_pipe_active_pct", 0.0) / 100.0 or None,
                 "source": os.path.relpath(p, ROOT) + " (ncu --set full of one launch)"}
    return j.get("dram_bytes_per_launch"), os.path.relpath(p, ROOT), pipes


def cpu_model() -> str:
    """The host CPU model (lscpu "Model name"), for the cpu_baseline / reference lines."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, seconds_target=10.0):
    """The oracle port (TTO_SEQ32 sampler + functionals, and the circus stage
    when the workload has it; OpenMP over lines) on a bounded sample of the
    same workload: a prefix of the angles of one image, repeated until about
    `seconds_target` of CPU work on all host threads, then the same sample on
    one thread (the 1-core figure)."""
    import oracle as O
    n, A = wl["n"], wl["angles"]
    img = O.synth(O.DISK, n)
    c, s, w = O.tables(n, A)
    cores = os.cpu_count() or 1

    def run(a_count, threads):
        out, _, _, _ = O.transform(img, n, c, s, w, a0=0, a_count=a_count, mode=O.SEQ32, nthreads=threads)
        if wl.get("features"):
            O.circus(out, nthreads=threads)

    a_count, t = 1, 0.0
    while True:
        t0 = time.perf_counter()
        run(a_count, cores)
        t = time.perf_counter() - t0
        if t >= seconds_target / 4 or a_count >= A:
            break
        a_count = min(A, max(a_count * 2, int(a_count * seconds_target / 4 / max(t, 1e-3))))
    reps = max(1, int(seconds_target / max(t, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        run(a_count, cores)
    t = time.perf_counter() - t0
    samples = 6 * a_count * n * reps
    # 1 core: the smallest angle prefix that takes >= ~2 s, one pass
    a1 = max(1, min(a_count, int(a_count * 2.0 / max(t / reps * cores, 1e-3)) + 1))
    t1 = time.perf_counter()
    run(a1, 1)
    t1 = time.perf_counter() - t1
    return {"value": samples / t, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "nproc": cores,
            "value_1core": 6 * a1 * n / t1,
            "sample": f"oracle TTO_SEQ32 (sequential fp32, pinned sampler){' + circus' if wl.get('features') else ''}"
                      f" on {a_count} of {A} angles x {n} lines of one {n}^2 image, repeated {reps}x "
                      f"({t:.1f} s wall, OpenMP {cores} threads); 1-core figure: {a1} angles, one pass "
                      f"({t1:.1f} s)",
            "seconds": t}


def run_ours(args, ws, rank, local):
    import ctypes as C

    import numpy as np
    import torch

    import paper_1604_03410_b200 as tt
    from paper_1604_03410_b200 import shard
    from paper_1604_03410_b200._lib import lib
    from paper_1604_03410_b200.sharded import ShardedTrace
    from paper_1604_03410_b200.trace import image_atlas, image_texture, image_texture_destroy, image_texture_update

    if args.dev_one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:  # NCCL async-error handling on, bounded timeout (sharded.init_process_group)
        from paper_1604_03410_b200.sharded import init_process_group
        dist = init_process_group("gloo" if args.dev_one_gpu else "nccl", local)
    wl = WORKLOADS[args.workload]
    n, A, full, feats_on = wl["n"], wl["angles"], wl["full"], wl["features"]
    F = 6 if full else 1
    batch_total = wl.get("batch", 1)
    orient = wl.get("orient", False) and ws > 1      # orientation shards assembled on rank 0 (strong)
    images = batch_total > 1                         # image shards (strong over a fixed batch)
    h = A // 2
    if orient:
        a0, cnt, pair = shard.orientation_shard(A, ws, rank)
        a_cnt = 2 * cnt
    else:
        a0, a_cnt, pair = 0, A, 0
    if images:
        b0, B = shard.image_shard(batch_total, ws, rank)
    else:
        b0, B = rank, 1  # c1/c2 under torchrun: one image per rank (weak scaling)

    ctab_h, stab_h, wtab_h = tt.make_tables(n, A)
    seed0 = tt.SEEDS[tt.DISK]
    img_h = np.stack([tt.synth_image(tt.DISK, n, seed0 + (0 if orient else b0 + b)) for b in range(B)])
    flush = torch.empty(int(256 << 20) // 4, device="cuda")  # > 126 MB L2
    tex = None
    st = None
    if orient:
        # the multi-GPU public call: shard kernels write rows into rank 0's sinogram over NVLink P2P,
        # per-chunk completion signals; the device leg starts with the image already on every GPU
        st = ShardedTrace(n, A, dist, local, full=full, chunks=args.chunks or 4, sampler=args.sampler,
                          assembly=args.assembly)  # falls back to "gather" if the IPC mapping fails
        st.img[0].copy_(torch.from_numpy(img_h[0]))
        torch.cuda.synchronize()
        stream = st.stream
        launches_per_step = st.chunks + (1 if args.sampler == 1 else 0)

        def step():
            st.run_device()

        def features():
            pass
    else:
        stream = torch.cuda.Stream()
        sptr = stream.cuda_stream
        with torch.cuda.stream(stream):
            img = torch.from_numpy(img_h).cuda()
            ctab, stab, wtab = (torch.from_numpy(x).cuda() for x in (ctab_h, stab_h, wtab_h))
            out = torch.empty((B, a_cnt, F, n), device="cuda")
            med = torch.empty((B, a_cnt, 2, n), dtype=torch.int32, device="cuda")
            circ = torch.empty((B, a_cnt, F, 3), device="cuda")
            wsoa = torch.empty(6 * n, device="cuda") if full else None  # pass-2 weight layout (constant of n)
            feats = torch.empty((ws * B, a_cnt, F, 3), device="cuda") if ws > 1 else None
        if args.sampler == 1:  # texture layout of this step's image(s); refreshed inside every timed step
            tex = image_atlas(img.data_ptr(), n, B, 0, sptr) if B > 1 else image_texture(img.data_ptr(), n, sptr)
        if full:
            tt.weights_soa(wtab.data_ptr(), n, wsoa.data_ptr(), sptr)
        # the P stage is a separate circus launch (measured faster than the fused form, DESIGN.md 3.2;
        # TT_FUSED_CIRCUS=1 selects the P stage inside the trace launch)
        fused = feats_on and os.environ.get("TT_FUSED_CIRCUS", "0") == "1"
        launches_per_step = 1 + (1 if feats_on and not fused else 0) + (1 if tex is not None and B > 1 else 0)

        def step():
            if tex is not None:
                image_texture_update(tex, img.data_ptr(), 0, sptr)
            tt.trace_device(img.data_ptr(), n, a0, a_cnt, ctab.data_ptr(), stab.data_ptr(), wtab.data_ptr(),
                            out.data_ptr(), med.data_ptr(), full=full, sampler=args.sampler, stream=sptr, tex=tex,
                            pair_stride=pair, batch=B, wsoa_ptr=wsoa.data_ptr() if full else 0,
                            circ_ptr=circ.data_ptr() if fused else 0, fused_p=fused)

        def features():
            if feats_on and not fused:  # P-functional (circus) stage consuming the sinograms
                tt.circus_device(out.data_ptr(), n, B * a_cnt * F, circ.data_ptr(), stream=sptr)
            if dist:      # image sharding: gather the per-image circus features
                with torch.cuda.stream(stream):
                    dist.all_gather_into_tensor(feats, circ)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
        features()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # ---- timed region (device events per step; L2 flushed between steps) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    with clocks:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            features()
            ev[i][2].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    step_ms = [e0.elapsed_time(e2) for e0, _, e2 in ev]
    kern_ms = [e0.elapsed_time(e1) for e0, e1, _ in ev]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    if orient:
        samples_step = F * A * n                     # one image, angles split over ranks
    elif images:
        samples_step = F * A * n * batch_total       # the whole batch, images split over ranks
    else:
        samples_step = F * A * n * ws                # one image per rank
    value = samples_step / (ms_per_step / 1e3)

    # ---- e2e through the public API (host buffers, copies in the timed region) ----
    e2e_steps = max(3, min(args.steps, 5 if images else 50))
    lat = []
    if orient:
        # ShardedTrace.submit: rank 0 uploads the pinned image, broadcasts it (NCCL), every shard's
        # kernels write into rank 0's sinogram (P2P), rank 0 downloads the rows chunk by chunk
        root = rank == 0
        h_img = torch.from_numpy(img_h[0]).pin_memory() if root else None
        h_out = torch.empty((A, F, n), pin_memory=True) if root else None
        h_med = torch.empty((A, 2, n), dtype=torch.int32, pin_memory=True) if root else None
        for _ in range(max(2, args.warmup)):
            st.submit(h_img, h_out, h_med)
        st.wait()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            st.submit(h_img, h_out, h_med)
        st.wait()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        for _ in range(min(10, e2e_steps)):
            dist.barrier()
            t1 = time.perf_counter()
            st.submit(h_img, h_out, h_med)
            st.wait()
            lat.append(time.perf_counter() - t1)
        nb_img = n * n * 4 if root else 0
        d2h = A * (F + (2 if full else 0)) * n * 4 if root else 0
        chunks_note = f"{st.chunks} chunks per shard"
        if st.assembly == "p2p":
            api = (f"ShardedTrace.submit/wait (per step: rank 0 pinned H2D of the image, NCCL broadcast, "
                   f"{chunks_note} of fused-kernel launches writing rows into rank 0's sinogram over NVLink P2P, "
                   f"a 4-byte completion all_reduce per chunk, rank 0 D2H of sinogram + medians overlapped "
                   f"chunk by chunk)")
        else:
            api = (f"ShardedTrace(assembly='gather').submit/wait (per step: rank 0 pinned H2D of the image, "
                   f"NCCL broadcast, {chunks_note} of fused-kernel launches into a local shard block, one NCCL "
                   f"all-gather of every shard, rank 0 reorders into angle order and downloads sinogram + "
                   f"medians)")
    else:
        ctx = tt.create_context(local)
        ctx.set_sampler(args.sampler)
        nb_img, nb_out = B * n * n * 4, B * a_cnt * F * n * 4
        nb_med, nb_circ = B * a_cnt * 2 * n * 4, B * a_cnt * F * 3 * 4
        # feature extraction (c4) returns the features; the sinogram workloads return sinograms + medians
        want_sino = not images
        # pinned host buffers: one image, two output sets (consecutive submissions are in flight together)
        nbs = (nb_img, nb_out if want_sino else 4, nb_med if want_sino else 4, nb_circ)
        hp = [C.c_void_p() for _ in range(7)]
        for hh, nb in zip(hp, nbs + nbs[1:]):
            if lib.tt_host_alloc(nb, C.byref(hh)) != 0:
                raise RuntimeError(f"tt_host_alloc({nb}) failed")
        h_img = np.ctypeslib.as_array((C.c_float * (B * n * n)).from_address(hp[0].value)).reshape(img_h.shape)
        h_img[:] = img_h
        outs = []
        for k in (1, 4):
            outs.append((np.ctypeslib.as_array((C.c_float * (nb_out // 4)).from_address(hp[k].value))
                         if want_sino else None,
                         np.ctypeslib.as_array((C.c_int32 * (nb_med // 4)).from_address(hp[k + 1].value))
                         if want_sino and full else None,
                         np.ctypeslib.as_array((C.c_float * (nb_circ // 4)).from_address(hp[k + 2].value))
                         if feats_on else None))
        img_arg = h_img if B > 1 else h_img[0]

        def measure(graph):
            """Pipelined throughput and one-call latency of a plan (graph: CUDA-graph replay per slot)."""
            plan = tt.Plan(ctx, n, A, full=full, a0=0, a_count=a_cnt, features=feats_on, batch=B, graph=graph)
            warm = max(2, min(args.warmup, 3) if images else args.warmup)
            for i in range(warm + warm % 2):  # both slots see their steady-state buffers (graph capture)
                plan.run(img_arg, *outs[i % 2])
            if dist:
                dist.barrier()
            # every step: H2D of the image, the chunked launches, D2H of sinograms + medians (+ features);
            # steps are submitted back to back (the next upload overlaps the current kernels) and drained
            t0 = time.perf_counter()
            for i in range(e2e_steps):
                plan.submit(img_arg, *outs[i % 2])
            plan.wait()
            per_step = (time.perf_counter() - t0) / e2e_steps
            # the latency of one synchronous call (submit + wait, nothing overlapped across calls)
            lt = []
            for i in range(min(10, e2e_steps) // 2 * 2):
                t1 = time.perf_counter()
                plan.run(img_arg, *outs[(e2e_steps + i) % 2])
                lt.append(time.perf_counter() - t1)
            chunks, caps = plan.chunks, plan.captures
            plan.destroy()
            return per_step, lt, chunks, caps

        # graph replay is the default e2e path; the enqueue-every-call form is measured beside it
        e2e_s, lat, chunks, caps = measure(True)
        e2e_ng, lat_ng, _, _ = measure(False)
        d2h = (nb_out + (nb_med if full else 0) if want_sino else 0) + (nb_circ if feats_on else 0)
        api = (f"tt.Plan(graph=True).submit/wait -> tt_plan_submit x steps + tt_plan_wait (per step: one "
               f"cudaGraphLaunch replaying the captured submission: pinned H2D, {chunks} chunked fused-kernel "
               f"launches with overlapped D2H of finished rows" + (" and the circus launch" if feats_on else "")
               + f"; two buffer slots, consecutive steps overlap; {caps} captures)")
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": samples_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nb_img, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_s * 1e3, "sync_call_latency_ms": statistics.median(lat) * 1e3, "api": api}
    if not orient:
        e2e["no_graph"] = {"ms_per_step": e2e_ng * 1e3, "sync_call_latency_ms": statistics.median(lat_ng) * 1e3,
                           "value": samples_step / e2e_ng}

    # ---- parity spot checks ----
    if orient:
        same = True
        if rank == 0:  # the P2P-assembled sinogram (device and host copies) against one whole 1-GPU launch
            ref = torch.empty((A, F, n), device="cuda")
            rmed = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
            rimg = torch.from_numpy(img_h[0]).cuda()
            tt.trace_device(rimg.data_ptr(), n, 0, A, st.ctab.data_ptr(), st.stab.data_ptr(), st.wtab.data_ptr(),
                            ref.data_ptr(), rmed.data_ptr(), full=full, sampler=0,
                            wsoa_ptr=st.wsoa.data_ptr() if full else 0)
            torch.cuda.synchronize()
            same = bool(torch.equal(st.out.view(torch.int32), ref.view(torch.int32)) and torch.equal(st.med, rmed)
                        and torch.equal(h_out.view(torch.int32), ref.cpu().view(torch.int32))
                        and torch.equal(h_med, rmed.cpu()))
            del ref, rmed
        st.close()
    elif not images:
        same = np.array_equal(outs[(e2e_steps - 1) % 2][0].reshape(out.shape), out.cpu().numpy())
    else:
        same = np.array_equal(outs[(e2e_steps - 1) % 2][2].reshape(circ.shape), circ.cpu().numpy())
    if not orient:
        ctx.destroy()
        for hh in hp:
            lib.tt_host_free(hh)

    # ---- roofline of the fused kernel (this rank's launches) ----
    if orient:
        taps = lib.tt_count_inbounds_taps(n, a0, cnt, ctab_h.ctypes.data, stab_h.ctypes.data) + \
            lib.tt_count_inbounds_taps(n, a0 + h, cnt, ctab_h.ctypes.data, stab_h.ctypes.data)
    else:
        taps = B * lib.tt_count_inbounds_taps(n, 0, A, ctab_h.ctypes.data, stab_h.ctypes.data)
    kern_s = statistics.mean(kern_ms) / 1e3
    peak = fp32_peak_tflops(torch, tt, stream)
    traffic, traffic_src, pipes = load_traffic(args.workload)
    # executed-flop model (SURVEY.md 8d without double credit): the 16 sampling flops of a tap are
    # executed once per mirrored PAIR of line taps -> 8 per line tap, + 18 per line tap for the
    # prefix sums and the T1..T5 accumulations = 26 (T0 only: 16 / 2 + 1 = 9)
    fpt = FLOPS_PER_TAP_EXEC[full]
    fp32 = {"achieved": fpt * taps / kern_s / 1e12, "peak": peak, "unit": "TFLOP/s",
            "frac": fpt * taps / kern_s / 1e12 / peak,
            "work": f"{fpt} executed flop per in-bounds line tap x {taps} taps (mirrored pairs share the sampling)",
            "peak_source": "measured in this run: tt_ffma_probe (8 independent FFMA chains x 148*8 CTAs)"}
    # mirrored angle pairs share one sampling pass, so a launch issues B * (a_cnt / 2) * n^2 gathers
    gpk = B * (a_cnt // 2) * n * n
    if args.sampler == 1:
        tpeak = tex_peak_gathers(torch, stream)
        roofline = {"bound": "tex", "achieved": gpk / kern_s, "peak": tpeak, "unit": "gathers/s",
                    "frac": gpk / kern_s / tpeak, "traffic": traffic,
                    "work": f"{gpk} TLD4 gathers per launch: one per distinct sampled tap (mirrored angle pairs "
                            f"share one sampling pass; in- and out-of-range taps)",
                    "peak_source": "measured in this run: tt_tld4_probe (8 independent TLD4 per thread, "
                                   "L1-resident texture, 148*8 CTAs)",
                    "binding_unit_note": "ncu: SM issue slots and the L1/TEX data path (texture gathers + line-"
                                         "buffer LDS/STS) are co-binding (see ncu_pipes); HBM is not (image "
                                         "L2-resident / line-blocked order), so the sampling pipe is the roofline",
                    "fp32_model": fp32}
    else:
        roofline = dict(bound="fp32", traffic=traffic, **fp32)
    roofline.update({"kernel_ms": kern_s * 1e3, "taps_per_s": taps / kern_s,
                     "hbm_algorithmic_bytes": B * (n * n * 4 + a_cnt * (F + 2) * n * 4),
                     "traffic_source": traffic_src})
    if pipes:
        roofline["ncu_pipes"] = pipes
    if orient:
        roofline["kernel_ms_note"] = ("per-rank step time incl. the chunk signals (no separate kernel-only "
                                      "event under orientation sharding)")
    scaling = "strong" if (orient or images) else "weak"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (disk-masked U[0,1) noise, seed 20160412 + image index)",
            "config": {"workload": args.workload, "desc": wl["desc"], "image": [n, n], "angles": A,
                       "images": batch_total if images else (1 if orient else ws),
                       "functionals": ("T0-T5" if full else "T0") + (" + P1-P3 circus" if feats_on else ""),
                       "sampler": ["ldg", "tex"][args.sampler],
                       "parallelism": ((f"orientations sharded x{ws}; fused kernels write sinogram rows into "
                                        "rank 0 over NVLink P2P + per-chunk 4-byte NCCL completion signal"
                                        if st.assembly == "p2p" else
                                        f"orientations sharded x{ws}; one NCCL all-gather of the shards per step")
                                       if orient else
                                       (f"images sharded x{ws} + NCCL feature gather" if images and ws > 1 else
                                        (f"one image per rank x{ws} + NCCL feature gather" if ws > 1 else
                                         "1 GPU"))),
                       "l2": "flushed (256 MiB memset) between timed steps",
                       "ms_per_image": ms_per_step / (batch_total if images else 1)},
            "e2e": e2e, "roofline": roofline, "clocks": clocks.summary(),
            "gpu_launches": args.steps * launches_per_step,
            "e2e_matches_device_result": bool(same)}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    if tex is not None:
        image_texture_destroy(tex)
    if dist:
        dist.destroy_process_group()
    return line if rank == 0 else None


# ---------------------------------------------------------- reference arm

def run_reference(args, ws, rank):
    """The reference's own execution engine on a bounded sample (rank 0 only).

    oracle/_ref/tt_tier2 is the reference's gridjit engine (cuda_launch ->
    specialize -> lower -> VPTX -> emulated run_kernel, /root/reference/proj/
    include/gridjit/autolaunch.hpp:167, emulator.hpp:747) compiled from its own
    headers, running the path written in the reference's kernel DSL
    (oracle/trace_t05.krn for T0..T5, oracle/circus.krn for the P-functionals
    of workloads that have them).  It is a separate process that generates its
    own inputs; nothing of the product package (or any in-tree .so) is loaded
    here.  Each step runs `threads` angles x `lines` lines of the trace kernel
    and `crow` circus rows, one DeviceContext per host thread, and reports the
    launch-only seconds; the step time of the WHOLE workload is extrapolated
    linearly from those rates (every line / row of the workload costs the same
    fixed-length loops: n taps twice per line, n samples twice per row)."""
    if rank != 0:
        return None
    import subprocess
    wl = WORKLOADS[args.workload]
    n, A, feats_on = wl["n"], wl["angles"], wl["features"]
    batch = wl.get("batch", 1)
    F = 6
    exe = os.path.join(ROOT, "oracle", "_ref", "tt_tier2")
    if not os.path.exists(exe):
        return {"impl": "reference", "unavailable": "oracle/_ref/tt_tier2 not built (needs /root/reference)"}
    cores = os.cpu_count() or 1
    threads = min(cores, A)
    lines = max(1, min(n, int(os.environ.get("TT_REF_LINES", "0")) or 16384 // n))
    crow = 4 * threads if feats_on else 0

    def one():
        r = subprocess.run([exe, "bench", str(n), str(A), str(threads), str(lines), str(crow), str(threads),
                            os.path.join(ROOT, "oracle", "_ref")], check=True, capture_output=True, text=True)
        return json.loads(r.stdout.strip().splitlines()[-1])

    for _ in range(args.warmup):
        one()
    steps = []
    for _ in range(args.steps):
        rep = one()
        t_line = rep["trace_seconds"] / rep["trace_lines"]           # s per line on `threads` threads
        t_row = rep["circus_seconds"] / rep["circus_rows"] if crow else 0.0
        steps.append((batch * A * n * t_line + (batch * A * F * t_row if feats_on else 0.0), rep))
    t = statistics.mean(x for x, _ in steps)
    samples = F * A * n * batch
    value = samples / t
    rep = steps[-1][1]
    sample = (f"reference gridjit engine (oracle/_ref/tt_tier2: cuda_launch of oracle/trace_t05.krn"
              + (" + oracle/circus.krn" if feats_on else "") + f") per step: {threads} angles x {lines} lines "
              f"x {n} taps" + (f" + {crow} circus rows of {n}" if feats_on else "")
              + f", one DeviceContext per host thread; launch-only seconds extrapolated to the whole workload "
              f"({batch} x {A} angles x {n} lines" + (f" + {batch * A * F} circus rows" if feats_on else "") + ")")
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (disk-masked U[0,1) noise, seed 20160412)",
            "config": {"workload": args.workload, "desc": wl["desc"], "image": [n, n], "angles": A,
                       "images": batch,
                       "functionals": "T0-T5" + (" + P1-P3 circus" if feats_on else "")},
            "impl": "reference", "same_config": True,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "cpu_model": cpu_model(), "nproc": cores, "sample": sample,
                             "measured_sample_seconds": rep["trace_seconds"] + rep["circus_seconds"],
                             "extrapolated": True},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(script: str, argv: list, nprocs: int, env=None) -> int:
    """Re-launch `script argv` as `nprocs` ranks on this node (one process per GPU), the
    way the driver does: python -m torch.distributed.run --nnodes=1 --nproc-per-node N
    --master-addr 127.0.0.1 --master-port P.  Rank 0's stdout (the JSON line) passes
    through; returns the launcher's exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sampler", type=int, default=int(os.environ.get("TT_BENCH_SAMPLER", "1")), choices=[0, 1])
    ap.add_argument("--chunks", type=int, default=0, help="angle chunks per shard (orientation sharding; 0: 4)")
    ap.add_argument("--assembly", default="p2p", choices=["p2p", "gather"],
                    help="orientation sharding: shard rows stored into rank 0 over P2P (default) or one NCCL "
                         "all-gather per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dev-one-gpu", action="store_true",
                    help="validation only: every rank on cuda:0 with gloo (exercises the multi-rank data path, "
                         "incl. the P2P shard writes, on a 1-GPU box; numbers are not a scaling measurement)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # plain `python bench.py --gpus N`: spawn the N ranks ourselves
        sys.exit(spawn_ranks(os.path.abspath(__file__), sys.argv[1:], args.gpus))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        sys.exit(2)
    line = run_reference(args, ws, rank) if args.impl == "reference" else run_ours(args, ws, rank, local)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
