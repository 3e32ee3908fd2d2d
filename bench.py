#!/usr/bin/env python
"""Trace-transform benchmark (contract: one JSON line from rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c1]
                  [--impl ours|reference] [--sampler 0|1]

Metric: sinogram samples/s = F*A*n per image per second (F = 6 for T0..T5),
whole job over all ranks.  A "step" is one pass of the hot path over one
image of the workload:
  c2 (default, BASELINE.json configs[1]): 1024^2 image, 720 angles, T0..T5;
     N>1: one image per rank ("image batches sharded", weak scaling), the
     per-rank feature summaries gathered to rank 0 over NCCL.
  c3: 4096^2 image, 1440 angles, T0..T5; N>1: orientations sharded across
     ranks (strong scaling), sinogram slices all-gathered over NCCL.
  c1: 256^2, 360 angles (the reference's CPU-runnable case).
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
    "c3": dict(n=4096, angles=1440, full=True, features=False, desc="4096^2 fp32, 1440 angles x 4096 lines, T0-T5"),
    "c4": dict(n=256, angles=360, full=True, features=True, batch=4096,
               desc="batched feature extraction: 4096 x 256^2 fp32, 360 angles, T0-T5 + circus"),
}
FLOPS_PER_TAP = {True: 34, False: 16}  # FMA = 2, in-bounds taps only
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


def cpu_baseline(wl, seconds_target=10.0):
    """The oracle port (TTO_SEQ32 sampler + functionals, and the circus stage
    when the workload has it; OpenMP over lines on all host threads) on a
    bounded sample of the same workload: whole images repeated (or a prefix of
    the angles) until about `seconds_target` of CPU work."""
    import oracle as O
    import paper_1604_03410_b200 as tt
    n, A = wl["n"], wl["angles"]
    img = tt.synth_image(tt.DISK, n)
    c, s, w = tt.make_tables(n, A)
    cores = os.cpu_count() or 1

    def run(a_count):
        out, _, _, _ = O.transform(img, n, c, s, w, a0=0, a_count=a_count, mode=O.SEQ32, nthreads=cores)
        if wl.get("features"):
            O.circus(out, nthreads=cores)

    a_count, t = 1, 0.0
    while True:
        t0 = time.perf_counter()
        run(a_count)
        t = time.perf_counter() - t0
        if t >= seconds_target / 4 or a_count >= A:
            break
        a_count = min(A, max(a_count * 2, int(a_count * seconds_target / 4 / max(t, 1e-3))))
    reps = max(1, int(seconds_target / max(t, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        run(a_count)
    t = time.perf_counter() - t0
    samples = 6 * a_count * n * reps
    return {"value": samples / t, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle TTO_SEQ32 (sequential fp32, pinned sampler){' + circus' if wl.get('features') else ''}"
                      f" on {a_count} of {A} angles x {n} lines of one {n}^2 image, repeated {reps}x "
                      f"({t:.1f} s wall, OpenMP {cores} threads)",
            "seconds": t}


def run_ours(args, ws, rank, local):
    import ctypes as C

    import numpy as np
    import torch

    import paper_1604_03410_b200 as tt
    from paper_1604_03410_b200 import shard
    from paper_1604_03410_b200._lib import lib
    from paper_1604_03410_b200.trace import image_atlas, image_texture, image_texture_destroy, image_texture_update

    if args.dev_one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if args.dev_one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.workload]
    n, A, full, feats_on = wl["n"], wl["angles"], wl["full"], wl["features"]
    F = 6 if full else 1
    batch_total = wl.get("batch", 1)
    orient = args.workload == "c3" and ws > 1        # orientation shards + sinogram gather (strong)
    images = batch_total > 1                         # image shards (strong over a fixed batch)
    h = A // 2
    if orient:
        # rank r owns angles [a0, a0+cnt) and their mirrors [A/2+a0, ...) -> rows [cnt] + [cnt]
        a0, cnt, pair = shard.orientation_shard(A, ws, rank)
        a_cnt = 2 * cnt
    else:
        a0, a_cnt, pair = 0, A, 0
    if images:
        b0, B = shard.image_shard(batch_total, ws, rank)
    else:
        b0, B = rank, 1  # c1/c2 under torchrun: one image per rank (weak scaling)

    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream
    ctab_h, stab_h, wtab_h = tt.make_tables(n, A)
    seed0 = tt.SEEDS[tt.DISK]
    img_h = np.stack([tt.synth_image(tt.DISK, n, seed0 + (0 if orient else b0 + b)) for b in range(B)])
    with torch.cuda.stream(stream):
        img = torch.from_numpy(img_h).cuda()
        ctab, stab, wtab = (torch.from_numpy(x).cuda() for x in (ctab_h, stab_h, wtab_h))
        out = torch.empty((B, a_cnt, F, n), device="cuda")
        med = torch.empty((B, a_cnt, 2, n), dtype=torch.int32, device="cuda")
        circ = torch.empty((B, a_cnt, F, 3), device="cuda")
        flush = torch.empty(int(256 << 20) // 4, device="cuda")  # > 126 MB L2
        wsoa = torch.empty(6 * n, device="cuda") if full else None  # pass-2 weight layout (constant of n)
        # orientation shards: rank 0 holds the assembled sinogram (+ medians); every rank's fused
        # kernel writes its rows straight into it over NVLink P2P (CUDA IPC mapping)
        gathered = torch.empty((A, F, n), device="cuda") if orient and rank == 0 else None
        gmed = torch.empty((A, 2, n), dtype=torch.int32, device="cuda") if orient and rank == 0 else None
        signal = torch.zeros(1, device="cuda") if orient else None
        feats = torch.empty((ws * B, a_cnt, F, 3), device="cuda") if (ws > 1 and not orient) else None
    tex = None
    if args.sampler == 1:  # texture layout of this step's image(s); refreshed inside every timed step
        tex = image_atlas(img.data_ptr(), n, B, 0, sptr) if B > 1 else image_texture(img.data_ptr(), n, sptr)
    if full:
        tt.weights_soa(wtab.data_ptr(), n, wsoa.data_ptr(), sptr)
    launches_per_step = 1 + (1 if feats_on else 0) + (1 if tex is not None and B > 1 else 0)

    close_peer = None
    if orient:
        peer, close_peer = shard.share_device_buffers(
            [gathered.data_ptr(), gmed.data_ptr()] if rank == 0 else [], dist, local)
        _, _, _, row0, prow = shard.direct_shard_rows(A, ws, rank, F, n)
        out_ptr, med_ptr = peer[0] + row0 * F * n * 4, peer[1] + row0 * 2 * n * 4
    else:
        out_ptr, med_ptr, prow = out.data_ptr(), med.data_ptr(), 0

    def step():
        if tex is not None:
            image_texture_update(tex, img.data_ptr(), 0, sptr)
        tt.trace_device(img.data_ptr(), n, a0, a_cnt, ctab.data_ptr(), stab.data_ptr(), wtab.data_ptr(),
                        out_ptr, med_ptr, full=full, sampler=args.sampler, stream=sptr, tex=tex,
                        pair_stride=pair, batch=B, wsoa_ptr=wsoa.data_ptr() if full else 0, partner_row=prow,
                        peer_out=orient and rank != 0)

    def features():
        if feats_on:  # P-functional (circus) stage consuming the sinograms
            tt.circus_device(out.data_ptr(), n, B * a_cnt * F, circ.data_ptr(), stream=sptr)

    def exchange():
        if not dist:
            return
        with torch.cuda.stream(stream):
            if orient:  # rows already written into rank 0's sinogram by the kernels: 4-byte completion signal
                dist.all_reduce(signal)
            else:       # image sharding: gather the per-image circus features
                dist.all_gather_into_tensor(feats, circ)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
        features()
        exchange()
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
            exchange()
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
    ctx = tt.create_context(local)
    ctx.set_sampler(args.sampler)
    # public API on this rank's share (contiguous angle block under torchrun c3)
    plan = tt.Plan(ctx, n, A, full=full, a0=rank * a_cnt if orient else 0, a_count=a_cnt, features=feats_on,
                   batch=B)
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
        outs.append((np.ctypeslib.as_array((C.c_float * (nb_out // 4)).from_address(hp[k].value)) if want_sino else None,
                     np.ctypeslib.as_array((C.c_int32 * (nb_med // 4)).from_address(hp[k + 1].value))
                     if want_sino and full else None,
                     np.ctypeslib.as_array((C.c_float * (nb_circ // 4)).from_address(hp[k + 2].value))
                     if feats_on else None))
    img_arg = h_img if B > 1 else h_img[0]
    for _ in range(max(2, min(args.warmup, 3) if images else args.warmup)):
        plan.run(img_arg, *outs[0])
    e2e_steps = max(3, min(args.steps, 5 if images else 50))
    if dist:
        dist.barrier()
    # every step: H2D of the image, the chunked launches, D2H of sinograms + medians (+ features);
    # steps are submitted back to back (the next upload overlaps the current kernels) and drained
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        plan.submit(img_arg, *outs[i % 2])
    plan.wait()
    e2e_pipelined_s = time.perf_counter() - t0
    # and the latency of one synchronous call (tt_plan_run: submit + wait, nothing overlapped across calls)
    lat = []
    for _ in range(min(10, e2e_steps)):
        t1 = time.perf_counter()
        plan.run(img_arg, *outs[0])
        lat.append(time.perf_counter() - t1)
    e2e_s = e2e_pipelined_s / e2e_steps  # pipelined throughput per step
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    d2h = (nb_out + (nb_med if full else 0) if want_sino else 0) + (nb_circ if feats_on else 0)
    e2e = {"value": samples_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nb_img, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_s * 1e3,
           "sync_call_latency_ms": statistics.median(lat) * 1e3,
           "api": f"tt.Plan.submit/wait -> tt_plan_submit x steps + tt_plan_wait (per step: pinned H2D, "
                  f"{plan.chunks} chunked fused-kernel launches with overlapped D2H of finished rows"
                  + (", circus" if feats_on else "") + "; two buffer slots, consecutive steps overlap)"}
    # parity spot checks: the e2e output against the device-resident one; under orientation
    # sharding, rank 0's P2P-assembled sinogram against one whole single-GPU launch
    if orient:
        same = True
        if rank == 0:
            ref = torch.empty((A, F, n), device="cuda")
            rmed = torch.empty((A, 2, n), dtype=torch.int32, device="cuda")
            tt.trace_device(img.data_ptr(), n, 0, A, ctab.data_ptr(), stab.data_ptr(), wtab.data_ptr(),
                            ref.data_ptr(), rmed.data_ptr(), full=full, sampler=args.sampler, stream=sptr, tex=tex,
                            wsoa_ptr=wsoa.data_ptr() if full else 0)
            torch.cuda.synchronize()
            same = bool(torch.equal(gathered.view(torch.int32), ref.view(torch.int32)) and torch.equal(gmed, rmed))
            del ref, rmed
        dist.barrier()
        close_peer()
    elif want_sino:
        same = np.array_equal(outs[(e2e_steps - 1) % 2][0].reshape(out.shape), out.cpu().numpy())
    else:
        same = np.array_equal(outs[(e2e_steps - 1) % 2][2].reshape(circ.shape), circ.cpu().numpy())
    plan.destroy()
    ctx.destroy()
    for hh in hp:
        lib.tt_host_free(hh)

    # ---- roofline of the fused kernel (this rank's launch) ----
    if orient:
        taps = lib.tt_count_inbounds_taps(n, a0, cnt, ctab_h.ctypes.data, stab_h.ctypes.data) + \
            lib.tt_count_inbounds_taps(n, a0 + h, cnt, ctab_h.ctypes.data, stab_h.ctypes.data)
    else:
        taps = B * lib.tt_count_inbounds_taps(n, 0, A, ctab_h.ctypes.data, stab_h.ctypes.data)
    kern_s = statistics.mean(kern_ms) / 1e3
    peak = fp32_peak_tflops(torch, tt, stream)
    achieved = FLOPS_PER_TAP[full] * taps / kern_s / 1e12
    traffic, traffic_src, pipes = load_traffic(args.workload)
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic,
                "peak_source": "measured in this run: tt_ffma_probe (8 independent FFMA chains x 148*8 CTAs), "
                               "FP32 is the bound (image L2-resident; no tensor-core work)",
                "work": f"{FLOPS_PER_TAP[full]} flop per in-bounds tap x {taps} taps (SURVEY.md 8d)",
                "kernel_ms": kern_s * 1e3, "taps_per_s": taps / kern_s,
                "hbm_algorithmic_bytes": B * (n * n * 4 + a_cnt * (F + 2) * n * 4),
                "traffic_source": traffic_src}
    if pipes:
        roofline["ncu_pipes"] = pipes
    # the sampling stage's own roofline: one TLD4 lane-gather per sampled tap; mirrored angle pairs
    # share one sampling pass, so a launch issues B * (a_cnt / 2) * n^2 gathers (in- and out-of-range)
    if tex is not None:
        gpk = B * (a_cnt // 2) * n * n
        tpeak = tex_peak_gathers(torch, stream)
        roofline["tex_gather"] = {"achieved": gpk / kern_s, "peak": tpeak, "unit": "gathers/s",
                                  "frac": gpk / kern_s / tpeak, "gathers_per_launch": gpk,
                                  "peak_source": "measured in this run: tt_tld4_probe (8 independent TLD4 per "
                                                 "thread, L1-resident texture, 148*8 CTAs)"}
    scaling = "strong" if (orient or images) else "weak"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (disk-masked U[0,1) noise, seed 20160412 + image index)",
            "config": {"workload": args.workload, "desc": wl["desc"], "image": [n, n], "angles": A,
                       "images": batch_total if images else (1 if orient else ws),
                       "functionals": ("T0-T5" if full else "T0") + (" + P1-P3 circus" if feats_on else ""),
                       "sampler": ["ldg", "tex"][args.sampler],
                       "parallelism": (f"orientations sharded x{ws}; fused kernels write sinogram rows into "
                                       "rank 0 over NVLink P2P + 4-byte NCCL completion signal" if orient else
                                       (f"images sharded x{ws} + NCCL feature gather" if ws > 1 else "1 GPU")),
                       "l2": "flushed (256 MiB memset) between timed steps",
                       "ms_per_image": ms_per_step / (batch_total if images else 1)},
            "e2e": e2e, "roofline": roofline, "clocks": clocks.summary(),
            "gpu_launches": args.steps * launches_per_step,
            "e2e_matches_device_result": None if orient else bool(same)}
    if orient:
        line["p2p_assembled_sinogram_matches_single_launch"] = bool(same)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    if tex is not None:
        image_texture_destroy(tex)
    if dist:
        dist.destroy_process_group()
    return line if rank == 0 else None


# ---------------------------------------------------------- reference arm

def run_reference(args, ws, rank):
    """The reference's own execution engine on a bounded sample (rank 0 only)."""
    if rank != 0:
        return None
    import numpy as np

    import oracle as O
    import paper_1604_03410_b200 as tt  # noqa: F401 (host inputs only: tables / image)
    wl = WORKLOADS[args.workload]
    n, A = wl["n"], wl["angles"]
    if not os.path.exists(O.TIER2_PATH):
        return {"impl": "reference", "unavailable": "oracle/_ref/tt_tier2 not built (needs /root/reference)"}
    cores = os.cpu_count() or 1
    img = tt.synth_image(tt.DISK, n)
    c, s, w = tt.make_tables(n, A)
    lines = int(os.environ.get("TT_REF_LINES", "32"))
    threads = min(cores, A)

    def one():
        out, med, rep = O.tier2_sample(img, n, c, s, w, angles=threads, lines=lines, threads=threads)
        return rep

    for _ in range(args.warmup):
        one()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rep = one()
        times.append(time.perf_counter() - t0)
    samples = 6 * threads * min(lines, n)
    t = statistics.mean(times)
    value = samples / t
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "desc": wl["desc"], "image": [n, n], "angles": A,
                       "functionals": "T0-T5"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"reference gridjit emulator (cuda_launch of oracle/trace_t05.krn) on "
                                       f"{threads} angles x {lines} lines x {n} taps per step, one DeviceContext "
                                       f"per host thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sampler", type=int, default=int(os.environ.get("TT_BENCH_SAMPLER", "1")), choices=[0, 1])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dev-one-gpu", action="store_true",
                    help="validation only: every rank on cuda:0 with gloo (exercises the multi-rank data path, "
                         "incl. the P2P shard writes, on a 1-GPU box; numbers are not a scaling measurement)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_env()
    line = run_reference(args, ws, rank) if args.impl == "reference" else run_ours(args, ws, rank, local)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
