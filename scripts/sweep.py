"""Config C5 sweep (BASELINE.json configs[4]): n in 128..8192 x angles in
180..2880, T0-only (Radon) vs T0-T5, one GPU.  Device-resident timing with
CUDA events on the launch stream, L2 flushed before every timed launch.
Prints one JSON line per point (ms, sinogram samples/s, taps/s, FLOP
fraction of the measured FFMA peak, fraction of the measured TLD4 gather peak).

  python scripts/sweep.py [--quick] [--sampler auto|tex|tma] > profiles/sweep_rNN.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1604_03410_b200 as tt  # noqa: E402
from paper_1604_03410_b200._lib import lib  # noqa: E402
from paper_1604_03410_b200.trace import image_texture, image_texture_destroy  # noqa: E402


def run_point(n, A, full, stream, flush, reps, peak, tpeak, sampler=1):
    F = 6 if full else 1
    c, s, w = tt.make_tables(n, A)
    img = torch.from_numpy(tt.synth_image(tt.DISK, n)).cuda()
    ct, st, wt = (torch.from_numpy(x).cuda() for x in (c, s, w))
    out = torch.empty((A, F, n), device="cuda")
    med = torch.empty((A, 2, n), dtype=torch.int32, device="cuda") if full else None
    sp = stream.cuda_stream
    tex = image_texture(img.data_ptr(), n, sp) if sampler == 1 else None
    wsoa = torch.empty(6 * n, device="cuda")
    tt.weights_soa(wt.data_ptr(), n, wsoa.data_ptr(), sp)

    def launch():
        tt.trace_device(img.data_ptr(), n, 0, A, ct.data_ptr(), st.data_ptr(), wt.data_ptr(), out.data_ptr(),
                        med.data_ptr() if full else 0, full=full, sampler=sampler, stream=sp, tex=tex,
                        wsoa_ptr=wsoa.data_ptr())

    for _ in range(2):
        launch()
    times = []
    for _ in range(reps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    if tex is not None:
        image_texture_destroy(tex)
    ms = sorted(times)[len(times) // 2]
    taps = lib.tt_count_inbounds_taps(n, 0, A, c.ctypes.data, s.ctypes.data)
    flops = bench.FLOPS_PER_TAP[full] * taps
    return {"n": n, "angles": A, "functionals": "T0-T5" if full else "T0", "ms": ms,
            "sampler": "tma" if sampler == 2 else "tex",
            "samples_per_s": F * A * n / (ms / 1e3), "taps_per_s": taps / (ms / 1e3),
            "tflops": flops / (ms / 1e3) / 1e12, "fp32_frac": flops / (ms / 1e3) / 1e12 / peak,
            # one TLD4 per sampled tap; mirrored angle pairs share a pass (A/2 passes of n^2 taps); for the
            # TMA tile kernel (no TLD4) this is the rate relative to the texture-gather ceiling (> 1: beyond it)
            "tex_gather_frac": (A // 2) * n * n / (ms / 1e3) / tpeak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--sampler", default="auto", choices=["auto", "tex", "tma"],
                    help="auto (the product default): TMA tiles for the T0 launches they serve of >= 1.5e8 taps, texture otherwise")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    flush = torch.empty(int(256 << 20) // 4, device="cuda")
    peak = bench.fp32_peak_tflops(torch, tt, stream)
    tpeak = bench.tex_peak_gathers(torch, stream)
    ns = [128, 256, 512, 1024, 2048, 4096, 8192]
    angles = [180, 360, 720, 1440, 2880]
    if args.quick:
        ns, angles = [256, 1024, 4096], [360, 1440]
    for n in ns:
        for A in angles:
            for full in (False, True):
                if full and n > tt.max_full_n():
                    continue
                reps = 5 if n * n * A > 4e10 else 10
                # the product rule (context sampler 3) for these (power-of-two) n: tiles from 1.5e8 taps
                tma_ok = not full and n > 704 and n % 4 == 0 and (A // 2) * n * n >= 1.5e8
                smp = 2 if (args.sampler == "tma" or (args.sampler == "auto" and tma_ok)) else 1
                pt = run_point(n, A, full, stream, flush, reps, peak, tpeak, smp)
                pt["fp32_peak_tflops"] = peak
                pt["tex_peak_gathers_per_s"] = tpeak
                print(json.dumps(pt), flush=True)


if __name__ == "__main__":
    main()
