"""Regenerate tests/golden/tier2_c1.npz: the REFERENCE engine's outputs at the
full C1 size (BASELINE.json configs[0]: 256^2, 360 angles, T0-T5).

Runs oracle/trace_t05.krn through gridjit's cuda_launch on the reference's
emulated device (oracle/_ref/tt_tier2, compiled from
/root/reference/proj/include by `make -C oracle ref`; the launch path is
/root/reference/proj/include/gridjit/autolaunch.hpp:167-245 ->
emulator.hpp:747-793) for the DISK and PHANTOM images, one DeviceContext per
host thread.  The fixtures let the GPU box (where /root/reference is absent)
compare the fused kernel DIRECTLY with the reference engine's sinograms and
medians (tests/test_reference_c1_gpu.py) and pin the SEQ32 oracle bit-exactly
at a real configuration size (tests/test_oracle.py).

Usage: python tests/golden/make_golden_c1.py [threads]   (~2-4 min on 8 cores)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

N, A = 256, 360
KINDS = (O.DISK, O.PHANTOM)
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tier2_c1.npz")


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    O.build()
    if not O.build_ref():
        raise SystemExit("oracle/_ref/tt_tier2 unavailable (needs /root/reference)")
    c, s, w = O.tables(N, A)
    arrays = {"meta": np.array([N, A], np.int64), "kinds": np.array(KINDS, np.int64),
              "seeds": np.array([O.SEEDS[k] for k in KINDS], np.int64)}
    for k in KINDS:
        img = O.synth(k, N)
        t0 = time.time()
        out, med, rep = O.tier2(img, N, c, s, w, threads=threads)
        seq, smed, _, _ = O.transform(img, N, c, s, w, mode=O.SEQ32)
        same = np.array_equal(seq.view(np.uint32), out.view(np.uint32)) and np.array_equal(smed, med)
        print(f"kind={k}: taps={rep['taps']} emulator {rep['seconds']:.1f}s (wall {time.time() - t0:.1f}s), "
              f"SEQ32 bit-exact: {same}", flush=True)
        if not same:
            raise SystemExit("SEQ32 oracle differs from the reference engine at C1")
        arrays[f"k{k}_out"] = out
        arrays[f"k{k}_med"] = med.astype(np.int16)  # indices < 256
    np.savez_compressed(OUT, **arrays)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
