"""Regenerate tests/golden/tier2_golden.npz from the REFERENCE's execution engine.

Runs oracle/trace_t05.krn through gridjit's cuda_launch on the reference's
emulated device (oracle/_ref/tt_tier2, built from /root/reference by
`make -C oracle ref`) for small fixed-seed cases and stores the outputs.
The fixtures pin oracle/tt_oracle.c (TTO_SEQ32) on machines where the
reference is absent (the GPU box).  Usage: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

CASES = [  # (n, A, kind)
    (16, 8, O.DISK), (24, 10, O.SPARSE), (31, 7, O.PHANTOM), (32, 12, O.PHANTOM),
    (48, 6, O.DISK), (64, 16, O.DISK), (40, 9, O.SPARSE),
]


def main():
    O.build()
    if not O.build_ref():
        raise SystemExit("oracle/_ref/tt_tier2 unavailable (needs /root/reference)")
    arrays = {}
    for i, (n, A, kind) in enumerate(CASES):
        img = O.synth(kind, n)
        c, s, w = O.tables(n, A)
        out, med, rep = O.tier2(img, n, c, s, w, threads=4)
        arrays[f"c{i}_meta"] = np.array([n, A, kind, O.SEEDS[kind]], np.int64)
        arrays[f"c{i}_out"] = out
        arrays[f"c{i}_med"] = med
        print(f"case {i}: n={n} A={A} kind={kind} taps={rep['taps']} {rep['seconds']:.2f}s")
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tier2_golden.npz"), **arrays)


if __name__ == "__main__":
    main()
