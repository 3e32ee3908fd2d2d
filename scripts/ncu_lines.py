"""Per-source-line stall samples / executed instructions from `ncu -i X --page source --csv
--print-source cuda,sass` (usage: ncu_lines.py cs.csv [top])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[2]
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows[3:]:
    if r and r[0].strip().isdigit():
        try:
            lines.append((int(r[0]), int(r[iS] or 0), int(r[iI] or 0), r[1].strip()))
        except ValueError:
            pass
ts, ti = sum(x[1] for x in lines), sum(x[2] for x in lines)
print(f"total samples {ts} warp instructions {ti}")
for ln, s, i, src in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{ln:5d} samp {100 * s / ts:5.1f}% inst {100 * i / ti:5.1f}%  {src[:95]}")
