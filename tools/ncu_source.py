#!/usr/bin/env python
"""Per-CUDA-source-line hot spots of an ncu --set full capture (needs
-lineinfo and --import-source on):  python tools/ncu_source.py <rep> [top] [inst]

Aggregates the SASS rows of `ncu --page source --print-source cuda,sass`
under the CUDA line they belong to: warp-stall samples and instructions."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0   # sort key: stalls (default) / instructions
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = {}
fname, cur, hdr = "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]), r[1].strip())
        continue
    if cur is None:
        continue
    def num(i):
        try:
            return float(r[i].replace(",", ""))
        except Exception:
            return 0.0
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += num(4)   # warp stall samples (all)
    a[1] += num(7)   # instructions executed (warp level)
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"# {rep}: {ti:.3e} warp instructions, {ts:.0f} stall samples")
print(f"{'file:line':>18} {'%stall':>7} {'%inst':>7}  source")
for (f, ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][by])[:top]:
    print(f"{f + ':' + str(ln):>18} {100 * s / ts:7.2f} {100 * i / ti:7.2f}  {src[:100]}")
