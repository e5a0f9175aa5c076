#!/usr/bin/env python
"""Per-source-line instruction and stall-sample totals of one kernel in an
.ncu-rep (ncu --page source --print-source=cuda), sorted by instructions."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        inst = int(d.get("Instructions Executed", "0") or 0)
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    if inst or samp:
        rows.append((inst, samp, fname, int(r[0]), r[1].strip()[:90]))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total warp-inst {ti/1e6:.1f} M, samples {ts}")
for inst, samp, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{f}:{ln:<5} inst {100*inst/ti:5.1f}%  samp {100*samp/ts:5.1f}%  {src}")

if len(sys.argv) > 3:  # phase ranges "name:file:lo-hi,..."
    for spec in sys.argv[3].split(","):
        name, f, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        si = sum(x[0] for x in rows if x[2] == f and lo <= x[3] <= hi)
        ss = sum(x[1] for x in rows if x[2] == f and lo <= x[3] <= hi)
        print(f"{name:12s} inst {100*si/ti:5.1f}%  samp {100*ss/ts:5.1f}%")
