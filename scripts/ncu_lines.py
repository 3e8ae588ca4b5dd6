"""Top source lines of one kernel in an ncu report by executed warp
instructions and stall samples.  Usage:
  python scripts/ncu_lines.py <report.ncu-rep> [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path, hdr, rows = "", None, []
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[:4], r[:4]))
        inst = float(r[hdr.index("Instructions Executed")] or 0)
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        rows.append((inst, samp, f"{path}:{r[0]}", r[1].strip()[:90]))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total warp instructions {ti:.3g}, stall samples {ts:.0f}")
for inst, samp, loc, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{inst / ti * 100:5.1f}% inst {samp / ts * 100:5.1f}% samples  {loc:18s} {src}")
