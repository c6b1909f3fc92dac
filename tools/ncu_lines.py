"""Summarise an ncu source page (cuda,sass csv) per CUDA source line:
instructions executed and warp-stall samples.  Usage: ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None; agg = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")]); inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    agg.append((samples, inst, f"{fname}:{r[0]}", r[1][:90]))
tot_s = sum(a[0] for a in agg) or 1; tot_i = sum(a[1] for a in agg) or 1
print(f"total stall samples {tot_s}, warp-instructions {tot_i}")
for s, i, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {loc:16s} {src}")
