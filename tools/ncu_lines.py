"""Per-source-line instruction and stall-sample shares of one kernel in an
.ncu-rep (`python tools/ncu_lines.py rep.ncu-rep [top] [launch index]`)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
extra = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
                     + extra, capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for x in csv.reader(io.StringIO(out)):
    if len(x) >= 2 and x[0] == "File Path":
        fname = x[1].split("/")[-1]
        continue
    if len(x) >= 2 and x[0] == "Line No":
        hdr = x
        continue
    if hdr and len(x) == len(hdr) and x[0] != "":
        rows.append([fname] + x)
hdr = ["file"] + hdr
ie = hdr.index("Instructions Executed")
smp = hdr.index("Warp Stall Sampling (All Samples)")


def f(v):
    return float(v) if v not in ("", "-") else 0.0


tot = sum(f(x[ie]) for x in rows)
ts = sum(f(x[smp]) for x in rows)
print(f"warp instructions {tot:.4g}")
rows.sort(key=lambda x: -f(x[ie]))
for x in rows[:top]:
    print("%-15s %4s %5.1f%% inst %5.1f%% smp  %s" % (x[0][:15], x[1], 100 * f(x[ie]) / tot,
                                                     100 * f(x[smp]) / ts, x[2].strip()[:80]))
