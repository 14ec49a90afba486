"""Aggregate an ncu 'source --print-source cuda,sass' CSV per CUDA line:
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kn = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep] + (kn.split() if kn else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, cur_file, hdr = [], None, None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = {k: i for i, k in enumerate(r)}; continue
    if r[0] == "Function Name" or hdr is None: continue
    if r[0] != "":  # a CUDA line row with aggregated metrics
        def g(k):
            try: return float(r[hdr[k]])
            except Exception: return 0.0
        res.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), cur_file, r[0], r[1]))
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
print(f"total samples {tot:.0f}, instructions {toti:.3g}")
for s, i, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% stall  {100*i/toti:5.1f}% inst  {f}:{ln}  {src.strip()[:90]}")
