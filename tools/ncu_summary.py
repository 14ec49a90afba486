"""Summarise ncu outputs into profiles/.
usage: python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <tag>
writes profiles/<tag>_launches.md (per-kernel share of a frame from the
launch list), profiles/<tag>_ncu_full.md (key --set full metrics per
launch) and profiles/ncu_traffic.json (dram bytes per launch per kernel
class, read by bench.py's roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
CLASS = {"stage_kernel<0,": "stage_first", "stage_kernel<1,": "stage_depth",
         "stage_kernel<2,": "stage_intensity", "stage_kernel<3,": "stage_tail",
         "apss_kernel": "apss", "apss_fit_kernel": "apss_fit", "apss_fit_split_kernel": "apss_fit",
         "zblock_kernel": "apss_fit", "knn_kernel": "knn"}


def kclass(name):
    n = name.replace(" ", "")
    for k, v in CLASS.items():
        if k.replace(" ", "") in n:
            return v
    return None


def launches(path):
    txt = Path(path).read_text()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["Metric Unit"]]
        a = agg[r["Kernel Name"]]
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total µs | µs/launch | share |", "|---|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k[:70]}` | {n} | {us:.1f} | {us / n:.1f} | {100 * us / tot:.1f}% |")
    return out, tot


def full(path):
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    want = OrderedDict([
        ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram rd"),
        ("dram__bytes_write.sum", "dram wr"), ("lts__t_bytes.sum", "L2 bytes"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__inst_executed.sum", "warp instr"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid")])
    lines = ["| kernel | " + " | ".join(want.values()) + " |", "|---" * (len(want) + 1) + "|"]
    traffic = defaultdict(list)
    for r in data:
        name = r[col["Kernel Name"]]
        vals = []
        for m in want:
            if m in col:
                vals.append(f"{r[col[m]]} {units[col[m]]}".strip())
            else:
                vals.append("-")
        lines.append(f"| `{name[:40]}` | " + " | ".join(vals) + " |")
        c = kclass(name)
        if c:
            rd = float(r[col["dram__bytes_read.sum"]]) * UNIT[units[col["dram__bytes_read.sum"]]]
            wr = float(r[col["dram__bytes_write.sum"]]) * UNIT[units[col["dram__bytes_write.sum"]]]
            traffic[c].append(rd + wr)
    return lines, {c: {"dram_bytes_per_launch": sum(v) / len(v), "launches_captured": len(v)}
                   for c, v in traffic.items()}


CMD = "python tools/profile_batch.py B 20 (one batch of 20 config-B frames, the bench step)"
FULL_ARGS = "--profile-from-start off -c 6"


def main():
    lpath, fpath, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    prof = ROOT / "profiles"
    l, tot = launches(lpath)
    (prof / f"{tag}_launches.md").write_text(
        f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n"
        f"Cold-cache, serialised per-launch times of `{CMD}`. "
        "Compare shares, not absolutes.\n\n"
        f"Total {tot:.1f} µs.\n\n" + "\n".join(l) + "\n")
    f, traffic = full(fpath)
    (prof / f"{tag}_ncu_full.md").write_text(
        f"# {tag}: ncu --set full (key metrics per captured launch)\n\n"
        f"`ncu --set full --clock-control none --import-source on -k "
        f"regex:\"apss_kernel|apss_fit|knn_kernel|stage_kernel\" {FULL_ARGS} {CMD}`\n\n"
        + "\n".join(f) + "\n")
    traffic["_source"] = f"{fpath} ({tag}), dram__bytes_read.sum + dram__bytes_write.sum"
    (prof / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    main()
