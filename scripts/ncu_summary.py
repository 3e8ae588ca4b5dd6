"""Summarise ncu outputs (gpurun_out/) into profiles/: launch-list shares and the
full-set metrics of the captured kernels.  Usage:
  python scripts/ncu_summary.py <launches.csv> <prof.ncu-rep> <round-tag>"""
import collections, csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launch_csv, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

rows = list(csv.reader(open(launch_csv)))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("ps::<unnamed>::", "").replace("<unnamed>::", "")
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"]) / 1e3
            seq.append((name, float(d["Metric Value"]) / 1e3, d.get("Grid Size", "")))
tot = sum(v[1] for v in agg.values())
lines = [f"# ncu launch list ({tag})", "",
         f"Source: `{os.path.basename(launch_csv)}` — `ncu --metrics gpu__time_duration.sum --clock-control none` over "
         f"`{os.environ.get('NCU_CMD', 'python bench.py --steps 1 --warmup 3 --no-cpu-baseline')}` (cold-cache, serialised: compare shares).", "",
         "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / tot * 100:.1f}% |")
lines.append("")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
want = ["Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum"]
units = r[1]
idx = [h.index(w) for w in want if w in h]
lines += [f"# ncu --set full ({tag})", "", "Source: `" + os.path.basename(rep) + "` (`--set full --clock-control none --import-source on`).", "",
          "| " + " | ".join(h[i] + (f" [{units[i]}]" if units[i] else "") for i in idx) + " |",
          "|" + "---|" * len(idx)]
traffic = {}
for row in r[2:]:
    lines.append("| " + " | ".join(row[i].replace("|", "/")[:60] for i in idx) + " |")
    name = row[h.index("Kernel Name")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(row[h.index("dram__bytes_read.sum")]) * scale.get(units[h.index("dram__bytes_read.sum")], 1)
    wr = float(row[h.index("dram__bytes_write.sum")]) * scale.get(units[h.index("dram__bytes_write.sum")], 1)
    key = "k_refine" if "k_refine" in name else ("k_raster" if "k_raster" in name else name[:40])
    traffic.setdefault(key, []).append(rd + wr)
open(os.path.join(out_dir, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
tpath = os.path.join(out_dir, "ncu_traffic.json")
merged = json.load(open(tpath)) if os.path.exists(tpath) else {}
merged.update({k: sum(v) / len(v) for k, v in traffic.items()})  # per launch, bytes
json.dump(merged, open(tpath, "w"), indent=1)
print("\n".join(lines))
