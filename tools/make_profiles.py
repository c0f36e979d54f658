"""Turn a gpurun ncu launch list + a --set full report into the committed
profile summaries under profiles/ (round-tagged).

    python tools/make_profiles.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_r01.ncu-rep c2-u32-asc
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

tag, launches, rep, workload = sys.argv[1:5]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(root, "profiles")
os.makedirs(out_dir, exist_ok=True)

# ---- launch list: per-kernel share of the sort (cold-cache, serialised)
rows = list(csv.reader(open(launches)))
hdr = None
per = defaultdict(lambda: [0, 0.0])
order = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    if not name.startswith("vxs::"):
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    us = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
    per[name][0] += 1
    per[name][1] += us
    order.append((name, d.get("Grid Size"), d.get("Block Size"), us))
tot = sum(v[1] for v in per.values())
with open(os.path.join(out_dir, f"{tag}_launches.md"), "w") as f:
    f.write(f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)\n\n")
    f.write(f"Command: `python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-e2e` (workload {workload}).\n")
    f.write("Times are cold-cache and serialised by ncu; compare shares, not absolutes.\n\n")
    f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
    for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        f.write(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |\n")
    f.write("\nFirst sort's launches (grid, block, us):\n\n")
    for name, g, b, us in order[:16]:
        f.write(f"- `{name}` grid {g} block {b}: {us:.1f} us\n")

# ---- full report: per-kernel metrics
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
stall_cols = [i for i, x in enumerate(h) if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued")]
summary = {"workload": workload, "report": os.path.basename(rep), "kernels": {}}
lines = [f"# {tag}: ncu --set full summary ({workload})\n", f"Report: `{os.path.basename(rep)}` (gpurun_out, not committed).\n"]


def scale(v, unit):
    v = float(v.replace(",", ""))
    return {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}.get(unit, 1) * v


agg = defaultdict(list)
for r in rr[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    m = {}
    for k in keys:
        if k in h:
            i = h.index(k)
            m[k] = (r[i], units[i])
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i].replace(",", "")), h[i].split("stalled_")[-1]))
        except ValueError:
            pass
    tot_s = sum(v for v, _ in st) or 1
    m["top_stalls"] = [(round(100 * v / tot_s, 1), n) for v, n in sorted(st, reverse=True)[:5]]
    agg[name].append(m)
    lines.append(f"\n## `{name}`\n")
    for k in keys:
        if k in m:
            lines.append(f"- {k}: {m[k][0]} {m[k][1]}")
    lines.append(f"- top stalls (% of samples): {m['top_stalls']}")
for name, ms in agg.items():
    by = []
    for m in ms:
        rd = scale(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else 0
        wr = scale(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else 0
        by.append(rd + wr)
    short = name.split("<")[0].replace("vxs::", "")
    summary["kernels"].setdefault(short, {})
    summary["kernels"][short][name] = {"dram_bytes_per_launch": sum(by) / len(by), "launches_captured": len(by)}
# dominant-kernel traffic for bench.py (per launch, averaged over captured launches)
for short in list(summary["kernels"].keys()):
    vals = [v["dram_bytes_per_launch"] for v in summary["kernels"][short].values()]
    summary["kernels"][short] = {"dram_bytes_per_launch": sum(vals) / len(vals), "variants": summary["kernels"][short]}
json.dump(summary, open(os.path.join(out_dir, "ncu_summary.json"), "w"), indent=1)
open(os.path.join(out_dir, f"{tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
print("wrote", out_dir)
