"""Summarise an ncu report: per-kernel key metrics, stall breakdown and the
hottest SASS lines.  Usage: python tools/ncu_summary.py rep.ncu-rep [kernel-substr] [--src N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
nsrc = int(sys.argv[sys.argv.index("--src") + 1]) if "--src" in sys.argv else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if kre and kre not in name:
        continue
    print("----", name[:70], "id", r[hdr.index("ID")] if "ID" in hdr else "")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w}: {r[i]} {units[i]}")
    vals = []
    for i in stall:
        try:
            vals.append((float(r[i].replace(",", "")), hdr[i].split("stalled_")[-1]))
        except ValueError:
            pass
    tot = sum(v for v, _ in vals) or 1
    print("  stalls%:", [(round(100 * v / tot, 1), h) for v, h in sorted(vals, reverse=True)[:8]])
    if nsrc and name not in seen:
        seen.add(name)
        short = name.split("(")[0].replace("void ", "", 1).strip()
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + short.split("<")[0],
                              "--print-source", "sass"], capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(src)))
        h2 = srows[1]
        i_src, i_s = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)")
        data, dup = [], set()
        for q in srows[2:]:
            if len(q) < len(h2) or q[0] in dup:
                continue
            dup.add(q[0])
            try:
                data.append((float(q[i_s] or 0), q[0], q[i_src]))
            except ValueError:
                pass
        t2 = sum(d[0] for d in data) or 1
        ops = Counter()
        for s_, a, t in data:
            parts = t.split()
            if parts:
                op = parts[1] if parts[0].startswith("@") else parts[0]
                ops[op.split(".")[0]] += s_
        print("  by opcode%:", [(o, round(100 * v / t2, 1)) for o, v in ops.most_common(12)])
        for s_, a, t in sorted(data, reverse=True)[:nsrc]:
            print(f"   {100 * s_ / t2:5.1f}% {a[-6:]} {t[:80]}")
