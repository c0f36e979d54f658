"""Per-CUDA-source-line instruction and stall totals from an ncu report
(--print-source cuda,sass).  Usage: python tools/ncu_lines.py rep kernel-regex [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur_file = ""
hdr = None
agg = []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        ie = float(r[7] or 0)
        st = float(r[4] or 0)
    except ValueError:
        continue
    agg.append((ie, st, f"{cur_file}:{r[0]}", r[1].strip()[:90]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total warp-inst {ti:.0f}")
for a in sorted(agg, reverse=True)[:n]:
    print(f"{100 * a[0] / ti:5.1f}% inst {100 * a[1] / ts:5.1f}% stall  {a[2]:22s} {a[3]}")
