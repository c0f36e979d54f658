"""Shared-memory wavefronts (and excess from bank conflicts) per CUDA source
line of one kernel in an ncu report.  Usage: python tools/ncu_smem_lines.py rep kernel-regex [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, agg, hdr, fname = None, {}, None, ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, r[0], r[1][:100])
    if r[2]:
        try:
            w = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
            e = float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
        except ValueError:
            continue
        if w:
            a = agg.setdefault(cur, [0.0, 0.0])
            a[0] += w
            a[1] += e
tot = sum(v[0] for v in agg.values()) or 1
print("total shared wavefronts", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * v[0] / tot:5.1f}% wf  excess {100 * v[1] / max(v[0], 1):4.0f}%  {k[0]}:{k[1]}  {k[2]}")
