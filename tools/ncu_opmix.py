"""Instruction mix of one kernel from an ncu --page source --csv --print-source sass dump:
per opcode executed count, smem wavefronts (actual / ideal) and stall samples.
    ncu -i rep --page source --csv --print-source sass -k regex:NAME --launch-count 1 > f.csv
    python tools/ncu_opmix.py f.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
print(rows[k - 1][:2] if k else "")
hdr = rows[k]
idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[k + 1:]:
    if len(r) != len(hdr) or r[0] == "Address":
        break
    data.append(r)


def I(r, key):
    try:
        return int(r[idx[key]])
    except (ValueError, KeyError):
        return 0


S = "Warp Stall Sampling (All Samples)"
agg = defaultdict(lambda: [0, 0, 0, 0])
for r in data:
    op = r[idx["Source"]].strip()
    op = re.sub(r'^@!?U?P\w+\s+', '', op).split()[0] if op else '?'
    a = agg[op]
    a[0] += I(r, "L1 Wavefronts Shared")
    a[1] += I(r, S)
    a[2] += I(r, "Instructions Executed")
    a[3] += I(r, "L1 Wavefronts Shared Ideal")
tot = max(1, sum(v[1] for v in agg.values()))
ex = max(1, sum(v[2] for v in agg.values()))
print("warp instructions executed", ex)
for op, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{op:20s} exec={v[2]:>11} ({v[2] * 100 / ex:4.1f}%)  stall-samples={v[1] * 100 / tot:5.1f}%  "
          f"smem wf={v[0]:>10} ideal={v[3]:>10}")
