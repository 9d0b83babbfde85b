"""Executed warp instructions per CUDA source line and per SASS opcode from an ncu
source page (--page source --csv --print-source cuda,sass).

    python tools/ncu_instr_lines.py src.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ops, lines, src = collections.Counter(), collections.Counter(), {}
cur, fname, col = None, None, 7
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        col = r.index("Instructions Executed")
        continue
    if r[0] == "Function Name":
        continue
    if r[0].strip():
        cur = (fname, r[0])
        src[cur] = r[1]
        continue
    if len(r) <= col or not r[3].strip():
        continue
    try:
        n = float(r[col] or 0)
    except ValueError:
        continue
    t = r[3].strip().split()
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += n
    lines[cur] += n
tot = sum(ops.values()) or 1
print(f"total {tot / 1e6:.1f} M warp instructions")
print(" ".join(f"{k}={100 * v / tot:.1f}%" for k, v in ops.most_common(20)))
for k, v in lines.most_common(top):
    print(f"{k[0][:14]:14s} {k[1]:>5} {100 * v / tot:5.1f}%  {src[k].strip()[:90]}")
