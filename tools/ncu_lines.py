"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, cur = None, None, None
agg, src, stall = {}, {}, {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    try:
        s = float(r[i_s] or 0)
    except ValueError:
        s = 0
    if cur is None:
        continue
    agg[cur] = agg.get(cur, 0) + s
    d = stall.setdefault(cur, {})
    for j, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                d[h] = d.get(h, 0) + float(r[j] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
for k, s in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    st = sorted(stall.get(k, {}).items(), key=lambda x: -x[1])[:2]
    sts = " ".join(f"{n[6:]}={100 * v / tot:.1f}" for n, v in st if v)
    print(f"{k[0][:14]:14s}{k[1]:5d} {100 * s / tot:5.1f}%  {src.get(k, '')[:70]:70s} {sts}")
