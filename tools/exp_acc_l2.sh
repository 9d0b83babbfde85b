# Does the fp16-row A L2 policy (XQ_A_HINT) slow the following accumulate kernel? Warm-cache launch times.
set -u
mkdir -p gpurun_out
for h in 0 1; do
  for cc in none all; do
  XQ_A_HINT=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control $cc --clock-control none --nvtx --nvtx-include "step/" -k regex:"k_cl_accumulate|k_decode_absorbed" --csv python tools/prof_step.py --config c3 --layers 8 > gpurun_out/accl2_${h}_${cc}.csv 2>/dev/null
  python - "$h" "$cc" gpurun_out/accl2_${h}_${cc}.csv <<'PY'
import csv, sys, collections
h, cc, f = sys.argv[1:4]
rows = [r for r in csv.reader(open(f)) if len(r) > 10]
hdr = rows[0]; ix = {n: i for i, n in enumerate(hdr)}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    agg[r[ix["Kernel Name"]].split("(")[0][-40:]][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
for k, m in agg.items():
    print(f"hint={h} cache={cc} {k}: " + " ".join(f"{n.split('__')[1][:12]}={sum(v)/len(v):.4g}({len(v)})" for n, v in m.items()))
PY
  done
done
