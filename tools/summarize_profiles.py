"""Turn the ncu outputs of tools/profile_round.sh into the committed summaries.

    python tools/summarize_profiles.py gpurun_out r01

writes profiles/<tag>_launches.csv (the raw launch list), profiles/<tag>_launch_shares.txt,
profiles/<tag>_decode_kernel.txt and updates profiles/decode_kernel_ncu.json (read by
bench.py for roofline.traffic).
"""

import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# where the summaries go (on the GPU box: a directory under gpurun_out/ that travels back)
OUT = os.environ.get("PROFILE_OUT", os.path.join(ROOT, "profiles"))


def launches(src, tag, cfg):
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list of `python bench.py --config {cfg} --steps 2 --warmup 1 --no-fp16 --no-cpu-baseline`",
             "# (gpu__time_duration.sum, --clock-control none; cold-cache serialised: compare SHARES)",
             f"# {len(data)} launches, {tot / 1e3:.2f} ms total",
             f"{'total_ms':>10} {'share':>6} {'count':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[1] / 1e3:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:6d}  {k}")
    out = os.path.join(OUT, f"{tag}_launch_shares.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    shutil.copy(src, os.path.join(OUT, f"{tag}_launches.csv"))
    print("\n".join(lines[:12]))


WANT = [
    "gpu__time_duration.sum", "gpc__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
]


def kernel(rep, tag, key, cfg):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    vals = {n: (v[i], u[i]) for i, n in enumerate(h)}
    lines = [f"# ncu --set full of {vals.get('Kernel Name', ('?', ''))[0]}",
             f"# one launch = one layer of the {cfg.upper()} bench step (tools/prof_step.py --config {cfg}, "
             "layer 3 = first layer at the config's bit width), --clock-control none"]
    for n in WANT:
        if n in vals:
            lines.append(f"{n:80s} {vals[n][0]:>16} {vals[n][1]}")
    # stall breakdown from the source page
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    ix = {n: i for i, n in enumerate(hh)}
    data = rows[2:]
    S = ix["Warp Stall Sampling (All Samples)"]
    tot = sum(float(x[S] or 0) for x in data)
    stalls = collections.Counter()
    for n in hh:
        if n.startswith("stall_") and "Not Issued" not in n:
            stalls[n] = sum(float(x[ix[n]] or 0) for x in data)
    lines.append("# warp stall sampling (all warps, all roles)")
    for n, c in stalls.most_common(8):
        lines.append(f"{n:30s} {100 * c / tot:5.1f}%")
    # hottest source lines (tools/ncu_lines.py over the cuda+sass source view)
    mix = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = os.path.join(ROOT, "build", f"{tag}_mix.csv")
    os.makedirs(os.path.dirname(tmp), exist_ok=True)
    open(tmp, "w").write(mix)
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "25"],
                         capture_output=True, text=True).stdout
    lines.append("# hottest source lines (share of all warp-stall samples, top two stall reasons)")
    lines.extend(hot.rstrip().splitlines())
    out = os.path.join(OUT, f"{tag}_decode_kernel.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

    def num(n, unit_scale):
        val, unit = vals[n]
        return float(val) * unit_scale.get(unit, 1.0)

    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    js_path = os.path.join(OUT, "decode_kernel_ncu.json")
    if not os.path.exists(js_path) and os.path.exists(os.path.join(ROOT, "profiles", "decode_kernel_ncu.json")):
        shutil.copy(os.path.join(ROOT, "profiles", "decode_kernel_ncu.json"), js_path)
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    js[key] = {
        "dram_bytes_per_launch": num("dram__bytes_read.sum", bscale) + num("dram__bytes_write.sum", bscale),
        "duration_ms": num("gpu__time_duration.sum", tscale),
        "tensor_pipe_active_pct": float(vals["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]),
        "source": f"profiles/{tag}_decode_kernel.txt",
    }
    json.dump(js, open(js_path, "w"), indent=1)


KEYS = {"c2": "xq-mha_3", "c3": "xq-cl-mha_2", "c4": "xq-gqa_3", "c1": "xq-mha_4"}

if __name__ == "__main__":
    # python tools/summarize_profiles.py gpurun_out r01 c2   (files of tools/profile_round.sh)
    src, tag = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
    os.makedirs(OUT, exist_ok=True)
    launches(os.path.join(src, f"launches_bench_{cfg}.csv"), f"{tag}_{cfg}", cfg)
    kernel(os.path.join(src, f"decode_full_{cfg}.ncu-rep"), f"{tag}_{cfg}", KEYS[cfg], cfg)
