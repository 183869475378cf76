#!/usr/bin/env python
"""Summarise a gpu_round.sh session (gpurun_out/<tag>_*) into profiles/ (tracked): the ncu launch list with
each kernel's share of the step, the full ncu capture of the replay kernel (time, DRAM bytes, pipes, issue,
stalls), and profiles/ncu_replay_summary.json (per-launch DRAM traffic, read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)
bench = json.load(open(os.path.join(go, f"{tag}_bench.json")))

# launch list
rows = list(csv.reader(open(os.path.join(go, f"{tag}_launches.csv"))))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")) / 1e3)
step = {k: sum(v) / len(v) for k, v in agg.items() if "gen_kernel" not in k}
tot = sum(step.values())
lines = [f"# ncu launch list ({rnd}, {tag}): `ncu --metrics gpu__time_duration.sum --clock-control none` over",
         "# `python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline` (cold-cache, serialised launches:",
         "# compare SHARES of the step, not absolutes).  Mean per launch; the generator runs once, untimed.", "",
         f"{'kernel':100s} {'launches':>8s} {'mean us':>9s} {'share':>6s}"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
    m = sum(v) / len(v)
    share = f"{100 * m / tot:5.1f}%" if k in step else "  --  "
    lines.append(f"{k[:100]:100s} {len(v):8d} {m:9.1f} {share}")
live = bench["kernel_ms"]
lines += ["", f"live CUDA-event split of the same bench (ms per step): {json.dumps(live)}",
          f"replay share of the step: ncu {100 * max(v for k, v in step.items() if 'magus_replay' in k) / tot:.1f}%"
          f" vs live {100 * live['replay_ms'] / bench['ms_per_step']:.1f}%"]
open(os.path.join(prof, f"{rnd}_launches.txt"), "w").write("\n".join(lines) + "\n")

# full capture
rep = os.path.join(go, f"{tag}_replay.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
d = {rr[0][i]: (rr[2][i], rr[1][i]) for i in range(len(rr[0]))}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_tma_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
out = [f"# ncu --set full --clock-control none of the replay kernel ({rnd}, {tag}), bench config "
       f"{bench['config']['workload']}", ""]
for k in keys:
    if k in d:
        out.append(f"{k:75s} {d[k][0]:>22s} {d[k][1]}")
st = sorted(((k, float(d[k][0].replace(",", ""))) for k in d
             if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
             and d[k][0].replace(",", "").replace(".", "").isdigit()), key=lambda t: -t[1])
out += ["", "warp stalls per issued instruction:"] + [f"   {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:40s} {x:7.3f}"
                                                   for k, x in st[:10] if x > 0.02]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rb = float(d["dram__bytes_read.sum"][0].replace(",", "")) * UNIT[d["dram__bytes_read.sum"][1]]
wb = float(d["dram__bytes_write.sum"][0].replace(",", "")) * UNIT[d["dram__bytes_write.sum"][1]]
alg = bench["roofline"]["bytes_per_launch"]
out += ["", f"DRAM traffic per launch {rb + wb:.4e} B vs algorithmic {alg:.4e} B (4 B per trace-sample): "
            f"x{(rb + wb) / alg:.3f}  (warm-up overlap of speculative segments + state/statistics writes)",
        f"bench roofline (live CUDA events): {json.dumps(bench['roofline'])}"]
open(os.path.join(prof, f"{rnd}_ncu_replay.txt"), "w").write("\n".join(out) + "\n")
json.dump({"config": bench["config"]["workload"], "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
           "source": f"profiles/{rnd}_ncu_replay.txt"}, open(os.path.join(prof, "ncu_replay_summary.json"), "w"),
          indent=1)
json.dump(bench, open(os.path.join(prof, f"{rnd}_bench.json"), "w"), indent=1)
print("\n".join(lines[-3:]))
print("\n".join(out[-3:]))
