#!/usr/bin/env python
"""Benchmark of the MAGUS batched replay on B200 (BASELINE.json metric: trace-samples/s and achieved
HBM GB/s vs peak at 1/2/4/8 GPUs).  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole hot path over one batch: the replay kernel,
the exact fix-up of speculative segments, the per-trace epilogue, the per-policy sums, the NCCL
allreduce (N > 1) and the argmin, for BASELINE.json config 2 (4,096 traces x 100,000 samples,
MAGUS default + static max) per GPU -- weak scaling, traces sharded by global id.

`value` is device-timed with CUDA events (inputs resident in HBM, 1.64 GB per GPU >> 126 MB L2, so
no flush is needed), max over ranks.  `e2e` is the same metric through magus_replay_run_host with
pinned host buffers: the H2D copy of each step's traces and the D2H read of its results are inside
the timed region.  `roofline` is the replay kernel's algorithmic HBM bytes (4 B per trace-sample)
over its CUDA-event duration, against MEASURED_PEAKS.json.  `cpu_baseline` is the oracle (oracle/,
test infrastructure, never tuned) on the host cores, on a bounded sample of the same workload.
`--impl reference` times that oracle alone (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace-samples/s"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU work of the oracle baseline")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: wall-time budget of warmup + steps (sizes each step's sample)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--open-loop", action="store_true", help="NEXT-3 observation model: the trace is a recorded "
                    "throughput observed as is (magus_model.observe = 1, DESIGN.md A30); not the headline")
    ap.add_argument("--wallclock", action="store_true", help="NEXT-1 time model: wall-clock governor rounds "
                    "(MAGUS_F_WALLCLOCK, DESIGN.md A32); not the headline configuration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl", action="store_true", help="run the cross-rank exchange (process group, MAGUS_F_NCCL: "
                    "chunk sums + NCCL allreduce inside the step's graph) even at N = 1")
    ap.add_argument("--policy-shards", type=int, default=1, help="parameter-grid split: this many columns of the "
                    "world replay disjoint policy slices (magus_grid_plan); the rest shard the traces (weak)")
    ap.add_argument("--preroll-ms", type=float, default=600.0, help="untimed load before the timed region "
                    "so the clock samples see the GPU under load")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms while the GPU is loaded."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.rows, self.proc, self.t = [], None, None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            if len(r) < 8:
                continue
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def alu_roofline(cfg, n, ns, n_pol, replay_ms, replay_ms_max):
    """Issue roofline of the unsegmented wide plan (the many-policy sweep): the replay is
    bound by instruction issue, not HBM (each trace byte feeds 64 recurrences).  achieved = lane instructions per
    second = chain-ticks of the launch x the replay kernels' executed instructions per chain-tick (ncu
    smsp__inst_executed x 32 / chain-ticks, profiles/ncu_wide_summary.json) / the replay time; peak = the issue
    ceiling 148 SMs x 4 sub-partitions x 32 lanes x one warp instruction per cycle at the measured max SM clock."""
    chain_ticks = float(n) * ns * n_pol
    ipt, src, traffic = None, None, None
    prof = os.path.join(ROOT, "profiles", "ncu_wide_summary.json")
    if os.path.exists(prof):
        pj = json.load(open(prof))
        if pj.get("config") == cfg["name"]:
            ipt, src, traffic = pj["lane_instr_per_chain_tick"], pj["source"], pj.get("dram_bytes_per_run")
    mhz = 1965.0
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        mhz = float(json.load(open(pk)).get("sm_max_mhz", mhz))
    peak = 148 * 4 * 32 * mhz * 1e6 / 1e9                      # Ginstr/s
    achieved = chain_ticks * ipt / (replay_ms / 1e3) / 1e9 if ipt else None
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Ginstr/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "kernel": "magus_replay_wide_kernel", "replay_ms": replay_ms, "replay_ms_max_over_ranks": replay_ms_max,
            "chain_ticks_per_launch": chain_ticks, "lane_instr_per_chain_tick": ipt,
            "peak_source": f"issue ceiling 148 x 4 x 32 lanes x {mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)",
            "instr_source": src}


def cpu_baseline(cfg, target_s):
    """The oracle as it stands, on all host cores, over a bounded sample (the first n traces of the
    workload, full length, all of the config's policies)."""
    from oracle import oracle as O
    ns = cfg["n_samples"]
    pols = [O.Policy(**d) for d in cfg["policies"]]
    cores = os.cpu_count() or 1

    def timed(n):
        tr, w = O.gen_traces(O.GenDesc(seed=cfg["seed"], n_traces=n, n_samples=ns, class_mix=cfg["class_mix"]))
        t0 = time.perf_counter()
        _, _, used = O.replay_batch(tr, w, pols, n_threads=0)
        return time.perf_counter() - t0, used

    n0 = min(cfg["n_traces"], cores)
    t0, _ = timed(n0)
    n = int(min(cfg["n_traces"], max(n0, n0 * target_s / max(t0, 1e-3))))
    n = max(1, (n // cores) * cores) if n >= cores else n
    dt, used = timed(n)
    return {"value": n * ns / dt, "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": f"first {n} of {cfg['n_traces']} traces x {ns} samples x {len(pols)} policies "
                      f"({cfg['name']}), {dt:.1f} s of wall time on {used} threads"}


def run_reference(args, cfg):
    """--impl reference: the oracle (this tier's reference arm) on the host cores; rank 0 only."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    ns = cfg["n_samples"]
    pols = [O.Policy(**d) for d in cfg["policies"]]
    cores = os.cpu_count() or 1
    # per-step sample sized so that warmup + steps finish in ~2-3 minutes
    per_step_s = max(0.05, args.ref_budget_s / max(1, args.steps + args.warmup))
    n = min(cfg["n_traces"], cores)
    tr, w = O.gen_traces(O.GenDesc(seed=cfg["seed"], n_traces=n, n_samples=ns,
                                   class_mix=cfg["class_mix"]))
    t0 = time.perf_counter()
    O.replay_batch(tr, w, pols)
    t1 = time.perf_counter() - t0
    n = int(min(cfg["n_traces"], max(1, n * per_step_s / max(t1, 1e-3))))
    n = max(1, (n // cores) * cores) if n >= cores else n
    tr, w = O.gen_traces(O.GenDesc(seed=cfg["seed"], n_traces=n, n_samples=ns, class_mix=cfg["class_mix"]))
    used = 1
    for _ in range(args.warmup):
        _, _, used = O.replay_batch(tr, w, pols)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, _, used = O.replay_batch(tr, w, pols)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = n * ns / (ms / 1e3)
    sample = f"first {n} of {cfg['n_traces']} traces x {ns} samples x {len(pols)} policies per step ({cfg['name']})"
    print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                      "config": {"workload": cfg["name"], "n_traces_per_step": n, "n_samples": ns,
                                 "policies": len(pols)},
                      "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "oracle", "sample": sample},
                      "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2502_03796_b200 import magus as M

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = world > 1 or args.nccl
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2502_03796_b200.sharding import grid_shard
    ps = args.policy_shards
    n_pol_glob = len(cfg["policies"])
    per_shard = cfg.get("per_gpu_traces", cfg["n_traces"])      # traces per trace shard (weak over trace shards)
    offset, n, p_off, n_pol = grid_shard(per_shard * (world // ps), n_pol_glob, rank, world, ps)   # global ids
    ns = cfg["n_samples"]
    stride = (n + 3) // 4 * 4
    tr = torch.empty((ns, stride), dtype=torch.float32, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)          # a capturable stream: the library runs each step as a CUDA graph
    M.gen_traces(cfg["seed"], n, ns, cfg["class_mix"], tr, w, trace_stride=stride, global_trace_offset=offset,
                 stream=stream)
    nccl_id = None
    if dist_on:
        obj = [M.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    pols = [M.Policy(**d) for d in cfg["policies"][p_off:p_off + n_pol]]
    R = M.Replay(n, ns, pols, M.Model(observe=1 if args.open_loop else 0), trace_stride=stride, global_trace_offset=offset, rank=rank, world=world,
                 nccl_id=nccl_id, n_policies_global=n_pol_glob, policy_offset=p_off,
                 flags=M.F_TIMING | (M.F_WALLCLOCK if args.wallclock else 0) | (M.F_NCCL if args.nccl else 0))
    geo = R.geometry()
    for _ in range(max(3, args.warmup)):
        R.run(tr, w, stream)
        R.results()
    # untimed pre-roll so that clock samples are taken under load, then the timed region
    sampler = ClockSampler(local)
    t_end = time.perf_counter() + args.preroll_ms / 1e3
    while time.perf_counter() < t_end:
        for _ in range(20):
            R.run(tr, w, stream)
        torch.cuda.synchronize(dev)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        R.run(tr, w, stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if dist_on:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    tsum = R.timing_summary(args.steps)          # per-kernel CUDA events of the same K runs, same stream
    per_run = R.run_times(args.steps)            # the replay kernel of each of those K runs (median / min)
    plan = R.plan_info()
    res = R.results()
    ms_t = torch.tensor([ms, tsum["replay_ms"]], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max, replay_ms_max = float(ms_t[0]), float(ms_t[1])
    total_samples = n * ns * (world // ps)     # trace-samples of the job (each under all of its policies)
    value = total_samples / (ms_max / 1e3)

    # roofline of the dominant kernel (the replay): 4 algorithmic bytes per trace-sample per launch
    peak, peak_src = peaks()
    bytes_per_launch = 4.0 * n * ns
    achieved = bytes_per_launch / (tsum["replay_ms"] / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_replay_summary.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("config") == cfg["name"]:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": ("magus_wallclock_em_kernel" if args.wallclock else
                           "magus_replay_fused_kernel" if plan["fused_magus_tdp"] else
                           "magus_replay_solo_kernel" if geo.get("solo_groups") else "magus_replay_kernel"),
                "replay_ms": tsum["replay_ms"], "replay_ms_max_over_ranks": replay_ms_max,
                "replay_ms_median": statistics.median(per_run) if per_run else None,
                "replay_ms_min": min(per_run) if per_run else None,
                "bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                # the algorithmic bytes count each sample once; every replay launch (one per chain kind, concurrent,
                # unless groups are combined) streams the trace itself, so DRAM reads ~ launches x bytes_per_launch
                # (config 5: MAGUS + TDP in the fused kernel = 1 -- DESIGN.md section 7)
                "launch_groups_streaming_trace": plan["replay_launches"]}
    if geo.get("wide_groups") and not args.wallclock:
        roofline = alu_roofline(cfg, n, ns, geo["lane_policies"], tsum["replay_ms"], replay_ms_max)

    e2e = None
    if not args.no_e2e:
        th = tr.cpu().pin_memory()
        wh = w.cpu().pin_memory()
        R.run_host(th, wh, stream)
        R.results()
        k_e2e = max(1, min(args.steps, 5))
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            R.run_host(th, wh, stream)
            R.results()                           # D2H of the step's totals + argmin (synchronising)
        e2e_ms = 1e3 * (time.perf_counter() - t0) / k_e2e
        e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_ms = float(e2e_t[0])
        e2e = {"value": total_samples / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms, "steps": k_e2e,
               "h2d_bytes_per_step": int(th.numel() * 4 + wh.numel() * 4),
               # magus_replay_results: one copy of the per-(policy, 256-trace chunk) partials + 4 flag words
               "d2h_bytes_per_step": int(len(pols) * ((n + 255) // 256) * M.N_TOTALS * 8 + 4 * 4),
               "path": "magus_replay_run_host + magus_replay_results (pinned host buffers)"}
        del th, wh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.wallclock and not args.open_loop:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    geo = R.geometry()                            # the plan actually timed (after any adaptive re-plan)
    launches_per_step = geo["kernels_per_run"]
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            # sweeps also report trace-sample-policy ticks/s (the replayed recurrences' ticks)
            "policy_ticks_per_s": value * geo["lane_policies"] if not args.wallclock else None,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak" if ps == 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"] + ("+wallclock" if args.wallclock else "") + ("+open-loop" if args.open_loop else ""), "n_traces_per_gpu": n, "n_samples": ns, "policies": len(pols),
                       "policies_global": n_pol_glob,
                       # STATIC_MAX (and a TDP_DEFAULT policy that can never leave f_max) have a closed-form record:
                       # replayed = the policies whose recurrence the kernels step
                       "replayed_policies": geo["lane_policies"] if not args.wallclock else None,
                       "closed_form_policies": "STATIC_MAX (+ TDP never reaching its budget at f_max)",
                       "parallelism": f"trace-sharded x{world // ps}" + (f", parameter grid x{ps}" if ps > 1 else "")
                                      + (", NCCL allreduce of per-policy totals" if dist_on else ""),
                       "l2": "inputs 1.64 GB/GPU >> 126 MB L2; no flush needed" if ns * n * 4 > 4e8 else "L2-resident"},
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "kernel_ms": {"replay_ms": round(tsum["replay_ms"], 5),
                          "rest_of_step_ms": round(ms - tsum["replay_ms"], 5)},
            "plan": plan,
            "segmentation": {"n_segments": res.n_segments, "warmup_ticks": res.warmup_ticks,
                             "mismatched_segments": res.n_mismatched_segments, "fixup_rounds": res.fixup_rounds,
                             "geometry": geo},
            "argmin_policy": res.argmin_policy,
        }
        print(json.dumps(out), flush=True)
    R.close()
    if dist_on:
        dist.destroy_process_group()


def main():
    args = parse()
    from paper_2502_03796_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
