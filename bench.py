#!/usr/bin/env python
"""Benchmark: symplectic Brouwer-Zimmermann distance (Saved_isometry route) on B200.

One *step* = one complete time-to-distance enumeration of BASELINE config 4
([[56,8]] seed 3, 64x112 normalizer, 9 levels x 3 Gamma_j, 9.8e10 candidates, d = 10),
sharded over the ranks' GPUs (combination-rank space split per level, one min-allreduce
per level). Metric (BASELINE.json): symplectic-weight combos/s and time-to-distance.

  value  combos/s with the Gamma_j already resident in HBM (Plan.run: the level loop),
         timed with CUDA events on the launching stream, max over ranks.
  e2e    the same metric through the public C-ABI call sdb_saved_isometry with the
         normalizer in host memory: validation, isometry, information sets, H2D, every
         level, the per-level D2H of the bound — inside the timed region, every step.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "symplectic-weight combos/sec and time-to-distance, random [[n,k]] codes"
R_POPC = 16  # nominal POPC results per clock per SM
R_POPC_MEASURED = 15.62  # measured on this pool's B200 (tools/microbench/pipes.cu, profiles/r01_pipes.log)
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 4])
    ap.add_argument("--no-extras", action="store_true", help="skip the per-config side measurements")
    ap.add_argument("--cpu-sample-levels", type=int, default=7)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference sample (profiling runs)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, s[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def flush_l2(torch, buf):
    buf.zero_()


def make_allreduce(torch, dist, device):
    import numpy as np

    def fn(values):
        v = (values.astype(np.uint64) ^ np.uint64(1 << 63)).view(np.int64)
        t = torch.tensor(v, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return (t.cpu().numpy().view(np.uint64) ^ np.uint64(1 << 63))

    return fn


def cpu_reference_sample(a, levels: int, workers: int) -> dict:
    import oracle as O

    lv = O.ref_isometry_levels(a, workers=workers, g_max=levels)
    cands = sum(lv["level_candidates"])
    secs = sum(lv["level_seconds"])
    return dict(candidates=cands, seconds=secs, trace=lv["trace"], prep_seconds=lv["prep_seconds"])


def load_profile_summary() -> dict:
    """Per-launch DRAM traffic of the dominant kernel from the committed ncu --set full
    capture (profiles/ncu_summary.json, written by tools/ncu_summary.py)."""
    try:
        with open(PROFILE_SUMMARY) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import paper_2408_10743_b200 as P
    import oracle as O

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsymdist_ref.so not built"}))
        return 0
    c = P.CONFIGS[args.config]
    a = O.generate(c["n"], c["k"], c["seed"])
    workers = os.cpu_count() or 1
    lv = args.cpu_sample_levels
    for _ in range(args.warmup):
        cpu_reference_sample(a, lv, workers)
    tot_c, tot_s = 0, 0.0
    for _ in range(args.steps):
        r = cpu_reference_sample(a, lv, workers)
        tot_c += r["candidates"]
        tot_s += r["seconds"]
    value = tot_c / tot_s
    sample = (f"config {args.config} [[{c['n']},{c['k']}]] seed {c['seed']}: levels g<={lv} of saved_isometry through "
              f"the reference's enumerate_generation (oracle/_ref, reference flags), {r['candidates']} candidates "
              f"per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "combos/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"config{args.config}", "n": c["n"], "k": c["k"], "seed": c["seed"],
                   "sample_levels": lv},
        "cpu_baseline": {"value": value, "unit": "combos/s", "cores": workers, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "combos/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    import paper_2408_10743_b200 as P

    if not P.device_available():
        raise RuntimeError("no CUDA device: " + P.library().sdb_last_error().decode())
    c = P.CONFIGS[args.config]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    stream = torch.cuda.current_stream(device)
    comm = None
    if world > 1:
        # NCCL communicator owned by the library: each sharded level's exchange is a
        # stream-ordered min-allreduce between the level kernel and level_close
        obj = [P.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(obj[0], rank, world, local)
    opts = P.RunOptions(device=local, rank=rank, world=world, comm=comm.handle if comm else 0,
                        stream=stream.cuda_stream)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- value: levels from HBM (Plan), CUDA events on the launching stream
    plan = P.Plan(a, opts)
    for _ in range(args.warmup):
        plan.run()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    reports = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for s in range(args.steps):
            flush_l2(torch, l2)
            ev0[s].record(stream)
            reports.append(plan.run())
            ev1[s].record(stream)
        torch.cuda.synchronize()
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in zip(ev0, ev1)]
    total_ms = max_over_ranks(sum(step_ms))
    r0 = reports[-1]
    cands = r0.candidates_enumerated
    value = args.steps * cands / (total_ms * 1e-3)
    launches = sum(r.kernel_launches for r in reports)
    # dominant kernel: the last (largest) level; its event time is measured inside the
    # library around the kernel on the same stream
    last = len(r0.level_seconds) - 1
    lvl_s = statistics.mean(r.level_seconds[last] for r in reports)
    lvl_s = max_over_ranks(lvl_s)
    g_last = r0.bounds_trace[last].g
    n_rows = a.shape[0]
    from math import comb

    lvl_cands = r0.n_gammas * comb(n_rows, g_last)
    clocks = clk.summary()
    f_mhz = clocks["sm_mhz"] or 1965.0
    props = torch.cuda.get_device_properties(device)
    n_sm = props.multi_processor_count
    w32 = (c["n"] + 31) // 32
    achieved = lvl_cands / lvl_s  # candidates/s of the dominant launch, this rank's share x world
    # XU pipe: the kernel spends exactly one POPC per candidate (one-word probe fold,
    # DESIGN.md §3), so candidates/s == POPC/s; peak = SMs x SM clock x measured POPC/clk/SM
    peak = n_sm * f_mhz * 1e6 * R_POPC_MEASURED * world
    survey_peak = n_sm * f_mhz * 1e6 * R_POPC / w32 * world
    prof = load_profile_summary()
    roofline = {
        "bound": "int-pipe (XU: POPC)",
        "kernel": f"tile_kernel<{w32}> level g={g_last}",
        "achieved": achieved, "peak": peak, "unit": "POPC/s (= candidates/s, 1 POPC per candidate)",
        "frac": achieved / peak,
        "peak_basis": (f"{n_sm} SMs x {f_mhz:.0f} MHz (median SM clock under load, nvidia-smi) x "
                       f"{R_POPC_MEASURED} POPC/clk/SM (measured, profiles/r01_pipes.log) x {world} GPU(s)"),
        "algorithmic_per_launch": f"{lvl_cands} candidates x 1 POPC + 2 LOP3 (W={w32}: {w32} LOP3) + 0.5 VIMNMX3",
        "traffic": prof.get("dram_bytes_per_launch"),
        "traffic_note": prof.get("source"),
        "survey_roofline": {"peak": survey_peak, "frac": achieved / survey_peak,
                            "basis": "SURVEY.md §8(d): N_SM x f x 16 / ceil(n/32) (ceil(n/32) POPC per candidate); "
                                     "the probe fold needs 1, so this fraction can exceed 1"},
    }
    plan.close()

    # ---------------- e2e: the public C-ABI call, host normalizer in, report out
    for _ in range(max(1, args.warmup)):
        P.saved_isometry(a, opts)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e2e_reps = []
    barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        flush_l2(torch, l2)
        e0[s].record(stream)
        e2e_reps.append(P.saved_isometry(a, opts))
        e1[s].record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(sum(x.elapsed_time(y) for x, y in zip(e0, e1)))
    e2e_value = args.steps * cands / (e2e_ms * 1e-3)
    for r in e2e_reps:
        assert r.distance == r0.distance and r.trace_tuples() == r0.trace_tuples()
    launches += sum(r.kernel_launches for r in e2e_reps)

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "combos/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": f"config{args.config}: full saved_isometry distance of [[{c['n']},{c['k']}]] seed "
                            f"{c['seed']} (BASELINE.md §2 xorshift64* transvection generator)",
                "n": c["n"], "k": c["k"], "seed": c["seed"], "distance": r0.distance,
                "trace": r0.trace_tuples(), "candidates_per_step": cands, "levels": len(r0.bounds_trace),
                "parallelism": (f"rank-space shard x{world} (levels >= 2^26 candidates; NCCL min-allreduce of the "
                                f"per-weight keys per sharded level)" if world > 1 else "single GPU"), "l2": "flushed (256 MB write) before every timed step",
                "time_to_distance_ms": {"device_levels": total_ms / args.steps, "e2e_c_abi": e2e_ms / args.steps},
            },
            "roofline": roofline,
            "e2e": {"value": e2e_value, "unit": "combos/s",
                    "h2d_bytes_per_step": int(statistics.mean(r.h2d_bytes for r in e2e_reps)),
                    "d2h_bytes_per_step": int(statistics.mean(r.d2h_bytes for r in e2e_reps)),
                    "ms_per_step": e2e_ms / args.steps},
            "clocks": clocks,
            "gpu_launches": launches,
            "level_ms": [round(1e3 * x, 4) for x in r0.level_seconds],
        }

    # ---------------- side measurements and the CPU baseline (rank 0 at N=1 only)
    if world == 1 and not args.no_extras:
        line["per_config"] = per_config(P, opts, torch)
    if world == 1 and not args.no_cpu:
        try:
            import oracle as O

            if O.ref_available():
                workers = os.cpu_count() or 1
                ra = O.generate(c["n"], c["k"], c["seed"])
                cs = cpu_reference_sample(ra, args.cpu_sample_levels, workers)
                line["cpu_baseline"] = {
                    "value": cs["candidates"] / cs["seconds"], "unit": "combos/s", "cores": workers,
                    "kind": "reference",
                    "sample": (f"config {args.config}: levels g<={args.cpu_sample_levels} ({cs['candidates']} "
                               f"candidates) through the reference's enumerate_generation, oracle/_ref built with "
                               f"the reference's flags, workers={workers}; trace {cs['trace']}"),
                    "cpu": cpu_model(),
                }
            else:
                line["cpu_baseline"] = {"value": None, "unavailable": "oracle/_ref not built"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unavailable": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
    return 0


def per_config(P, opts, torch):
    """Time-to-distance for the other BASELINE configs (rank 0, one GPU)."""
    out = {}
    for cid in (1, 2):
        c = P.CONFIGS[cid]
        a = P.generate_code(c["n"], c["k"], c["seed"])
        P.saved_isometry(a, opts)
        ts, r = [], None
        for _ in range(5):
            t0 = time.perf_counter()
            r = P.saved_isometry(a, opts)
            ts.append(time.perf_counter() - t0)
        out[f"config{cid}"] = {"distance": r.distance, "trace": r.trace_tuples(),
                               "e2e_time_to_distance_ms": 1e3 * statistics.median(ts),
                               "device_levels_ms": 1e3 * r.enum_seconds,
                               "combos_per_s_e2e": r.candidates_enumerated / statistics.median(ts)}
    c = P.CONFIGS[3]
    codes = [P.generate_code(c["n"], c["k"], s) for s in c["seeds"]]
    for _ in range(10):  # the first calls in a process run slower (host caches, clocks)
        P.saved_isometry_batch(codes, opts)
    runs = [P.saved_isometry_batch(codes, opts) for _ in range(15)]
    res = sorted(runs, key=lambda x: x.elapsed_seconds)[len(runs) // 2]  # the median run
    hist = {}
    for d in res.distances:
        hist[str(int(d))] = hist.get(str(int(d)), 0) + 1
    out["config3"] = {"codes": len(codes), "codes_per_s_e2e": len(codes) / res.elapsed_seconds,
                      "e2e_ms": 1e3 * res.elapsed_seconds, "device_ms": 1e3 * res.device_seconds,
                      "runs": len(runs), "statistic": "median of the runs (elapsed normalizers-in-host-memory to results)",
                      "histogram": hist}
    # the package routes on config 4, and the device brute force
    c = P.CONFIGS[4]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for name in ("saved_1_gamma", "saved_2_gamma"):
        fn = getattr(P, name)
        fn(a, opts)
        ts, r = [], None
        for _ in range(3):
            t0 = time.perf_counter()
            r = fn(a, opts)
            ts.append(time.perf_counter() - t0)
        out[f"config4_{name}"] = {"distance": r.distance, "trace": r.trace_tuples(), "candidates": r.candidates_enumerated,
                                  "e2e_time_to_distance_ms": 1e3 * statistics.median(ts),
                                  "device_levels_ms": 1e3 * r.enum_seconds,
                                  "combos_per_s": r.candidates_enumerated / r.enum_seconds}
    c = P.CONFIGS[1]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    r = P.compute_distance(a, P.Algorithm.brute_force, opts)
    out["config1_brute_force"] = {"distance": r.distance, "combinations": r.candidates_enumerated,
                                  "device_ms": 1e3 * r.enum_seconds}
    c = P.CONFIGS[5]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    o5 = P.RunOptions(device=opts.device, stream=opts.stream, max_generation=9)
    with P.Plan(a, o5) as pl:
        pl.run()
        r = pl.run()
    out["config5_g9"] = {"trace": r.trace_tuples(), "candidates": r.candidates_enumerated,
                         "device_levels_ms": 1e3 * r.enum_seconds,
                         "combos_per_s": r.candidates_enumerated / r.enum_seconds,
                         "level_ms": [round(1e3 * x, 3) for x in r.level_seconds]}
    # the K = 3 tile kernel (W = 3) on its g = 9 launch against the same 1-POPC bound, at the
    # B200's 1965 MHz SM clock (the clock the main run records under load)
    import torch

    n_sm = torch.cuda.get_device_properties(opts.device).multi_processor_count
    g9 = 3 * math.comb(c["n"] + c["k"], 9)
    out["config5_g9"]["g9_popc_roofline_frac"] = g9 / r.level_seconds[8] / (n_sm * 1965e6 * R_POPC_MEASURED)
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
