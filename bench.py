#!/usr/bin/env python
"""Benchmark: symplectic Brouwer-Zimmermann distance (Saved_isometry route) on B200.

One *step* = one complete time-to-distance enumeration of BASELINE config 4
([[56,8]] seed 3, 64x112 normalizer, 9 levels x 3 Gamma_j, 9.8e10 candidates, d = 10),
sharded over the ranks' GPUs (combination-rank space split per level, one min-allreduce
per sharded level). Metric (BASELINE.json): symplectic-weight combos/s and time-to-distance.

  value  combos/s with the Gamma_j already resident in HBM (Plan.run: the level loop),
         timed with CUDA events on the launching stream, max over ranks.
  e2e    the same metric through the public C-ABI call sdb_saved_isometry with the
         normalizer in host memory, timed with the host clock around the (synchronous)
         call: validation, isometry, information sets, H2D, every level, the D2H of the
         bound and the report.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL); it refuses to run when the box has
fewer than N GPUs or when WORLD_SIZE disagrees with --gpus.
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
R_POPC_MEASURED = 15.62  # POPC/clk/SM measured on this pool's B200 (tools/microbench/pipes.cu, profiles/r01_pipes.log)
# int8 tcgen05.mma: a 128 x 256 x 32 MMA retires in 128 SM cycles (tools/microbench/tc_i8.cu,
# profiles/r02_tc_i8_microbench_v2.log: KT=4 mma-only 512 cycles) = 8192 MAC = 16384 ops/clk/SM
TC_I8_OPS_PER_CLK_SM = 16384
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
KERNEL_NAMES = {1: "walk_kernel", 2: "tile_kernel (POPC)", 3: "tc_tile_kernel (tcgen05 int8)", 4: "pkg_kernel",
                5: "ptile_kernel"}
SAMPLE_LEVELS = 7  # the CPU arms' bounded sample: config 4 levels g <= 7 (2.1e9 candidates)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 4])
    ap.add_argument("--no-extras", action="store_true", help="skip the per-config side measurements")
    ap.add_argument("--cpu-sample-levels", type=int, default=SAMPLE_LEVELS)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference runs (profiling runs)")
    ap.add_argument("--no-cpu-config4", action="store_true", help="skip the CPU's full config-4 distance (~80 s)")
    ap.add_argument("--master-port", type=int, default=29517)
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def gpu_count() -> int:
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return sum(1 for ln in out.splitlines() if ln.startswith("GPU "))
    except (OSError, subprocess.SubprocessError):
        return 0


def launch_ranks(args, argv, script: str = "") -> int:
    """--gpus N > 1 without a torchrun environment: re-run this script (or `script`, tests) as N ranks."""
    have = gpu_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}; "
              f"refusing to time fewer GPUs than requested", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator's init lines (nranks) go to stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(args.master_port), script or os.path.abspath(__file__), *argv]
    return subprocess.run(cmd, env=env).returncode


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


def workload_config(P, cid: int) -> dict:
    c = P.CONFIGS[cid]
    return {"workload": f"config{cid}: full saved_isometry distance of [[{c['n']},{c['k']}]] seed {c['seed']} "
                        f"(BASELINE.md §2 xorshift64* transvection generator)",
            "n": c["n"], "k": c["k"], "seed": c["seed"]}


# ------------------------------------------------------------------ CPU (reference) legs
def cpu_sample(a, levels: int, workers: int, native: bool) -> dict:
    """Levels g <= `levels` of saved_isometry through the reference library's own
    enumerate_generation (oracle/_ref), all host threads."""
    import oracle as O

    lv = O.ref_isometry_levels(a, workers=workers, g_max=levels, native=native)
    return dict(candidates=sum(lv["level_candidates"]), seconds=sum(lv["level_seconds"]), trace=lv["trace"],
                prep_seconds=lv["prep_seconds"])


def cpu_time_to_distance(P, workers: int, config4: bool) -> dict:
    """The reference's compute_distance(saved_isometry) wall time per config (its own
    DistanceReport.elapsed_seconds, distance.cpp:136,148), both builds."""
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor

    out = {}
    for cid in (1, 2):
        c = P.CONFIGS[cid]
        a = O.generate(c["n"], c["k"], c["seed"])
        row = {}
        for native in (False, True):
            best = min(O.ref_compute_distance(a, "saved_isometry", workers=workers, native=native).elapsed_seconds
                       for _ in range(3))
            row["native_s" if native else "reference_flags_s"] = best
        out[f"config{cid}"] = row
    # config 3: 4096 independent codes, one code per host thread at a time (ctypes drops the GIL)
    c = P.CONFIGS[3]
    codes = [O.generate(c["n"], c["k"], s) for s in c["seeds"]]
    row = {"codes": len(codes), "threads": workers}
    for native in (False, True):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(lambda x: O.ref_compute_distance(x, "saved_isometry", workers=1, native=native), codes))
        dt = time.perf_counter() - t0
        key = "native" if native else "reference_flags"
        row[key + "_s"] = dt
        row[key + "_codes_per_s"] = len(codes) / dt
    out["config3"] = row
    if config4:
        c = P.CONFIGS[4]
        a = O.generate(c["n"], c["k"], c["seed"])
        r = O.ref_compute_distance(a, "saved_isometry", workers=workers, native=False)
        out["config4"] = {"reference_flags_s": r.elapsed_seconds, "distance": r.distance,
                          "candidates": r.candidates, "combos_per_s": r.candidates / r.elapsed_seconds}
    return out


def run_reference(args):
    """The reference arm: the reference's own CPU library on the box's host cores, a bounded
    sample of our arm's workload per step (config 4 levels g <= 7)."""
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
        cpu_sample(a, lv, workers, native=False)
    tot_c, tot_s, r = 0, 0.0, None
    for _ in range(args.steps):
        r = cpu_sample(a, lv, workers, native=False)
        tot_c += r["candidates"]
        tot_s += r["seconds"]
    value = tot_c / tot_s
    sample = (f"config {args.config} [[{c['n']},{c['k']}]] seed {c['seed']}: levels g<={lv} of saved_isometry "
              f"through the reference's enumerate_generation (oracle/_ref, reference flags -O3), "
              f"{r['candidates']} candidates per step; the GPU arm's per_config.like_for_like times the same levels")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "combos/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {**workload_config(P, args.config), "sample_levels": lv},
        "cpu_baseline": {"value": value, "unit": "combos/s", "cores": workers, "kind": "reference",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "combos/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch

    world, rank, local = dist_env()
    dist = None
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=device)
    import paper_2408_10743_b200 as P

    if os.path.realpath(P.library_path()) != os.path.realpath(P.IN_TREE_LIBRARY):
        raise RuntimeError(f"bench.py times the in-tree library only, not {P.library_path()}")
    if not P.device_available():
        raise RuntimeError("no CUDA device: " + P.library().sdb_last_error().decode())
    c = P.CONFIGS[args.config]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    # one dedicated stream: the L2 flush, the CUDA events and every library call run on it
    stream = torch.cuda.Stream(device)
    comm = None
    if world > 1:
        # NCCL communicator owned by the library: each sharded level's exchange is a
        # stream-ordered min-allreduce between the level kernel and level_close
        obj = [P.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = P.Comm(obj[0], rank, world, local)
    opts = P.RunOptions(device=local, rank=rank, world=world, comm=comm.handle if comm else 0,
                        stream=stream.cuda_stream)
    assert stream.cuda_stream != 0
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

    def device_timed(plan, steps):
        """K plan.run() steps, each after an L2 flush, CUDA events on the library's stream."""
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        reps = []
        barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for s in range(steps):
                l2.zero_()
                ev0[s].record(stream)
                reps.append(plan.run())
                ev1[s].record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in zip(ev0, ev1))), reps

    # ---------------- value: levels from HBM (Plan), CUDA events on the launching stream
    plan = P.Plan(a, opts)
    for _ in range(args.warmup):
        plan.run()
    with ClockSampler(local) as clk:
        total_ms, reports = device_timed(plan, args.steps)
    r0 = reports[-1]
    cands = r0.candidates_enumerated
    value = args.steps * cands / (total_ms * 1e-3)
    launches = sum(r.kernel_launches for r in reports)
    for r in reports:
        assert r.distance == r0.distance and r.trace_tuples() == r0.trace_tuples()
    # dominant kernel: the last (largest) level, timed inside the library with CUDA events
    # around its kernel on the same stream
    last = len(r0.level_seconds) - 1
    lvl_s = max_over_ranks(statistics.mean(r.level_seconds[last] for r in reports))
    g_last = r0.bounds_trace[last].g
    lvl_cands = r0.n_gammas * math.comb(a.shape[0], g_last)
    clocks = clk.summary()
    f_mhz = clocks["sm_mhz"] or 1965.0
    n_sm = torch.cuda.get_device_properties(device).multi_processor_count
    roofline = dominant_roofline(P, a, r0.last_level_kernel, g_last, lvl_cands, lvl_s, n_sm, f_mhz, world)
    plan.close()

    # ---------------- e2e: the public C-ABI call, host normalizer in, report out (host clock)
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            P.saved_isometry(a, opts)
        e2e_s, e2e_reps = 0.0, []
        barrier()
        for s in range(args.steps):
            l2.zero_()
            stream.synchronize()
            t0 = time.perf_counter()
            e2e_reps.append(P.saved_isometry(a, opts))  # returns after the report's D2H
            e2e_s += time.perf_counter() - t0
        barrier()
    e2e_ms = max_over_ranks(1e3 * e2e_s)
    e2e_value = args.steps * cands / (e2e_ms * 1e-3)
    for r in e2e_reps:
        assert r.distance == r0.distance and r.trace_tuples() == r0.trace_tuples()

    # ---------------- config 5 through g = 9 (the largest code; its sharded levels carry 99.99%)
    o5 = P.RunOptions(device=local, rank=rank, world=world, comm=opts.comm, stream=opts.stream, max_generation=9)
    c5 = P.CONFIGS[5]
    with P.Plan(P.generate_code(c5["n"], c5["k"], c5["seed"]), o5) as pl5:
        pl5.run()
        c5_ms, c5_reps = device_timed(pl5, 2)
    r5 = c5_reps[-1]
    config5 = {"trace": r5.trace_tuples(), "candidates": r5.candidates_enumerated,
               "device_ms": c5_ms / 2, "combos_per_s": 2 * r5.candidates_enumerated / (c5_ms * 1e-3),
               "level_ms": [round(1e3 * x, 3) for x in r5.level_seconds], "n_gpus": world}
    # the same roofline for the largest code's dominant launch (its g = 9 level, K = 96)
    a5 = P.generate_code(c5["n"], c5["k"], c5["seed"])
    last5 = len(r5.level_seconds) - 1
    lvl5_s = max_over_ranks(statistics.mean(r.level_seconds[last5] for r in c5_reps))
    g5 = r5.bounds_trace[last5].g
    rf5 = dominant_roofline(P, a5, r5.last_level_kernel, g5, r5.n_gammas * math.comb(a5.shape[0], g5), lvl5_s, n_sm,
                            f_mhz, world)
    rf5["traffic"], rf5["traffic_note"] = None, "profiles/r02_tc_c5_g9_ncu.txt: 0.25 MB per launch (not re-read here)"
    config5["roofline"] = rf5

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "combos/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                **workload_config(P, args.config),
                "distance": r0.distance, "trace": r0.trace_tuples(), "candidates_per_step": cands,
                "levels": len(r0.bounds_trace),
                "parallelism": (f"rank-space shard x{world} (levels >= 2^26 candidates; NCCL min-allreduce of the "
                                f"per-weight keys per sharded level)" if world > 1 else "single GPU"),
                "l2": "flushed (256 MB write on the library's stream) before every timed step",
                "time_to_distance_ms": {"device_levels": total_ms / args.steps, "e2e_c_abi": e2e_ms / args.steps},
            },
            "roofline": roofline,
            "e2e": {"value": e2e_value, "unit": "combos/s",
                    "h2d_bytes_per_step": int(statistics.mean(r.h2d_bytes for r in e2e_reps)),
                    "d2h_bytes_per_step": int(statistics.mean(r.d2h_bytes for r in e2e_reps)),
                    "ms_per_step": e2e_ms / args.steps, "timer": "host perf_counter around each synchronous call"},
            "clocks": clocks,
            "gpu_launches": launches,
            "level_ms": [round(1e3 * x, 4) for x in r0.level_seconds],
            "config5_g9": config5,
        }

    # ---------------- side measurements and the CPU baseline (rank 0 at N=1 only)
    if world == 1 and not args.no_extras:
        line["per_config"] = per_config(P, opts, a, args)
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(P, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
    return 0


def dominant_roofline(P, a, kind, g_last, lvl_cands, lvl_s, n_sm, f_mhz, world) -> dict:
    prof = load_profile_summary()
    achieved_c = lvl_cands / lvl_s  # candidates/s of the dominant launch (this rank's share x world)
    popc_peak = n_sm * f_mhz * 1e6 * R_POPC_MEASURED * world
    base = {"kernel": f"{KERNEL_NAMES.get(kind, '?')} level g={g_last}", "candidates_per_launch": lvl_cands,
            "launch_ms": 1e3 * lvl_s, "traffic": prof.get("dram_bytes_per_launch"),
            "traffic_note": prof.get("source"), "sm_mhz": f_mhz}
    if kind == 3:
        # tensor-core tile kernel: each candidate is one int8 dot product of K exact ±1
        # coordinates (csrc/tcenc.cpp) -> 2K int8 ops
        _, ks = P.tc_encoding_check(a, trials=1)
        k = max(ks)
        achieved = 2 * k * achieved_c
        peak = n_sm * f_mhz * 1e6 * TC_I8_OPS_PER_CLK_SM * world
        return {**base, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "int8 OP/s", "frac": achieved / peak,
                "peak_basis": (f"{n_sm} SMs x {f_mhz:.0f} MHz x {TC_I8_OPS_PER_CLK_SM} int8 ops/clk/SM (tcgen05.mma "
                               f"kind::i8, measured: 128 x 256 x 32 per 128 cycles) x {world} GPU(s)"),
                "algorithmic_per_launch": f"{lvl_cands} candidates x 2 x K={k} int8 ops",
                "candidates_per_s": achieved_c,
                "vs_cuda_core_popc_roofline": {"peak": popc_peak, "frac": achieved_c / popc_peak,
                                               "basis": f"1 POPC per candidate at {R_POPC_MEASURED} POPC/clk/SM: "
                                                        f"the CUDA-core kernel's ceiling"}}
    return {**base, "bound": "int-pipe (XU: POPC)", "achieved": achieved_c, "peak": popc_peak,
            "unit": "POPC/s (= candidates/s, 1 POPC per candidate)", "frac": achieved_c / popc_peak,
            "peak_basis": f"{n_sm} SMs x {f_mhz:.0f} MHz x {R_POPC_MEASURED} POPC/clk/SM x {world} GPU(s)"}


def cpu_baseline(P, args) -> dict:
    try:
        import oracle as O

        if not O.ref_available():
            return {"value": None, "unavailable": "oracle/_ref not built"}
        workers = os.cpu_count() or 1
        c = P.CONFIGS[args.config]
        ra = O.generate(c["n"], c["k"], c["seed"])
        cs = cpu_sample(ra, args.cpu_sample_levels, workers, native=False)
        out = {
            "value": cs["candidates"] / cs["seconds"], "unit": "combos/s", "cores": workers, "kind": "reference",
            "sample": (f"config {args.config}: levels g<={args.cpu_sample_levels} ({cs['candidates']} candidates) "
                       f"through the reference's enumerate_generation, oracle/_ref built with the reference's "
                       f"flags, workers={workers}; trace {cs['trace']}"),
            "cpu": cpu_model(),
        }
        if O.ref_available(native=True):
            cn = cpu_sample(ra, args.cpu_sample_levels, workers, native=True)
            out["native_value"] = cn["candidates"] / cn["seconds"]
            out["native_note"] = "same sample, the reference sources built with -march=native (BASELINE.md §3)"
        out["time_to_distance"] = cpu_time_to_distance(P, workers, config4=not args.no_cpu_config4)
        return out
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unavailable": repr(e)}


def per_config(P, opts, a4, args):
    """Time-to-distance for the other BASELINE configs (rank 0, one GPU), host clock."""
    out = {}
    # like for like with the CPU arms: the same config-4 levels g <= 7 sample, device-timed
    o7 = P.RunOptions(device=opts.device, stream=opts.stream, max_generation=args.cpu_sample_levels)
    with P.Plan(a4, o7) as pl:
        pl.run()
        reps = [pl.run() for _ in range(5)]
    r = min(reps, key=lambda x: x.enum_seconds)
    out["like_for_like"] = {"sample": f"config 4 levels g<={args.cpu_sample_levels}", "trace": r.trace_tuples(),
                            "candidates": r.candidates_enumerated, "device_ms": 1e3 * r.enum_seconds,
                            "combos_per_s": r.candidates_enumerated / r.enum_seconds, "statistic": "best of 5"}

    def host_timed(fn, reps):
        fn()
        ts, res = [], None
        for _ in range(reps):
            t0 = time.perf_counter()
            res = fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), res

    for cid in (1, 2):
        c = P.CONFIGS[cid]
        a = P.generate_code(c["n"], c["k"], c["seed"])
        t, r = host_timed(lambda: P.saved_isometry(a, opts), 5)
        out[f"config{cid}"] = {"distance": r.distance, "trace": r.trace_tuples(),
                               "e2e_time_to_distance_ms": 1e3 * t, "device_levels_ms": 1e3 * r.enum_seconds,
                               "combos_per_s_e2e": r.candidates_enumerated / t}
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
    for name in ("saved_1_gamma", "saved_2_gamma"):
        fn = getattr(P, name)
        t, r = host_timed(lambda: fn(a4, opts), 3)
        out[f"config4_{name}"] = {"distance": r.distance, "trace": r.trace_tuples(), "candidates": r.candidates_enumerated,
                                  "e2e_time_to_distance_ms": 1e3 * t, "device_levels_ms": 1e3 * r.enum_seconds,
                                  "combos_per_s": r.candidates_enumerated / r.enum_seconds}
    c = P.CONFIGS[1]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    r = P.compute_distance(a, P.Algorithm.brute_force, opts)
    out["config1_brute_force"] = {"distance": r.distance, "combinations": r.candidates_enumerated,
                                  "device_ms": 1e3 * r.enum_seconds}
    return out


def main():
    argv = sys.argv[1:]
    args = parse(argv)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and not world:
        return launch_ranks(args, argv)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
