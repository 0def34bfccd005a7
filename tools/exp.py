"""Experiment driver (GPU box; not product code, not used by tests or bench.py).

  python tools/exp.py time   [--kernel K] [--configs 2,4,5] [--lib PATH]   level timings (Plan, 2nd run)
  python tools/exp.py check  [--kernels 4,2,0] [--configs 1,2,4,5]         traces vs the reference goldens
  python tools/exp.py e2e    [--configs 1,2,4]                              saved_isometry wall vs device time
  python tools/exp.py shard  [--configs 4,5]                               1-GPU emulation of the P-rank split
  python tools/exp.py sweep  --config 4 --levels 6,7,8                      (t, tchunk) sweep, SDB_TILE_FORCE
  python tools/exp.py config5                                              config 5 to its distance (~10 min)

--lib loads another build of the same C ABI (tools/build_variant.sh) for A/B runs; config 5 is
run through g = 9 unless --gmax says otherwise.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from math import comb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2408_10743_b200 as P  # noqa: E402


def code(cid):
    c = P.CONFIGS[cid]
    return P.generate_code(c["n"], c["k"], c["seed"])


def ms(xs):
    return [round(x * 1e3, 3) for x in xs]


def cmd_time(a):
    for cid in a.configs:
        gmax = a.gmax if cid == 5 or a.gmax != 9 else 0
        with P.Plan(code(cid), P.RunOptions(kernel=a.kernel, max_generation=gmax)) as pl:
            pl.run()
            r = pl.run()
        print(os.path.basename(os.path.dirname(P.library_path())), f"k{a.kernel}", cid, r.distance,
              r.trace_tuples()[-1], round(r.enum_seconds * 1e3, 3), "ms",
              f"{r.candidates_enumerated / r.enum_seconds:.3e}", ms(r.level_seconds), flush=True)


def cmd_check(a):
    for cid in a.configs:
        gname = {5: "config5_g9.json"}.get(cid, f"config{cid}.json")
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", gname)))
        gmax = 9 if cid == 5 else 0
        want = [tuple(x) for x in gold["trace"]]
        for k in a.kernels:
            with P.Plan(code(cid), P.RunOptions(kernel=k, max_generation=gmax)) as pl:
                pl.run()
                r = pl.run()
            ok = r.trace_tuples() == want
            print(f"config {cid} kernel {k}: trace {'OK' if ok else 'MISMATCH'} d={r.distance} "
                  f"{r.enum_seconds * 1e3:.3f} ms {r.candidates_enumerated / max(r.enum_seconds, 1e-12):.3e} cand/s "
                  f"visited==enum {r.candidates_visited == r.candidates_enumerated} best (g={r.best_generation}, "
                  f"j={r.best_gamma}, r={r.best_rank}) levels_ms={ms(r.level_seconds)}", flush=True)


def cmd_e2e(a):
    for cid in a.configs:
        x = code(cid)
        P.saved_isometry(x)
        ts, r = [], None
        for _ in range(10):
            t = time.perf_counter()
            r = P.saved_isometry(x)
            ts.append(time.perf_counter() - t)
        print(cid, f"wall {statistics.median(ts) * 1e3:.3f} ms", f"elapsed {r.elapsed_seconds * 1e3:.3f}",
              f"prep {r.prep_seconds * 1e3:.3f}", f"levels {r.enum_seconds * 1e3:.3f}", "launches", r.kernel_launches,
              flush=True)


class GlobalAnswer:
    """allreduce_min stand-in for the shard emulation: level g's exchange returns the global
    level minimum known from the one-GPU run, so each rank sees a real run's thresholds."""

    NONE = np.uint64(2**64 - 1)

    def __init__(self, trace, sentinel, levels):
        self.mins, prev = [], sentinel
        for (_, _, U) in trace:
            self.mins.append(U if U < prev else None)
            prev = U
        self.levels, self.calls = levels, 0

    def __call__(self, v):
        lvl = self.levels[self.calls // 2]
        first = self.calls % 2 == 0
        self.calls += 1
        m = self.mins[lvl - 1]
        if first:
            return np.array([np.uint64(m) if m is not None else self.NONE], dtype=np.uint64)
        return v


def cmd_shard(a):
    """Each rank of world P runs its own share alone on one GPU, one after another (nothing
    waits on another rank); the slowest rank per level estimates the P-GPU step."""
    shard_min = 1 << 26
    for cid in a.configs:
        c = P.CONFIGS[cid]
        gmax = a.gmax if cid == 5 else 0
        x = code(cid)
        with P.Plan(x, P.RunOptions(max_generation=gmax)) as pl:
            pl.run()
            base = pl.run()
        t1, nl = sum(base.level_seconds), len(base.level_seconds)
        N = c["n"] + c["k"]
        sharded = [g for g in range(1, nl + 1) if 3 * comb(N, g) >= shard_min]
        for world in (2, 4, 8):
            per_level = None
            for r in range(world):
                ga = GlobalAnswer(base.trace_tuples(), 3 * c["n"] + 1, sharded)
                o = P.RunOptions(rank=r, world=world, allreduce_min=ga, max_generation=gmax, shard_min=shard_min)
                with P.Plan(x, o) as pl:
                    pl.run()
                    ga.calls = 0
                    rep = pl.run()
                assert rep.trace_tuples() == base.trace_tuples()
                lv = rep.level_seconds[:nl]
                per_level = lv if per_level is None else [max(p, q) for p, q in zip(per_level, lv)]
            tp = sum(per_level)
            print(f"config {cid} g<={gmax or 'all'} world {world}: 1-GPU {t1 * 1e3:.2f} ms, slowest rank "
                  f"{tp * 1e3:.2f} ms, efficiency {t1 / (world * tp):.3f}", ms(per_level), flush=True)


def cmd_sweep(a):
    x = code(a.config)
    gmax = max(a.levels)

    def run(force):
        if force:
            os.environ["SDB_TILE_FORCE"] = force
        else:
            os.environ.pop("SDB_TILE_FORCE", None)
        with P.Plan(x, P.RunOptions(kernel=2, max_generation=gmax)) as pl:
            best = None
            for _ in range(4):
                lv = pl.run().level_seconds
                best = lv if best is None else [min(p, q) for p, q in zip(best, lv)]
        return ms(best)

    print("default", run(None), flush=True)
    for g in a.levels:
        for t in range(1, g):
            for tc in (64, 128, 256, 512, 1024):
                print(g, t, tc, run(f"{g}:{t}:{tc}")[g - 1], flush=True)


def cmd_config5(a):
    t0 = time.perf_counter()
    rep = P.saved_isometry(code(5), P.RunOptions(max_generation=a.gmax if a.gmax != 9 else 0))
    wall = time.perf_counter() - t0
    print(json.dumps({"config": 5, "distance": rep.distance, "trace": rep.trace_tuples(), "complete": rep.complete,
                      "candidates": rep.candidates_enumerated, "visited": rep.candidates_visited,
                      "device_levels_s": rep.enum_seconds, "time_to_distance_s": wall,
                      "level_s": rep.level_seconds, "combos_per_s": rep.candidates_enumerated / rep.enum_seconds,
                      "best": [rep.best_generation, rep.best_gamma, rep.best_rank]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["time", "check", "e2e", "shard", "sweep", "config5"])
    ap.add_argument("--configs", default="")
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--kernels", default="4,2,0")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--levels", default="6,7,8")
    ap.add_argument("--gmax", type=int, default=9)
    ap.add_argument("--lib", default="")
    a = ap.parse_args()
    if a.lib:
        P.use_variant_library(a.lib)
    defaults = {"time": "2,4,5", "check": "1,2,4,5", "e2e": "1,2,4", "shard": "4,5"}
    a.configs = [int(x) for x in (a.configs or defaults.get(a.cmd, "4")).split(",")]
    a.kernels = [int(x) for x in a.kernels.split(",")]
    a.levels = [int(x) for x in a.levels.split(",")]
    globals()["cmd_" + a.cmd](a)


if __name__ == "__main__":
    main()
