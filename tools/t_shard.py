"""Single-GPU emulation of the sharded level loop: every rank of world P runs its own share
alone (one after another; nothing waits on another rank). The exchange is replaced by the
global answer known from the one-GPU run (the level minimum that lowered U, else none), so
every rank sees the thresholds a real P-GPU run would. The slowest rank's level time then
estimates the P-GPU step; prints the estimated strong-scaling efficiency (NCCL latency, ~10-20
us per sharded level, not included)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P

NONE = np.uint64(2**64 - 1)


class GlobalAnswer:
    """allreduce_min stand-in: level g's exchange returns the global level minimum."""

    def __init__(self, trace, sentinel, levels):
        self.mins = []
        prev = sentinel
        for (g, L, U) in trace:
            self.mins.append(U if U < prev else None)
            prev = U
        self.levels = levels  # which levels exchange (sharded ones), in order
        self.calls = 0

    def __call__(self, v):
        lvl = self.levels[self.calls // 2]
        first = self.calls % 2 == 0
        self.calls += 1
        m = self.mins[lvl - 1]
        if first:
            return np.array([np.uint64(m) if m is not None else NONE], dtype=np.uint64)
        return v  # the key: this rank's own (timing only)


for cid, gmax in ((4, 0), (5, 9)):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    with P.Plan(a, P.RunOptions(max_generation=gmax)) as pl:
        pl.run()
        base = pl.run()
    t1 = sum(base.level_seconds)
    n_levels = len(base.level_seconds)
    sentinel = 3 * c["n"] + 1
    # levels with fewer candidates than shard_min run whole on every rank (no exchange)
    shard_min = int(os.environ.get("SHARD_MIN", str(1 << 26)))
    from math import comb
    N = c["n"] + c["k"]
    sharded = [g for g in range(1, n_levels + 1) if 3 * comb(N, g) >= shard_min]
    for world in (2, 4, 8):
        per_level = None
        for r in range(world):
            ga = GlobalAnswer(base.trace_tuples(), sentinel, sharded)
            o = P.RunOptions(rank=r, world=world, allreduce_min=ga, max_generation=gmax, shard_min=shard_min)
            with P.Plan(a, o) as pl:
                pl.run()
                ga.calls = 0
                rep = pl.run()
            assert rep.trace_tuples() == base.trace_tuples()
            lv = rep.level_seconds[:n_levels]
            if os.environ.get("SHARD_VERBOSE"):
                print("  rank", r, [round(x * 1e3, 3) for x in lv], flush=True)
            per_level = lv if per_level is None else [max(x, y) for x, y in zip(per_level, lv)]
        tp = sum(per_level)
        print(f"config {cid} g<={gmax or 'all'} world {world}: 1-GPU {t1*1e3:.2f} ms, slowest rank {tp*1e3:.2f} ms, "
              f"efficiency {t1 / (world * tp):.3f}", [round(x * 1e3, 3) for x in per_level], flush=True)
