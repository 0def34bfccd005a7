"""Sweep (t, tchunk) of the packaged tile kernel per level on config 4's package routes
(SDB_TILE_FORCE); prints the route's device time for each forced level shape."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[4]
a = P.generate_code(c["n"], c["k"], c["seed"])


def dev(fn, force):
    if force:
        os.environ["SDB_TILE_FORCE"] = force
    else:
        os.environ.pop("SDB_TILE_FORCE", None)
    ts = []
    for _ in range(3):
        ts.append(fn(a).enum_seconds)
    return round(1e3 * statistics.median(ts), 3)


for alg in sys.argv[1:] or ["saved_1_gamma", "saved_2_gamma"]:
    fn = getattr(P, alg)
    r = fn(a)
    print(alg, "default", dev(fn, None), "levels", len(r.trace_tuples()), flush=True)
    for g in range(4, len(r.trace_tuples()) + 1):
        for t in range(1, g):
            for tc in (64, 256, 1024):
                print(alg, g, t, tc, dev(fn, f"{g}:{t}:{tc}"), flush=True)
