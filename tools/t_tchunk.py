"""Sweep (t, tchunk) of the tile kernel on some levels of a config (SDB_TILE_FORCE).
Usage: t_tchunk.py [config] [levels, e.g. 6,7,8]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
levels = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [6, 7, 8]
gmax = max(levels)
c = P.CONFIGS[cid]
a = P.generate_code(c["n"], c["k"], c["seed"])


def run(force):
    if force:
        os.environ["SDB_TILE_FORCE"] = force
    else:
        os.environ.pop("SDB_TILE_FORCE", None)
    with P.Plan(a, P.RunOptions(max_generation=gmax)) as pl:
        best = None
        for _ in range(4):
            r = pl.run()
            lv = r.level_seconds
            best = lv if best is None else [min(x, y) for x, y in zip(best, lv)]
    return [round(x * 1e3, 4) for x in best]


print("default", run(None), flush=True)
for g in levels:
    for t in range(1, g):
        for tc in (64, 128, 256, 512, 1024):
            lv = run(f"{g}:{t}:{tc}")
            print(g, t, tc, lv[g - 1], flush=True)
