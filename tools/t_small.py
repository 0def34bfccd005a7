"""Config 2 / config 4 plan runs (for launch lists of the small levels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
for cid in (2, 4):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    with P.Plan(a) as pl:
        for _ in range(3):
            r = pl.run()
        print(cid, [round(x * 1e3, 4) for x in r.level_seconds], flush=True)
