"""Config 1/2 breakdown: per-level device times (Plan) and the host trace of saved_isometry."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
for cid in (1, 2):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    with P.Plan(a) as pl:
        for _ in range(3):
            r = pl.run()
    print(cid, "levels ms", [round(x * 1e3, 4) for x in r.level_seconds], "launches", r.kernel_launches, flush=True)
    for _ in range(3):
        r = P.saved_isometry(a)
    print(cid, "saved_isometry device ms", round(r.enum_seconds * 1e3, 4), flush=True)
