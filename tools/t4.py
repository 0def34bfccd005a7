"""Kernel timing across configs (variant experiments): python tools/t4.py [kernel]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfgs = ((2, 0), (4, 0), (5, 9)) if len(sys.argv) <= 2 else tuple((int(x), 9 if int(x) == 5 else 0) for x in sys.argv[2].split(","))
lib = os.environ.get("SDB_LIBRARY", "default")
for cid, gmax in cfgs:
    c = P.CONFIGS[cid]
    a = P.generate_code(c['n'], c['k'], c['seed'])
    with P.Plan(a, P.RunOptions(kernel=kern, max_generation=gmax)) as pl:
        r = pl.run(); r = pl.run()
        print(lib, f"k{kern}", cid, r.distance, r.trace_tuples()[-1], round(r.enum_seconds * 1e3, 3), "ms", f"{r.candidates_enumerated/r.enum_seconds:.3e}",
              [round(x*1e3,3) for x in r.level_seconds], flush=True)
