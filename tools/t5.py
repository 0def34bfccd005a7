"""Config 5 through g = 10 (timing experiments): python tools/t5.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
lib = os.environ.get("SDB_LIBRARY", "default")
c = P.CONFIGS[5]
a = P.generate_code(c['n'], c['k'], c['seed'])
for gmax in (9, 10):
    with P.Plan(a, P.RunOptions(max_generation=gmax)) as pl:
        r = pl.run(); r = pl.run()
        print(lib, gmax, r.trace_tuples()[-1], round(r.enum_seconds * 1e3, 3), "ms", f"{r.candidates_enumerated/r.enum_seconds:.3e}",
              [round(x*1e3,3) for x in r.level_seconds], flush=True)
