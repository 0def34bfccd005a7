"""One run of a config with a given kernel (profiling target): python tools/tc_one.py CONFIG KERNEL [GMAX]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
cid, k = int(sys.argv[1]), int(sys.argv[2])
gmax = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = P.CONFIGS[cid]
a = P.generate_code(c["n"], c["k"], c["seed"])
with P.Plan(a, P.RunOptions(kernel=k, max_generation=gmax)) as pl:
    r = pl.run()
print(cid, k, r.trace_tuples()[-1], round(r.enum_seconds * 1e3, 3), "ms", [round(x * 1e3, 3) for x in r.level_seconds])
