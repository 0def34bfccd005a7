import sys, time, paper_2408_10743_b200 as P
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for cid in (2, 4):
    c = P.CONFIGS[cid]
    a = P.generate_code(c['n'], c['k'], c['seed'])
    with P.Plan(a, P.RunOptions(kernel=kern)) as pl:
        r = pl.run(); r = pl.run()
        print(cid, r.distance, r.trace_tuples(), r.enum_seconds, r.candidates_enumerated/r.enum_seconds, [round(x*1e3,3) for x in r.level_seconds], flush=True)
