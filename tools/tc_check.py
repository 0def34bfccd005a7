"""Tensor-core tile kernel vs the POPC tile kernel and the reference goldens:
python tools/tc_check.py [configs, e.g. 1,2,4,5] [kernels, e.g. 4,2,0]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_10743_b200 as P

cfgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,5").split(",")]
kerns = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,2").split(",")]
for cid in cfgs:
    gname = {5: "config5_g8.json"}.get(cid, f"config{cid}.json")
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", gname)))
    gmax = 8 if cid == 5 else 0
    want = [tuple(x) for x in gold["trace"]]
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for k in kerns:
        with P.Plan(a, P.RunOptions(kernel=k, max_generation=gmax)) as pl:
            r = pl.run()
            r = pl.run()
        tr = r.trace_tuples()
        ok = tr == want
        print(f"config {cid} kernel {k}: trace {'OK' if ok else 'MISMATCH'} d={r.distance} "
              f"{r.enum_seconds*1e3:.3f} ms {r.candidates_enumerated/max(r.enum_seconds,1e-12):.3e} cand/s "
              f"visited==enum {r.candidates_visited == r.candidates_enumerated} ({r.candidates_visited} vs {r.candidates_enumerated}) "
              f"best (g={r.best_generation}, j={r.best_gamma}, r={r.best_rank}) levels_ms={[round(x*1e3,3) for x in r.level_seconds]}",
              flush=True)
        if not ok:
            print("   got ", tr)
            print("   want", want)
