"""Where the e2e time of one saved_isometry call goes (config 4 and 2)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
for cid in (2, 4):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for validate in (True, False):
        o = P.RunOptions(validate=validate)
        P.saved_isometry(a, o)
        ts, r = [], None
        for _ in range(10):
            t = time.perf_counter(); r = P.saved_isometry(a, o); ts.append(time.perf_counter() - t)
        wall = statistics.median(ts)
        print(cid, "validate" if validate else "no-validate", f"wall {wall*1e3:.3f} ms", f"elapsed {r.elapsed_seconds*1e3:.3f}",
              f"prep {r.prep_seconds*1e3:.3f}", f"levels {r.enum_seconds*1e3:.3f}", flush=True)
