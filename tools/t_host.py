import os, sys, time
sys.path.insert(0, "/root/repo")
os.environ["SDB_TRACE_HOST"] = "1"
import paper_2408_10743_b200 as P
for cid in (2, 4):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for _ in range(4):
        t = time.perf_counter(); r = P.saved_isometry(a); w = time.perf_counter() - t
        print(cid, f"wall {w*1e3:.3f} elapsed {r.elapsed_seconds*1e3:.3f} enum {r.enum_seconds*1e3:.3f}", file=sys.stderr, flush=True)
