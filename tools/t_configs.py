"""Time-to-distance of configs 1, 2 and 4 through saved_isometry (median of 5), with launches."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
for cid in (1, 2, 4):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    P.saved_isometry(a)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        r = P.saved_isometry(a)
        ts.append(time.perf_counter() - t0)
    print(cid, "d", r.distance, "e2e ms", round(1e3 * statistics.median(ts), 3), "device ms", round(1e3 * r.enum_seconds, 3),
          "launches", r.kernel_launches, flush=True)
