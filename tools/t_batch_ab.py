"""Config 3 batch e2e, median of 15 runs, with the host phase trace of the last one."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[3]
codes = [P.generate_code(c["n"], c["k"], s) for s in c["seeds"]]
e2e = []
for _ in range(15):
    r = P.saved_isometry_batch(codes)
    e2e.append(r.elapsed_seconds * 1e3)
print(os.environ.get("SDB_LIBRARY", "default"), "e2e median ms", round(statistics.median(e2e), 4),
      "min", round(min(e2e), 4), "device ms", round(r.device_seconds * 1e3, 4), flush=True)
