"""Config 3 batch timing with every code stopped at a fixed level (kernel experiments)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[3]
codes = [P.generate_code(c["n"], c["k"], s) for s in c["seeds"]]
mg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(3):
    r = P.saved_isometry_batch(codes, P.RunOptions(max_generation=mg))
print(os.environ.get("SDB_LIBRARY", "default")[-40:], "max_g", mg, "e2e ms", round(r.elapsed_seconds * 1e3, 3),
      "device ms", round(r.device_seconds * 1e3, 3))
