"""Config 3 batch (4096 [[20,2]] codes) timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[3]
codes = [P.generate_code(c["n"], c["k"], s) for s in c["seeds"]]
for _ in range(3):
    r = P.saved_isometry_batch(codes)
print("e2e ms", r.elapsed_seconds * 1e3, "device ms", r.device_seconds * 1e3)
