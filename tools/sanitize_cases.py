"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): configs 1-2 on every
kernel family (walk, POPC tile, tensor-core tile), a small config-3 batch (device prep +
meet-in-the-middle batch kernel), the package routes and brute force on config 1.
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P  # noqa: E402

want = {1: 5, 2: 7}
for cid in (1, 2):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for kernel in (0, 1, 2, 4):
        r = P.saved_isometry(a, P.RunOptions(kernel=kernel))
        assert r.distance == want[cid], (cid, kernel, r.distance)
        print(f"config {cid} kernel {kernel}: d={r.distance}", flush=True)
    for fn in (P.saved_1_gamma, P.saved_2_gamma):
        r = fn(a, P.RunOptions())
        assert r.distance == want[cid]
        print(f"config {cid} {fn.__name__}: d={r.distance}", flush=True)
c = P.CONFIGS[3]
codes = [P.generate_code(c["n"], c["k"], s) for s in c["seeds"][:128]]
res = P.saved_isometry_batch(codes)
assert (res.statuses == 0).all()
print("config 3 batch (128 codes): distances", sorted(set(int(d) for d in res.distances)), flush=True)
c = P.CONFIGS[1]
r = P.compute_distance(P.generate_code(c["n"], c["k"], c["seed"]), P.Algorithm.brute_force)
assert r.distance == 5
print("config 1 brute force: d=5\nsanitize cases done", flush=True)
