"""Package-route timings (Saved_1_Gamma / Saved_2_Gamma) on BASELINE configs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
for cid, algs in ((2, ("saved_1_gamma", "saved_2_gamma")), (4, ("saved_1_gamma", "saved_2_gamma"))):
    c = P.CONFIGS[cid]
    a = P.generate_code(c["n"], c["k"], c["seed"])
    for alg in algs:
        fn = getattr(P, alg)
        fn(a)
        t = time.perf_counter(); r = fn(a); el = time.perf_counter() - t
        print(cid, alg, r.distance, r.trace_tuples(), r.candidates_enumerated, f"e2e {el*1e3:.2f} ms",
              f"dev {r.enum_seconds*1e3:.2f} ms", f"{r.candidates_enumerated / r.enum_seconds:.3e} cand/s", flush=True)
b = P.compute_distance(P.generate_code(24, 4, 1), P.Algorithm.brute_force)
print("brute config1", b.distance, f"{b.enum_seconds*1e3:.2f} ms", f"{b.candidates_enumerated/b.enum_seconds:.3e}")
