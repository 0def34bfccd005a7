"""Saved_2_Gamma on config 4 with each kernel choice (per-run device time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[4]
a = P.generate_code(c["n"], c["k"], c["seed"])
for kern in (0, 2, 1):
    for mg in (6, 7, 8):
        r = P.saved_2_gamma(a, P.RunOptions(kernel=kern, max_generation=mg))
        print("kernel", kern, "g<=", mg, f"{r.enum_seconds*1e3:.2f} ms", r.candidates_enumerated, flush=True)
gs = P.prepare_packages(a, P.Algorithm.saved_2_gamma)
print([(g.matrix.shape, len(g.packages), g.n_pp, sum(len(p) == 3 for p in g.packages)) for g in gs])
