"""Full time-to-distance of BASELINE config 5 ([[80,10]] seed 4) on one GPU.
Levels past g = 9 cannot be checked against the CPU reference (SURVEY.md §0 finding 3);
g <= 8 is pinned by tests/golden/config5_g8.json."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10743_b200 as P
c = P.CONFIGS[5]
a = P.generate_code(c["n"], c["k"], c["seed"])
t0 = time.perf_counter()
rep = P.saved_isometry(a, P.RunOptions())
wall = time.perf_counter() - t0
print(json.dumps({"config": 5, "distance": rep.distance, "trace": rep.trace_tuples(), "complete": rep.complete,
                  "candidates": rep.candidates_enumerated, "visited": rep.candidates_visited,
                  "device_levels_s": rep.enum_seconds, "time_to_distance_s": wall,
                  "combos_per_s": rep.candidates_enumerated / rep.enum_seconds,
                  "best": [rep.best_generation, rep.best_gamma, rep.best_rank]}), flush=True)
