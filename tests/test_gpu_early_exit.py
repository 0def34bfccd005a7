"""The mid-level early exit (kernels.cu early_key): once a level's minimum reaches L(g-1) it
is the distance, and units / segments whose keys all exceed the current best key are left
out. On codes where the distance is found exactly at L(g-1) (found by scanning seeded random
codes with the oracle), trace and best codeword must still equal the reference's, and
visited + skipped must equal the analytic count (reference engine.cpp:327-335, 182-189)."""
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

# (n, k, seed, level at which U drops to L(g-1))
CASES = [(16, 2, 153, 3), (18, 3, 2, 3), (18, 3, 119, 3), (18, 3, 292, 3), (16, 4, 96, 3), (16, 4, 153, 3),
         (12, 2, 225, 2), (14, 2, 74, 2), (18, 3, 31, 2)]


@pytest.mark.parametrize("kernel", [0, 1, 2, 4])
def test_early_exit_codes_match_the_reference(gpu, kernel):
    skipped = 0
    for n, k, seed, g_hit in CASES:
        a = O.generate(n, k, seed)
        ref = O.run_levels(a)
        rep, best = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel), return_best=True)
        trace = [e.astuple() for e in rep.bounds_trace]
        assert trace == ref["trace"], (n, k, seed)
        assert trace[g_hit - 1][2] <= trace[g_hit - 2][1]  # U reached L(g-1) at that level
        assert rep.candidates_visited + rep.candidates_skipped == rep.candidates_enumerated
        if O.ref_available():
            rb = O.ref_isometry_best(a, workers=1)
            assert list(best) == list(rb["best"][:len(best)]), (n, k, seed, kernel)
        skipped += rep.candidates_skipped
    # whether work is left out depends on timing; the count identity above holds either way
    print(f"kernel {kernel}: {skipped} candidates skipped over {len(CASES)} codes")
