"""Randomized parity against the reference library itself (oracle/_ref, built from
/root/reference/proj/src and shipped with the repo): every algorithm, every kernel choice,
random codes from the reference's own random_stabilizer and from the BASELINE generator.
Bit-exact: distance, (g, L, U) trace, candidates_enumerated."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

ALGS = ["saved_isometry", "saved_1_gamma", "saved_2_gamma"]


def _needs_ref():
    if not O.ref_available():
        pytest.fail("oracle/_ref (the reference library) is missing")


@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_random_codes_all_algorithms(gpu, kernel):
    _needs_ref()
    rng = np.random.default_rng(1000 + kernel)
    checked = 0
    for it in range(60):
        n = int(rng.integers(2, 26))
        k = int(rng.integers(0, n + 1))
        if it % 2:
            a = gpu.random_stabilizer(n, k, int(rng.integers(1, 1 << 40))).a
        else:
            a = gpu.generate_code(n, k, int(rng.integers(1, 1 << 40)))
        for alg in ALGS:
            ref = O.ref_compute_distance(a, alg)
            mine = gpu.compute_distance(a, gpu.Algorithm[alg], gpu.RunOptions(kernel=kernel))
            assert mine.distance == ref.distance, (n, k, alg)
            assert mine.trace_tuples() == [tuple(t) for t in ref.trace], (n, k, alg)
            assert mine.candidates_enumerated == ref.candidates, (n, k, alg)
            checked += 1
    assert checked == 180


def test_random_codes_filter_off_and_auto(gpu):
    _needs_ref()
    rng = np.random.default_rng(77)
    for _ in range(30):
        n = int(rng.integers(2, 20))
        k = int(rng.integers(0, n + 1))
        a = gpu.random_stabilizer(n, k, int(rng.integers(1, 1 << 40))).a
        for alg in ALGS + ["auto"]:
            ref = O.ref_compute_distance(a, alg, dual_filter=False)
            algo = gpu.Algorithm.auto_select if alg == "auto" else gpu.Algorithm[alg]
            mine = gpu.compute_distance(a, algo, gpu.RunOptions(dual_filter=False))
            assert mine.distance == ref.distance and mine.trace_tuples() == [tuple(t) for t in ref.trace]
            assert gpu.Algorithm(mine.algorithm).name == ref.algorithm or alg != "auto"
