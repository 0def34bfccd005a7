"""CPU: pin the oracle (our C restatement) to the reference.

1. against the golden fixtures frozen from the reference build (tests/golden/*.json);
2. against the reference library itself (oracle/_ref, compiled from
   /root/reference/proj/src) on random instances, when it is present here.
"""
import numpy as np
import pytest

import oracle as O
from conftest import hex_to_mat, load_golden


def test_generator_c_matches_python_twin():
    for n, k, seed in [(24, 4, 1), (40, 6, 2), (20, 2, 1000), (33, 3, 7), (5, 0, 9), (7, 7, 3)]:
        assert (O.generate(n, k, seed) == O.py_generate(n, k, seed)).all()


@pytest.mark.parametrize("cid", [1, 2, 4, 5])
def test_generator_matches_golden_normalizer(cid):
    name = {1: "config1.json", 2: "config2.json", 4: "config4.json", 5: "config5_g8.json"}[cid]
    gd = load_golden(name)
    a = O.generate(gd["n"], gd["k"], gd["seed"])
    assert (a == hex_to_mat(gd["normalizer"], 2 * gd["n"])).all()
    assert O.validate(a) == 0


@pytest.mark.parametrize("cid", [1, 2, 4, 5])
def test_information_sets_match_golden_gammas(cid):
    name = {1: "config1.json", 2: "config2.json", 4: "config4.json", 5: "config5_g8.json"}[cid]
    gd = load_golden(name)
    n = gd["n"]
    a = hex_to_mat(gd["normalizer"], 2 * n)
    gammas = O.information_sets(O.isometry(a))
    assert len(gammas) == len(gd["gammas"]) == 3
    for mine, ref in zip(gammas, gd["gammas"]):
        assert mine["rank_deficit"] == ref["rank_deficit"]
        assert mine["pivots"] == ref["pivots"]
        assert (mine["matrix"] == hex_to_mat(ref["matrix"], 3 * n)).all()


@pytest.mark.parametrize("name", ["config1.json", "config2.json"])
def test_oracle_trace_matches_golden(name):
    gd = load_golden(name)
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    res = O.run_levels(a, threads=4)
    assert [tuple(t) for t in gd["trace"]] == res["trace"]
    assert res["upper"] == 2 * gd["distance"]


def test_oracle_config5_first_levels_match_golden():
    gd = load_golden("config5_g8.json")
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    res = O.run_levels(a, g_max=4, threads=4)
    assert res["trace"] == [tuple(t) for t in gd["trace"][:4]]


def test_oracle_batch_sample_matches_golden():
    gd = load_golden("config3.json")
    for code in gd["codes"][::64]:
        a = O.generate(gd["n"], gd["k"], code["seed"])
        res = O.run_levels(a)
        assert res["trace"] == [tuple(t) for t in code["trace"]]
        assert res["upper"] == 2 * code["distance"]


def test_batch_histogram_matches_survey_probe():
    gd = load_golden("config3.json")
    assert gd["histogram"] == {"2": 24, "3": 442, "4": 2753, "5": 877}


def test_oracle_reference_kats():
    gd = load_golden("reference_kats.json")
    for case in gd["cases"]:
        n = case["n"]
        a = hex_to_mat(case["normalizer"], 2 * n)
        res = O.run_levels(a)
        assert res["trace"] == [tuple(t) for t in case["trace"]], case["src"]
        assert res["upper"] == 2 * case["distance"]
        assert case["brute"] == case["distance"]
        if a.shape[0] <= 22:
            assert O.brute_force(a) == case["distance"]


# ---------------------------------------------------------------- live reference, when built here

ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@ref
def test_oracle_matches_live_reference_random():
    rng = np.random.default_rng(5)
    for _ in range(25):
        n = int(rng.integers(3, 14))
        k = int(rng.integers(0, n + 1))
        a = O.ref_random_stabilizer(n, k, int(rng.integers(1, 1 << 40)))
        r = O.ref_compute_distance(a, "saved_isometry")
        mine = O.run_levels(a)
        assert mine["trace"] == r.trace
        assert mine["upper"] == 2 * r.distance


@ref
def test_oracle_best_matches_live_reference_best():
    # the reference's single-worker best codeword == first minimal candidate in
    # (level, Gamma, lexicographic) order, which is what the oracle's best key records
    for cid in (1, 2):
        c = O.CONFIGS[cid]
        a = O.generate(c["n"], c["k"], c["seed"])
        rb = O.ref_isometry_best(a)
        res = O.run_levels(a)
        g = max(i for i, (gj, _) in enumerate(res["best"]) if gj >= 0) + 1
        j, rank = res["best"][g - 1]
        gam = O.information_sets(O.isometry(a))[j]["matrix"]
        # lexicographic unrank
        N = gam.shape[0]
        r, v, rows = rank, 0, []
        for i in range(g):
            while True:
                cnt = O.binom(N - 1 - v, g - 1 - i)
                if r < cnt:
                    break
                r -= cnt
                v += 1
            rows.append(v)
            v += 1
        cw = np.bitwise_xor.reduce(gam[rows], axis=0)
        assert (cw == rb["best"]).all()


@ref
def test_oracle_validation_agrees_with_reference():
    cases = [np.array(m, dtype=np.uint8) for m in (
        [[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]],
        [[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]],
        [[1, 0, 0, 0], [0, 0, 1, 0]],
    )]
    for a in cases:
        ok, _ = O.ref_validate(a)
        assert ok == (O.validate(a) == 0)


@ref
def test_enumerate_generation_golden_matches_live_reference():
    # the fixture the GPU parity test reads was produced by the reference's own
    # enumerate_generation; a sample of it is re-answered live here
    gd = load_golden("enumerate_generation.json")
    for case in gd["cases"][::7]:
        m = hex_to_mat(case["matrix"], case["cols"])
        frows = hex_to_mat(case["filter"], case["filter_cols"]) if case["filter"] else None
        r = O.ref_enumerate_generation(m, case["mode"], case["g"], upper=case["upper_in"],
                                       packages=case["packages"] or None, filter_rows=frows, filter_k=case["k"])
        assert r["upper"] == case["upper"] and r["candidates"] == case["candidates"], case["src"]
        best = hex_to_mat([case["best"]], case["cols"])[0] if case["best"] else np.zeros(0, np.uint8)
        assert np.array_equal(r["best"], best), case["src"]
