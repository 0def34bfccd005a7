"""GPU parity of the per-level seam enumerate_generation (reference engine.hpp:53-54,
engine.cpp:296-301) through sdb_enumerate_generation: one matrix, one
generation, folded into a bound state. Answers come from the reference library
(tests/golden/enumerate_generation.json, make_golden.py --only enumgen): the new upper bound, the
candidate count and the first minimal codeword, entered with upper = 0 (unset), with the previous
level's bound and with a tight bound, in Hamming mode (information sets) and symplectic mode
(1- and 3-packages)."""
import numpy as np
import pytest

from conftest import hex_to_mat, load_golden

pytestmark = pytest.mark.gpu


def _gamma(gpu, case):
    m = hex_to_mat(case["matrix"], case["cols"])
    mode = gpu.WeightMode.hamming if case["mode"] == "hamming" else gpu.WeightMode.symplectic
    gm = gpu.singleton_gamma(m, mode)
    gm.packages = [list(p) for p in case["packages"]]
    filt = (gpu.AdmissibilityFilter.for_rows(hex_to_mat(case["filter"], case["filter_cols"]), case["k"])
            if case["filter"] else gpu.AdmissibilityFilter.disabled())
    return gm, filt


def test_enumerate_generation_matches_reference(gpu):
    gd = load_golden("enumerate_generation.json")
    assert len(gd["cases"]) > 100
    for case in gd["cases"]:
        gm, filt = _gamma(gpu, case)
        st = gpu.BoundsState(upper=case["upper_in"], candidates_enumerated=7)
        gpu.enumerate_generation(gm, case["g"], st, filt)
        key = (case["src"], case["g"], case["upper_in"])
        assert st.upper == case["upper"], key
        assert st.candidates_enumerated == 7 + case["candidates"], key
        if case["best"]:
            want = hex_to_mat([case["best"]], case["cols"])[0]
            assert np.array_equal(st.best, want), key
        else:
            assert st.best.size == 0, key  # no improvement: best untouched


def test_enumerate_generation_errors(gpu):
    gd = load_golden("enumerate_generation.json")
    case = next(c for c in gd["cases"] if c["mode"] == "hamming" and c["filter"])
    gm, filt = _gamma(gpu, case)
    np_ = gm.n_p()
    for g in (0, np_ + 1):  # engine.cpp:276-278: generation out of range
        with pytest.raises(ValueError, match="generation out of range"):
            gpu.enumerate_generation(gm, g, gpu.BoundsState(), filt)
    bad = gpu.AdmissibilityFilter.for_rows(np.ones((2, case["filter_cols"] + 2), dtype=np.uint8), 1)
    with pytest.raises(ValueError, match="filter frame mismatch"):  # engine.cpp:279-281
        gpu.enumerate_generation(gm, 1, gpu.BoundsState(), bad)


def test_generation_loop_over_the_seam_equals_run_bz(gpu):
    # run_bz (engine.cpp:303-343) rebuilt on the host from enumerate_generation and
    # lower_bound reproduces saved_isometry's trace and candidate count (config 1)
    gd = load_golden("config1.json")
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    gammas = gpu.information_sets(gpu.isometry_transform(a))
    filt = gpu.AdmissibilityFilter.for_rows(a, gd["k"])
    st = gpu.BoundsState()
    trace = []
    for g in range(1, min(gm.n_p() for gm in gammas) + 1):
        for gm in gammas:
            gpu.enumerate_generation(gm, g, st, filt)
        lower = gpu.lower_bound(g, gammas)
        trace.append((g, lower, st.upper))
        if lower >= st.upper:
            break
    assert trace == [tuple(t) for t in gd["trace"]]
    assert st.candidates_enumerated == gd["candidates"]
    rep = gpu.saved_isometry(a)
    assert st.upper == 2 * rep.distance
