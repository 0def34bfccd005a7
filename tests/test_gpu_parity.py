"""GPU parity: the CUDA enumeration path (through the C ABI) against the golden fixtures
frozen from the reference and against the oracle, on the BASELINE configs and the
reference's own test instances. Bit-exact: distance, (g, L, U) trace, candidate counts,
best codeword."""
import numpy as np
import pytest

import oracle as O
from conftest import hex_to_mat, load_golden

pytestmark = pytest.mark.gpu


def tr(rep):
    return [e.astuple() for e in rep.bounds_trace]


# kernel: 0 auto (tensor-core tiles on levels >= 2^24 candidates), 1 lexicographic walk,
# 2 POPC head x tail tiles, 4 tensor-core tiles on every level g >= 2
@pytest.mark.parametrize("kernel", [0, 1, 2, 4])
@pytest.mark.parametrize("name", ["config1.json", "config2.json"])
def test_small_configs_bit_exact(gpu, name, kernel):
    gd = load_golden(name)
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    rep, best = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel), return_best=True)
    assert rep.distance == gd["distance"]
    assert tr(rep) == [tuple(t) for t in gd["trace"]]
    assert rep.candidates_enumerated == gd["candidates"]
    assert rep.generations == gd["generations"]
    assert rep.complete
    # BoundsState::best of the single-worker reference = first minimal candidate in visiting order
    assert (best == hex_to_mat([gd["best"]], gd["best_len"])[0]).all()


@pytest.mark.parametrize("kernel", [0, 2, 4])
def test_config4_bit_exact(gpu, kernel):
    gd = load_golden("config4.json")
    gb = load_golden("config4_iso_best.json")  # the single-worker reference's best (engine.cpp:182-189)
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    rep, best = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel), return_best=True)
    assert rep.distance == gd["distance"] == 10
    assert tr(rep) == [tuple(t) for t in gd["trace"]]
    assert rep.candidates_enumerated == gd["candidates"]
    assert rep.candidates_visited + rep.candidates_skipped == rep.candidates_enumerated
    assert 2 * rep.distance == gb["upper"]
    assert (best == hex_to_mat([gb["best"]], gb["best_len"])[0]).all()


def test_config5_first_eight_levels_bit_exact(gpu):
    gd = load_golden("config5_g8.json")
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    rep = gpu.saved_isometry(a, gpu.RunOptions(max_generation=8))
    assert not rep.complete
    assert tr(rep) == [tuple(t) for t in gd["trace"]]
    assert rep.candidates_enumerated == sum(gd["level_candidates"])


@pytest.mark.parametrize("kernel", [0, 2])
def test_config5_first_nine_levels_bit_exact(gpu, kernel):
    # g = 9 alone is 2.1e12 candidates, 99.99% of the levels through g = 9; the reference
    # (native build, 6 workers) took 2066 s on it (tests/golden/config5_g9.json)
    gd = load_golden("config5_g9.json")
    a = hex_to_mat(gd["normalizer"], 2 * gd["n"])
    rep = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel, max_generation=9))
    assert not rep.complete
    assert tr(rep) == [tuple(t) for t in gd["trace"]]
    assert rep.candidates_enumerated == rep.candidates_visited + rep.candidates_skipped == sum(gd["level_candidates"])


def test_batch_config3_bit_exact(gpu):
    gd = load_golden("config3.json")
    codes = [gpu.generate_code(gd["n"], gd["k"], c["seed"]) for c in gd["codes"]]
    res = gpu.saved_isometry_batch(codes)
    assert (res.statuses == 0).all()
    assert [int(x) for x in res.distances] == [c["distance"] for c in gd["codes"]]
    for got, c in zip(res.traces, gd["codes"]):
        assert got == [tuple(t) for t in c["trace"]]


def test_reference_kats(gpu):
    gd = load_golden("reference_kats.json")
    for case in gd["cases"]:
        a = hex_to_mat(case["normalizer"], 2 * case["n"])
        rep = gpu.saved_isometry(a)
        assert rep.distance == case["distance"] == case["brute"], case
        assert tr(rep) == [tuple(t) for t in case["trace"]], case
        assert rep.candidates_enumerated == case["candidates"], case


def test_reference_kats_batched(gpu):
    gd = load_golden("reference_kats.json")
    by_shape = {}
    for case in gd["cases"]:
        by_shape.setdefault((case["n"], case["k"]), []).append(case)
    for (n, k), cases in by_shape.items():
        mats = [hex_to_mat(c["normalizer"], 2 * n) for c in cases]
        res = gpu.saved_isometry_batch(mats)
        assert [int(x) for x in res.distances] == [c["distance"] for c in cases]
        assert res.traces == [[tuple(t) for t in c["trace"]] for c in cases]


def test_engine_singleton_kats_both_modes(gpu):
    # proj/tests/test_engine.cpp:121-161 shapes, answers from the reference's run_bz
    gd = load_golden("engine_kats.json")
    for case in gd["cases"]:
        if "matrix" not in case:
            continue
        n = case["n"]
        m = hex_to_mat(case["matrix"], 2 * n)
        sym = gpu.run_bz([gpu.singleton_gamma(m, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.disabled())
        assert sym.trace == [tuple(t) for t in case["symplectic"]["trace"]]
        assert sym.upper == case["symplectic"]["upper"]
        assert sym.candidates_enumerated == case["symplectic"]["candidates"]
        img = gpu.isometry_transform(m)
        ham = gpu.run_bz([gpu.singleton_gamma(img, gpu.WeightMode.hamming)], gpu.AdmissibilityFilter.disabled())
        assert ham.trace == [tuple(t) for t in case["hamming"]["trace"]]
        assert ham.upper == case["hamming"]["upper"]
        # general Hamming layout (not an isometry image): shuffle the columns
        perm = np.random.default_rng(n).permutation(3 * n)
        ham2 = gpu.run_bz([gpu.singleton_gamma(img[:, perm], gpu.WeightMode.hamming)],
                          gpu.AdmissibilityFilter.disabled())
        assert ham2.trace == ham.trace


def test_planted_distance_one_wide(gpu):
    # proj/tests/test_engine.cpp:163-182: scrambled (I_70 | 0), three words per half
    gd = load_golden("engine_kats.json")
    case = [c for c in gd["cases"] if "planted" in c][0]
    a = hex_to_mat(case["planted"], 2 * case["n"])
    rep = gpu.saved_isometry(a)
    assert rep.distance == 1 == case["distance"]
    assert tr(rep) == [tuple(t) for t in case["trace"]]


@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_oracle_agreement_random_instances(gpu, kernel):
    rng = np.random.default_rng(73)
    for _ in range(30):
        n = int(rng.integers(2, 30))
        k = int(rng.integers(0, n + 1))
        a = gpu.generate_code(n, k, int(rng.integers(1, 1 << 40)))
        mine, best = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel), return_best=True)
        if kernel:
            base, best0 = gpu.saved_isometry(a, return_best=True)
            assert (best == best0).all()
        ref = O.run_levels(a, threads=4)
        assert tr(mine) == ref["trace"]
        assert 2 * mine.distance == ref["upper"]
        if a.shape[0] <= 22:
            assert mine.distance == O.brute_force(a)


def test_filter_off_and_self_dual(gpu):
    # k = 0: filter disabled by construction (engine.cpp:19); dual_filter=False: plain minimum
    ident = np.zeros((5, 10), dtype=np.uint8)
    for i in range(5):
        ident[i, i] = 1
    assert gpu.saved_isometry(ident).distance == 1
    a = gpu.generate_code(16, 3, 99)
    plain = gpu.saved_isometry(a, gpu.RunOptions(dual_filter=False))
    ref = O.run_levels(a, dual_filter=False)
    assert tr(plain) == ref["trace"]
    filt = gpu.saved_isometry(a)
    assert plain.distance <= filt.distance


def test_worked_example_and_errors(gpu):
    ex = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8)
    assert gpu.saved_isometry(ex).distance == 1
    # raw matrix as singleton packages stops at 2 (test_engine.cpp:213-218)
    plain = gpu.run_bz([gpu.singleton_gamma(ex, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.for_rows(ex, 1))
    assert plain.upper == 2 and plain.generation == 1
    # exhaustion without an admissible codeword (test_engine.cpp:260-269)
    m = np.array([[1, 0, 0, 0]], dtype=np.uint8)
    with pytest.raises(gpu.InternalError):
        gpu.run_bz([gpu.singleton_gamma(m, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.for_rows(m, 1))
    # malformed calls (test_engine.cpp:271-285)
    g2 = gpu.singleton_gamma(np.array([[1, 0, 0, 1]]), gpu.WeightMode.symplectic)
    g3 = gpu.singleton_gamma(np.array([[1, 0, 0, 1, 1, 1]]), gpu.WeightMode.symplectic)
    with pytest.raises(ValueError):
        gpu.run_bz([], gpu.AdmissibilityFilter.disabled())
    with pytest.raises(ValueError):
        gpu.run_bz([g2, g3], gpu.AdmissibilityFilter.disabled())
    with pytest.raises(ValueError):
        gpu.run_bz([g2], gpu.AdmissibilityFilter.for_rows(np.array([[1, 0, 0, 1, 1, 1]]), 1))
    # validation gate (test_distance.cpp:93-100)
    with pytest.raises(gpu.ValidationError):
        gpu.saved_isometry(np.array([[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]]))


def test_visit_count_single_candidate(gpu):
    # test_engine.cpp:66-78: g = n_p on all-singleton packages visits one candidate
    m = np.eye(6, dtype=np.uint8)
    st = gpu.run_bz([gpu.singleton_gamma(m, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.disabled())
    assert st.report.candidates_visited == st.candidates_enumerated


@pytest.mark.parametrize("kernel", [1, 2])
def test_engine_kats_forced_kernels(gpu, kernel):
    gd = load_golden("engine_kats.json")
    for case in gd["cases"]:
        if "matrix" not in case:
            continue
        n = case["n"]
        m = hex_to_mat(case["matrix"], 2 * n)
        o = gpu.RunOptions(kernel=kernel)
        sym = gpu.run_bz([gpu.singleton_gamma(m, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.disabled(),
                         opts=o)
        assert sym.trace == [tuple(t) for t in case["symplectic"]["trace"]]
        ham = gpu.run_bz([gpu.singleton_gamma(gpu.isometry_transform(m), gpu.WeightMode.hamming)],
                         gpu.AdmissibilityFilter.disabled(), opts=o)
        assert ham.trace == [tuple(t) for t in case["hamming"]["trace"]]


def test_batch_host_prep_path_matches_device_prep(gpu):
    # kernel=3 forces the host prep (validation, isometry, information sets on the CPU);
    # the default batch path runs them on the device, one warp per code
    gd = load_golden("config3.json")
    codes = [gpu.generate_code(gd["n"], gd["k"], c["seed"]) for c in gd["codes"][:512]]
    dev = gpu.saved_isometry_batch(codes)
    host = gpu.saved_isometry_batch(codes, gpu.RunOptions(kernel=3))
    assert (dev.statuses == 0).all() and (host.statuses == 0).all()
    assert (dev.distances == host.distances).all()
    assert dev.traces == host.traces == [[tuple(t) for t in c["trace"]] for c in gd["codes"][:512]]


def test_batch_device_prep_rejects_what_the_host_rejects(gpu):
    rng = np.random.default_rng(5)
    good = [gpu.generate_code(12, 3, s) for s in range(1, 9)]
    dep = good[0].copy()
    dep[1] = dep[0]                                   # dependent rows
    rnd = rng.integers(0, 2, size=(15, 24), dtype=np.uint8)  # random rows: not a normalizer
    batch = good[:3] + [dep, rnd] + good[3:]
    for filt in (True, False):
        for validate in (True, False):
            o = gpu.RunOptions(validate=validate, dual_filter=filt)
            dev = gpu.saved_isometry_batch(batch, o)
            host = gpu.saved_isometry_batch(batch, gpu.RunOptions(validate=validate, dual_filter=filt, kernel=3))
            assert (dev.statuses == host.statuses).all(), (validate, filt, dev.statuses, host.statuses)
            ok = dev.statuses == 0
            assert (dev.distances[ok] == host.distances[ok]).all()
            assert [t for t, g in zip(dev.traces, ok) if g] == [t for t, g in zip(host.traces, ok) if g]
    st = gpu.saved_isometry_batch(batch).statuses
    assert st[3] == 2 and st[4] == 2 and (np.delete(st, [3, 4]) == 0).all()


@pytest.mark.parametrize("nk", [(20, 2), (12, 3), (30, 4), (40, 6), (33, 31), (3, 1)])
def test_batch_meet_in_the_middle_matches_walk(gpu, nk):
    # default: levels whose half-lists fit in shared memory pair A_h x B_(g-h); kernel=1 runs
    # every level on the per-thread lexicographic walk
    n, k = nk
    codes = [gpu.generate_code(n, k, s) for s in range(200, 200 + (256 if n <= 20 else 16))]
    o = dict(max_generation=4) if n > 30 else {}
    mitm = gpu.saved_isometry_batch(codes, gpu.RunOptions(**o))
    walk = gpu.saved_isometry_batch(codes, gpu.RunOptions(kernel=1, **o))
    assert (mitm.statuses == walk.statuses).all()
    assert (mitm.distances == walk.distances).all()
    assert mitm.traces == walk.traces


@pytest.mark.parametrize("nk", [(30, 4), (40, 6), (64, 0), (33, 31), (62, 2)])
def test_batch_device_prep_shapes(gpu, nk):
    # multi-word rows (n > 32), k = 0 (filter off), n + k = 64 rows (two rows per lane)
    n, k = nk
    codes = [gpu.generate_code(n, k, s) for s in range(100, 104)]
    dev = gpu.saved_isometry_batch(codes, gpu.RunOptions(max_generation=3) if n > 40 else None)
    host = gpu.saved_isometry_batch(codes, gpu.RunOptions(kernel=3, max_generation=3 if n > 40 else 0))
    assert (dev.statuses == host.statuses).all()
    assert dev.traces == host.traces


@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_wide_rows_first_levels(gpu, kernel):
    # n up to 256 (W = 4..8 words per half, the kernels' limit): the reference's first levels
    gd = load_golden("wide_codes.json")
    for case in gd["cases"]:
        a = hex_to_mat(case["normalizer"], 2 * case["n"])
        rep = gpu.saved_isometry(a, gpu.RunOptions(kernel=kernel, max_generation=case["g_max"]))
        assert tr(rep) == [tuple(t) for t in case["trace"]], (case["n"], case["k"], kernel)
        assert rep.candidates_enumerated == sum(case["level_candidates"])
        assert rep.candidates_visited + rep.candidates_skipped == rep.candidates_enumerated


def test_edge_shapes(gpu):
    # n = 1 codes, k = n (no stabilizer), k = 0, a single row, rows exactly on a word boundary
    for n, k in [(1, 0), (1, 1), (2, 2), (32, 0), (32, 1), (64, 0), (31, 1), (33, 2)]:
        a = gpu.generate_code(n, k, 5)
        rep = gpu.saved_isometry(a, gpu.RunOptions(max_generation=4))
        ref = O.run_levels(a, g_max=4)
        assert tr(rep) == ref["trace"], (n, k)
    with pytest.raises(gpu.ValidationError):  # validate_normalizer: "matrix has no rows"
        gpu.saved_isometry(np.zeros((0, 4), dtype=np.uint8))
    with pytest.raises(ValueError):
        gpu.saved_isometry(np.zeros((2, 3), dtype=np.uint8))  # odd column count
    with pytest.raises(ValueError):
        gpu.saved_isometry_batch([])
