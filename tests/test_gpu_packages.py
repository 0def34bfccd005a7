"""GPU parity of the package routes (Saved_1_Gamma / Saved_2_Gamma)
against the reference's own answers (tests/golden/package_routes.json, make_golden.py):
distance, the (g, L, U) trace, candidates_enumerated and the best codeword (the
single-worker BoundsState::best), through the C ABI."""
import numpy as np
import pytest

from conftest import hex_to_mat, load_golden

pytestmark = pytest.mark.gpu


def tr(rep):
    return [e.astuple() for e in rep.bounds_trace]


def _run(gpu, case, kernel=0, **kw):
    a = hex_to_mat(case["normalizer"], 2 * case["n"])
    o = gpu.RunOptions(validate=case.get("validate", True), dual_filter=case.get("dual_filter", True), kernel=kernel,
                       **kw)
    fn = gpu.saved_1_gamma if case["alg"] == "saved_1_gamma" else gpu.saved_2_gamma
    return fn(a, o, return_best=True)




@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("which", ["configs", "examples", "random"])
def test_package_routes_bit_exact(gpu, which, kernel):
    gd = load_golden("package_routes.json")
    sel = {"configs": lambda c: c["src"].startswith("config"),
           "examples": lambda c: c["src"].startswith("test_prep") or c["src"].startswith("test_distance.cpp:57"),
           "random": lambda c: c["src"].startswith("test_distance.cpp:1")}[which]
    cases = [c for c in gd["cases"] if sel(c)]
    assert cases
    for case in cases:
        if kernel == 1 and case["candidates"] > 2e10:
            continue  # the walk kernel alone takes seconds there
        rep, best = _run(gpu, case, kernel=kernel)
        assert rep.distance == case["distance"], case["src"]
        assert tr(rep) == [tuple(t) for t in case["trace"]], (case["src"], case["alg"])
        assert rep.candidates_enumerated == case["candidates"]
        assert rep.candidates_visited == case["candidates"]
        assert rep.generations == case["generations"]
        if "best" in case:
            assert (best == hex_to_mat([case["best"]], case["best_len"])[0]).all(), (case["src"], case["alg"])
        if "brute" in case:
            assert rep.distance == case["brute"]


@pytest.mark.parametrize("kernel", [0, 2])
def test_config4_saved_2_gamma_bit_exact(gpu, kernel):
    # the reference's saved_2_gamma on config 4 (distance.cpp:115-133; 1.5e11 candidates,
    # 195 s on 8 threads: tests/golden/config4_s2g.json); the best codeword when its
    # single-worker golden (config4_s2g_best.json) exists
    gd = load_golden("config4_s2g.json")
    c = gpu.CONFIGS[4]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    rep, best = gpu.saved_2_gamma(a, gpu.RunOptions(kernel=kernel), return_best=True)
    assert rep.distance == gd["distance"] == 10
    assert tr(rep) == [tuple(t) for t in gd["trace"]]
    assert rep.candidates_enumerated == rep.candidates_visited == gd["candidates"]
    assert rep.generations == gd["generations"]
    try:
        gb = load_golden("config4_s2g_best.json")
    except pytest.skip.Exception:
        return
    assert (best == hex_to_mat([gb["best"]], gb["best_len"])[0]).all()


def test_auto_dispatch_sends_small_k_to_two_gamma(gpu):
    gd = load_golden("package_routes.json")["config3_auto"]
    for c in gd["codes"][:64]:
        a = gpu.generate_code(gd["n"], gd["k"], c["seed"])
        rep = gpu.compute_distance(a, gpu.Algorithm.auto_select)
        assert rep.algorithm == gpu.Algorithm.saved_2_gamma
        assert rep.distance == c["distance"]
        assert tr(rep) == [tuple(t) for t in c["trace"]]
        assert rep.candidates_enumerated == c["candidates"]


def test_run_bz_with_prepared_packages(gpu):
    # the engine seam (engine.hpp:60-61) with the routes' prepared matrices, and the additive
    # example of test_engine.cpp:184-203: bounds (1, 2, 3), (2, 3, 2), best = (a2, a, 0, 0)
    add = np.array([[int(ch) for ch in r] for r in ("11110000", "00001011", "01110111")], dtype=np.uint8)
    b, _ = gpu.prepare_packages(add, gpu.Algorithm.saved_2_gamma)
    st = gpu.run_bz([b], gpu.AdmissibilityFilter.disabled())
    assert st.trace == [(1, 2, 3), (2, 3, 2)]
    assert st.upper == 2
    assert st.best.tolist() == [int(ch) for ch in "10001100"]
    naive = gpu.run_bz([gpu.singleton_gamma(add, gpu.WeightMode.symplectic)], gpu.AdmissibilityFilter.disabled())
    assert naive.upper == 3
    # test_engine.cpp:205-219: the 3x4 example through diagonalize_f2
    ex = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8)
    g = gpu.diagonalize_f2(ex)
    st = gpu.run_bz([g], gpu.AdmissibilityFilter.for_rows(g.matrix[:3], 1))
    assert st.upper == 1 and st.generation == 1 and st.candidates_enumerated == 4
    # sharded packaged levels merge to the single-rank answer
    c = gpu.CONFIGS[2]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    one = gpu.saved_2_gamma(a)
    import threading

    vals, barrier = {}, threading.Barrier(2)

    def fn_for(r):
        def fn(v):
            vals[r] = v.copy()
            barrier.wait()
            out = np.minimum(vals[0], vals[1])
            barrier.wait()
            return out
        return fn

    out = [None, None]

    def run(r):
        out[r] = gpu.saved_2_gamma(a, gpu.RunOptions(rank=r, world=2, allreduce_min=fn_for(r), shard_min=1))

    ths = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for rep in out:
        assert tr(rep) == tr(one) and rep.distance == one.distance == 7
    assert out[0].candidates_visited + out[1].candidates_visited == one.candidates_visited


def test_package_route_errors(gpu):
    dup = np.array([[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]], dtype=np.uint8)
    for fn in (gpu.saved_1_gamma, gpu.saved_2_gamma):
        with pytest.raises(gpu.ValidationError):
            fn(dup)
    with pytest.raises(gpu.ValidationError):
        gpu.compute_distance(dup, gpu.Algorithm.brute_force)


def test_brute_force_on_the_device(gpu):
    # brute_force_distance (distance.cpp:151-224): the reference's own brute-force answers
    gd = load_golden("reference_kats.json")
    for case in gd["cases"]:
        a = hex_to_mat(case["normalizer"], 2 * case["n"])
        rep = gpu.compute_distance(a, gpu.Algorithm.brute_force)
        assert rep.distance == case["brute"]
        assert rep.algorithm == gpu.Algorithm.brute_force
        assert rep.candidates_enumerated == (1 << a.shape[0]) - 1 and rep.generations == 0
    # config 1 (28 rows, the reference's limit) and the limit itself
    c1 = load_golden("config1.json")
    a = hex_to_mat(c1["normalizer"], 2 * c1["n"])
    assert gpu.compute_distance(a, gpu.Algorithm.brute_force).distance == c1["distance"]
    with pytest.raises(ValueError):
        gpu.compute_distance(gpu.generate_code(25, 4, 1), gpu.Algorithm.brute_force)
    # filter off: plain minimum weight over the whole row space
    a = gpu.generate_code(10, 3, 77)
    plain = gpu.compute_distance(a, gpu.Algorithm.brute_force, gpu.RunOptions(dual_filter=False))
    import oracle as O
    assert plain.distance == O.brute_force(a, dual_filter=False)
