"""CPU: the product's native host side (C-ABI entry points that need no device) against
the golden fixtures and the oracle; the C-ABI library loads and exports every symbol
include/symdist_b200.h declares."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2408_10743_b200 as P
from conftest import ROOT, hex_to_mat, load_golden

HEADER = os.path.join(ROOT, "include", "symdist_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sdb_[a-z0-9_]+)\s*\(", src)) - {"sdb_allreduce_min_fn"})


def test_library_exports_every_declared_symbol():
    lib = P.library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.sdb_abi_version() == 2
    # the Python mirror binds exactly the header's symbols
    assert set(P._EXPORTS) == set(syms)


def test_pack_roundtrip():
    rng = np.random.default_rng(1)
    for cols in (1, 63, 64, 65, 130, 240):
        m = rng.integers(0, 2, size=(7, cols), dtype=np.uint8)
        w = P.pack_rows(m)
        assert w.shape == (7, max(1, (cols + 63) // 64))
        assert (P.unpack_rows(w, cols) == m).all()
        for r in range(7):
            v = sum(int(m[r, c]) << c for c in range(cols))
            assert v == sum(int(w[r, i]) << (64 * i) for i in range(w.shape[1]))


@pytest.mark.parametrize("name", ["config1.json", "config2.json", "config4.json", "config5_g8.json"])
def test_native_prep_matches_golden(name):
    gd = load_golden(name)
    n, k = gd["n"], gd["k"]
    a = P.generate_code(n, k, gd["seed"])
    assert (a == hex_to_mat(gd["normalizer"], 2 * n)).all()
    assert P.validate_normalizer(a).ok
    img = P.isometry_transform(a)
    assert (img == O.isometry(a)).all()
    gs = P.information_sets(img)
    assert len(gs) == len(gd["gammas"])
    for mine, ref in zip(gs, gd["gammas"]):
        assert mine.rank_deficit == ref["rank_deficit"]
        assert mine.pivots == ref["pivots"]
        assert (mine.matrix == hex_to_mat(ref["matrix"], 3 * n)).all()


def test_native_prep_matches_oracle_on_random_codes():
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(2, 40))
        k = int(rng.integers(0, n + 1))
        seed = int(rng.integers(1, 1 << 62))
        a = P.generate_code(n, k, seed)
        assert (a == O.generate(n, k, seed)).all()
        assert P.validate_normalizer(a).ok and O.validate(a) == 0
        mine = P.information_sets(P.isometry_transform(a))
        ref = O.information_sets(O.isometry(a))
        assert len(mine) == len(ref)
        for x, y in zip(mine, ref):
            assert x.rank_deficit == y["rank_deficit"] and x.pivots == y["pivots"]
            assert (x.matrix == y["matrix"]).all()


def test_validation_messages_match_reference_text():
    # proj/tests/test_distance.cpp:27-47
    ex = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8)
    assert P.validate_normalizer(ex).ok
    ident = np.zeros((4, 8), dtype=np.uint8)
    for i in range(4):
        ident[i, i] = 1
    assert P.validate_normalizer(ident).ok
    dup = np.array([[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]], dtype=np.uint8)
    r = P.validate_normalizer(dup)
    assert not r.ok and "dependent" in r.message
    thin = np.array([[1, 0, 0, 1, 0, 1, 1, 0]], dtype=np.uint8)
    assert not P.validate_normalizer(thin).ok
    askew = np.array([[1, 0, 0, 0], [0, 0, 1, 0]], dtype=np.uint8)
    r = P.validate_normalizer(askew)
    assert not r.ok and "outside the rowspace" in r.message
    if O.ref_available():
        for m in (ex, ident, dup, thin, askew):
            ok, msg = O.ref_validate(m)
            mine = P.validate_normalizer(m)
            assert mine.ok == ok and mine.message == msg


def test_isometry_transform_cases():
    # proj/tests/test_prep.cpp:183-188
    assert (P.isometry_transform(np.array([[1, 0, 0, 1]])) == np.array([[1, 0, 0, 1, 1, 1]])).all()
    assert (P.isometry_transform(np.zeros((1, 8))) == 0).all()
    with pytest.raises(ValueError):
        P.isometry_transform(np.zeros((1, 5)))


def test_isometry_weight_identity():
    # acceptance.cpp:159-187: Hamming weight of an image combination = 2 x symplectic weight
    rng = np.random.default_rng(2024)
    for _ in range(300):
        n = int(rng.integers(1, 51))
        rows = int(rng.integers(1, 7))
        a = rng.integers(0, 2, size=(rows, 2 * n), dtype=np.uint8)
        img = P.isometry_transform(a)
        sel = rng.integers(0, 2, size=rows).astype(bool)
        comb = np.bitwise_xor.reduce(a[sel], axis=0) if sel.any() else np.zeros(2 * n, np.uint8)
        ic = np.bitwise_xor.reduce(img[sel], axis=0) if sel.any() else np.zeros(3 * n, np.uint8)
        sym = int(np.count_nonzero(comb[:n] | comb[n:]))
        assert int(ic.sum()) == 2 * sym


def test_information_sets_examples():
    # proj/tests/test_prep.cpp:212-238
    n = 5
    b = np.zeros((n, 3 * n), dtype=np.uint8)
    for i in range(n):
        b[i, i] = b[i, n + i] = b[i, 2 * n + i] = 1
    gs = P.information_sets(b)
    assert len(gs) == 3 and all(g.rank_deficit == 0 and g.n_p() == n for g in gs)
    a = np.zeros((4, 8), dtype=np.uint8)
    for i in range(4):
        a[i, i] = 1
    gs = P.information_sets(P.isometry_transform(a))
    assert len(gs) == 2 and gs[0].rank_deficit == 0 and gs[1].rank_deficit == 0
    with pytest.raises(P.ValidationError):
        P.information_sets(np.array([[1, 0, 1], [1, 0, 1]]))


def test_information_sets_invariants_random():
    # proj/tests/test_prep.cpp:240-270: disjoint pivots, unit pivot columns, deficits
    for seed in range(1, 30):
        n = 2 + seed % 6
        k = seed % (n + 1)
        a = P.generate_code(n, k, seed)
        gs = P.information_sets(P.isometry_transform(a))
        assert gs[0].rank_deficit == 0
        seen = set()
        for g in gs:
            piv = [p for p in g.pivots if p >= 0]
            assert g.rank_deficit == g.matrix.shape[0] - len(piv)
            for p in piv:
                assert p not in seen
                seen.add(p)
                assert int(g.matrix[:, p].sum()) == 1


def test_lower_bound_formulas():
    # proj/tests/test_engine.cpp:35-64
    one = P.PackagedGamma(matrix=np.zeros((5, 4), np.uint8), mode=P.WeightMode.symplectic)
    assert P.lower_bound(1, [one]) == 2
    assert P.lower_bound(3, [one]) == 4
    h = [P.PackagedGamma(matrix=np.zeros((6, 6), np.uint8), mode=P.WeightMode.hamming, rank_deficit=d)
         for d in (0, 2, 5)]
    assert P.lower_bound(2, h) == 3 + 1 + 0
    with pytest.raises(ValueError):
        P.lower_bound(1, [])
    with pytest.raises(ValueError):
        P.lower_bound(1, [one, one, one])
    # isometry configs: L(g) = 2(g+1) + max(0, g+1-3k)
    for g in range(1, 14):
        assert P.lower_bound(g, [P.PackagedGamma(np.zeros((90, 1), np.uint8), P.WeightMode.hamming, 80, d)
                                 for d in (0, 0, 30)]) == 2 * (g + 1) + max(0, g + 1 - 30)


def test_bad_arguments_fail_before_the_device():
    with pytest.raises(ValueError):
        P.StabilizerInstance.from_matrix(np.zeros((2, 3)))
    lib = P.library()
    # null report
    rc = lib.sdb_saved_isometry(None, 0, 4, 1, None, None, None, 0, None)
    assert rc == 5 and b"null report" in lib.sdb_last_error()
    with pytest.raises(ValueError):
        P.generate_code(4, 5, 1)
    with pytest.raises(ValueError):
        P.generate_code(4, 1, 0)
    with pytest.raises(P.ValidationError):
        P.saved_isometry(np.array([[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]]))


def test_library_has_no_oracle_dependency():
    """The product .so must not link or embed the oracle / reference code."""
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", P.library_path()], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_" not in out and "symdist::" not in out
    deps = subprocess.run(["ldd", P.library_path()], capture_output=True, text=True).stdout
    assert "symdist_ref" not in deps and "symdist_oracle" not in deps


def test_package_prep_matches_reference_on_random_codes():
    # diagonalize_f2 (prep.cpp:155-254) and diagonalize_f4 + second_gamma (prep.cpp:256-297):
    # same matrices, packages and n_pp as the reference library built from its sources
    import oracle as O

    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(8)
    for _ in range(120):
        n = int(rng.integers(2, 24))
        k = int(rng.integers(0, n + 1))
        a = P.generate_code(n, k, int(rng.integers(1, 1 << 40)))
        for alg in ("saved_1_gamma", "saved_2_gamma"):
            ref = O.ref_prepare_packages(a, alg)
            mine = P.prepare_packages(a, P.Algorithm[alg])
            assert len(ref) == len(mine)
            for r, m in zip(ref, mine):
                assert (r["matrix"] == m.matrix).all()
                assert r["packages"] == m.packages
                assert r["n_pp"] == m.n_pp


def test_package_prep_worked_examples():
    # test_prep.cpp:24-46: the 3x4 example; test_prep.cpp:84-99 / 131-152: the additive example
    ex = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8)
    g = P.diagonalize_f2(ex)
    assert g.matrix.tolist() == [[1, 0, 0, 1], [0, 1, 0, 1], [0, 0, 1, 1], [1, 0, 1, 0]]
    assert g.packages == [[0, 2, 3], [1]] and g.pair_count == 2
    add = np.array([[int(c) for c in r] for r in ("11110000", "00001011", "01110111")], dtype=np.uint8)
    b, d = P.prepare_packages(add, P.Algorithm.saved_2_gamma)
    assert b.matrix.tolist() == [[int(c) for c in r] for r in ("11110000", "00001011", "01110111", "11111011")]
    assert b.packages == [[0, 1, 3], [2]]
    assert d.matrix.tolist() == [[int(c) for c in r] for r in ("11110000", "10000111", "10001100", "01110111")]
    assert len(d.packages) == 2 and d.n_pp == 1 and [len(p) for p in d.packages] == [3, 1]
    with pytest.raises(P.ValidationError):
        P.diagonalize_f2(np.array([[1, 0, 0, 1], [1, 0, 0, 1], [0, 0, 1, 1]], dtype=np.uint8))


def test_tensor_core_encoding_is_exact_on_the_configs():
    """The tensor-core tile kernel scores head x tail sums as an int8 dot product of exact ±1
    coordinates (csrc/tcenc.cpp); the host check compares it with popc(x|z) on random splits."""
    for i, kexp in ((1, 32), (2, 64), (4, 64), (5, 96)):
        c = P.CONFIGS[i]
        a = P.generate_code(c["n"], c["k"], c["seed"])
        mism, ks = P.tc_encoding_check(a, trials=512)
        assert mism == 0
        assert len(ks) == 3 and all(k == kexp for k in ks), ks
    # random small codes, isometry route and the raw symplectic matrix
    for seed in range(20):
        a = P.generate_code(12 + seed % 9, 1 + seed % 4, 500 + seed)
        assert P.tc_encoding_check(a, trials=128)[0] == 0
        assert P.tc_encoding_check(a, isometry=False, trials=128)[0] == 0
