"""Freeze golden vectors from the REFERENCE library (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile). Run in the build container:

    make -C oracle && python tests/golden/make_golden.py [--heavy]

Writes small JSON fixtures next to this script. The GPU box never runs this
(it has no /root/reference); tests only read the JSON.

Matrices are stored one hex string per row: the row's bits as an integer,
column c at bit c (little-endian), so ``int(h, 16) >> c & 1`` is entry c.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def hexrows(m) -> list[str]:
    m = np.asarray(m, dtype=np.uint8)
    out = []
    for row in m:
        v = 0
        for c in np.nonzero(row)[0]:
            v |= 1 << int(c)
        out.append(format(v, "x"))
    return out


def dump(name: str, obj) -> None:
    path = os.path.join(OUT, name)
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes", flush=True)


def gammas_of(a):
    img = O.ref_isometry_transform(a)
    return [dict(matrix=hexrows(g["matrix"]), rank_deficit=g["rank_deficit"], pivots=g["pivots"])
            for g in O.ref_information_sets(img)]


def single_config(cid: int, workers: int, g_max: int = 0, with_best: bool = False) -> dict:
    c = O.CONFIGS[cid]
    n, k, seed = c["n"], c["k"], c["seed"]
    a = O.generate(n, k, seed)
    t0 = time.time()
    if g_max:
        lv = O.ref_isometry_levels(a, workers=workers, g_max=g_max, native=True)
        res = dict(trace=lv["trace"], level_candidates=lv["level_candidates"], complete=False,
                   levels_run=len(lv["trace"]), ref_level_seconds=lv["level_seconds"], ref_workers=workers,
                   ref_build="native")
    else:
        r = O.ref_compute_distance(a, "saved_isometry", workers=workers)
        res = dict(trace=r.trace, distance=r.distance, candidates=r.candidates, generations=r.generations,
                   complete=True, ref_elapsed_seconds=r.elapsed_seconds, ref_workers=workers, ref_build="default")
    if with_best:
        b = O.ref_isometry_best(a, workers=1)
        res["best"] = hexrows([b["best"]])[0]
        res["best_len"] = int(len(b["best"]))
    res.update(config=cid, n=n, k=k, seed=seed, transvections=4 * n, normalizer=hexrows(a), gammas=gammas_of(a),
               wall_seconds=time.time() - t0)
    return res


def batch_config() -> dict:
    c = O.CONFIGS[3]
    n, k = c["n"], c["k"]
    codes = []
    hist: dict = {}
    for s in c["seeds"]:
        a = O.generate(n, k, s)
        r = O.ref_compute_distance(a, "saved_isometry", workers=1)
        codes.append(dict(seed=s, distance=r.distance, trace=r.trace, candidates=r.candidates))
        hist[r.distance] = hist.get(r.distance, 0) + 1
    return dict(config=3, n=n, k=k, seeds=[c["seeds"][0], c["seeds"][-1]], codes=codes,
                histogram={str(d): v for d, v in sorted(hist.items())})


def reference_kats() -> dict:
    """Instances from the reference's own tests, reproduced through its own
    random_stabilizer (mt19937_64) and answered by its own algorithms."""
    cases = []
    # proj/tests/test_distance.cpp:122-125 mid-size instances (oracle agreement)
    for n, k, seed in [(16, 1, 11), (18, 2, 12), (20, 0, 13), (22, 2, 14)]:
        a = O.ref_random_stabilizer(n, k, seed)
        iso = O.ref_compute_distance(a, "saved_isometry")
        brute = O.ref_compute_distance(a, "brute_force")
        cases.append(dict(src="test_distance.cpp:122-125", n=n, k=k, seed=seed, normalizer=hexrows(a),
                          distance=iso.distance, brute=brute.distance, trace=iso.trace, candidates=iso.candidates))
    # proj/tests/acceptance.cpp:124-157 criterion 3 sweep: seeds 10000 + 97*i
    count = 0
    for rep in range(3):
        for n in range(4, 13):
            for k in range(0, n + 1):
                seed = 10000 + 97 * count
                count += 1
                a = O.ref_random_stabilizer(n, k, seed)
                iso = O.ref_compute_distance(a, "saved_isometry")
                brute = O.ref_compute_distance(a, "brute_force")
                cases.append(dict(src="acceptance.cpp:124-157", n=n, k=k, seed=seed, normalizer=hexrows(a),
                                  distance=iso.distance, brute=brute.distance, trace=iso.trace,
                                  candidates=iso.candidates))
    # proj/tests/acceptance.cpp:56-79 worked 3x4 example; test_distance.cpp:57-64 (I_5 | 0)
    ex = np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8)
    r = O.ref_compute_distance(ex, "saved_isometry")
    cases.append(dict(src="acceptance.cpp:56-79", n=2, k=1, seed=None, normalizer=hexrows(ex), distance=r.distance,
                      brute=O.ref_compute_distance(ex, "brute_force").distance, trace=r.trace,
                      candidates=r.candidates))
    ident = np.zeros((5, 10), dtype=np.uint8)
    for i in range(5):
        ident[i, i] = 1
    r = O.ref_compute_distance(ident, "saved_isometry")
    cases.append(dict(src="test_distance.cpp:57-64", n=5, k=0, seed=None, normalizer=hexrows(ident),
                      distance=r.distance, brute=O.ref_compute_distance(ident, "brute_force").distance,
                      trace=r.trace, candidates=r.candidates))
    return dict(cases=cases)


def engine_kats() -> dict:
    """Singleton-package run_bz cases in both weight modes across word boundaries, the
    shape of proj/tests/test_engine.cpp:121-161 (n 60..79, 5 rows), inputs from a seeded
    numpy generator, answers from the reference's run_bz."""
    rng = np.random.default_rng(103)
    cases = []
    for it in range(6):
        n = 60 + int(rng.integers(0, 20))
        m = rng.integers(0, 2, size=(5, 2 * n), dtype=np.uint8)
        sym = O.ref_run_bz_singleton(m, "symplectic")
        img = O.ref_isometry_transform(m)
        ham = O.ref_run_bz_singleton(img, "hamming")
        cases.append(dict(src="test_engine.cpp:121-161", n=n, matrix=hexrows(m), symplectic=dict(
            trace=sym["trace"], upper=sym["upper"], generation=sym["generation"], candidates=sym["candidates"]),
            hamming=dict(trace=ham["trace"], upper=ham["upper"], generation=ham["generation"],
                         candidates=ham["candidates"])))
    # planted d=1 at n=70 (test_engine.cpp:163-182): scrambled (I_n | 0)
    n = 70
    a = np.zeros((n, 2 * n), dtype=np.uint8)
    for i in range(n):
        a[i, i] = 1
    for _ in range(400):
        r1, r2 = (int(x) for x in rng.integers(0, n, size=2))
        if r1 != r2:
            a[r2] ^= a[r1]
    r = O.ref_compute_distance(a, "saved_isometry")
    cases.append(dict(src="test_engine.cpp:163-182", n=n, planted=hexrows(a), distance=r.distance, trace=r.trace))
    # filtered singleton runs with the reference's exhaustion error (test_engine.cpp:260-269)
    return dict(cases=cases)


def package_routes(heavy: bool, workers: int) -> dict:
    """Saved_1_Gamma / Saved_2_Gamma answered by the reference:
    BASELINE configs 1-2 (config 4 for 1-Gamma with --heavy), the reference tests' worked
    examples, random instances with the brute-force distance, auto dispatch (k <= 2 sends
    to saved_2_gamma, distance.cpp:233-237) and the first 256 config-3 codes."""
    cases = []

    def add(src, a, algs=("saved_1_gamma", "saved_2_gamma"), best=True, brute=False, validate=True, filt=True,
            **extra):
        for alg in algs:
            r = O.ref_compute_distance(a, alg, workers=workers if a.shape[1] > 60 else 1, validate=validate,
                                       dual_filter=filt)
            case = dict(src=src, alg=alg, n=a.shape[1] // 2, k=a.shape[0] - a.shape[1] // 2, normalizer=hexrows(a),
                        distance=r.distance, trace=r.trace, candidates=r.candidates, generations=r.generations,
                        validate=validate, dual_filter=filt, **extra)
            if best:
                b = O.ref_package_best(a, alg)
                case["best"] = hexrows([b["best"]])[0]
                case["best_len"] = int(len(b["best"]))
            if brute:
                case["brute"] = O.ref_compute_distance(a, "brute_force").distance
            cases.append(case)

    for cid in (1, 2):
        c = O.CONFIGS[cid]
        add(f"config{cid}", O.generate(c["n"], c["k"], c["seed"]), config=cid)
    if heavy:
        c = O.CONFIGS[4]
        add("config4", O.generate(c["n"], c["k"], c["seed"]), algs=("saved_1_gamma",), best=False, config=4)
    # proj/tests/test_engine.cpp:205-219 / test_prep.cpp:14: the 3x4 example
    add("test_prep.cpp:14", np.array([[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]], dtype=np.uint8), brute=True)
    # test_prep.cpp:17-19 additive example rows (1,1,1,1), (a,0,a,a), (0,a2,a2,a2) as (a | b)
    add("test_prep.cpp:17-19", np.array([[int(ch) for ch in row] for row in
                                         ("11110000", "00001011", "01110111")], dtype=np.uint8),
        algs=("saved_2_gamma",), validate=False, filt=False)
    for n in (2, 6):  # test_distance.cpp:57-64 style (I_n | 0)
        ident = np.zeros((n, 2 * n), dtype=np.uint8)
        for i in range(n):
            ident[i, i] = 1
        add("test_distance.cpp:57-64", ident, brute=True)
    # test_distance.cpp:102-117 style: random instances against the brute-force oracle
    for i in range(40):
        n = 3 + i % 10
        k = (7 * i) % (n + 1)
        add("test_distance.cpp:102-117", O.ref_random_stabilizer(n, k, 20000 + 31 * i), brute=True, seed=20000 + 31 * i)
    for n, k, seed in [(16, 1, 11), (18, 2, 12), (20, 0, 13), (22, 2, 14)]:  # test_distance.cpp:122-125
        add("test_distance.cpp:122-125", O.ref_random_stabilizer(n, k, seed), seed=seed)
    # auto dispatch on the first 256 config-3 codes (k = 2: saved_2_gamma)
    c = O.CONFIGS[3]
    batch = []
    for s in c["seeds"][:256]:
        a = O.generate(c["n"], c["k"], s)
        r = O.ref_compute_distance(a, "auto")
        batch.append(dict(seed=s, alg=r.algorithm, distance=r.distance, trace=r.trace, candidates=r.candidates))
    return dict(cases=cases, config3_auto=dict(n=c["n"], k=c["k"], codes=batch))


def enumerate_generation_cases() -> dict:
    """The per-level seam enumerate_generation (engine.hpp:53-54) answered by the reference on
    single matrices: the isometry route's information sets (Hamming mode, filter from the
    normalizer), the package routes' prepared matrices (symplectic mode, 1- and 3-packages, their
    routes' filters) and unfiltered symplectic singletons across word boundaries, each entered
    with upper = 0 (unset), the previous level's bound and a tight bound."""
    cases = []

    def add(src, m, mode, g, upper, packages=None, frows=None, k=0):
        r = O.ref_enumerate_generation(m, mode, g, upper=upper, packages=packages, filter_rows=frows, filter_k=k)
        cases.append(dict(src=src, cols=int(m.shape[1]), matrix=hexrows(m), mode=mode, g=g, upper_in=upper,
                          packages=packages or [], filter=hexrows(frows) if frows is not None else [],
                          filter_cols=int(frows.shape[1]) if frows is not None else 0, k=k,
                          upper=r["upper"], candidates=r["candidates"],
                          best=hexrows(r["best"].reshape(1, -1))[0] if r["best"].size else ""))
        return r["upper"]

    codes = [("config1", O.generate(24, 4, 1), 4)]
    codes += [(f"random n={n} k={k}", O.generate(n, k, 31 + n), k) for n, k in [(12, 3), (20, 2), (30, 4), (40, 1)]]
    for src, a, k in codes:
        img = O.ref_isometry_transform(a)
        for j, gm in enumerate(O.ref_information_sets(img)):
            up = 0
            for g in (1, 2, 3):
                prev = add(f"{src} isometry gamma {j}", gm["matrix"], "hamming", g, up, frows=a, k=k)
                up = prev
            add(f"{src} isometry gamma {j} tight", gm["matrix"], "hamming", 3, max(2, up - 4), frows=a, k=k)
        n = a.shape[1] // 2
        for alg in ("saved_1_gamma", "saved_2_gamma"):
            gs = O.ref_prepare_packages(a, alg)
            for j, gm in enumerate(gs):
                frows = gm["matrix"][: a.shape[0]] if alg == "saved_1_gamma" else a
                up = 0
                for g in (1, 2, 3):
                    if g > len(gm["packages"]):
                        break
                    up = add(f"{src} {alg} gamma {j}", gm["matrix"], "symplectic", g, up, packages=gm["packages"],
                             frows=frows, k=k)
    rng = np.random.default_rng(211)
    for n in (31, 32, 33, 64, 65):
        m = rng.integers(0, 2, size=(6, 2 * n), dtype=np.uint8)
        for g in (1, 2, 3):
            add(f"singleton symplectic n={n}", m, "symplectic", g, 0)
    return dict(cases=cases)


def wide_codes() -> dict:
    """Wide rows (n up to 256: 4-8 u32 words per half, the kernels' upper limit) through the
    first levels of saved_isometry, answered by the reference (levels g <= g_max)."""
    cases = []
    for n, k, g in [(100, 5, 4), (130, 7, 3), (160, 0, 3), (200, 10, 2), (256, 0, 2), (256, 12, 2)]:
        a = O.generate(n, k, 11)
        lv = O.ref_isometry_levels(a, workers=os.cpu_count() or 1, g_max=g, native=True)
        cases.append(dict(n=n, k=k, seed=11, g_max=g, normalizer=hexrows(a), trace=lv["trace"],
                          level_candidates=lv["level_candidates"]))
    return dict(cases=cases)


def config4_extra(part: str, workers: int) -> dict:
    """Config 4 answers the full-run fixture (config4.json) leaves out, each from the reference
    (native build; the results do not depend on the flags):
      iso_best  - saved_isometry's best codeword with ONE worker (engine.cpp:182-189: the first
                  minimum in the single-worker visiting order, the one the GPU keys reproduce);
      s2g       - saved_2_gamma (distance.cpp:115-133): distance, trace, candidates, generations;
      s2g_best  - saved_2_gamma's best codeword with one worker;
      s1g_best  - saved_1_gamma's best codeword with one worker (its trace is in package_routes.json).
    """
    c = O.CONFIGS[4]
    a = O.generate(c["n"], c["k"], c["seed"])
    t0 = time.time()
    res: dict = dict(config=4, n=c["n"], k=c["k"], seed=c["seed"], part=part)
    if part == "iso_best":
        b = O.ref_isometry_best(a, workers=1, native=True)
        res.update(alg="saved_isometry", best=hexrows([b["best"]])[0], best_len=int(len(b["best"])),
                   upper=int(b["upper"]))
    elif part == "s2g":
        r = O.ref_compute_distance(a, "saved_2_gamma", workers=workers, native=True)
        res.update(alg="saved_2_gamma", distance=r.distance, trace=r.trace, candidates=r.candidates,
                   generations=r.generations, ref_elapsed_seconds=r.elapsed_seconds, ref_workers=workers)
    elif part in ("s2g_best", "s1g_best"):
        alg = "saved_2_gamma" if part == "s2g_best" else "saved_1_gamma"
        b = O.ref_package_best(a, alg, workers=1, native=True)
        res.update(alg=alg, best=hexrows([b["best"]])[0], best_len=int(len(b["best"])), upper=int(b["upper"]))
    res["wall_seconds"] = time.time() - t0
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--heavy", action="store_true", help="also config 4 (full) and config 5 (g<=8)")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None

    def want(x):
        return only is None or x in only

    if want("c1"):
        dump("config1.json", single_config(1, 1, with_best=True))
    if want("c2"):
        dump("config2.json", single_config(2, args.workers, with_best=True))
    if want("c3"):
        dump("config3.json", batch_config())
    if want("kats"):
        dump("reference_kats.json", reference_kats())
    if want("engine"):
        dump("engine_kats.json", engine_kats())
    if want("wide"):
        dump("wide_codes.json", wide_codes())
    if want("enumgen"):
        dump("enumerate_generation.json", enumerate_generation_cases())
    if want("packages"):
        dump("package_routes.json", package_routes(args.heavy, args.workers))
    if args.heavy and want("c4"):
        dump("config4.json", single_config(4, args.workers))
    if args.heavy and want("c5"):
        dump("config5_g8.json", single_config(5, args.workers, g_max=8))
    if args.heavy and want("c5g9"):
        dump("config5_g9.json", single_config(5, args.workers, g_max=9))
    for part in ("iso_best", "s2g", "s2g_best", "s1g_best"):
        if args.heavy and want("c4_" + part):
            dump(f"config4_{part}.json", config4_extra(part, args.workers))


if __name__ == "__main__":
    main()
