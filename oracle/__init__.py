"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two libraries live under ``oracle/``:

* ``_ref/libsymdist_ref.so`` — the UNMODIFIED reference library
  (``/root/reference/proj/src/*.cpp``) compiled in place by ``oracle/Makefile``
  with the reference's own flags, plus ``ref_shim.cpp`` (an ``extern "C"``
  wrapper over its public C++ API). ``_ref/libsymdist_ref_native.so`` is the
  same with ``-march=native``.
* ``_build/libsymdist_oracle.so`` — ``symdist_oracle.c``, our plain-C
  restatement of the Saved_isometry route (each function cites the reference
  file:line it follows).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package. The product (``paper_2408_10743_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsymdist_ref.so")
REF_NATIVE_SO = os.path.join(HERE, "_ref", "libsymdist_ref_native.so")
ORACLE_SO = os.path.join(HERE, "_build", "libsymdist_oracle.so")

# BASELINE.json configs: (n, k, seed); config 3 is a batch.
CONFIGS = {
    1: dict(n=24, k=4, seed=1),
    2: dict(n=40, k=6, seed=2),
    3: dict(n=20, k=2, seeds=list(range(1000, 5096))),
    4: dict(n=56, k=8, seed=3),
    5: dict(n=80, k=10, seed=4),
}

ALG = {"auto": 0, "saved_1_gamma": 1, "saved_2_gamma": 2, "saved_isometry": 3, "brute_force": 4}
ALG_NAME = {v: k for k, v in ALG.items()}


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Trace(C.Structure):
    _fields_ = [("g", C.c_int), ("lower", C.c_long), ("upper", C.c_long)]


class _Report(C.Structure):
    _fields_ = [
        ("distance", C.c_int),
        ("algorithm", C.c_int),
        ("generations", C.c_int),
        ("candidates", C.c_ulonglong),
        ("elapsed_seconds", C.c_double),
        ("workers", C.c_int),
        ("trace_len", C.c_int),
    ]


_libs: dict = {}


def _load(path: str):
    if path not in _libs:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        _libs[path] = C.CDLL(path)
    return _libs[path]


def ref_available(native: bool = False) -> bool:
    return os.path.exists(REF_NATIVE_SO if native else REF_SO)


def _u8(mat) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(mat, dtype=np.uint8))
    assert a.ndim == 2
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _err():
    return C.create_string_buffer(512)


def _check(rc: int, err) -> None:
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"))


# ----------------------------------------------------------------- reference (oracle/_ref)


@dataclass
class RefReport:
    distance: int
    algorithm: str
    generations: int
    candidates: int
    elapsed_seconds: float
    workers: int
    trace: list = field(default_factory=list)


def ref_compute_distance(mat, alg: str = "saved_isometry", workers: int = 1, validate: bool = True,
                         dual_filter: bool = True, native: bool = False) -> RefReport:
    lib = _load(REF_NATIVE_SO if native else REF_SO)
    a = _u8(mat)
    rep = _Report()
    tr = (_Trace * 512)()
    err = _err()
    rc = lib.ref_compute_distance(_ptr(a), a.shape[0], a.shape[1], ALG[alg], workers, int(validate),
                                  int(dual_filter), C.byref(rep), tr, 512, err, 512)
    _check(rc, err)
    trace = [(tr[i].g, tr[i].lower, tr[i].upper) for i in range(min(rep.trace_len, 512))]
    return RefReport(rep.distance, ALG_NAME.get(rep.algorithm, "?"), rep.generations, rep.candidates,
                     rep.elapsed_seconds, rep.workers, trace)


def ref_validate(mat) -> tuple[bool, str]:
    lib = _load(REF_SO)
    a = _u8(mat)
    ok = C.c_int(0)
    msg = _err()
    rc = lib.ref_validate(_ptr(a), a.shape[0], a.shape[1], C.byref(ok), msg, 512)
    _check(rc, msg)
    return bool(ok.value), msg.value.decode()


def ref_random_stabilizer(n: int, k: int, seed: int) -> np.ndarray:
    lib = _load(REF_SO)
    out = np.zeros((n + k, 2 * n), dtype=np.uint8)
    err = _err()
    rc = lib.ref_random_stabilizer(n, k, C.c_ulonglong(seed), _ptr(out), err, 512)
    _check(rc, err)
    return out


def ref_isometry_transform(mat) -> np.ndarray:
    lib = _load(REF_SO)
    a = _u8(mat)
    out = np.zeros((a.shape[0], a.shape[1] // 2 * 3), dtype=np.uint8)
    err = _err()
    _check(lib.ref_isometry_transform(_ptr(a), a.shape[0], a.shape[1], _ptr(out), err, 512), err)
    return out


def ref_information_sets(image) -> list[dict]:
    lib = _load(REF_SO)
    b = _u8(image)
    rows, cols = b.shape
    cap = 16
    out = np.zeros((cap, rows, cols), dtype=np.uint8)
    defs = np.zeros(cap, dtype=np.int32)
    piv = np.zeros((cap, rows), dtype=np.int32)
    ng = C.c_int(0)
    err = _err()
    rc = lib.ref_information_sets(_ptr(b), rows, cols, cap, _ptr(out), defs.ctypes.data_as(C.POINTER(C.c_int)),
                                  piv.ctypes.data_as(C.POINTER(C.c_int)), C.byref(ng), err, 512)
    _check(rc, err)
    return [dict(matrix=out[j].copy(), rank_deficit=int(defs[j]), pivots=[int(x) for x in piv[j]])
            for j in range(min(ng.value, cap))]


def ref_isometry_levels(mat, workers: int = 1, validate: bool = True, dual_filter: bool = True,
                        g_max: int = 0, native: bool = False) -> dict:
    lib = _load(REF_NATIVE_SO if native else REF_SO)
    a = _u8(mat)
    cap = 512
    tr = (_Trace * cap)()
    secs = (C.c_double * cap)()
    cands = (C.c_ulonglong * cap)()
    nlev = C.c_int(0)
    upper = C.c_long(0)
    prep = C.c_double(0)
    err = _err()
    rc = lib.ref_isometry_levels(_ptr(a), a.shape[0], a.shape[1], workers, int(validate), int(dual_filter),
                                 g_max, tr, secs, cands, cap, C.byref(nlev), C.byref(upper), C.byref(prep),
                                 err, 512)
    _check(rc, err)
    n = min(nlev.value, cap)
    return dict(trace=[(tr[i].g, tr[i].lower, tr[i].upper) for i in range(n)],
                level_seconds=[secs[i] for i in range(n)], level_candidates=[int(cands[i]) for i in range(n)],
                upper=upper.value, prep_seconds=prep.value)


def ref_run_bz_singleton(mat, mode: str, filter_rows=None, filter_k: int = 0, workers: int = 1) -> dict:
    lib = _load(REF_SO)
    a = _u8(mat)
    if filter_rows is None:
        f = np.zeros((1, 1), dtype=np.uint8)
        fr, fc = 0, 0
    else:
        f = _u8(filter_rows)
        fr, fc = f.shape
    cap = 512
    tr = (_Trace * cap)()
    tl, gen = C.c_int(0), C.c_int(0)
    upper = C.c_long(0)
    cands = C.c_ulonglong(0)
    best = np.zeros(4096, dtype=np.uint8)
    blen = C.c_int(0)
    err = _err()
    rc = lib.ref_run_bz_singleton(_ptr(a), a.shape[0], a.shape[1], 1 if mode == "hamming" else 0, _ptr(f), fr, fc,
                                  filter_k, workers, tr, cap, C.byref(tl), C.byref(upper), C.byref(gen),
                                  C.byref(cands), _ptr(best), 4096, C.byref(blen), err, 512)
    _check(rc, err)
    return dict(trace=[(tr[i].g, tr[i].lower, tr[i].upper) for i in range(min(tl.value, cap))],
                upper=upper.value, generation=gen.value, candidates=int(cands.value),
                best=best[: blen.value].copy())


def ref_enumerate_generation(mat, mode: str, g: int, upper: int = 0, packages=None, filter_rows=None,
                             filter_k: int = 0, workers: int = 1) -> dict:
    """The reference's enumerate_generation (engine.hpp:53-54) on one matrix with a bound state
    entering at `upper` (0: unset) and no best."""
    lib = _load(REF_SO)
    a = _u8(mat)
    if filter_rows is None:
        f = np.zeros((1, 1), dtype=np.uint8)
        fr, fc = 0, 0
    else:
        f = _u8(filter_rows)
        fr, fc = f.shape
    enc = []
    for pk in packages or []:
        enc += [len(pk)] + list(pk)
    enc = np.array(enc or [0], dtype=np.int32)
    up = C.c_long(upper)
    cands = C.c_ulonglong(0)
    best = np.zeros(4096, dtype=np.uint8)
    blen = C.c_int(0)
    err = _err()
    rc = lib.ref_enumerate_generation(_ptr(a), a.shape[0], a.shape[1], 1 if mode == "hamming" else 0,
                                      len(packages or []), enc.ctypes.data_as(C.POINTER(C.c_int)), g, _ptr(f), fr, fc,
                                      filter_k, workers, C.byref(up), C.byref(cands), _ptr(best), 4096, C.byref(blen),
                                      err, 512)
    _check(rc, err)
    return dict(upper=up.value, candidates=int(cands.value), best=best[: blen.value].copy())


def ref_isometry_best(mat, workers: int = 1, native: bool = False) -> dict:
    lib = _load(REF_NATIVE_SO if native else REF_SO)
    a = _u8(mat)
    best = np.zeros(4096, dtype=np.uint8)
    blen = C.c_int(0)
    upper = C.c_long(0)
    err = _err()
    rc = lib.ref_isometry_best(_ptr(a), a.shape[0], a.shape[1], workers, _ptr(best), 4096, C.byref(blen),
                               C.byref(upper), err, 512)
    _check(rc, err)
    return dict(upper=upper.value, best=best[: blen.value].copy())


def ref_prepare_packages(mat, alg: str) -> list[dict]:
    """The reference's package-route prep: diagonalize_f2 (saved_1_gamma) or diagonalize_f4 +
    second_gamma (saved_2_gamma)."""
    lib = _load(REF_SO)
    a = _u8(mat)
    rows, cols = a.shape
    max_rows = 2 * rows + 2
    out = np.zeros((2, max_rows, cols), dtype=np.uint8)
    gr, npk, npp = (np.zeros(2, dtype=np.int32) for _ in range(3))
    pk = np.zeros(16 * rows + 16, dtype=np.int32)
    ng = C.c_int(0)
    err = _err()
    ip = lambda x: x.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    rc = lib.ref_prepare_packages(_ptr(a), rows, cols, ALG[alg], max_rows, _ptr(out), ip(gr), ip(npk), ip(npp),
                                  ip(pk), len(pk), C.byref(ng), err, 512)
    _check(rc, err)
    res, pos = [], 0
    for j in range(ng.value):
        pkgs = []
        for _ in range(int(npk[j])):
            sz = int(pk[pos])
            pkgs.append([int(x) for x in pk[pos + 1:pos + 1 + sz]])
            pos += 1 + sz
        res.append(dict(matrix=out[j, :int(gr[j])].copy(), packages=pkgs, n_pp=int(npp[j])))
    return res


def ref_package_best(mat, alg: str, workers: int = 1, native: bool = False) -> dict:
    lib = _load(REF_NATIVE_SO if native else REF_SO)
    a = _u8(mat)
    best = np.zeros(a.shape[1], dtype=np.uint8)
    bl, up = C.c_int(0), C.c_long(0)
    err = _err()
    rc = lib.ref_package_best(_ptr(a), a.shape[0], a.shape[1], ALG[alg], workers, _ptr(best), len(best),
                              C.byref(bl), C.byref(up), err, 512)
    _check(rc, err)
    return dict(best=best[:bl.value].copy(), upper=int(up.value))


# ----------------------------------------------------------------- C restatement (oracle/_build)


def _olib():
    lib = _load(ORACLE_SO)
    lib.orc_lower_bound.restype = C.c_long
    return lib


def generate(n: int, k: int, seed: int, transvections: int | None = None) -> np.ndarray:
    """BASELINE.md §2 config generator (xorshift64* transvections), C restatement."""
    out = np.zeros((n + k, 2 * n), dtype=np.uint8)
    rc = _olib().orc_generate(n, k, C.c_uint64(seed), 4 * n if transvections is None else transvections, _ptr(out))
    if rc:
        raise RefError(rc, "orc_generate: bad arguments")
    return out


def py_generate(n: int, k: int, seed: int, transvections: int | None = None) -> np.ndarray:
    """Pure-Python twin of ``generate`` (cross-check of the C restatement)."""
    M = (1 << 64) - 1
    rows = []
    for i in range(n - k):
        rows.append((0, 1 << i))
    for i in range(n - k, n):
        rows.append((1 << i, 0))
    for i in range(n - k, n):
        rows.append((0, 1 << i))
    s = seed
    mask = (1 << (2 * n)) - 1
    words = (2 * n + 63) // 64
    for _ in range(4 * n if transvections is None else transvections):
        while True:
            v = 0
            for w in range(words):
                s ^= s >> 12
                s ^= (s << 25) & M
                s ^= s >> 27
                v |= ((s * 0x2545F4914F6CDD1D) & M) << (64 * w)
            v &= mask
            if v:
                break
        vx, vz = v & ((1 << n) - 1), v >> n
        for i, (ux, uz) in enumerate(rows):
            if (bin(ux & vz).count("1") + bin(uz & vx).count("1")) & 1:
                rows[i] = (ux ^ vx, uz ^ vz)
    out = np.zeros((n + k, 2 * n), dtype=np.uint8)
    for i, (ux, uz) in enumerate(rows):
        for c in range(n):
            out[i, c] = (ux >> c) & 1
            out[i, n + c] = (uz >> c) & 1
    return out


def rank(mat) -> int:
    a = _u8(mat)
    return int(_olib().orc_rank(_ptr(a), a.shape[0], a.shape[1]))


def validate(mat) -> int:
    """0 when ``mat`` is a valid normalizer (restated validate_normalizer)."""
    a = _u8(mat)
    return int(_olib().orc_validate(_ptr(a), a.shape[0], a.shape[1]))


def isometry(mat) -> np.ndarray:
    a = _u8(mat)
    out = np.zeros((a.shape[0], a.shape[1] // 2 * 3), dtype=np.uint8)
    _olib().orc_isometry(_ptr(a), a.shape[0], a.shape[1], _ptr(out))
    return out


def information_sets(image) -> list[dict]:
    b = _u8(image)
    rows, cols = b.shape
    cap = 64
    out = np.zeros((cap, rows, cols), dtype=np.uint8)
    defs = np.zeros(cap, dtype=np.int32)
    piv = np.zeros((cap, rows), dtype=np.int32)
    ng = C.c_int(0)
    rc = _olib().orc_information_sets(_ptr(b), rows, cols, cap, _ptr(out), defs.ctypes.data_as(C.POINTER(C.c_int)),
                                      piv.ctypes.data_as(C.POINTER(C.c_int)), C.byref(ng))
    if rc:
        raise RefError(rc, "information_sets: rows are linearly dependent")
    return [dict(matrix=out[j].copy(), rank_deficit=int(defs[j]), pivots=[int(x) for x in piv[j]])
            for j in range(min(ng.value, cap))]


def lower_bound(g: int, deficits) -> int:
    d = np.ascontiguousarray(np.asarray(deficits, dtype=np.int32))
    return int(_olib().orc_lower_bound(g, d.ctypes.data_as(C.POINTER(C.c_int)), len(d)))


def run_levels(mat, validate: bool = True, dual_filter: bool = True, g_max: int = 0, threads: int = 1) -> dict:
    """Saved_isometry through run_bz's level loop (restated). Returns trace, per-level best
    (Gamma index, lexicographic rank) and the final upper bound in Hamming units."""
    a = _u8(mat)
    cap = 512
    tg = np.zeros(cap, dtype=np.int32)
    tl = np.zeros(cap, dtype=np.int64)
    tu = np.zeros(cap, dtype=np.int64)
    bg = np.zeros(cap, dtype=np.int32)
    br = np.zeros(cap, dtype=np.uint64)
    nlev = C.c_int(0)
    upper = C.c_long(0)
    rc = _olib().orc_run_levels(_ptr(a), a.shape[0], a.shape[1], int(validate), int(dual_filter), g_max, threads,
                                tg.ctypes.data_as(C.POINTER(C.c_int)), tl.ctypes.data_as(C.POINTER(C.c_long)),
                                tu.ctypes.data_as(C.POINTER(C.c_long)), bg.ctypes.data_as(C.POINTER(C.c_int)),
                                br.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(nlev), C.byref(upper))
    if rc:
        raise RefError(rc, {2: "validation error", 3: "no admissible codeword", 5: "bad arguments"}.get(rc, "?"))
    n = min(nlev.value, cap)
    return dict(trace=[(int(tg[i]), int(tl[i]), int(tu[i])) for i in range(n)],
                best=[(int(bg[i]), int(br[i])) for i in range(n)], upper=int(upper.value))


def brute_force(mat, dual_filter: bool = True) -> int:
    a = _u8(mat)
    d = C.c_int(0)
    rc = _olib().orc_brute_force(_ptr(a), a.shape[0], a.shape[1], int(dual_filter), C.byref(d))
    if rc:
        raise RefError(rc, "brute_force: bad arguments or no admissible codeword")
    return int(d.value)


def binom(n: int, k: int) -> int:
    from math import comb
    return comb(n, k) if 0 <= k <= n else 0
