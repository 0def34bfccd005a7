"""symdist-b200: the symplectic Brouwer-Zimmermann distance hot path on B200 (sm_100a).

Python mirror of the reference's public C++ API (``/root/reference/proj/include/symdist``)
over the C-ABI library ``libsymdist_b200.so`` (``include/symdist_b200.h``):

=====================================  ==================================================
this module                            reference
=====================================  ==================================================
``StabilizerInstance.from_matrix``     ``StabilizerInstance::from_matrix`` distance.cpp:49-58
``RunOptions``                         ``RunOptions`` distance.hpp:33-37
``DistanceReport``                     ``DistanceReport`` distance.hpp:44-52
``saved_isometry``                     ``saved_isometry`` distance.cpp:135-149
``saved_1_gamma`` / ``saved_2_gamma``  ``saved_1_gamma`` / ``saved_2_gamma`` distance.cpp:95-133
``diagonalize_f2``                     ``diagonalize_f2`` prep.cpp:155-254
``diagonalize_f4`` / ``second_gamma``  prep.cpp:256-297 (F4 package routes)
``compute_distance``                   ``compute_distance`` distance.cpp:226-240
``validate_normalizer``                ``validate_normalizer`` distance.cpp:71-93
``isometry_transform``                 ``isometry_transform`` prep.cpp:299-315
``information_sets``                   ``information_sets`` prep.cpp:317-364
``singleton_gamma``                    ``singleton_gamma`` prep.cpp:366-383
``AdmissibilityFilter``                ``AdmissibilityFilter`` engine.hpp:18-25
``lower_bound``                        ``lower_bound`` engine.cpp:31-47
``run_bz``                             ``run_bz`` engine.cpp:303-343 (singleton packages)
``saved_isometry_batch``               (loop of saved_isometry; one code per CTA)
``random_stabilizer``                  ``random_stabilizer`` distance.cpp:242-294
``parse_matrix_text`` / ``format_matrix``  matrix_io.cpp:26-106
``cli_path()`` (``symdist_b200``)      the CLI, tools/symdist_main.cpp
=====================================  ==================================================

Errors: ``ValidationError``, ``InternalError``, ``ParseError`` mirror symdist/errors.hpp;
``std::invalid_argument`` becomes ``ValueError``; CUDA/NCCL failures raise ``DeviceError``.
There is no CPU fallback: every distance call runs the CUDA kernels and fails loudly when
the native library or the GPU is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "Algorithm", "WeightMode", "StabilizerInstance", "RunOptions", "DistanceReport", "BoundsTraceEntry",
    "BoundsState", "PackagedGamma", "AdmissibilityFilter", "ValidationResult", "ParseError", "ValidationError",
    "InternalError", "DeviceError", "saved_isometry", "saved_1_gamma", "saved_2_gamma", "compute_distance",
    "diagonalize_f2", "prepare_packages", "random_stabilizer", "parse_matrix_text", "parse_matrix_file",
    "format_matrix", "cli_path", "Comm", "saved_isometry_batch", "run_bz", "enumerate_generation",
    "lower_bound", "validate_normalizer", "isometry_transform", "information_sets", "singleton_gamma",
    "generate_code", "Plan", "pack_rows", "unpack_rows", "library", "library_path", "device_available", "CONFIGS",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# the product library, built in-tree; tools/ A/B experiments call use_variant_library() explicitly
IN_TREE_LIBRARY = os.path.join(HERE, "libsymdist_b200.so")
_LIB_PATH = IN_TREE_LIBRARY

# BASELINE.json configs: (n, k, seed); 3 is the 4096-code batch.
CONFIGS = {
    1: dict(n=24, k=4, seed=1),
    2: dict(n=40, k=6, seed=2),
    3: dict(n=20, k=2, seeds=list(range(1000, 5096))),
    4: dict(n=56, k=8, seed=3),
    5: dict(n=80, k=10, seed=4),
}


class ParseError(RuntimeError):
    pass


class ValidationError(RuntimeError):
    pass


class InternalError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


class Algorithm(enum.IntEnum):
    auto_select = 0
    saved_1_gamma = 1
    saved_2_gamma = 2
    saved_isometry = 3
    brute_force = 4


class WeightMode(enum.IntEnum):
    symplectic = 0
    hamming = 1


# ------------------------------------------------------------------ ctypes structures


class _Trace(C.Structure):
    _fields_ = [("g", C.c_int), ("lower", C.c_longlong), ("upper", C.c_longlong)]


_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int)


class _Options(C.Structure):
    _fields_ = [
        ("workers", C.c_int), ("validate", C.c_int), ("dual_filter", C.c_int), ("device", C.c_int),
        ("max_generation", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("allreduce_min", _ALLREDUCE),
        ("allreduce_ctx", C.c_void_p), ("kernel", C.c_int), ("stream", C.c_void_p), ("comm", C.c_void_p),
        ("shard_min", C.c_longlong), ("reserved", C.c_int * 4),
    ]


class _Report(C.Structure):
    _fields_ = [
        ("distance", C.c_int), ("algorithm", C.c_int), ("generations", C.c_int),
        ("candidates_enumerated", C.c_ulonglong), ("elapsed_seconds", C.c_double), ("workers", C.c_int),
        ("trace_len", C.c_int), ("complete", C.c_int), ("upper", C.c_longlong),
        ("candidates_visited", C.c_ulonglong), ("prep_seconds", C.c_double), ("enum_seconds", C.c_double),
        ("n_gammas", C.c_int), ("kernel_launches", C.c_int), ("best_generation", C.c_int), ("best_gamma", C.c_int),
        ("best_rank", C.c_ulonglong), ("h2d_bytes", C.c_ulonglong), ("d2h_bytes", C.c_ulonglong),
        ("last_level_kernel", C.c_int), ("reserved", C.c_int), ("candidates_skipped", C.c_ulonglong),
    ]


_lib = None

_EXPORTS = [
    "sdb_default_options", "sdb_last_error", "sdb_abi_version", "sdb_device_available", "sdb_saved_isometry",
    "sdb_compute_distance", "sdb_saved_isometry_batch", "sdb_run_bz", "sdb_lower_bound", "sdb_validate_normalizer",
    "sdb_isometry_transform", "sdb_information_sets", "sdb_generate_code", "sdb_plan_create", "sdb_plan_run",
    "sdb_plan_destroy", "sdb_saved_1_gamma", "sdb_saved_2_gamma", "sdb_run_bz_packaged", "sdb_prepare_packages",
    "sdb_random_stabilizer", "sdb_parse_matrix_text", "sdb_format_matrix", "sdb_comm_unique_id", "sdb_comm_create",
    "sdb_comm_destroy", "sdb_comm_allreduce_min", "sdb_enumerate_generation", "sdb_tc_encoding_check",
]


def library_path() -> str:
    return _LIB_PATH


def use_variant_library(path: str) -> None:
    """Kernel-variant A/B experiments only (tools/): load another build of the same C ABI.
    Must be called before the first library() call; bench.py refuses to run on a variant."""
    global _LIB_PATH
    if _lib is not None:
        raise RuntimeError("use_variant_library: the library is already loaded")
    _LIB_PATH = os.path.abspath(path)


def library():
    """Load libsymdist_b200.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (or `make -C paper_2408_10743_b200`)")
        lib = C.CDLL(_LIB_PATH)
        lib.sdb_last_error.restype = C.c_char_p
        lib.sdb_plan_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(_Options),
                                        C.POINTER(C.c_void_p)]
        lib.sdb_plan_run.argtypes = [C.c_void_p, C.POINTER(_Report), C.POINTER(_Trace), C.c_int,
                                     C.POINTER(C.c_double)]
        lib.sdb_plan_destroy.argtypes = [C.c_void_p]
        lib.sdb_comm_destroy.argtypes = [C.c_void_p]
        lib.sdb_comm_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        lib.sdb_comm_allreduce_min.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        lib.sdb_generate_code.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_void_p, C.c_int]
        lib.sdb_random_stabilizer.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_int]
        lib.sdb_parse_matrix_text.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_int, C.c_int,
                                              C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _lib = lib
    return _lib


def device_available() -> bool:
    return bool(library().sdb_device_available())


def _raise(rc: int) -> None:
    if rc == 0:
        return
    msg = library().sdb_last_error().decode(errors="replace")
    if rc == 1:
        raise ParseError(msg)
    if rc == 2:
        raise ValidationError(msg)
    if rc == 3:
        raise InternalError(msg)
    if rc == 4:
        raise DeviceError(msg)
    if rc == 5:
        raise ValueError(msg)
    raise RuntimeError(f"sdb status {rc}: {msg}")


# ------------------------------------------------------------------ bit packing


def pack_rows(mat) -> np.ndarray:
    """0/1 matrix (rows x cols) -> uint64 words (rows x ceil(cols/64)), column c at bit c%64
    of word c/64 (the reference BitVector layout)."""
    a = np.ascontiguousarray(np.asarray(mat, dtype=np.uint8))
    if a.ndim != 2:
        raise ValueError("matrix must be 2-D")
    rows, cols = a.shape
    words = max(1, (cols + 63) // 64)
    padded = np.zeros((rows, words * 64), dtype=np.uint8)
    padded[:, :cols] = a & 1
    packed = np.packbits(padded, axis=1, bitorder="little")
    return np.ascontiguousarray(packed.view("<u8").reshape(rows, words))


def unpack_rows(words, cols: int) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(words, dtype="<u8"))
    if w.ndim == 1:
        w = w.reshape(1, -1)
    bits = np.unpackbits(w.view(np.uint8).reshape(w.shape[0], -1), axis=1, bitorder="little")
    return np.ascontiguousarray(bits[:, :cols])


def _wptr(w: np.ndarray):
    return w.ctypes.data_as(C.POINTER(C.c_uint64))


# ------------------------------------------------------------------ reference-shaped types


@dataclass
class StabilizerInstance:
    a: np.ndarray
    n: int
    k: int

    @staticmethod
    def from_matrix(m) -> "StabilizerInstance":
        a = np.ascontiguousarray(np.asarray(m, dtype=np.uint8))
        if a.ndim != 2 or a.shape[1] == 0 or a.shape[1] % 2:
            raise ValueError("StabilizerInstance: column count must be even and nonzero")
        n = a.shape[1] // 2
        return StabilizerInstance(a=a, n=n, k=a.shape[0] - n)


@dataclass
class RunOptions:
    workers: int = 1
    validate: bool = True
    dual_filter: bool = True
    device: int = 0
    max_generation: int = 0
    rank: int = 0
    world: int = 1
    allreduce_min: Optional[Callable[[np.ndarray], np.ndarray]] = None
    kernel: int = 0  # 0 auto, 1 walk, 2 POPC tile, 4 tensor-core tile
    stream: int = 0  # cudaStream_t handle (e.g. torch.cuda.current_stream().cuda_stream); 0 = private
    comm: int = 0  # Comm.handle (NCCL): the level exchange runs on the stream, no host round trip
    shard_min: int = 0  # levels below this many candidates run whole on every rank (0: 2^26)

    def _c(self) -> tuple[_Options, object]:
        o = _Options()
        o.workers = self.workers
        o.validate = int(self.validate)
        o.dual_filter = int(self.dual_filter)
        o.device = self.device
        o.max_generation = self.max_generation
        o.rank = self.rank
        o.world = self.world
        o.kernel = self.kernel
        o.stream = self.stream or None
        o.comm = self.comm or None
        o.shard_min = self.shard_min
        keep = None
        if self.allreduce_min is not None:
            fn = self.allreduce_min

            def _cb(ctx, values, count):
                try:
                    arr = np.ctypeslib.as_array(values, shape=(count,))
                    arr[:] = np.asarray(fn(arr.copy()), dtype=np.uint64)
                    return 0
                except Exception:  # noqa: BLE001 - reported as a device error by the library
                    return 1

            keep = _ALLREDUCE(_cb)
            o.allreduce_min = keep
        return o, keep


@dataclass
class BoundsTraceEntry:
    g: int
    lower: int
    upper: int

    def astuple(self):
        return (self.g, self.lower, self.upper)


@dataclass
class DistanceReport:
    distance: int
    algorithm: Algorithm
    generations: int
    candidates_enumerated: int
    elapsed_seconds: float
    workers: int
    bounds_trace: list = field(default_factory=list)
    # GPU-side extras
    complete: bool = True
    upper: int = 0
    candidates_visited: int = 0
    prep_seconds: float = 0.0
    enum_seconds: float = 0.0
    n_gammas: int = 0
    kernel_launches: int = 0
    best_generation: int = -1
    best_gamma: int = -1
    best_rank: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    level_seconds: list = field(default_factory=list)
    last_level_kernel: int = 0  # 1 walk, 2 POPC tile, 3 tensor-core tile, 4 package walk, 5 package tile
    candidates_skipped: int = 0  # left out by the mid-level early exit (visited + skipped = enumerated)

    def trace_tuples(self):
        return [e.astuple() for e in self.bounds_trace]


def _report(r: _Report, tr, cap: int) -> DistanceReport:
    alg = Algorithm(r.algorithm) if r.algorithm in (0, 1, 2, 3, 4) else Algorithm.saved_isometry
    n = min(r.trace_len, cap)
    return DistanceReport(
        distance=r.distance, algorithm=alg, generations=r.generations,
        candidates_enumerated=int(r.candidates_enumerated), elapsed_seconds=r.elapsed_seconds, workers=r.workers,
        bounds_trace=[BoundsTraceEntry(tr[i].g, tr[i].lower, tr[i].upper) for i in range(n)],
        complete=bool(r.complete), upper=int(r.upper), candidates_visited=int(r.candidates_visited),
        prep_seconds=r.prep_seconds, enum_seconds=r.enum_seconds, n_gammas=r.n_gammas,
        kernel_launches=r.kernel_launches, best_generation=r.best_generation, best_gamma=r.best_gamma,
        best_rank=int(r.best_rank), h2d_bytes=int(r.h2d_bytes), d2h_bytes=int(r.d2h_bytes),
        last_level_kernel=r.last_level_kernel, candidates_skipped=int(r.candidates_skipped))


_TRACE_CAP = 512


def _inst(x) -> StabilizerInstance:
    return x if isinstance(x, StabilizerInstance) else StabilizerInstance.from_matrix(x)


def saved_isometry(inst, opts: Optional[RunOptions] = None, return_best: bool = False):
    """Saved_isometry distance of a normalizer (distance.cpp:135-149) on the GPU."""
    inst = _inst(inst)
    opts = opts or RunOptions()
    w = pack_rows(inst.a)
    o, keep = opts._c()
    rep = _Report()
    tr = (_Trace * _TRACE_CAP)()
    best = np.zeros(max(1, (3 * inst.n + 63) // 64), dtype=np.uint64)
    rc = library().sdb_saved_isometry(_wptr(w), w.shape[0], inst.a.shape[1], w.shape[1], C.byref(o), C.byref(rep), tr,
                                      _TRACE_CAP, _wptr(best) if return_best else None)
    del keep
    _raise(rc)
    out = _report(rep, tr, _TRACE_CAP)
    if return_best:
        return out, unpack_rows(best.reshape(1, -1), 3 * inst.n)[0]
    return out


def _package_route(fn_name: str, inst, opts: Optional[RunOptions], return_best: bool):
    inst = _inst(inst)
    opts = opts or RunOptions()
    w = pack_rows(inst.a)
    o, keep = opts._c()
    rep = _Report()
    tr = (_Trace * _TRACE_CAP)()
    best = np.zeros(max(1, (2 * inst.n + 63) // 64), dtype=np.uint64)
    rc = getattr(library(), fn_name)(_wptr(w), w.shape[0], inst.a.shape[1], w.shape[1], C.byref(o), C.byref(rep), tr,
                                     _TRACE_CAP, _wptr(best) if return_best else None)
    del keep
    _raise(rc)
    out = _report(rep, tr, _TRACE_CAP)
    if return_best:
        return out, unpack_rows(best.reshape(1, -1), 2 * inst.n)[0]
    return out


def saved_1_gamma(inst, opts: Optional[RunOptions] = None, return_best: bool = False):
    """Saved_1_Gamma (distance.cpp:95-113): diagonalize_f2 packages, one matrix, L = g + 1."""
    return _package_route("sdb_saved_1_gamma", inst, opts, return_best)


def saved_2_gamma(inst, opts: Optional[RunOptions] = None, return_best: bool = False):
    """Saved_2_Gamma (distance.cpp:115-133): two F4-diagonalized matrices, the 2-matrix bound."""
    return _package_route("sdb_saved_2_gamma", inst, opts, return_best)


def prepare_packages(inst, alg: Algorithm) -> list:
    """The package routes' prepared matrices: diagonalize_f2 (saved_1_gamma) or
    diagonalize_f4 + second_gamma (saved_2_gamma), as PackagedGamma objects."""
    inst = _inst(inst)
    w = pack_rows(inst.a)
    rows, cols = inst.a.shape
    max_rows, cap = 2 * rows + 2, 16 * rows + 16
    ow = max(1, (cols + 63) // 64)
    out = np.zeros((2 * max_rows, ow), dtype=np.uint64)
    gr, npk, npp = (np.zeros(2, dtype=np.int32) for _ in range(3))
    pk = np.zeros(cap, dtype=np.int32)
    ng = C.c_int(0)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    _raise(library().sdb_prepare_packages(_wptr(w), rows, cols, w.shape[1], int(alg), 2, max_rows, _wptr(out), ow,
                                          ip(gr), ip(npk), ip(npp), ip(pk), cap, C.byref(ng)))
    res, pos = [], 0
    for j in range(ng.value):
        pkgs = []
        for _ in range(int(npk[j])):
            sz = int(pk[pos])
            pkgs.append([int(x) for x in pk[pos + 1:pos + 1 + sz]])
            pos += 1 + sz
        mat = unpack_rows(out[j * max_rows:j * max_rows + int(gr[j])], cols)
        res.append(PackagedGamma(matrix=mat, mode=WeightMode.symplectic, pair_count=cols // 2, rank_deficit=0,
                                 pivots=[], packages=pkgs, n_pp=int(npp[j])))
    return res


def diagonalize_f2(a) -> PackagedGamma:
    return prepare_packages(a, Algorithm.saved_1_gamma)[0]


def compute_distance(inst, alg: Algorithm = Algorithm.saved_isometry, opts: Optional[RunOptions] = None):
    inst = _inst(inst)
    opts = opts or RunOptions()
    w = pack_rows(inst.a)
    o, keep = opts._c()
    rep = _Report()
    tr = (_Trace * _TRACE_CAP)()
    rc = library().sdb_compute_distance(_wptr(w), w.shape[0], inst.a.shape[1], w.shape[1], int(alg), C.byref(o),
                                        C.byref(rep), tr, _TRACE_CAP)
    del keep
    _raise(rc)
    return _report(rep, tr, _TRACE_CAP)


@dataclass
class BatchResult:
    distances: np.ndarray
    statuses: np.ndarray
    generations: np.ndarray
    traces: list
    elapsed_seconds: float
    device_seconds: float


def saved_isometry_batch(codes, opts: Optional[RunOptions] = None) -> BatchResult:
    """Many same-shape normalizers, one code per CTA (BASELINE config 3)."""
    arrs = [np.asarray(c.a if isinstance(c, StabilizerInstance) else c, dtype=np.uint8) for c in codes]
    if not arrs:
        raise ValueError("empty batch")
    rows, cols = arrs[0].shape
    for a in arrs:
        if a.shape != (rows, cols):
            raise ValueError("batch codes must share one shape")
    words = max(1, (cols + 63) // 64)
    packed = np.ascontiguousarray(np.stack([pack_rows(a) for a in arrs]).reshape(len(arrs) * rows, words))
    return saved_isometry_batch_packed(packed, len(arrs), rows, cols, opts)


def saved_isometry_batch_packed(packed: np.ndarray, n_codes: int, rows: int, cols: int,
                                opts: Optional[RunOptions] = None, trace_cap: int = 64) -> BatchResult:
    opts = opts or RunOptions()
    words = packed.shape[-1]
    o, keep = opts._c()
    dist = np.zeros(n_codes, dtype=np.int32)
    stat = np.zeros(n_codes, dtype=np.int32)
    gens = np.zeros(n_codes, dtype=np.int32)
    tl = np.zeros(n_codes, dtype=np.int32)
    tr = (_Trace * (n_codes * trace_cap))()
    el, dev = C.c_double(0), C.c_double(0)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    rc = library().sdb_saved_isometry_batch(_wptr(packed), n_codes, rows, cols, words, C.byref(o), ip(dist), ip(stat),
                                            ip(gens), tr, ip(tl), trace_cap, C.byref(el), C.byref(dev))
    del keep
    _raise(rc)
    traces = [[(tr[c * trace_cap + i].g, tr[c * trace_cap + i].lower, tr[c * trace_cap + i].upper)
               for i in range(min(int(tl[c]), trace_cap))] for c in range(n_codes)]
    return BatchResult(dist, stat, gens, traces, el.value, dev.value)


@dataclass
class ValidationResult:
    ok: bool
    message: str


def validate_normalizer(inst) -> ValidationResult:
    inst = _inst(inst)
    w = pack_rows(inst.a)
    ok = C.c_int(0)
    msg = C.create_string_buffer(8192)
    _raise(library().sdb_validate_normalizer(_wptr(w), w.shape[0], inst.a.shape[1], w.shape[1], C.byref(ok), msg,
                                             8192))
    return ValidationResult(bool(ok.value), msg.value.decode())


def isometry_transform(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.uint8)
    if a.shape[1] % 2:
        raise ValueError("isometry_transform: column count must be even")
    w = pack_rows(a)
    n = a.shape[1] // 2
    ow = max(1, (3 * n + 63) // 64)
    out = np.zeros((a.shape[0], ow), dtype=np.uint64)
    _raise(library().sdb_isometry_transform(_wptr(w), w.shape[0], a.shape[1], w.shape[1], _wptr(out), ow))
    return unpack_rows(out, 3 * n)


@dataclass
class PackagedGamma:
    """Generator matrix with its package partition (prep.hpp:25-35). packages = [] means every
    row is its own package (singleton_gamma / information_sets)."""
    matrix: np.ndarray
    mode: WeightMode = WeightMode.hamming
    pair_count: int = 0
    rank_deficit: int = 0
    pivots: list = field(default_factory=list)
    packages: list = field(default_factory=list)
    n_pp: int = -1

    def n_p(self) -> int:
        return len(self.packages) if self.packages else int(self.matrix.shape[0])


def singleton_gamma(m, mode: WeightMode) -> PackagedGamma:
    m = np.ascontiguousarray(np.asarray(m, dtype=np.uint8))
    cols = m.shape[1]
    if mode == WeightMode.symplectic:
        if cols % 2:
            raise ValueError("singleton_gamma: column count must be even")
        pc = cols // 2
    else:
        pc = cols // 3 if cols % 3 == 0 else 0
    return PackagedGamma(matrix=m, mode=WeightMode(mode), pair_count=pc, rank_deficit=0, pivots=[-1] * m.shape[0])


def information_sets(b) -> list[PackagedGamma]:
    b = np.asarray(b, dtype=np.uint8)
    rows, cols = b.shape
    w = pack_rows(b)
    cap = 64
    out = np.zeros((cap * rows, w.shape[1]), dtype=np.uint64)
    defs = np.zeros(cap, dtype=np.int32)
    piv = np.zeros(cap * rows, dtype=np.int32)
    ng = C.c_int(0)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    _raise(library().sdb_information_sets(_wptr(w), rows, cols, w.shape[1], cap, _wptr(out), w.shape[1], ip(defs),
                                          ip(piv), C.byref(ng)))
    res = []
    for j in range(min(ng.value, cap)):
        mat = unpack_rows(out[j * rows:(j + 1) * rows], cols)
        res.append(PackagedGamma(matrix=mat, mode=WeightMode.hamming, pair_count=cols // 3 if cols % 3 == 0 else 0,
                                 rank_deficit=int(defs[j]), pivots=[int(x) for x in piv[j * rows:(j + 1) * rows]]))
    return res


def tc_encoding_check(a, isometry: bool = True, seed: int = 1, trials: int = 256):
    """Host-only check of the tensor-core tile kernel's exact ±1 coordinate encoding
    (csrc/tcenc.cpp): on `trials` random head/tail splits per Gamma, the encoded dot product
    must reproduce popc(x|z). Returns (mismatches, [K per Gamma]); mismatches == -1 means the
    code has no tensor-core encoding (more than 128 coordinates)."""
    a = np.asarray(a, dtype=np.uint8)
    rows, cols = a.shape
    w = pack_rows(a)
    mism = C.c_int(0)
    ks = np.zeros(64, dtype=np.int32)
    ng = C.c_int(0)
    ip = lambda x: x.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    _raise(library().sdb_tc_encoding_check(_wptr(w), rows, cols, w.shape[1], int(bool(isometry)), C.c_uint64(seed),
                                           trials, C.byref(mism), ip(ks), 64, C.byref(ng)))
    return mism.value, [int(x) for x in ks[:min(ng.value, 64)]]


@dataclass
class AdmissibilityFilter:
    normalizer: Optional[np.ndarray] = None
    enabled: bool = False
    k: int = 0

    @staticmethod
    def disabled() -> "AdmissibilityFilter":
        return AdmissibilityFilter()

    @staticmethod
    def for_rows(rows, k: int) -> "AdmissibilityFilter":
        return AdmissibilityFilter(normalizer=np.asarray(rows, dtype=np.uint8), enabled=k >= 1, k=k)


@dataclass
class BoundsState:
    """symdist::BoundsState (engine.hpp:33-40); upper = 0 means unset (the sentinel)."""
    lower: int = 1
    upper: int = 0
    generation: int = 0
    candidates_enumerated: int = 0
    trace: list = field(default_factory=list)
    best: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint8))
    report: Optional[DistanceReport] = None


class _BoundsC(C.Structure):
    _fields_ = [("upper", C.c_longlong), ("candidates_enumerated", C.c_ulonglong), ("improved", C.c_int)]


def enumerate_generation(gamma: PackagedGamma, g: int, state: BoundsState, filt: AdmissibilityFilter,
                         workers: int = 1, opts: Optional[RunOptions] = None) -> None:
    """enumerate_generation (engine.hpp:53-54, engine.cpp:296-301) on the GPU: every g-combination
    of one matrix (one member per package) folded into `state` — upper (set to the sentinel when
    0), best (the first minimal codeword, when it improved upper) and candidates_enumerated."""
    opts = opts or RunOptions(workers=workers)
    m = np.asarray(gamma.matrix, dtype=np.uint8)
    rows, cols = m.shape
    w = pack_rows(m)
    enc = []
    for pk in gamma.packages:
        enc += [len(pk)] + list(pk)
    enc = np.array(enc or [0], dtype=np.int32)
    if filt.normalizer is not None and filt.enabled:
        fw = pack_rows(filt.normalizer)
        fr, fc, fwords = filt.normalizer.shape[0], filt.normalizer.shape[1], fw.shape[1]
    else:
        fw = np.zeros((1, 1), dtype=np.uint64)
        fr, fc, fwords = 0, 0, 1
    st = _BoundsC(int(state.upper), int(state.candidates_enumerated), 0)
    best = np.zeros(w.shape[1], dtype=np.uint64)
    o, keep = opts._c()
    rc = library().sdb_enumerate_generation(_wptr(w), rows, cols, w.shape[1], int(gamma.mode), gamma.pair_count,
                                            len(gamma.packages), enc.ctypes.data_as(C.POINTER(C.c_int)), int(g),
                                            _wptr(fw), fr, fc, fwords, int(filt.enabled), filt.k if filt.enabled else 0,
                                            C.byref(o), C.byref(st), _wptr(best))
    del keep
    _raise(rc)
    state.upper = int(st.upper)
    state.candidates_enumerated = int(st.candidates_enumerated)
    if st.improved:
        state.best = unpack_rows(best.reshape(1, -1), cols)[0]


def lower_bound(g: int, gammas: Sequence[PackagedGamma]) -> int:
    if not gammas:
        raise ValueError("lower_bound: no generator matrices")
    defs = np.array([gm.rank_deficit for gm in gammas], dtype=np.int32)
    nps = np.array([gm.n_p() for gm in gammas], dtype=np.int32)
    npp = np.array([gm.n_pp if gm.n_pp >= 0 else gm.n_p() for gm in gammas], dtype=np.int32)
    out = C.c_longlong(0)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    _raise(library().sdb_lower_bound(g, int(gammas[0].mode), len(gammas), ip(defs), ip(nps), ip(npp), C.byref(out)))
    return int(out.value)


def run_bz(gammas: Sequence[PackagedGamma], filt: AdmissibilityFilter, workers: int = 1,
           opts: Optional[RunOptions] = None) -> BoundsState:
    """run_bz (engine.cpp:303-343) over singleton-package matrices on the GPU."""
    if not gammas:
        raise ValueError("run_bz: need at least one generator matrix")
    opts = opts or RunOptions(workers=workers)
    g0 = gammas[0]
    rows, cols = g0.matrix.shape
    if any(gm.packages for gm in gammas) or len({gm.matrix.shape[0] for gm in gammas}) > 1:
        return _run_bz_packaged(gammas, filt, opts)
    for gm in gammas:
        if gm.matrix.shape[1] != cols or gm.mode != g0.mode or gm.pair_count != g0.pair_count:
            raise ValueError("run_bz: generator matrices must share one codeword frame")
        if gm.matrix.shape[0] == 0:
            raise ValueError("run_bz: matrix with no packages")
        if gm.matrix.shape[0] != rows:
            raise ValueError("run_bz: this build needs equal package counts across matrices")
    words = max(1, (cols + 63) // 64)
    packed = np.ascontiguousarray(np.concatenate([pack_rows(gm.matrix) for gm in gammas], axis=0))
    defs = np.array([gm.rank_deficit for gm in gammas], dtype=np.int32)
    if filt.normalizer is not None and filt.enabled:
        fw = pack_rows(filt.normalizer)
        fr, fc, fwords = filt.normalizer.shape[0], filt.normalizer.shape[1], fw.shape[1]
    else:
        fw = np.zeros((1, 1), dtype=np.uint64)
        fr, fc, fwords = 0, 0, 1
    o, keep = opts._c()
    rep = _Report()
    tr = (_Trace * _TRACE_CAP)()
    best = np.zeros(words, dtype=np.uint64)
    rc = library().sdb_run_bz(_wptr(packed), len(gammas), rows, cols, words, int(g0.mode), g0.pair_count,
                              defs.ctypes.data_as(C.POINTER(C.c_int)), _wptr(fw), fr, fc, fwords, int(filt.enabled),
                              filt.k if filt.enabled else 0, C.byref(o), C.byref(rep), tr, _TRACE_CAP, _wptr(best))
    del keep
    _raise(rc)
    r = _report(rep, tr, _TRACE_CAP)
    lower = r.bounds_trace[-1].lower if r.bounds_trace else 1
    return BoundsState(lower=lower, upper=r.upper, generation=r.generations,
                       candidates_enumerated=r.candidates_enumerated, trace=r.trace_tuples(),
                       best=unpack_rows(best.reshape(1, -1), cols)[0] if r.best_generation > 0 else np.zeros(0, np.uint8),
                       report=r)


def _run_bz_packaged(gammas, filt, opts):
    g0 = gammas[0]
    cols = g0.matrix.shape[1]
    for gm in gammas:
        if gm.matrix.shape[1] != cols or gm.mode != g0.mode or gm.pair_count != g0.pair_count:
            raise ValueError("run_bz: generator matrices must share one codeword frame")
        if gm.n_p() == 0:
            raise ValueError("run_bz: matrix with no packages")
    words = max(1, (cols + 63) // 64)
    max_rows = max(gm.matrix.shape[0] for gm in gammas)
    packed = np.zeros((len(gammas) * max_rows, words), dtype=np.uint64)
    enc, npk = [], []
    for j, gm in enumerate(gammas):
        packed[j * max_rows:j * max_rows + gm.matrix.shape[0]] = pack_rows(gm.matrix)
        pk = gm.packages or [[r] for r in range(gm.matrix.shape[0])]
        npk.append(len(pk))
        for p in pk:
            enc += [len(p)] + list(p)
    gr = np.array([gm.matrix.shape[0] for gm in gammas], dtype=np.int32)
    npk = np.array(npk, dtype=np.int32)
    npp = np.array([gm.n_pp for gm in gammas], dtype=np.int32)
    defs = np.array([gm.rank_deficit for gm in gammas], dtype=np.int32)
    enc = np.array(enc, dtype=np.int32)
    if filt.normalizer is not None and filt.enabled:
        fw = pack_rows(filt.normalizer)
        fr, fc, fwords = filt.normalizer.shape[0], filt.normalizer.shape[1], fw.shape[1]
    else:
        fw = np.zeros((1, 1), dtype=np.uint64)
        fr, fc, fwords = 0, 0, 1
    o, keep = opts._c()
    rep = _Report()
    tr = (_Trace * _TRACE_CAP)()
    best = np.zeros(words, dtype=np.uint64)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    rc = library().sdb_run_bz_packaged(_wptr(packed), len(gammas), ip(gr), max_rows, cols, words, int(g0.mode),
                                       g0.pair_count, ip(defs), ip(npk), ip(npp), ip(enc), _wptr(fw), fr, fc, fwords,
                                       int(filt.enabled), filt.k if filt.enabled else 0, C.byref(o), C.byref(rep), tr,
                                       _TRACE_CAP, _wptr(best))
    del keep
    _raise(rc)
    r = _report(rep, tr, _TRACE_CAP)
    lower = r.bounds_trace[-1].lower if r.bounds_trace else 1
    return BoundsState(lower=lower, upper=r.upper, generation=r.generations,
                       candidates_enumerated=r.candidates_enumerated, trace=r.trace_tuples(),
                       best=unpack_rows(best.reshape(1, -1), cols)[0] if r.best_generation > 0 else np.zeros(0, np.uint8),
                       report=r)


def random_stabilizer(n: int, k: int, seed: int) -> StabilizerInstance:
    """The reference's instance generator (distance.cpp:242-294), same mt19937_64 draws."""
    words = max(1, (2 * n + 63) // 64)
    out = np.zeros((max(n + k, 1), words), dtype=np.uint64)
    _raise(library().sdb_random_stabilizer(n, k, C.c_uint64(seed), out.ctypes.data, words))
    return StabilizerInstance.from_matrix(unpack_rows(out[:n + k], 2 * n))


def parse_matrix_text(text: str, origin: str = "<input>") -> StabilizerInstance:
    """matrix_io.cpp:26-89: "K N" header then K rows of N '0'/'1' (ParseError on bad input)."""
    t = text.encode()
    o = origin.encode()
    nr, nc = C.c_int(0), C.c_int(0)
    lib = library()
    _raise(lib.sdb_parse_matrix_text(t, o, None, 0, 0, C.byref(nr), C.byref(nc)))
    words = max(1, (nc.value + 63) // 64)
    out = np.zeros((max(nr.value, 1), words), dtype=np.uint64)
    _raise(lib.sdb_parse_matrix_text(t, o, out.ctypes.data, words, nr.value, C.byref(nr), C.byref(nc)))
    return StabilizerInstance.from_matrix(unpack_rows(out[:nr.value], nc.value))


def parse_matrix_file(path: str) -> StabilizerInstance:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ParseError(f"{path}: cannot open file") from None
    return parse_matrix_text(text, path)


def format_matrix(m) -> str:
    a = np.asarray(m.a if isinstance(m, StabilizerInstance) else m, dtype=np.uint8)
    w = pack_rows(a)
    ln = C.c_int(0)
    lib = library()
    _raise(lib.sdb_format_matrix(_wptr(w), a.shape[0], a.shape[1], w.shape[1], None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    _raise(lib.sdb_format_matrix(_wptr(w), a.shape[0], a.shape[1], w.shape[1], buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode()


class Comm:
    """NCCL communicator for the per-level exchange across GPUs (one per process/GPU).
    ``Comm.unique_id()`` on rank 0, shared out of band, then ``Comm(uid, rank, world, device)``
    on every rank; pass ``comm.handle`` as ``RunOptions.comm``."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _raise(library().sdb_comm_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, rank: int, world: int, device: int = 0):
        h = C.c_void_p()
        _raise(library().sdb_comm_create(uid, rank, world, device, C.byref(h)))
        self.handle = h.value
        self.device = device

    def allreduce_min(self, values) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64)).copy()
        _raise(library().sdb_comm_allreduce_min(self.handle, v.ctypes.data, len(v), self.device))
        return v

    def close(self):
        if getattr(self, "handle", None):
            library().sdb_comm_destroy(self.handle)
            self.handle = None


def torch_allreduce_min(dist, device="cpu"):
    """RunOptions.allreduce_min over a torch.distributed process group (gloo or nccl): the
    host-callback form of the per-level exchange (MIN on order-preserving int64 views of the
    uint64 values), for callers without an NCCL communicator handle (Comm)."""
    import torch

    def fn(values):
        v = (np.asarray(values, dtype=np.uint64) ^ np.uint64(1 << 63)).view(np.int64)
        t = torch.tensor(v, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return t.cpu().numpy().view(np.uint64) ^ np.uint64(1 << 63)

    return fn


def cli_path() -> str:
    """The symdist_b200 CLI (compute / verify / bench, reference tools/symdist_main.cpp)."""
    return os.path.join(HERE, "symdist_b200")


def generate_code(n: int, k: int, seed: int, transvections: int = 0) -> np.ndarray:
    """BASELINE.md §2 generator (xorshift64* transvections), computed by the native host code."""
    words = max(1, (2 * n + 63) // 64)
    out = np.zeros((n + k, words), dtype=np.uint64)
    _raise(library().sdb_generate_code(n, k, seed, transvections, out.ctypes.data, words))
    return unpack_rows(out, 2 * n)


class Plan:
    """Device-resident saved_isometry: prep + H2D once, then ``run()`` executes the level loop
    from HBM (used to time the kernels alone)."""

    def __init__(self, inst, opts: Optional[RunOptions] = None):
        inst = _inst(inst)
        self.inst = inst
        self.opts = opts or RunOptions()
        w = pack_rows(inst.a)
        o, self._keep = self.opts._c()
        self._o = o
        h = C.c_void_p()
        _raise(library().sdb_plan_create(w.ctypes.data, w.shape[0], inst.a.shape[1], w.shape[1], C.byref(o),
                                         C.byref(h)))
        self._h = h

    def run(self) -> DistanceReport:
        rep = _Report()
        tr = (_Trace * _TRACE_CAP)()
        secs = (C.c_double * _TRACE_CAP)()
        _raise(library().sdb_plan_run(self._h, C.byref(rep), tr, _TRACE_CAP, secs))
        r = _report(rep, tr, _TRACE_CAP)
        r.level_seconds = [secs[i] for i in range(min(rep.trace_len, _TRACE_CAP))]
        return r

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            library().sdb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
