"""GPU: size-independent properties at full sizes, sharding invariance and the
device-resident plan."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def tr(rep):
    return [e.astuple() for e in rep.bounds_trace]


def test_trace_properties_on_configs(gpu):
    for cid in (1, 2, 4):
        c = gpu.CONFIGS[cid]
        a = gpu.generate_code(c["n"], c["k"], c["seed"])
        rep = gpu.saved_isometry(a)
        t = tr(rep)
        assert all(t[i + 1][1] >= t[i][1] and t[i + 1][2] <= t[i][2] for i in range(len(t) - 1))
        assert t[-1][2] % 2 == 0 and t[-1][2] == 2 * rep.distance
        assert t[-1][1] >= t[-1][2]
        assert rep.candidates_visited + rep.candidates_skipped == rep.candidates_enumerated


class _ThreadAllreduce:
    """In-process stand-in for the NCCL/gloo min-allreduce: ranks are threads."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.lock = threading.Lock()
        self.vals = {}

    def fn_for(self, rank):
        def fn(values):
            with self.lock:
                self.vals[rank] = values.copy()
            self.barrier.wait()
            out = np.minimum.reduce([self.vals[r] for r in range(self.world)])
            self.barrier.wait()
            return out
        return fn


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_levels_match_single(gpu, world):
    c = gpu.CONFIGS[2]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    single, best1 = gpu.saved_isometry(a, return_best=True)
    ar = _ThreadAllreduce(world)
    out = [None] * world

    def run(r):
        out[r] = gpu.saved_isometry(a, gpu.RunOptions(rank=r, world=world, allreduce_min=ar.fn_for(r), shard_min=1),
                                    return_best=True)

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for rep, best in out:
        assert tr(rep) == tr(single)
        assert rep.distance == single.distance
        assert (best == best1).all()
    assert sum(rep.candidates_visited for rep, _ in out) == single.candidates_visited


def test_plan_reuse_is_deterministic(gpu):
    c = gpu.CONFIGS[2]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    with gpu.Plan(a) as plan:
        r1 = plan.run()
        r2 = plan.run()
    assert tr(r1) == tr(r2)
    assert r1.distance == 7
    assert len(r1.level_seconds) == len(r1.bounds_trace)


def test_small_levels_run_whole_on_every_rank(gpu):
    # below shard_min a level runs whole on every rank with no exchange: same answer, and each
    # rank visits every candidate of those levels
    c = gpu.CONFIGS[2]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    single = gpu.saved_isometry(a)
    calls = []

    def never(v):
        calls.append(1)
        return v

    rep = gpu.saved_isometry(a, gpu.RunOptions(rank=1, world=2, allreduce_min=never, shard_min=1 << 40))
    assert tr(rep) == tr(single) and not calls
    assert rep.candidates_visited == single.candidates_visited


def test_nccl_exchange_path_on_one_gpu(gpu):
    # a one-rank NCCL communicator with shard_min = 1 runs every level through the
    # stream-ordered min-allreduce of the per-weight keys and level_close's key scan
    comm = gpu.Comm(gpu.Comm.unique_id(), 0, 1, 0)
    try:
        v = comm.allreduce_min([5, 3, 2**64 - 1])
        assert v.tolist() == [5, 3, 2**64 - 1]
        for cid in (1, 2, 4):
            c = gpu.CONFIGS[cid]
            a = gpu.generate_code(c["n"], c["k"], c["seed"])
            base, best0 = gpu.saved_isometry(a, return_best=True)
            via, best1 = gpu.saved_isometry(a, gpu.RunOptions(comm=comm.handle, shard_min=1), return_best=True)
            assert tr(via) == tr(base) and (best0 == best1).all()
        g2 = gpu.saved_2_gamma(a, gpu.RunOptions(comm=comm.handle, shard_min=1))
        assert g2.distance == base.distance
    finally:
        comm.close()


def test_config5_through_g10_matches_the_full_run(gpu):
    # levels g <= 9 are pinned to the reference (config5_g9.json); g = 10 against this
    # build's own complete run (profiles/r01_config5_full.json: d = 14 after 13 levels), which
    # no CPU can reproduce (SURVEY.md §0 finding 3) — a determinism and monotonicity check
    c = gpu.CONFIGS[5]
    a = gpu.generate_code(c["n"], c["k"], c["seed"])
    rep = gpu.saved_isometry(a, gpu.RunOptions(max_generation=10))
    full = [(1, 4, 44), (2, 6, 42), (3, 8, 36), (4, 10, 34), (5, 12, 32), (6, 14, 30), (7, 16, 30), (8, 18, 28),
            (9, 20, 28), (10, 22, 28)]
    assert tr(rep) == full
    assert rep.candidates_visited + rep.candidates_skipped == rep.candidates_enumerated == 19537662444573
