"""CPU, world_size 2 over gloo: the multi-rank level loop's host logic.

Each rank takes the product's shard of every level — lexicographic segments of each Gamma_j's
rank space, segment s to rank s % world (csrc/engine.cpp prepare_level, kernels.cu
walk_kernel) — scores its candidates on the CPU (the oracle's Gamma_j, the reference's
admissibility rule engine.cpp:23-29), and merges the level minimum with the product's
exchange: paper_2408_10743_b200.torch_allreduce_min (torch.distributed MIN on order-preserving int64 views), then
the key of the winning weight only (Plan::run). The merged trace and best key must equal the
reference's single-process ones (tests/golden/config1.json).
"""
import itertools
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

KEY_BITS = 58
NO_KEY = (1 << 64) - 1
SEG_LEN = 64


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows_as_ints(m) -> list:
    return [int("".join(str(int(b)) for b in row[::-1]), 2) for row in m]


def _sym_ip(u: int, v: int, n: int) -> int:
    ua, ub = u & ((1 << n) - 1), (u >> n) & ((1 << n) - 1)
    va, vb = v & ((1 << n) - 1), (v >> n) & ((1 << n) - 1)
    return (bin(ua & vb).count("1") + bin(ub & va).count("1")) & 1


def _worker(rank: int, world: int, port: int, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import paper_2408_10743_b200 as P
        import oracle as O
        from conftest import hex_to_mat, load_golden

        gd = load_golden("config1.json")
        n, k = gd["n"], gd["k"]
        a = hex_to_mat(gd["normalizer"], 2 * n)
        gammas = O.information_sets(O.isometry(a))
        rows = [_rows_as_ints(gm["matrix"]) for gm in gammas]
        defs = [gm["rank_deficit"] for gm in gammas]
        filt = _rows_as_ints(a)
        mask2n = (1 << (2 * n)) - 1
        N, G = a.shape[0], len(gammas)
        allreduce = P.torch_allreduce_min(dist, "cpu")
        U, trace, best, visited = 3 * n + 1, [], None, 0
        for g in range(1, N + 1):
            per = len(list(itertools.combinations(range(N), g)))
            segs = (per + SEG_LEN - 1) // SEG_LEN
            wmin, keys = None, {}
            for j in range(G):
                for r, combo in enumerate(itertools.combinations(range(N), g)):
                    if (j * segs + r // SEG_LEN) % world != rank:
                        continue
                    visited += 1
                    c = 0
                    for i in combo:
                        c ^= rows[j][i]
                    w = bin(c).count("1")  # Hamming weight of (a|b|a^b) = 2 popc(a|b)
                    if w >= U:
                        continue
                    if not any(_sym_ip(c & mask2n, f, n) for f in filt):
                        continue  # in C: not admissible
                    key = (j << KEY_BITS) | r
                    keys[w] = min(keys.get(w, NO_KEY), key)
                    wmin = w if wmin is None else min(wmin, w)
            # the product's exchange (Plan::run): weight first, then the key of that weight
            mine = NO_KEY if wmin is None else wmin
            v = int(allreduce(np.array([mine], dtype=np.uint64))[0])
            key = keys[v] if (v != NO_KEY and v == mine) else NO_KEY
            key = int(allreduce(np.array([key], dtype=np.uint64))[0])
            if v != NO_KEY and v < U:
                U, best = v, (g, key >> KEY_BITS, key & ((1 << KEY_BITS) - 1))
            L = sum(max(0, g + 1 - d) for d in defs)
            trace.append((g, L, U))
            if L >= U:
                break
        # BoundsState::best: the first minimal candidate in the reference's visiting order
        bg, bj, br = best
        combo = list(itertools.combinations(range(N), bg))[br]
        word = 0
        for i in combo:
            word ^= rows[bj][i]
        best = format(word, "x")
        tot = torch.tensor([visited], dtype=torch.int64)
        dist.all_reduce(tot)
        q.put((rank, trace, best, int(tot.item())))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), 0))


def test_two_rank_sharded_levels_merge_to_the_reference_trace():
    from conftest import load_golden

    gd = load_golden("config1.json")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, trace, best, visited in res:
        assert trace != "error", best
        assert trace == [tuple(t) for t in gd["trace"]]
        assert visited == gd["candidates"]  # the shards cover every candidate exactly once
        assert best == gd["best"]  # the reference's BoundsState::best
