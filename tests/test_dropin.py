"""The drop-in proof: integration/_build/dropin_check links the UNMODIFIED
reference library (oracle/_ref) and the reference-side adapter over libsymdist_b200, parses
each matrix with the reference's own parser, and runs symdist::saved_isometry (and the
package routes / auto dispatch) beside the adapter's saved_isometry_b200 on the same
StabilizerInstance. Every DistanceReport field the reference defines must agree
(distance, algorithm, generations, candidates_enumerated, workers, bounds_trace); errors
agree by exception class."""
import json
import os
import subprocess

import pytest

from conftest import ROOT, hex_to_mat, load_golden

BIN = os.path.join(ROOT, "integration", "_build", "dropin_check")


def _bin():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/dropin_check not built (needs /root/reference at build time)")
    return BIN


def _write(tmp_path, name, a):
    import paper_2408_10743_b200 as P

    p = tmp_path / f"{name}.txt"
    p.write_text(P.format_matrix(a))
    return str(p)


def _run(files, algs, workers=None, timeout=1800):
    cmd = [_bin(), "--algs", algs, *files]
    if workers:
        cmd[1:1] = ["--workers", str(workers)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    return r.returncode, [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]


def test_dropin_binary_runs_the_reference_side(tmp_path):
    # CPU: the reference half answers like the golden; the GPU half fails loudly (no device)
    import paper_2408_10743_b200 as P

    gd = load_golden("config1.json")
    f = _write(tmp_path, "c1", hex_to_mat(gd["normalizer"], 2 * gd["n"]))
    rc, lines = _run([f], "isometry", workers=2)
    assert len(lines) == 1
    ref = lines[0]["reference"]
    assert ref["distance"] == gd["distance"] and [tuple(t) for t in ref["trace"]] == [tuple(t) for t in gd["trace"]]
    assert ref["candidates_enumerated"] == gd["candidates"]
    if not P.device_available():
        assert rc == 1 and "CUDA" in lines[0]["b200"]["message"]


@pytest.mark.gpu
def test_dropin_reports_equal_on_the_configs(gpu, tmp_path):
    files = []
    for cid in (1, 2, 4):
        c = gpu.CONFIGS[cid]
        files.append(_write(tmp_path, f"config{cid}", gpu.generate_code(c["n"], c["k"], c["seed"])))
    rc, lines = _run(files, "isometry")
    assert len(lines) == 3 and all(x["equal"] for x in lines), [x for x in lines if not x["equal"]]
    assert rc == 0
    # the package routes and auto dispatch on the small configs
    rc, lines = _run(files[:2], "1g,2g,auto")
    assert len(lines) == 6 and all(x["equal"] for x in lines), [x for x in lines if not x["equal"]]


@pytest.mark.gpu
def test_dropin_reports_equal_on_config3_codes(gpu, tmp_path):
    c = gpu.CONFIGS[3]
    files = [_write(tmp_path, f"c3_{s}", gpu.generate_code(c["n"], c["k"], s)) for s in c["seeds"][:64]]
    rc, lines = _run(files, "isometry,auto", workers=1)
    assert len(lines) == 128 and all(x["equal"] for x in lines), [x for x in lines if not x["equal"]][:3]


@pytest.mark.gpu
def test_dropin_reports_equal_on_the_reference_kats(gpu, tmp_path):
    cases = load_golden("reference_kats.json")["cases"]
    files = []
    for i, c in enumerate(cases):
        rows = eval(c["normalizer"]) if isinstance(c["normalizer"], str) else c["normalizer"]  # noqa: S307
        files.append(_write(tmp_path, f"kat{i}", hex_to_mat(rows, 2 * int(c["n"]))))
    rc, lines = _run(files, "isometry,1g,2g", workers=1)
    assert len(lines) == 3 * len(cases)
    bad = [x for x in lines if not x["equal"]]
    assert not bad, bad[:3]
