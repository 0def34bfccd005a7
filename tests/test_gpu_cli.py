"""The symdist_b200 CLI end to end on the GPU (proj/tests/test_io_cli.cpp:90-190): compute
with every algorithm, --json/--trace output, exit codes, verify and bench."""
import json
import re
import subprocess

import pytest

import paper_2408_10743_b200 as P

pytestmark = pytest.mark.gpu

EXAMPLE = "3 4\n1001\n0110\n0011\n"


def _cli(*args):
    r = subprocess.run([P.cli_path(), *args], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout + r.stderr


def test_cli_compute_every_algorithm(tmp_path):
    f = tmp_path / "example.mat"
    f.write_text(EXAMPLE)
    code, out = _cli("compute", str(f))
    assert code == 0 and "distance 1\n" in out
    for alg in ("1gamma", "2gamma", "isometry", "brute"):
        code, out = _cli("compute", str(f), "--alg", alg)
        assert code == 0 and "distance 1\n" in out, (alg, out)


def test_cli_threads_do_not_change_the_output(tmp_path):
    f = tmp_path / "threads.mat"
    f.write_text(P.format_matrix(P.random_stabilizer(8, 3, 12345)))
    assert _cli("compute", str(f), "--threads", "1") == _cli("compute", str(f), "--threads", "8")


def test_cli_json_and_trace(tmp_path):
    f = tmp_path / "json.mat"
    f.write_text(EXAMPLE)
    code, out = _cli("compute", str(f), "--json", "--trace", "--alg", "1gamma")
    assert code == 0
    assert "g=1 L=2 U=1" in out
    rep = json.loads(out[out.index("{"):])
    assert rep["distance"] == 1 and rep["algorithm"] == "saved_1_gamma"
    assert rep["bounds_trace"] == [{"L": 2, "U": 1, "g": 1}]
    assert set(rep) == {"algorithm", "bounds_trace", "candidates_enumerated", "distance", "elapsed_seconds",
                        "generations", "k", "n", "workers"}
    # the config-1 isometry trace matches the reference's
    c = P.CONFIGS[1]
    f2 = tmp_path / "c1.mat"
    f2.write_text(P.format_matrix(P.generate_code(c["n"], c["k"], c["seed"])))
    code, out = _cli("compute", str(f2), "--alg", "isometry", "--trace")
    assert code == 0
    assert re.findall(r"g=(\d+) L=(\d+) U=(\d+)", out) == [("1", "4", "14"), ("2", "6", "10"), ("3", "8", "10"),
                                                          ("4", "10", "10")]


def test_cli_exit_codes(tmp_path):
    dup = tmp_path / "dup.mat"
    dup.write_text("3 4\n1001\n1001\n0011\n")
    code, out = _cli("compute", str(dup))
    assert code == 2 and "dependent" in out
    ill = tmp_path / "illustrative.mat"
    ill.write_text("3 8\n11110000\n00001011\n01110111\n")
    assert _cli("compute", str(ill), "--alg", "2gamma")[0] == 2
    code, out = _cli("compute", str(ill), "--alg", "2gamma", "--no-validate", "--no-dual-filter")
    assert code == 0 and "distance 2\n" in out


def test_cli_verify_and_bench(tmp_path):
    f = tmp_path / "verify.mat"
    f.write_text(P.format_matrix(P.random_stabilizer(8, 3, 777)))
    code, out = _cli("verify", str(f))
    assert code == 0 and "AGREE d=" in out
    big = tmp_path / "verify_big.mat"
    big.write_text(P.format_matrix(P.random_stabilizer(15, 15, 3)))
    code, out = _cli("verify", str(big))
    assert code == 0 and "oracle skipped" in out and "AGREE d=" in out
    code, out = _cli("bench", "--n", "6", "--k", "2", "--count", "3", "--seed", "42")
    assert code == 0
    for needle in ("median_s", "mean_s", "saved_1_gamma", "saved_2_gamma", "saved_isometry"):
        assert needle in out
