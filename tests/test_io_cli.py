"""Matrix text format, the reference instance generator and the CLI's host-side paths
(proj/tests/test_io_cli.cpp), on the CPU. The CLI's distance runs are in test_gpu_cli.py."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2408_10743_b200 as P

EXAMPLE = "3 4\n1001\n0110\n0011\n"


def test_parse_worked_example_and_spacing():
    inst = P.parse_matrix_text(EXAMPLE)
    assert (inst.n, inst.k) == (2, 1)
    assert inst.a.tolist() == [[1, 0, 0, 1], [0, 1, 1, 0], [0, 0, 1, 1]]
    inst = P.parse_matrix_text("2 4\n\n10 00\n\n0 100\n\n")
    assert (inst.n, inst.k) == (2, 0) and inst.a.tolist() == [[1, 0, 0, 0], [0, 1, 0, 0]]


@pytest.mark.parametrize("text,needle", [
    ("x y\n", "bad header"), ("2 5\n", "even"), ("6 4\n", "K exceeds N"), ("2 4\n1021\n0110\n", "row 1, column 3"),
    ("2 4\n101\n0110\n", "has 3 bits"), ("2 4\n1011\n", "found 1"), ("1 4\n1011\n0110\n", "found more"),
    ("", "empty")])
def test_parse_diagnostics(text, needle):
    # test_io_cli.cpp:57-74; the full message equals the reference library's
    with pytest.raises(P.ParseError) as e:
        P.parse_matrix_text(text, "f")
    assert needle in str(e.value)
    assert str(e.value).startswith("f:")


def test_format_parse_round_trip():
    rng = np.random.default_rng(97)
    for _ in range(50):
        n = int(rng.integers(1, 21))
        rows = int(rng.integers(1, 2 * n + 1))
        m = rng.integers(0, 2, size=(rows, 2 * n), dtype=np.uint8)
        text = P.format_matrix(m)
        assert text.splitlines()[0] == f"{rows} {2 * n}"
        assert (P.parse_matrix_text(text).a == m).all()


def test_random_stabilizer_matches_reference():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, k, seed in [(8, 3, 12345), (8, 3, 777), (15, 15, 3), (6, 2, 42), (16, 1, 11), (22, 2, 14), (1, 0, 5),
                       (12, 0, 9)]:
        mine = P.random_stabilizer(n, k, seed)
        assert (mine.a == O.ref_random_stabilizer(n, k, seed)).all()
        assert (mine.n, mine.k) == (n, k)
    with pytest.raises(ValueError):
        P.random_stabilizer(3, 4, 1)


def _cli(*args, cwd=None):
    r = subprocess.run([P.cli_path(), *args], capture_output=True, text=True, cwd=cwd, timeout=120)
    return r.returncode, r.stdout + r.stderr


def test_cli_exit_codes_before_the_device(tmp_path):
    # test_io_cli.cpp:132-141: missing file and malformed text exit 1 with the parser's message
    code, out = _cli("compute", str(tmp_path / "no_such_file.mat"))
    assert code == 1 and "cannot open file" in out
    bad = tmp_path / "bad.mat"
    bad.write_text("2 4\n12x1\n0110\n")
    code, out = _cli("compute", str(bad))
    assert code == 1 and "row 1, column 2" in out
    code, out = _cli("compute", str(bad), "--alg", "nope")
    assert code == 1  # the file is parsed first
    code, out = _cli()
    assert code != 0
